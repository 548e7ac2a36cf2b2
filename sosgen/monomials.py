"""Monomial bases in graded-lexicographic order.

Input-generation code (SURVEY §2 status GEN). Holds none of the ADMM arithmetic; it is
shared by the oracle and the GPU tests only as a source of problem bytes.

Order (reading C2, after PAPER.md P:65-68 "v_d(x) = [1, x1, ..., xn, x1^2, x1x2, ...]"
and SPEC.md S:33): degree ascending; inside one degree, exponent vectors in DESCENDING
lexicographic order (x1^2 > x1x2 > ... > x2^2).  A monomial of degree k is represented by its
sorted tuple of variable indices (x1^2 x3 -> (0, 0, 2)); descending lex on exponent vectors is
exactly ascending lex on these sorted index tuples, which is what we sort by.
"""
from __future__ import annotations

from itertools import combinations_with_replacement
from math import comb

import numpy as np


def basis_tuples(n: int, dmin: int, dmax: int) -> list[tuple[int, ...]]:
    """All monomials with dmin <= degree <= dmax in graded-lex order, as sorted var-index tuples."""
    out: list[tuple[int, ...]] = []
    for deg in range(dmin, dmax + 1):
        out.extend(combinations_with_replacement(range(n), deg))
    return out


def count(n: int, dmin: int, dmax: int) -> int:
    return sum(comb(n + k - 1, k) for k in range(dmin, dmax + 1))


def exponents(tuples: list[tuple[int, ...]], n: int) -> np.ndarray:
    """Exponent matrix (len(tuples) x n) of the given index tuples."""
    e = np.zeros((len(tuples), n), dtype=np.int64)
    for r, t in enumerate(tuples):
        for v in t:
            e[r, v] += 1
    return e


class MonomialIndex:
    """Maps exponent vectors to row positions of a fixed, ordered monomial list."""

    def __init__(self, expo: np.ndarray):
        self.expo = np.ascontiguousarray(expo, dtype=np.int64)
        self.n = self.expo.shape[1]
        self.keys = self.encode(self.expo)
        self._order = np.argsort(self.keys, kind="stable")
        self._sorted = self.keys[self._order]
        if len(self._sorted) > 1 and np.any(self._sorted[1:] == self._sorted[:-1]):
            raise ValueError("duplicate monomials in index")

    def encode(self, expo: np.ndarray) -> np.ndarray:
        """Exact byte key of each exponent row (exponents < 128)."""
        expo = np.asarray(expo)
        if expo.size and (expo.max() > 127 or expo.min() < 0):
            raise ValueError("exponent out of range")
        e8 = np.ascontiguousarray(expo.reshape(-1, self.n).astype(np.int8))
        return e8.view(np.dtype((np.void, self.n))).ravel()

    def lookup(self, expo: np.ndarray) -> np.ndarray:
        """Row index of each exponent vector (any leading shape), -1 where absent."""
        expo = np.asarray(expo)
        lead = expo.shape[:-1]
        k = self.encode(expo)
        pos = np.searchsorted(self._sorted, k)
        pos = np.clip(pos, 0, len(self._sorted) - 1)
        hit = self._sorted[pos] == k
        return np.where(hit, self._order[pos], -1).reshape(lead)


def poly_eval(coef: np.ndarray, expo: np.ndarray, x: np.ndarray) -> float:
    """Evaluate sum_r coef[r] * x^expo[r]."""
    return float(np.sum(coef * np.prod(np.power(x[None, :], expo), axis=1)))

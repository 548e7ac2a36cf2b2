"""Brute-force partial-orthogonality structure (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md P:224-230 (`eq:coeff`): (B_alpha)_{beta,gamma} = 1 iff beta + gamma = alpha, over the
Gram basis v_d.  Proposition 1: A2 A2^T = diag(n_1, ..., n_m), n_alpha = number of
nonzero entries of B_alpha.  This module enumerates every ORDERED pair (beta_i, beta_j) of the
Gram basis with plain Python loops and a dict — no sparse algebra, no A at all — and returns

* alpha_map[p] for every svec position p = (i, j), i <= j: the row index of beta_i + beta_j;
* n_alpha per row: the ordered-pair count, i.e. the exact integer D of Proposition 1.

It is used only for the bit-exact structure check against the library's `get_structure`.
"""
from __future__ import annotations

import numpy as np


def brute_force_structure(row_expo: np.ndarray, blocks: list[dict], m: int):
    """row_expo: (m x nvars) monomial of each row; blocks: dicts with 'basis', 'row_offset',
    'weighted' (weighted blocks are not orthogonal and are skipped, §VI).

    Returns (alpha_map per block (list of int arrays, or None for weighted blocks),
             n_alpha (length-m int64 array summed over the orthogonal blocks))."""
    # rows of one SOS constraint form a contiguous range starting at its row_offset
    offsets = sorted({int(b["row_offset"]) for b in blocks} | {m})
    n_alpha = np.zeros(m, dtype=np.int64)
    maps = []
    for blk in blocks:
        if blk["weighted"]:
            maps.append(None)
            continue
        lo = int(blk["row_offset"])
        hi = offsets[offsets.index(lo) + 1]
        row_of = {tuple(int(v) for v in row_expo[a]): a for a in range(lo, hi)}
        basis = [tuple(int(v) for v in r) for r in blk["basis"]]
        N = len(basis)
        amap = np.empty(N * (N + 1) // 2, dtype=np.int64)
        for j in range(N):
            for i in range(N):
                alpha = tuple(a + b for a, b in zip(basis[i], basis[j]))
                r = row_of[alpha]
                assert blk["row_offset"] <= r
                n_alpha[r] += 1  # ordered pair (i, j): B_alpha entry (i, j) is 1
                if i <= j:
                    amap[i + j * (j + 1) // 2] = r
        maps.append(amap)
    return maps, n_alpha

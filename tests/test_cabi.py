"""CPU checks of the boundary: the C-ABI library builds, loads and exports every symbol that
include/sosadmm.h declares; workspace sizing works without a GPU."""
import ctypes
import os
import re

import numpy as np

from paper_1708_04174_b200 import EXPORTS, load_library
from paper_1708_04174_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sosadmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # declarations only, not the comments
    return sorted(set(re.findall(r"\b(sosadmm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    build()
    lib = load_library()
    decl = declared_symbols()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(EXPORTS)
    # the stage-level debug entry points of include/sosadmm_debug.h as well
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "sosadmm_debug.h")).read(), flags=re.S)
    dbg = sorted(set(re.findall(r"\b(sosadmm_debug_[a-z_]+)\s*\(", src)))
    assert len(dbg) >= 5
    for name in dbg:
        assert hasattr(lib, name), name


def test_workspace_size_cpu():
    from paper_1708_04174_b200.sosadmm import _Problem, _dptr
    from sosgen import make_config

    lib = load_library()
    prob = make_config("pop6")
    A = prob.A.tocsc()
    cp = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.indices, dtype=np.int32)
    va = np.ascontiguousarray(A.data, dtype=np.float64)
    dims = np.array(prob.psd_dims, dtype=np.int32)
    p = _Problem(prob.m, prob.n_free, len(dims), dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                 cp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ri.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                 _dptr(va), _dptr(prob.b), _dptr(prob.c))
    nb = lib.sosadmm_workspace_size(ctypes.byref(p))
    assert nb > 8 * (2 * prob.n + 2 * prob.m)
    # a block larger than SOSADMM_MAX_BLOCK is refused (E_STRUCT at setup, 0 bytes here)
    big = np.array([1281], dtype=np.int32)
    pb = _Problem(prob.m, prob.n_free, 1, big.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  cp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ri.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  _dptr(va), _dptr(prob.b), _dptr(prob.c))
    assert lib.sosadmm_workspace_size(ctypes.byref(pb)) == 0
    # malformed input: decreasing column pointers
    bad = cp.copy()
    bad[3] = bad[2] - 1
    p.A_colptr = bad.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    assert lib.sosadmm_workspace_size(ctypes.byref(p)) == 0


def test_strerror():
    lib = load_library()
    assert lib.sosadmm_strerror(0) == b"ok"
    assert lib.sosadmm_strerror(-6) == b"non-finite iterate"


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1708_04174_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+(oracle|sosgen)\b", txt, re.M), f


def _problem(prob, m=None, n_free=None, dims=None, colptr=None, rowidx=None):
    from paper_1708_04174_b200.sosadmm import _Problem, _dptr

    A = prob.A.tocsc()
    keep = {}
    keep["cp"] = np.ascontiguousarray(A.indptr if colptr is None else colptr, dtype=np.int64)
    keep["ri"] = np.ascontiguousarray(A.indices if rowidx is None else rowidx, dtype=np.int32)
    keep["va"] = np.ascontiguousarray(A.data, dtype=np.float64)
    keep["dims"] = np.array(prob.psd_dims if dims is None else dims, dtype=np.int32)
    p = _Problem(prob.m if m is None else m, prob.n_free if n_free is None else n_free, len(keep["dims"]),
                 keep["dims"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                 keep["cp"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                 keep["ri"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dptr(keep["va"]), _dptr(prob.b),
                 _dptr(prob.c))
    return p, keep


def test_setup_rejects_malformed_problems_before_any_device_work():
    """include/sosadmm.h error contract: analysis runs on the host first, so malformed or unsupported
    input fails with E_ARG / E_STRUCT and a message, with no GPU needed (this runs on CPU)."""
    from paper_1708_04174_b200.sosadmm import _Settings
    from sosgen import make_config

    lib = load_library()
    prob = make_config("pop6")
    st = _Settings(1e-4, 100, 1, 0, None, None, 0)
    A = prob.A.tocsc()
    bad_rows = A.indices.copy()
    bad_rows[5] = prob.m  # row index out of range
    cases = [
        (dict(dims=[1281]), -2),          # block > SOSADMM_MAX_BLOCK
        (dict(m=0), -1),                  # empty row space
        (dict(n_free=-1), -1),            # negative size
        (dict(rowidx=bad_rows), -1),      # CSC row index out of range
    ]
    for kw, want in cases:
        p, keep = _problem(prob, **kw)
        ctx = ctypes.c_void_p()
        err = lib.sosadmm_setup(ctypes.byref(p), ctypes.byref(st), ctypes.byref(ctx))
        assert err == want, (kw.keys(), err)
        assert lib.sosadmm_workspace_size(ctypes.byref(p)) == 0
        assert len(lib.sosadmm_last_error_message(ctx)) > 0
        lib.sosadmm_destroy(ctx)
    ctx = ctypes.c_void_p()
    assert lib.sosadmm_setup(None, ctypes.byref(st), ctypes.byref(ctx)) == -1
    lib.sosadmm_destroy(ctx)
    assert lib.sosadmm_setup(ctypes.byref(_problem(prob)[0]), ctypes.byref(st), None) == -1

"""Thin ctypes binding of the C ABI in include/sosadmm.h (argument marshalling only).

Every step of the ADMM iteration runs in the CUDA kernels of `libsosadmm.so`; this module only
converts arrays to pointers, allocates the device workspace with PyTorch (device memory and a
dedicated stream are the only things PyTorch provides) and decodes results.  There is no CPU
fallback: if the library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsosadmm.so")

STATUS = {0: "RUNNING", 1: "OPTIMAL", 2: "PRIMAL_INFEASIBLE", 3: "DUAL_INFEASIBLE", 4: "MAX_ITERS",
          5: "INCONCLUSIVE"}

EXPORTS = ["sosadmm_workspace_size", "sosadmm_setup", "sosadmm_setup_sharded", "sosadmm_nccl_unique_id",
           "sosadmm_iterate", "sosadmm_iterate_async", "sosadmm_set_shared_gpu", "sosadmm_iterate_profiled",
           "sosadmm_get_info", "sosadmm_get_iterate", "sosadmm_set_iterate", "sosadmm_get_structure",
           "sosadmm_project_affine", "sosadmm_project_psd", "sosadmm_launches_per_iter", "sosadmm_psd_work", "sosadmm_warm_stats", "sosadmm_residual_history",
           "sosadmm_destroy",
           "sosadmm_strerror", "sosadmm_last_error_message"]


class _Problem(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n_free", ctypes.c_int64), ("n_psd", ctypes.c_int32),
                ("psd_dim", ctypes.POINTER(ctypes.c_int32)), ("A_colptr", ctypes.POINTER(ctypes.c_int64)),
                ("A_rowidx", ctypes.POINTER(ctypes.c_int32)), ("A_val", ctypes.POINTER(ctypes.c_double)),
                ("b", ctypes.POINTER(ctypes.c_double)), ("c", ctypes.POINTER(ctypes.c_double))]


class _Settings(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iters", ctypes.c_int64), ("check_every", ctypes.c_int32),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t)]


class _Info(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int64), ("status", ctypes.c_int32), ("res_pri", ctypes.c_double),
                ("res_dual", ctypes.c_double), ("res_gap", ctypes.c_double), ("pobj", ctypes.c_double),
                ("dobj", ctypes.c_double), ("tau", ctypes.c_double), ("kappa", ctypes.c_double),
                ("pinf", ctypes.c_double), ("dinf", ctypes.c_double)]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["status_name"] = STATUS.get(self.status, str(self.status))
        return d


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libsosadmm.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: build it with `python -m paper_1708_04174_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, D, I32, I64, V = (ctypes.POINTER(ctypes.c_double), ctypes.c_double, ctypes.c_int32, ctypes.c_int64,
                         ctypes.c_void_p)
    lib.sosadmm_workspace_size.argtypes = [ctypes.POINTER(_Problem)]
    lib.sosadmm_workspace_size.restype = ctypes.c_size_t
    lib.sosadmm_setup.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Settings), ctypes.POINTER(V)]
    lib.sosadmm_setup_sharded.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Settings), ctypes.c_char_p, I32,
                                          I32, ctypes.POINTER(I32), ctypes.POINTER(V)]
    lib.sosadmm_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.sosadmm_iterate.argtypes = [V, I64, ctypes.POINTER(_Info)]
    lib.sosadmm_iterate_profiled.argtypes = [V, I64, ctypes.POINTER(_Info), P]
    lib.sosadmm_iterate_async.argtypes = [V, I64]
    lib.sosadmm_set_shared_gpu.argtypes = [V, I32]
    lib.sosadmm_get_info.argtypes = [V, ctypes.POINTER(_Info)]
    lib.sosadmm_get_iterate.argtypes = [V, P, P, P, P, P, P, ctypes.POINTER(I64)]
    lib.sosadmm_set_iterate.argtypes = [V, P, P, P, P, D, D, I64]
    lib.sosadmm_get_structure.argtypes = [V, ctypes.POINTER(I32), P, ctypes.POINTER(I64)]
    lib.sosadmm_project_affine.argtypes = [V, P, P, D, P, P, P]
    lib.sosadmm_project_psd.argtypes = [V, I32, P, P]
    lib.sosadmm_psd_work.argtypes = [V, P, ctypes.POINTER(I32)]
    lib.sosadmm_psd_work.restype = ctypes.c_int
    lib.sosadmm_warm_stats.argtypes = [V, ctypes.POINTER(I64), ctypes.POINTER(I32)]
    lib.sosadmm_warm_stats.restype = ctypes.c_int
    lib.sosadmm_residual_history.argtypes = [V, P, ctypes.POINTER(I32)]
    lib.sosadmm_residual_history.restype = ctypes.c_int
    lib.sosadmm_launches_per_iter.argtypes = [V]
    lib.sosadmm_launches_per_iter.restype = I64
    lib.sosadmm_destroy.argtypes = [V]
    lib.sosadmm_destroy.restype = None
    lib.sosadmm_strerror.argtypes = [ctypes.c_int]
    lib.sosadmm_strerror.restype = ctypes.c_char_p
    lib.sosadmm_last_error_message.argtypes = [V]
    lib.sosadmm_debug_setup_emulated.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Settings), I32, I32,
                                                 ctypes.POINTER(I32), ctypes.POINTER(V)]
    lib.sosadmm_debug_setup_emulated.restype = ctypes.c_int
    lib.sosadmm_debug_group_iterate.argtypes = [ctypes.POINTER(V), ctypes.c_int, I64]
    lib.sosadmm_debug_group_iterate.restype = ctypes.c_int
    lib.sosadmm_debug_group_get_iterate.argtypes = [ctypes.POINTER(V), ctypes.c_int, P, P, P, P, P, P,
                                                    ctypes.POINTER(I64)]
    lib.sosadmm_debug_group_get_iterate.restype = ctypes.c_int
    lib.sosadmm_debug_group_link_peers.argtypes = [ctypes.POINTER(V), ctypes.c_int]
    lib.sosadmm_debug_group_link_peers.restype = ctypes.c_int
    lib.sosadmm_last_error_message.restype = ctypes.c_char_p
    for f in ["sosadmm_setup", "sosadmm_setup_sharded", "sosadmm_nccl_unique_id", "sosadmm_iterate", "sosadmm_iterate_profiled", "sosadmm_get_info",
              "sosadmm_get_iterate", "sosadmm_set_iterate", "sosadmm_get_structure", "sosadmm_project_affine",
              "sosadmm_project_psd"]:
        getattr(lib, f).restype = ctypes.c_int
    _lib = lib
    return lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


NCCL_ID_BYTES = 128
NPHASE = 7  # SOSADMM_NPHASE
PHASES = ["affine", "scatter", "jacobi", "tridiag", "dc", "backtransform_recon", "pack"]


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 of a sharded solve creates it; the caller broadcasts it)."""
    import torch  # noqa: F401  (loads torch's libnccl.so.2 first, so the library resolves the same NCCL)

    lib = load_library()
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    err = lib.sosadmm_nccl_unique_id(buf)
    if err != 0:
        raise RuntimeError(f"sosadmm_nccl_unique_id: {lib.sosadmm_strerror(err).decode()} ({err})")
    return buf.raw


class SosAdmm:
    """One SOS-derived SDP on one GPU: setup(A, b, c, cone dims) once, then iterate(k)."""

    def __init__(self, A, b, c, n_free: int, psd_dims, tol: float = 1e-4, max_iters: int = 2000,
                 device: int = 0, shard=None):
        """shard = (rank, world, nccl_id, block_owner) runs the multi-GPU block-sharded mode
        (sosadmm_setup_sharded); iterate / info / get_iterate are then collectives."""
        import torch  # device memory + stream only

        if not torch.cuda.is_available():
            raise RuntimeError("SosAdmm needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self._A = A.tocsc() if hasattr(A, "tocsc") else A
        self._A.sort_indices()
        self.m, self.n = self._A.shape
        self._colptr = np.ascontiguousarray(self._A.indptr, dtype=np.int64)
        self._rowidx = np.ascontiguousarray(self._A.indices, dtype=np.int32)
        self._val = np.ascontiguousarray(self._A.data, dtype=np.float64)
        self._b = np.ascontiguousarray(b, dtype=np.float64)
        self._c = np.ascontiguousarray(c, dtype=np.float64)
        self._dims = np.ascontiguousarray(psd_dims, dtype=np.int32)
        self.n_free = int(n_free)
        self.psd_dims = [int(d) for d in psd_dims]
        self._prob = _Problem(self.m, self.n_free, len(self._dims),
                              self._dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                              self._colptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              self._rowidx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                              _dptr(self._val), _dptr(self._b), _dptr(self._c))
        nbytes = self.lib.sosadmm_workspace_size(ctypes.byref(self._prob))
        if nbytes == 0:
            raise ValueError("malformed problem (sosadmm_workspace_size returned 0)")
        self.device = device
        self._torch_dev = torch.device("cuda", device)
        self._ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self._torch_dev)
        self.stream = torch.cuda.Stream(device=self._torch_dev)
        st = _Settings(tol, max_iters, 1, device, ctypes.c_void_p(self.stream.cuda_stream),
                       ctypes.c_void_p(self._ws.data_ptr()), int(nbytes))
        self._ctx = ctypes.c_void_p()
        self.shard = shard
        if shard is None:
            err = self.lib.sosadmm_setup(ctypes.byref(self._prob), ctypes.byref(st), ctypes.byref(self._ctx))
        else:
            rank, world, nccl_id, owner = shard
            self._owner = np.ascontiguousarray(owner, dtype=np.int32)
            if len(self._owner) != len(self._dims) or (nccl_id is not None and len(nccl_id) != NCCL_ID_BYTES):
                raise ValueError("shard: block_owner needs one entry per PSD block and a 128-byte NCCL id")
            own_p = self._owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            if nccl_id is None:  # one-GPU emulation of rank `rank` (include/sosadmm_debug.h; tests only)
                err = self.lib.sosadmm_debug_setup_emulated(ctypes.byref(self._prob), ctypes.byref(st), int(rank),
                                                            int(world), own_p, ctypes.byref(self._ctx))
            else:
                err = self.lib.sosadmm_setup_sharded(ctypes.byref(self._prob), ctypes.byref(st), bytes(nccl_id),
                                                     int(rank), int(world), own_p, ctypes.byref(self._ctx))
        self._check(err, "setup")
        self.workspace_bytes = int(nbytes)

    @staticmethod
    def from_problem(prob, **kw) -> "SosAdmm":
        return SosAdmm(prob.A, prob.b, prob.c, prob.n_free, prob.psd_dims, **kw)

    def _check(self, err: int, what: str):
        if err != 0:
            msg = self.lib.sosadmm_last_error_message(self._ctx).decode() if self._ctx else ""
            raise RuntimeError(f"sosadmm_{what}: {self.lib.sosadmm_strerror(err).decode()} ({err}): {msg}")

    def iterate(self, k: int) -> dict:
        info = _Info()
        self._check(self.lib.sosadmm_iterate(self._ctx, int(k), ctypes.byref(info)), "iterate")
        return info.as_dict()

    def iterate_async(self, k: int) -> None:
        """Enqueue k iterations on this instance's stream and return at once (see iterate_batch)."""
        self._check(self.lib.sosadmm_iterate_async(self._ctx, int(k)), "iterate_async")

    def set_shared_gpu(self, shared: bool) -> None:
        """Scheduling hint (sosadmm_set_shared_gpu): other instances iterate on this GPU at the same time."""
        self._check(self.lib.sosadmm_set_shared_gpu(self._ctx, 1 if shared else 0), "set_shared_gpu")

    def iterate_profiled(self, k: int):
        info = _Info()
        ms = np.zeros(NPHASE)
        self._check(self.lib.sosadmm_iterate_profiled(self._ctx, int(k), ctypes.byref(info), _dptr(ms)),
                    "iterate_profiled")
        return info.as_dict(), ms

    def psd_work(self) -> list:
        """Per large block: dict of the algorithmic FP64 flops of the last projection (sosadmm_psd_work)."""
        n = ctypes.c_int32(0)
        self._check(self.lib.sosadmm_psd_work(self._ctx, None, ctypes.byref(n)), "psd_work")
        w = np.zeros(6 * max(n.value, 1))
        self._check(self.lib.sosadmm_psd_work(self._ctx, _dptr(w), ctypes.byref(n)), "psd_work")
        keys = ["tridiag", "dc_gemm", "backtransform", "recon", "r", "dc_zero_merges"]
        return [dict(zip(keys, w[6 * b:6 * b + 6].tolist())) for b in range(n.value)]

    def residual_history(self, cap: int = 1024) -> np.ndarray:
        """Rows (k, pres, dres, gap, pobj) of the last iterates u^k, oldest first (sosadmm_residual_history)."""
        out = np.zeros(5 * cap)
        n = ctypes.c_int32(cap)
        self._check(self.lib.sosadmm_residual_history(self._ctx, _dptr(out), ctypes.byref(n)), "residual_history")
        return out[:5 * n.value].reshape(n.value, 5)[::-1].copy()

    def warm_stats(self) -> list:
        """Per large block: the warm-start counters (sosadmm_warm_stats, csrc/warm.cuh)."""
        n = ctypes.c_int32(0)
        self._check(self.lib.sosadmm_warm_stats(self._ctx, None, ctypes.byref(n)), "warm_stats")
        w = np.zeros(10 * max(n.value, 1), dtype=np.int64)
        self._check(self.lib.sosadmm_warm_stats(self._ctx, w.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                ctypes.byref(n)), "warm_stats")
        keys = ["warm", "cold", "updates", "failed", "enabled", "r", "N", "last_evals", "seeds", "last_fail_reason"]
        return [dict(zip(keys, w[10 * b:10 * b + 10].tolist())) for b in range(n.value)]

    def info(self) -> dict:
        info = _Info()
        self._check(self.lib.sosadmm_get_info(self._ctx, ctypes.byref(info)), "get_info")
        return info.as_dict()

    def get_iterate(self, out: dict | None = None):
        """The iterate (u, v) = (xi, y, tau, z, s, kappa) on the host.  out: preallocated float64 arrays
        {"xi", "y", "z", "s"} (e.g. views of pinned host tensors, so the copies run at full DMA rate)."""
        if out is not None:
            xi, y, z, s = (out[k] for k in ("xi", "y", "z", "s"))
            for arr, size in ((xi, self.n), (z, self.n), (y, self.m), (s, self.m)):
                if arr.dtype != np.float64 or arr.size != size or not arr.flags.c_contiguous:
                    raise ValueError("get_iterate(out=...): contiguous float64 arrays of the iterate's sizes")
        else:
            xi, z = np.empty(self.n), np.empty(self.n)
            y, s = np.empty(self.m), np.empty(self.m)
        tau, kappa, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.sosadmm_get_iterate(self._ctx, _dptr(xi), _dptr(y), _dptr(z), _dptr(s),
                                                 ctypes.byref(tau), ctypes.byref(kappa), ctypes.byref(it)),
                    "get_iterate")
        return dict(xi=xi, y=y, z=z, s=s, tau=tau.value, kappa=kappa.value, iter=it.value)

    def set_iterate(self, xi, y, z, s=None, tau=1.0, kappa=0.0, iter=0):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.ascontiguousarray(z, dtype=np.float64)
        sp_ = None if s is None else _dptr(np.ascontiguousarray(s, dtype=np.float64))
        if s is not None:
            s = np.ascontiguousarray(s, dtype=np.float64)
            sp_ = _dptr(s)
        self._check(self.lib.sosadmm_set_iterate(self._ctx, _dptr(xi), _dptr(y), _dptr(z), sp_, float(tau),
                                                 float(kappa), int(iter)), "set_iterate")

    def get_structure(self):
        row_of = np.empty(self.n, dtype=np.int32)
        D = np.empty(self.m)
        t = ctypes.c_int64()
        self._check(self.lib.sosadmm_get_structure(self._ctx, row_of.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                   _dptr(D), ctypes.byref(t)), "get_structure")
        return row_of, D, t.value

    def project_affine(self, w1, w2, w3: float):
        w1 = np.ascontiguousarray(w1, dtype=np.float64)
        w2 = np.ascontiguousarray(w2, dtype=np.float64)
        u1, u2, u3 = np.empty(self.n), np.empty(self.m), ctypes.c_double()
        self._check(self.lib.sosadmm_project_affine(self._ctx, _dptr(w1), _dptr(w2), float(w3), _dptr(u1),
                                                    _dptr(u2), ctypes.byref(u3)), "project_affine")
        return u1, u2, u3.value

    def project_psd(self, block: int, a_svec):
        a = np.ascontiguousarray(a_svec, dtype=np.float64)
        out = np.empty_like(a)
        self._check(self.lib.sosadmm_project_psd(self._ctx, int(block), _dptr(a), _dptr(out)), "project_psd")
        return out

    @property
    def launches_per_iter(self) -> int:
        return int(self.lib.sosadmm_launches_per_iter(self._ctx))

    def close(self):
        if getattr(self, "_ctx", None):
            self.lib.sosadmm_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def iterate_batch(solvers, k: int, chunk: int = 256) -> list:
    """k iterations of independent instances on one GPU.  Each SosAdmm owns a stream,
    so every instance's graph replays are enqueued before any is waited on and the instances run
    concurrently (the per-instance iterates are exactly those of solo runs).  Replays are enqueued in
    rounds of `chunk` per instance; after each round the instances that reached a terminal status
    (their replays would be device-side no-ops) drop out, so solving a batch to convergence with a
    large k costs at most one round past each instance's stop.  Returns every instance's info."""
    if k < 0 or chunk < 1:
        raise ValueError("k must be >= 0 and chunk >= 1")
    left = [int(k)] * len(solvers)
    active = list(range(len(solvers)))
    if len(solvers) > 1:
        for s in solvers:
            s.set_shared_gpu(True)  # scheduling hint only: the iterates do not change
    while active:
        for i in active:
            n = min(chunk, left[i])
            solvers[i].iterate_async(n)
            left[i] -= n
        active = [i for i in active if left[i] > 0 and solvers[i].info()["status"] == 0]
    return [s.info() for s in solvers]


def group_iterate(solvers, k: int) -> None:
    """k iterations of an emulated block-sharded group (solvers[r] = rank r, set up with shard=(r, world,
    None, owner)): the world >= 2 arithmetic on one GPU, the partial sums added by a device kernel."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    err = lib.sosadmm_debug_group_iterate(arr, len(solvers), int(k))
    if err != 0:
        raise RuntimeError(f"sosadmm_debug_group_iterate: {lib.sosadmm_strerror(err).decode()} ({err})")


def group_link_peers(solvers) -> None:
    """Switch an emulated group to the peer-memory reduction fused into k_gather_fin_peer (f4)."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    err = lib.sosadmm_debug_group_link_peers(arr, len(solvers))
    if err != 0:
        raise RuntimeError(f"sosadmm_debug_group_link_peers: {lib.sosadmm_strerror(err).decode()} ({err})")


def group_get_iterate(solvers) -> dict:
    lib = load_library()
    s0 = solvers[0]
    out = {k: np.zeros(s0.n) for k in ("xi", "z")}
    out.update({k: np.zeros(s0.m) for k in ("y", "s")})
    tau, kappa, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    arr = (ctypes.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    err = lib.sosadmm_debug_group_get_iterate(arr, len(solvers), _dptr(out["xi"]), _dptr(out["y"]), _dptr(out["z"]),
                                              _dptr(out["s"]), ctypes.byref(tau), ctypes.byref(kappa),
                                              ctypes.byref(it))
    if err != 0:
        raise RuntimeError(f"sosadmm_debug_group_get_iterate: {lib.sosadmm_strerror(err).decode()} ({err})")
    out.update(tau=tau.value, kappa=kappa.value, iter=it.value)
    return out

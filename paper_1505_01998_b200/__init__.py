"""B200-native all-pairs kernel-sum engine for the KDE bandwidth selectors of arxiv 1505.01998.

Thin ctypes binding over the C ABI in include/kde.h (libkde_b200.so, built in-tree by
paper_1505_01998_b200.build).  Argument marshalling only: every step of the path (moments,
data prep, pair sums, reductions, the NCCL all-reduce) runs in the library.  PyTorch provides
device memory, the CUDA stream and (for world > 1) the process group used to broadcast the
NCCL unique id.  Sample matrices may be CUDA tensors or host arrays (the library copies host
arrays to the GPU inside the call).  There is no CPU fallback: if the library is missing this
module raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkde_b200.so")

PLUGIN, LSCV_h, LSCV_H = 0, 1, 2
SUM_PSI4, SUM_PSI6, SUM_PSI8, SUM_LSCV_h, SUM_LSCV_H = 4, 6, 8, 1, 2

STATUS = {
    0: "KDE_OK", 1: "KDE_E_INVALID", 2: "KDE_E_NOT_UNIVARIATE", 3: "KDE_E_INSUFFICIENT_SAMPLES",
    4: "KDE_E_DEGENERATE", 5: "KDE_E_SINGULAR_COV", 6: "KDE_E_NONPOSITIVE_BW",
    7: "KDE_E_DIM_MISMATCH", 8: "KDE_E_NUMERIC", 9: "KDE_E_NO_FEASIBLE", 10: "KDE_E_CUDA",
    11: "KDE_E_NCCL", 12: "KDE_E_OOM",
}

# Every symbol include/kde.h declares (checked by tests/test_abi.py).
EXPORTS = ["kde_create", "kde_destroy", "kde_last_error", "kde_nccl_unique_id",
           "kde_workspace_bytes", "kde_set_workspace", "kde_default_opts", "kde_psi_r",
           "kde_plugin_h", "kde_lscv_h_scores", "kde_lscv_H_scores", "kde_select_bandwidth",
           "kde_raw_sums", "kde_fixed_value", "kde_fixed_add", "kde_tile_coords",
           "kde_last_profile", "kde_set_profiling", "kde_shard_tiles", "kde_shard_tile", "kde_psi_skip_gap", "kde_lscv_skip_theta", "kde_evaluate", "kde_aqp_1d",
           "kde_lscv_h_scores_materialized", "kde_last_aux_ms", "kde_set_host_allreduce", "kde_set_precision",
           "kde_last_fp64_passes", "kde_last_psi_kappa", "kde_last_psi_gaps"]


class KDEError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class PluginTrace(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in
                ("V_hat", "sigma_hat", "psi8_ns", "g1", "psi6", "g2", "psi4", "h")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SelectOpts(ctypes.Structure):
    _fields_ = [("n_grid", ctypes.c_int32), ("range_factor", ctypes.c_double),
                ("max_iter", ctypes.c_int32), ("tol_rel", ctypes.c_double),
                ("penalty", ctypes.c_double), ("speculative", ctypes.c_int32),
                ("refine_steps", ctypes.c_int32), ("refine_tol", ctypes.c_double),
                ("nm_starts", ctypes.c_int32), ("nm_loop", ctypes.c_int32), ("nm_param", ctypes.c_int32)]


class Bandwidth(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("d", ctypes.c_int32), ("h", ctypes.c_double),
                ("vechH", ctypes.c_double * 136), ("objective", ctypes.c_double),
                ("iterations", ctypes.c_int32), ("evaluations", ctypes.c_int32),
                ("stop_reason", ctypes.c_int32), ("trace", PluginTrace)]


class Fixed(ctypes.Structure):
    _fields_ = [("hi", ctypes.c_int64), ("mid", ctypes.c_int64), ("lo", ctypes.c_int64),
                ("scale_exp", ctypes.c_int32), ("pad_", ctypes.c_int32)]

    def key(self):
        """Exact identity of the value: the integer hi 2^80 + mid 2^40 + lo and the scale (limb
        layouts that differ only by carries, e.g. a sum of shards, compare equal)."""
        return (self.hi * (1 << 80) + self.mid * (1 << 40) + self.lo, self.scale_exp)


_lib = None

# int (*)(int64_t* data, size_t count, void* user): the test transport's all-reduce callback
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_size_t, ctypes.c_void_p)


def lib():
    """Load libkde_b200.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1505_01998_b200.build` "
                          "(the CUDA path is the only implementation)")
    L = ctypes.CDLL(LIB_PATH)
    vp, dp, i32, i64, f64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.kde_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int]
    L.kde_destroy.argtypes = [vp]; L.kde_destroy.restype = None
    L.kde_last_error.argtypes = [vp]; L.kde_last_error.restype = ctypes.c_char_p
    L.kde_nccl_unique_id.argtypes = [vp]
    L.kde_workspace_bytes.argtypes = [i64, i32, i32]; L.kde_workspace_bytes.restype = ctypes.c_size_t
    L.kde_set_workspace.argtypes = [vp, vp, ctypes.c_size_t]
    L.kde_default_opts.argtypes = [ctypes.POINTER(SelectOpts)]; L.kde_default_opts.restype = None
    L.kde_psi_r.argtypes = [vp, vp, i64, i32, dp, i32, dp]
    L.kde_plugin_h.argtypes = [vp, vp, i64, dp, ctypes.POINTER(PluginTrace)]
    L.kde_lscv_h_scores.argtypes = [vp, vp, i64, i32, dp, i32, dp]
    L.kde_lscv_H_scores.argtypes = [vp, vp, i64, i32, dp, i32, f64, dp]
    L.kde_select_bandwidth.argtypes = [vp, ctypes.c_int, vp, i64, i32, ctypes.POINTER(SelectOpts), ctypes.POINTER(Bandwidth)]
    L.kde_raw_sums.argtypes = [vp, ctypes.c_int, vp, i64, i32, dp, i32, i32, i32, ctypes.POINTER(Fixed)]
    L.kde_fixed_value.argtypes = [ctypes.POINTER(Fixed)]; L.kde_fixed_value.restype = f64
    L.kde_fixed_add.argtypes = [Fixed, Fixed]; L.kde_fixed_add.restype = Fixed
    L.kde_tile_coords.argtypes = [i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]; L.kde_tile_coords.restype = None
    L.kde_last_profile.argtypes = [vp, ctypes.POINTER(i32), dp, dp, ctypes.POINTER(i32)]
    L.kde_set_profiling.argtypes = [vp, i32]
    L.kde_shard_tiles.argtypes = [ctypes.c_int, i64, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i64),
                                  ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.kde_shard_tiles.restype = ctypes.c_int
    L.kde_shard_tile.argtypes = [i64, i32, i32]; L.kde_shard_tile.restype = i64
    L.kde_psi_skip_gap.argtypes = [i32, f64, f64]; L.kde_psi_skip_gap.restype = f64
    L.kde_lscv_skip_theta.argtypes = [i64]; L.kde_lscv_skip_theta.restype = f64
    L.kde_evaluate.argtypes = [vp, vp, i64, i32, vp, i64, dp, dp]
    L.kde_evaluate.restype = ctypes.c_int
    L.kde_aqp_1d.argtypes = [vp, vp, i64, f64, dp, dp, i32, dp, dp, dp]
    L.kde_aqp_1d.restype = ctypes.c_int
    L.kde_lscv_h_scores_materialized.argtypes = [vp, vp, i64, i32, dp, i32, i32, dp]
    L.kde_lscv_h_scores_materialized.restype = ctypes.c_int
    L.kde_last_aux_ms.argtypes = [vp]
    L.kde_last_aux_ms.restype = f64
    L.kde_set_precision.argtypes = [vp, i32]
    L.kde_set_precision.restype = ctypes.c_int
    L.kde_last_fp64_passes.argtypes = [vp]
    L.kde_last_fp64_passes.restype = i32
    L.kde_last_psi_kappa.argtypes = [vp]
    L.kde_last_psi_kappa.restype = f64
    L.kde_last_psi_gaps.argtypes = [vp, dp, i32]
    L.kde_last_psi_gaps.restype = i32
    L.kde_set_host_allreduce.argtypes = [vp, HOST_ALLREDUCE_FN, vp]
    L.kde_set_host_allreduce.restype = ctypes.c_int
    for f in ("kde_create", "kde_nccl_unique_id", "kde_set_workspace", "kde_psi_r", "kde_plugin_h",
              "kde_lscv_h_scores", "kde_lscv_H_scores", "kde_select_bandwidth", "kde_raw_sums",
              "kde_last_profile", "kde_set_profiling"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _dbuf(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def tile_coords(bx: int):
    l, q = ctypes.c_int64(), ctypes.c_int64()
    lib().kde_tile_coords(int(bx), ctypes.byref(l), ctypes.byref(q))
    return l.value, q.value


def psi_skip_gap(r: int, g: float, var: float) -> float:
    return lib().kde_psi_skip_gap(int(r), float(g), float(var))


def lscv_skip_theta(n: int) -> float:
    return lib().kde_lscv_skip_theta(int(n))


def fixed_value(f: Fixed) -> float:
    return lib().kde_fixed_value(ctypes.byref(f))


def fixed_add(a: Fixed, b: Fixed) -> Fixed:
    return lib().kde_fixed_add(a, b)


def shard_tiles(kind: int, n: int, d: int, rank: int, world: int):
    """(tile edge T, total tiles, rank's tile count, chunk) of `rank`'s share (host-only query); the
    rank's local index i is tile id shard_tile(i, rank, world) (round-robin chunks)."""
    T, tot, cnt, ch = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    rc = lib().kde_shard_tiles(int(kind), int(n), int(d), int(rank), int(world), ctypes.byref(T),
                               ctypes.byref(tot), ctypes.byref(cnt), ctypes.byref(ch))
    if rc != 0:
        raise KDEError(rc, "bad shard query")
    return T.value, tot.value, cnt.value, ch.value


def shard_tile(i: int, rank: int, world: int) -> int:
    """Tile id of local index i of `rank` of `world` (kde_shard_tile)."""
    return int(lib().kde_shard_tile(int(i), int(rank), int(world)))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().kde_nccl_unique_id(buf)
    if rc != 0:
        raise KDEError(rc, "ncclGetUniqueId failed")
    return buf.raw


def default_opts() -> SelectOpts:
    o = SelectOpts()
    lib().kde_default_opts(ctypes.byref(o))
    return o


class _Samples:
    """A (d, n) fp64 sample matrix as the C ABI sees it: pointer, d, n (plus a reference that
    keeps the memory alive for the duration of the call)."""
    __slots__ = ("ptr", "d", "n", "host", "_keep")

    def __init__(self, ptr, d, n, host, keep):
        self.ptr, self.d, self.n, self.host, self._keep = ctypes.c_void_p(ptr), d, n, host, keep

    @property
    def shape(self):
        return (self.d, self.n)


def _samples(X) -> _Samples:
    """Marshal a sample matrix, (n,) or (d, n) fp64.  A CUDA tensor is passed as a device
    pointer; a host array (numpy, or a CPU tensor, pinned or not) as a host pointer, which the
    library copies to the GPU inside the call (include/kde.h).  There is no CPU compute path."""
    import torch
    if isinstance(X, torch.Tensor):
        if X.dtype != torch.float64:
            raise TypeError("sample matrix must be float64")
        if X.dim() == 1:
            X = X.unsqueeze(0)
        if X.dim() != 2:
            raise ValueError("sample matrix must be (n,) or (d, n)")
        X = X.contiguous()
        return _Samples(X.data_ptr(), X.shape[0], X.shape[1], not X.is_cuda, X)
    if not isinstance(X, np.ndarray):
        raise TypeError("sample matrix must be a torch.Tensor or a numpy array")
    if X.dtype != np.float64:
        raise TypeError("sample matrix must be float64")
    if X.ndim == 1:
        X = X[None, :]
    if X.ndim != 2:
        raise ValueError("sample matrix must be (n,) or (d, n)")
    X = np.ascontiguousarray(X)
    return _Samples(X.ctypes.data, X.shape[0], X.shape[1], True, X)


def to_device(X, device=None, pinned: bool = True):
    """Copy a host array to the GPU (pinned staging, non-blocking on the current stream)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(X, dtype=np.float64)))
    if pinned:
        t = t.pin_memory()
    return t.to(device or torch.device("cuda", torch.cuda.current_device()), non_blocking=True)


class Context:
    """One library context = one GPU, one stream, optionally one NCCL communicator."""

    def __init__(self, device: int | None = None, stream=None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, profiling: bool = False):
        import torch
        L = lib()
        if device is None:
            device = torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device, self.stream, self.rank, self.world = device, stream, rank, world
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        rc = L.kde_create(ctypes.byref(h), int(device), ctypes.c_void_p(stream.cuda_stream),
                          idbuf, int(rank), int(world))
        if rc != 0:
            raise KDEError(rc, "kde_create failed")
        self._h = h
        if profiling:
            self.set_profiling(True)

    @classmethod
    def distributed(cls, device: int | None = None, profiling: bool = False):
        """SPMD context over the default torch.distributed process group (NCCL id broadcast)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return cls(device=device, rank=rank, world=world, nccl_id=obj[0] if world > 1 else None,
                   profiling=profiling)

    @classmethod
    def distributed_host(cls, device: int | None = None, profiling: bool = False):
        """SPMD context whose per-pass partial sums are summed with torch.distributed on the host
        (any backend, e.g. gloo): a test transport for several ranks sharing one GPU, where NCCL
        refuses to run.  All compute stays on the GPU; only the int64 partial sums (24 bytes per
        output) travel through host memory."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        ctx = cls(device=device, rank=rank, world=world, profiling=profiling)

        def _allreduce(ptr, count, _user):
            try:
                arr = np.ctypeslib.as_array(ptr, shape=(count,))
                t = torch.from_numpy(arr)          # shares the pinned staging buffer
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
                return 0
            except Exception:
                return 1

        ctx._har = HOST_ALLREDUCE_FN(_allreduce)  # keep the callback alive
        ctx._check(lib().kde_set_host_allreduce(ctx._h, ctx._har, None))
        return ctx

    def close(self):
        if getattr(self, "_h", None):
            lib().kde_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            raise KDEError(rc, lib().kde_last_error(self._h).decode(errors="replace"))

    def set_workspace(self, buf):
        """Hand the library a caller-owned device workspace (a CUDA tensor that must outlive its
        use; kde_workspace_bytes tells the size a call needs)."""
        self._ws = buf
        self._check(lib().kde_set_workspace(self._h, ctypes.c_void_p(buf.data_ptr()),
                                            buf.numel() * buf.element_size()))

    def set_precision(self, fp64_terms):
        """Psi_r term precision (kde_set_precision): True / 1 = fp64 terms (exact-parity mode),
        False / 0 = automatic (fp32 terms, fp64 re-run of a pass that cancels too much),
        -1 = fp32 terms only (diagnostics)."""
        mode = int(fp64_terms) if not isinstance(fp64_terms, bool) else (1 if fp64_terms else 0)
        self._check(lib().kde_set_precision(self._h, mode))

    def last_fp64_passes(self) -> int:
        """Psi passes of the last call re-run with fp64 terms by the automatic precision."""
        return int(lib().kde_last_fp64_passes(self._h))

    def last_psi_kappa(self) -> float:
        """Largest cancellation estimate 2A/|2S + n He_r(0)| of the last call's fp32 Psi passes."""
        return float(lib().kde_last_psi_kappa(self._h))

    def last_psi_gaps(self):
        """Far-tile skip thresholds of the last call's fp32-term Psi passes (kde_last_psi_gaps)."""
        buf = (ctypes.c_double * 8)()
        cnt = lib().kde_last_psi_gaps(self._h, buf, 8)
        return [buf[k] for k in range(min(cnt, 8))]

    def set_profiling(self, on: bool):
        self._check(lib().kde_set_profiling(self._h, 1 if on else 0))

    def last_profile(self) -> dict:
        a, b = ctypes.c_int32(), ctypes.c_int32()
        ms, ev = ctypes.c_double(), ctypes.c_double()
        self._check(lib().kde_last_profile(self._h, ctypes.byref(a), ctypes.byref(ms), ctypes.byref(ev), ctypes.byref(b)))
        return {"pair_launches": a.value, "pair_ms": ms.value, "pair_evals": ev.value, "kernel_launches": b.value}

    # ---- the five entry points
    def psi_r(self, x, r: int, g) -> np.ndarray:
        X = _samples(x)
        if X.shape[0] != 1:
            raise KDEError(2, "Psi_r needs univariate data")
        gb, gp = _dbuf(np.atleast_1d(g))
        out = np.zeros(gb.size)
        self._check(lib().kde_psi_r(self._h, X.ptr, X.shape[1], int(r), gp,
                                    gb.size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def plugin_h(self, x):
        X = _samples(x)
        if X.shape[0] != 1:
            raise KDEError(2, "PLUGIN needs univariate data")
        h = ctypes.c_double()
        tr = PluginTrace()
        self._check(lib().kde_plugin_h(self._h, X.ptr, X.shape[1],
                                       ctypes.byref(h), ctypes.byref(tr)))
        return h.value, tr.as_dict()

    def lscv_h_scores(self, X, h) -> np.ndarray:
        X = _samples(X)
        hb, hp = _dbuf(np.atleast_1d(h))
        out = np.zeros(hb.size)
        self._check(lib().kde_lscv_h_scores(self._h, X.ptr, X.shape[1], X.shape[0],
                                            hp, hb.size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def lscv_H_scores(self, X, vechs, penalty: float = float("nan")) -> np.ndarray:
        X = _samples(X)
        d = X.shape[0]
        vb, vp = _dbuf(np.atleast_2d(vechs))
        if vb.shape[1] != d * (d + 1) // 2:
            raise KDEError(7, "vech length does not match d")
        out = np.zeros(vb.shape[0])
        self._check(lib().kde_lscv_H_scores(self._h, X.ptr, X.shape[1], d, vp,
                                            vb.shape[0], float(penalty),
                                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def select_bandwidth(self, method: int, X, **opts) -> dict:
        X = _samples(X)
        o = default_opts()
        for k, v in opts.items():
            setattr(o, k, v)
        r = Bandwidth()
        self._check(lib().kde_select_bandwidth(self._h, int(method), X.ptr, X.shape[1],
                                               X.shape[0], ctypes.byref(o), ctypes.byref(r)))
        d = X.shape[0]
        out = {"method": r.method, "d": r.d, "h": r.h, "objective": r.objective,
               "iterations": r.iterations, "evaluations": r.evaluations, "stop_reason": r.stop_reason}
        if method == LSCV_H:
            out["vechH"] = np.array(r.vechH[: d * (d + 1) // 2])
        if method == PLUGIN:
            out["trace"] = r.trace.as_dict()
        return out

    def lscv_h_scores_materialized(self, X, h, h_per_pass: int = 1) -> np.ndarray:
        """LSCV_h scores via the paper's two-phase algorithm (materialised S(v) buffer)."""
        X = _samples(X)
        hb, hp = _dbuf(np.atleast_1d(h))
        out = np.zeros(hb.size)
        self._check(lib().kde_lscv_h_scores_materialized(self._h, X.ptr, X.shape[1],
                                                         X.shape[0], hp, hb.size, int(h_per_pass),
                                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def last_aux_ms(self) -> float:
        return lib().kde_last_aux_ms(self._h)

    def evaluate(self, X, Y, H) -> np.ndarray:
        """fhat at the columns of Y (both CUDA tensors, d x n and d x m); H: d x d or vech."""
        Xd, Yd = _samples(X), _samples(Y)
        d = Xd.shape[0]
        if Yd.shape[0] != d:
            raise KDEError(7, "query dimension differs from the sample dimension")
        Hn = np.asarray(H, dtype=np.float64)
        vh = Hn if Hn.ndim == 1 else np.array([Hn[i, j] for j in range(d) for i in range(j, d)])
        vb, vp = _dbuf(vh)
        out = np.zeros(Yd.shape[1])
        self._check(lib().kde_evaluate(self._h, Xd.ptr, Xd.shape[1], d,
                                       Yd.ptr, Yd.shape[1], vp,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def aqp_1d(self, x, h: float, lo, hi):
        """(COUNT, SUM, AVG) arrays over the intervals [lo_q, hi_q] (univariate)."""
        Xd = _samples(x)
        if Xd.shape[0] != 1:
            raise KDEError(2, "AQP closed forms are univariate")
        lb, lp = _dbuf(np.atleast_1d(lo))
        hb, hp = _dbuf(np.atleast_1d(hi))
        cnt, sm, av = (np.zeros(lb.size) for _ in range(3))
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self._check(lib().kde_aqp_1d(self._h, Xd.ptr, Xd.shape[1], float(h), lp, hp,
                                     lb.size, P(cnt), P(sm), P(av)))
        return cnt, sm, av

    def raw_sums(self, kind: int, X, cand, shard=None):
        """Exact fixed-point pair sums (list of Fixed).  shard=(rank, world) computes one shard
        without the collective; None = this context's rank/world, all-reduced."""
        Xd = _samples(X)
        cb, cp = _dbuf(cand)
        d = Xd.shape[0]
        nc = cb.size if kind in (SUM_PSI4, SUM_PSI6, SUM_PSI8, SUM_LSCV_h) else cb.reshape(-1, d * (d + 1) // 2).shape[0]
        nout = nc if kind in (SUM_PSI4, SUM_PSI6, SUM_PSI8) else 2 * nc
        out = (Fixed * nout)()
        sr, sw = (0, 0) if shard is None else shard
        self._check(lib().kde_raw_sums(self._h, int(kind), Xd.ptr, Xd.shape[1], d,
                                       cp, nc, int(sr), int(sw), out))
        return list(out)


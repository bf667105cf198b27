"""paper_1202_6168_b200 -- B200-native D-iteration diffusion sweep (arXiv 1202.6168).

Thin ctypes binding over ``libditer.so`` (C ABI in ``include/diter.h``): the
functions below have the C names and only marshal arguments; every step of the
path runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library is missing or no CUDA device is present, the calls raise.

    ctx = di_create(n, col_ptr, row_idx, values=None, b=None, d=0.85, options=None)
    di_run(ctx, 1e-9)
    H = di_get_history(ctx)
    r = di_get_residual(ctx)
    di_destroy(ctx)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DITER_LIB: another build of this library (A/B experiments, scripts/build_variant.py)
LIB_PATH = os.environ.get("DITER_LIB") or os.path.join(_HERE, "libditer.so")

DI_OK, DI_ERR_INVALID_ARG, DI_ERR_CONTRACTION, DI_ERR_OOM, DI_ERR_CUDA, DI_ERR_NCCL, \
    DI_ERR_NOT_CONVERGED, DI_ERR_STATE, DI_ERR_UNSUPPORTED = range(9)
DI_POLICY_GEOM, DI_POLICY_HYBRID = 0, 1
DI_EXCHANGE_SYNC, DI_EXCHANGE_ASYNC, DI_EXCHANGE_P2P = 0, 1, 2
DI_KEY_RAW, DI_KEY_EDGE, DI_KEY_PAPER = 0, 1, 2
DI_REMOTE_PER_DIFFUSION, DI_REMOTE_INCREMENT, DI_REMOTE_RECEIVER = 0, 1, 2

STATUS_NAMES = {0: "DI_OK", 1: "DI_ERR_INVALID_ARG", 2: "DI_ERR_CONTRACTION", 3: "DI_ERR_OOM",
                4: "DI_ERR_CUDA", 5: "DI_ERR_NCCL", 6: "DI_ERR_NOT_CONVERGED", 7: "DI_ERR_STATE",
                8: "DI_ERR_UNSUPPORTED"}

# every symbol include/diter.h declares (checked by tests/test_abi.py)
EXPORTS = ["di_default_options", "di_struct_size", "di_create", "di_create_dist", "di_get_unique_id", "di_reset",
           "di_set_state", "di_set_profile", "di_run",
           "di_get_history", "di_get_fluid", "di_get_history_device", "di_get_fluid_device",
           "di_get_pagerank", "di_get_pagerank_device", "di_rebalance", "di_get_bounds",
           "di_get_residual", "di_get_stats", "di_get_pass_log", "di_last_error", "di_destroy",
           "di_csc_from_coo", "di_partition_cb"]


class DiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class di_options(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("check_interval", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("hybrid_frac", ctypes.c_double),
                ("t0", ctypes.c_double), ("max_passes", ctypes.c_int64),
                ("exchange_mode", ctypes.c_int32), ("device", ctypes.c_int32),
                ("scatter_kernel", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("pass_kernel", ctypes.c_int32), ("hot_window", ctypes.c_int32),
                ("scatter_run", ctypes.c_int32), ("scatter_stripes", ctypes.c_int32),
                ("far_push", ctypes.c_int32), ("far_warm_log2", ctypes.c_int32),
                ("select_key", ctypes.c_int32), ("remote_push", ctypes.c_int32),
                ("receive_rescale", ctypes.c_int32), ("adapt_rounds", ctypes.c_int32),
                ("l2_persist", ctypes.c_int32), ("p2p_sleep", ctypes.c_int32),
                ("far_defer", ctypes.c_int32), ("sweep", ctypes.c_int32),
                ("key_offset", ctypes.c_int32)]


class di_pass_log(ctypes.Structure):
    _fields_ = [("pass_", ctypes.c_int64), ("T", ctypes.c_double), ("r", ctypes.c_double),
                ("frontier", ctypes.c_int64), ("edges", ctypes.c_int64),
                ("dangling", ctypes.c_int64), ("bin_low", ctypes.c_int64),
                ("bin_mid", ctypes.c_int64), ("bin_hub", ctypes.c_int64),
                ("t_select_us", ctypes.c_double), ("t_scatter_us", ctypes.c_double)]


class di_stats(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int64), ("edges", ctypes.c_int64), ("nodes", ctypes.c_int64),
                ("residual", ctypes.c_double), ("threshold", ctypes.c_double),
                ("run_ms", ctypes.c_double), ("run_ms_total", ctypes.c_double),
                ("alg_bytes", ctypes.c_int64), ("exchanged_bytes", ctypes.c_int64),
                ("exchanges", ctypes.c_int64), ("n_local", ctypes.c_int64),
                ("nnz_local", ctypes.c_int64), ("graph_launches", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("kt_select_ms", ctypes.c_double),
                ("kt_scatter_ms", ctypes.c_double), ("kt_finalize_ms", ctypes.c_double),
                ("kt_passes", ctypes.c_int64), ("scatter_bytes", ctypes.c_int64),
                ("remote_pushes", ctypes.c_int64), ("rebalances", ctypes.c_int64),
                ("l2_window_bytes", ctypes.c_int64), ("l2_window_row", ctypes.c_int64),
                ("dangling", ctypes.c_int64), ("run_kernel_launches", ctypes.c_int64),
                ("collectives", ctypes.c_int64), ("confirms", ctypes.c_int64),
                ("exchange_bytes_resident", ctypes.c_int64), ("sleep_rounds", ctypes.c_int64),
                ("far_flushes", ctypes.c_int64), ("far_edges", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load_library() -> ctypes.CDLL:
    """Load libditer.so (built by __graft_entry__.build() / paper_1202_6168_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1202_6168_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    st = ctypes.c_int
    sig = {
        "di_default_options": (None, [ctypes.POINTER(di_options)]),
        "di_struct_size": (ctypes.c_size_t, [i32]),
        "di_create": (st, [ctypes.POINTER(vp), i64, vp, vp, vp, vp, f64, ctypes.POINTER(di_options)]),
        "di_create_dist": (st, [ctypes.POINTER(vp), i32, i32, vp, vp, i64, vp, vp, vp, vp, f64,
                                ctypes.POINTER(di_options)]),
        "di_get_unique_id": (st, [vp]),
        "di_reset": (st, [vp]),
        "di_set_state": (st, [vp, vp, vp]),
        "di_set_profile": (st, [vp, i32]),
        "di_run": (st, [vp, f64]),
        "di_get_history": (st, [vp, vp]),
        "di_get_fluid": (st, [vp, vp]),
        "di_get_history_device": (st, [vp, vp]),
        "di_get_pagerank": (st, [vp, vp]),
        "di_rebalance": (st, [vp, vp]),
        "di_get_bounds": (st, [vp, vp]),
        "di_get_pagerank_device": (st, [vp, vp]),
        "di_get_fluid_device": (st, [vp, vp]),
        "di_get_residual": (st, [vp, ctypes.POINTER(f64)]),
        "di_get_stats": (st, [vp, ctypes.POINTER(di_stats)]),
        "di_get_pass_log": (st, [vp, i64, i64, vp, ctypes.POINTER(i64)]),
        "di_last_error": (ctypes.c_char_p, [vp]),
        "di_destroy": (None, [vp]),
        "di_csc_from_coo": (st, [i64, i64, vp, vp, vp, vp, ctypes.POINTER(i64)]),
        "di_partition_cb": (st, [i64, vp, i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)           # a library missing a declared entry point fails here
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int, ctx=None):
    if status != DI_OK:
        msg = load_library().di_last_error(ctx)
        raise DiError(status, msg.decode() if msg else "")


def _arr(a, dtype):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _hostptr(a, dtype):
    """numpy array -> (keepalive, pointer); torch CPU tensors (pinned or not) pass through."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        if a.is_cuda:
            raise TypeError("di_create takes HOST arrays (the library copies them)")
        return a, ctypes.c_void_p(a.data_ptr())
    arr = _arr(a, dtype)
    return arr, _p(arr)


def default_options(**kw) -> di_options:
    o = di_options()
    load_library().di_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(k)
        setattr(o, k, v)
    return o


class Context:
    """Owning handle of a di_ctx*; the functions below take it as first argument."""

    def __init__(self, handle: ctypes.c_void_p, n_local: int):
        self.handle = handle
        self.n_local = n_local

    def __del__(self):
        try:
            if self.handle:
                di_destroy(self)
        except Exception:
            pass


def di_create(n, col_ptr, row_idx, values=None, b=None, d=0.85, options=None) -> Context:
    lib = load_library()
    kc, pc = _hostptr(col_ptr, np.int64)
    kr, pr = _hostptr(row_idx, np.int32)
    kv, pv = _hostptr(values, np.float64)
    kb, pb = _hostptr(b, np.float64)
    h = ctypes.c_void_p()
    opt = options if options is not None else default_options()
    s = lib.di_create(ctypes.byref(h), int(n), pc, pr, pv, pb, float(d), ctypes.byref(opt))
    _check(s)
    return Context(h, int(n))


def di_create_dist(rank, world, comm_id: bytes, bounds, n_global, col_ptr_local, row_idx_local,
                   values_local=None, b_local=None, d=0.85, options=None) -> Context:
    lib = load_library()
    bnd = _arr(bounds, np.int64)
    kc, pc = _hostptr(col_ptr_local, np.int64)
    kr, pr = _hostptr(row_idx_local, np.int32)
    kv, pv = _hostptr(values_local, np.float64)
    kb, pb = _hostptr(b_local, np.float64)
    idbuf = ctypes.create_string_buffer(bytes(comm_id), 128)
    h = ctypes.c_void_p()
    opt = options if options is not None else default_options()
    s = lib.di_create_dist(ctypes.byref(h), int(rank), int(world), idbuf, _p(bnd), int(n_global),
                           pc, pr, pv, pb, float(d), ctypes.byref(opt))
    _check(s)
    ctx = Context(h, int(bnd[rank + 1] - bnd[rank]))
    ctx.world = int(world)
    return ctx


def di_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().di_get_unique_id(buf))
    return buf.raw


def di_run(ctx: Context, residual_target: float, raise_on_not_converged: bool = True) -> int:
    s = load_library().di_run(ctx.handle, float(residual_target))
    if getattr(ctx, "world", 1) > 1:          # options.adapt_rounds may move ownership
        ctx.n_local = int(di_get_stats(ctx)["n_local"])
    if s == DI_ERR_NOT_CONVERGED and not raise_on_not_converged:
        return s
    _check(s, ctx.handle)
    return s


def di_reset(ctx: Context):
    _check(load_library().di_reset(ctx.handle), ctx.handle)


def di_set_state(ctx: Context, F, H):
    """Load (F, H) (n_local float64 each) and restart the schedule from them (include/diter.h)."""
    kf, pf = _hostptr(F, np.float64)
    kh, ph = _hostptr(H, np.float64)
    if len(kf) != ctx.n_local or len(kh) != ctx.n_local:
        raise ValueError(f"F and H must hold n_local = {ctx.n_local} values")
    _check(load_library().di_set_state(ctx.handle, pf, ph), ctx.handle)


def di_set_profile(ctx: Context, on: bool):
    _check(load_library().di_set_profile(ctx.handle, 1 if on else 0), ctx.handle)


def _get_vec(fn, ctx: Context, out=None):
    if out is None:
        out = np.empty(ctx.n_local, dtype=np.float64)
    if hasattr(out, "data_ptr"):
        ptr = ctypes.c_void_p(out.data_ptr())
    else:
        assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == ctx.n_local
        ptr = _p(out)
    _check(fn(ctx.handle, ptr), ctx.handle)
    return out


def di_get_history(ctx: Context, out=None):
    return _get_vec(load_library().di_get_history, ctx, out)


def di_get_fluid(ctx: Context, out=None):
    return _get_vec(load_library().di_get_fluid, ctx, out)


def di_get_history_device(ctx: Context, out):
    """out: a CUDA tensor (torch) of n_local float64 on the context's device."""
    return _get_vec(load_library().di_get_history_device, ctx, out)


def di_get_fluid_device(ctx: Context, out):
    return _get_vec(load_library().di_get_fluid_device, ctx, out)


def di_get_pagerank(ctx: Context, out=None):
    """Completed PageRank H / |H|_1."""
    return _get_vec(load_library().di_get_pagerank, ctx, out)


def di_get_pagerank_device(ctx: Context, out):
    return _get_vec(load_library().di_get_pagerank_device, ctx, out)


def di_rebalance(ctx: Context, new_bounds):
    """Collective: move ownership to new_bounds (world + 1 int64, same on every rank)."""
    nb = np.ascontiguousarray(new_bounds, dtype=np.int64)
    _check(load_library().di_rebalance(ctx.handle, _p(nb)), ctx.handle)
    ctx.n_local = int(di_get_stats(ctx)["n_local"])


def di_get_bounds(ctx: Context):
    out = np.zeros(max(2, getattr(ctx, "world", 1) + 1), dtype=np.int64)
    _check(load_library().di_get_bounds(ctx.handle, _p(out)), ctx.handle)
    return out


def di_get_residual(ctx: Context) -> float:
    r = ctypes.c_double()
    _check(load_library().di_get_residual(ctx.handle, ctypes.byref(r)), ctx.handle)
    return r.value


def di_get_stats(ctx: Context) -> dict:
    s = di_stats()
    _check(load_library().di_get_stats(ctx.handle, ctypes.byref(s)), ctx.handle)
    return s.as_dict()


def di_get_pass_log(ctx: Context, first: int = 0, count: int | None = None) -> np.ndarray:
    """Pass records as a structured numpy array (fields of di_pass_log)."""
    if count is None:
        count = di_get_stats(ctx)["passes"] - first
    count = max(0, int(count))
    buf = (di_pass_log * max(count, 1))()
    got = ctypes.c_int64()
    _check(load_library().di_get_pass_log(ctx.handle, int(first), count, buf, ctypes.byref(got)),
           ctx.handle)
    dt = np.dtype([("pass", np.int64), ("T", np.float64), ("r", np.float64), ("frontier", np.int64),
                   ("edges", np.int64), ("dangling", np.int64), ("bin_low", np.int64),
                   ("bin_mid", np.int64), ("bin_hub", np.int64), ("t_select_us", np.float64),
                   ("t_scatter_us", np.float64)])
    arr = np.frombuffer(bytes(buf), dtype=dt, count=max(count, 1))[: got.value].copy()
    return arr


def di_last_error(ctx: Context | None = None) -> str:
    m = load_library().di_last_error(ctx.handle if ctx else None)
    return m.decode() if m else ""


def di_destroy(ctx: Context):
    if ctx.handle:
        load_library().di_destroy(ctx.handle)
        ctx.handle = None


def di_csc_from_coo(n, src, dst):
    """GPU COO -> CSC (sort, dedup, scan); returns (col_ptr int64[n+1], row_idx int32[nnz])."""
    ks, ps = _hostptr(src, np.int32)
    kd, pd = _hostptr(dst, np.int32)
    m = len(src)
    col_ptr = np.empty(int(n) + 1, dtype=np.int64)
    row_idx = np.empty(max(m, 1), dtype=np.int32)
    nnz = ctypes.c_int64()
    _check(load_library().di_csc_from_coo(int(n), m, ps, pd, _p(col_ptr), _p(row_idx),
                                          ctypes.byref(nnz)))
    return col_ptr, row_idx[: nnz.value]


def di_partition_cb(cost_prefix, K: int):
    cp = _arr(cost_prefix, np.int64)
    b = np.empty(int(K) + 1, dtype=np.int64)
    _check(load_library().di_partition_cb(len(cp) - 1, _p(cp), int(K), _p(b)))
    return b


def solve(n, col_ptr, row_idx, target, values=None, b=None, d=0.85, **opts):
    """Convenience: create, run to |F|_1 < target, return (H, stats, log)."""
    ctx = di_create(n, col_ptr, row_idx, values, b, d, default_options(**opts))
    try:
        di_run(ctx, target)
        return di_get_history(ctx), di_get_stats(ctx), di_get_pass_log(ctx)
    finally:
        di_destroy(ctx)

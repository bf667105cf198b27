"""CPU oracle of the D-iteration diffusion sweep (arXiv 1202.6168).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1202_6168_b200``) never imports it and
shares no code with it.  See ``oracle.c`` for the citations of every function.

Thin ctypes marshalling over ``liboracle.so`` (plain single-threaded C, fp64).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

GEOM, HYBRID = 0, 1
KEY_RAW, KEY_EDGE, KEY_PAPER = 0, 1, 2
OK, ERR_ARG, ERR_OOM, ERR_NOT_CONVERGED, ERR_SINGULAR = 0, 1, 2, 3, 4


class PassLog(ctypes.Structure):
    _fields_ = [("pass_", ctypes.c_int64), ("T", ctypes.c_double), ("r", ctypes.c_double),
                ("frontier", ctypes.c_int64), ("edges", ctypes.c_int64),
                ("dangling", ctypes.c_int64)]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    hdr = os.path.join(_HERE, "oracle.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-std=c11", "-Wall", "-o", _SO, src, "-lm"], cwd=_HERE)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.orc_csc_from_coo.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        lib.orc_partition_uniform.argtypes = [i64, i32, vp]
        lib.orc_partition_cb.argtypes = [i64, vp, i32, vp]
        lib.orc_diffuse_node.argtypes = [i64, vp, vp, vp, f64, i64, vp, vp]
        lib.orc_diffuse_node.restype = i64
        lib.orc_l1.argtypes = [i64, vp]
        lib.orc_l1.restype = f64
        lib.orc_init.argtypes = [i64, vp, f64, vp, vp]
        lib.orc_init.restype = f64
        lib.orc_dit_snapshot.argtypes = [i64, vp, vp, vp, f64, f64, i32, f64, f64, i64,
                                         vp, vp, vp, vp, vp, i64, vp]
        lib.orc_key_weights.argtypes = [i64, vp, vp, i32, vp]
        lib.orc_init_key.argtypes = [i64, vp, f64, vp, vp, vp]
        lib.orc_init_key.restype = f64
        lib.orc_dit_snapshot_key.argtypes = [i64, vp, vp, vp, f64, f64, i32, f64, f64, i64, vp,
                                             vp, vp, vp, vp, vp, i64, vp]
        lib.orc_dit_sequential.argtypes = [i64, vp, vp, vp, f64, f64, f64, i64, vp, vp, vp, vp]
        lib.orc_jacobi.argtypes = [i64, vp, vp, vp, f64, vp, f64, i64, vp, vp]
        lib.orc_dense_solve.argtypes = [i64, vp, vp, vp, f64, vp, vp]
        lib.orc_completed_pagerank_dense.argtypes = [i64, vp, vp, f64, vp]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------------ graph ---

def csc_from_coo(n: int, src, dst):
    """COO (src -> dst) to CSC: counting sort by source, rows ascending, dedup."""
    src = _c(src, np.int32)
    dst = _c(dst, np.int32)
    m = len(src)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    row_idx = np.empty(max(m, 1), dtype=np.int32)
    nnz = ctypes.c_int64(0)
    rc = _L().orc_csc_from_coo(n, m, _p(src), _p(dst), _p(col_ptr), _p(row_idx), ctypes.byref(nnz))
    if rc:
        raise ValueError(f"orc_csc_from_coo rc={rc}")
    return col_ptr, row_idx[: nnz.value].copy()


def partition_uniform(n: int, K: int):
    b = np.zeros(K + 1, dtype=np.int64)
    if _L().orc_partition_uniform(n, K, _p(b)):
        raise ValueError("bad partition args")
    return b


def partition_cb(cost_prefix, K: int):
    """Cost-balanced contiguous ranges from an int64 prefix sum of per-node cost."""
    cp = _c(cost_prefix, np.int64)
    n = len(cp) - 1
    b = np.zeros(K + 1, dtype=np.int64)
    if _L().orc_partition_cb(n, _p(cp), K, _p(b)):
        raise ValueError("bad partition args")
    return b


# --------------------------------------------------------------- iteration ---

@dataclass
class State:
    """(F, H, T, pass) of a D-iteration run plus its per-pass log."""
    F: np.ndarray
    H: np.ndarray
    T: float
    passes: int = 0
    edges: int = 0
    log: list = field(default_factory=list)


def key_weights(n, col_ptr, row_idx, key: int):
    """fp32 selection-key weights w_i (orc_key_weights)."""
    w = np.empty(int(n), dtype=np.float32)
    cp = _c(col_ptr, np.int64)
    ri = _c(row_idx, np.int32) if len(row_idx) else np.zeros(1, np.int32)
    if _L().orc_key_weights(int(n), _p(cp), _p(ri), int(key), _p(w)):
        raise ValueError("bad key args")
    return w


class Problem:
    """Marshalled (P, B, d): CSC column j = out-edges of j.  `key`
    selects the selection key of init/snapshot/solve (KEY_RAW default)."""

    def __init__(self, n, col_ptr, row_idx, values=None, b=None, d=0.85, key: int = KEY_RAW):
        self.n = int(n)
        self.col_ptr = _c(col_ptr, np.int64)
        self.row_idx = _c(row_idx, np.int32) if len(row_idx) else np.zeros(1, np.int32)
        self.values = _c(values, np.float64)
        self.d = float(d)
        self.b = _c(b, np.float64) if b is not None else np.full(self.n, (1.0 - self.d) / self.n)
        self.key = int(key)
        self.kw = None if self.key == KEY_RAW else key_weights(self.n, self.col_ptr, self.row_idx, self.key)

    def _args(self):
        return (self.n, _p(self.col_ptr), _p(self.row_idx), _p(self.values), self.d)

    def init(self, alpha: float = 1.5) -> State:
        F = np.empty(self.n)
        H = np.empty(self.n)
        T = _L().orc_init_key(self.n, _p(self.b), alpha, _p(self.kw), _p(F), _p(H))
        return State(F, H, T)

    def snapshot(self, st: State, target: float, policy: int = HYBRID, alpha: float = 1.5,
                 hybrid_frac: float = 0.05, max_passes: int = 1_000_000) -> int:
        """Run snapshot passes until |F|_1 < target (or max_passes); returns status."""
        cap = max(0, min(max_passes, 1_000_000))
        log = (PassLog * max(cap, 1))()
        T = ctypes.c_double(st.T)
        p0 = st.passes
        p = ctypes.c_int64(0)              # log indices relative to this call
        e = ctypes.c_int64(st.edges)
        n, cpp, rip, vp, d = self._args()
        rc = _L().orc_dit_snapshot_key(n, cpp, rip, vp, d, target, policy, alpha, hybrid_frac,
                                       max_passes, _p(self.kw), _p(st.F), _p(st.H), ctypes.byref(T),
                                       ctypes.byref(p), log, cap, ctypes.byref(e))
        for k in range(min(p.value, cap)):
            L = log[k]
            st.log.append((p0 + k, L.T, L.r, L.frontier, L.edges, L.dangling))
        st.T = T.value
        st.passes = p0 + p.value
        st.edges = e.value
        return rc

    def sequential(self, st: State, target: float, alpha: float = 1.5,
                   max_cycles: int = 10_000_000) -> int:
        T = ctypes.c_double(st.T)
        ops = ctypes.c_int64(st.edges)
        n, cpp, rip, vp, d = self._args()
        rc = _L().orc_dit_sequential(n, cpp, rip, vp, d, target, alpha, max_cycles,
                                     _p(st.F), _p(st.H), ctypes.byref(T), ctypes.byref(ops))
        st.T = T.value
        st.edges = ops.value
        return rc

    def diffuse_node(self, st: State, i: int) -> int:
        n, cpp, rip, vp, d = self._args()
        return _L().orc_diffuse_node(n, cpp, rip, vp, d, i, _p(st.F), _p(st.H))

    def jacobi(self, tol: float, max_iter: int = 100_000):
        X = np.empty(self.n)
        it = ctypes.c_int64(0)
        n, cpp, rip, vp, d = self._args()
        rc = _L().orc_jacobi(n, cpp, rip, vp, d, _p(self.b), tol, max_iter, _p(X), ctypes.byref(it))
        if rc:
            raise RuntimeError(f"orc_jacobi rc={rc}")
        return X, it.value

    def dense_solve(self):
        X = np.empty(self.n)
        n, cpp, rip, vp, d = self._args()
        rc = _L().orc_dense_solve(n, cpp, rip, vp, d, _p(self.b), _p(X))
        if rc:
            raise RuntimeError(f"orc_dense_solve rc={rc}")
        return X

    def completed_pagerank_dense(self):
        """X' of the completed (dangling -> 1/N) PageRank system, dense."""
        X = np.empty(self.n)
        rc = _L().orc_completed_pagerank_dense(self.n, _p(self.col_ptr), _p(self.row_idx), self.d, _p(X))
        if rc:
            raise RuntimeError(f"orc_completed_pagerank_dense rc={rc}")
        return X

    def solve(self, target: float, policy: int = HYBRID, alpha: float = 1.5,
              hybrid_frac: float = 0.05, max_passes: int = 1_000_000) -> State:
        st = self.init(alpha)
        rc = self.snapshot(st, target, policy, alpha, hybrid_frac, max_passes)
        if rc not in (OK,):
            raise RuntimeError(f"oracle did not converge rc={rc}")
        return st


def l1(v) -> float:
    v = _c(v, np.float64)
    return float(_L().orc_l1(len(v), _p(v)))

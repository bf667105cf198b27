"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: it only draws graphs / right-hand
sides from the recipes of BASELINE.json configs[0..4].
The CSC arrays it returns for the "uniform", "web" and "signed" kinds are
generated column by column (the recipe draws each node's out-edges), so no
COO->CSC construction happens here; R-MAT returns raw COO (duplicates kept),
whose CSC construction is method-side (oracle.csc_from_coo vs di_csc_from_coo).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdigen.so")

DG_UNIFORM, DG_WEB, DG_RMAT, DG_SIGNED = 1, 2, 3, 5


class _Params(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("_pad0", ctypes.c_int32),
        ("n", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("deg_lo", ctypes.c_int32), ("deg_hi", ctypes.c_int32),
        ("x_min", ctypes.c_double), ("p_dangling", ctypes.c_double), ("p_local", ctypes.c_double),
        ("window", ctypes.c_int32), ("max_deg", ctypes.c_int32),
        ("nnz_per_col", ctypes.c_int32), ("_pad1", ctypes.c_int32),
        ("col_abs_sum", ctypes.c_double),
        ("scale", ctypes.c_int32), ("edge_factor", ctypes.c_int32),
        ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "digen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "digen.h"))):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-Wall", "-o", _SO, src, "-lm"], cwd=_HERE)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.POINTER(_Params)
        vp = ctypes.c_void_p
        lib.dg_csc_count.argtypes = [P, vp]
        lib.dg_csc_fill.argtypes = [P, vp, vp, vp]
        lib.dg_b_signed.argtypes = [P, vp]
        lib.dg_rmat_edges.argtypes = [P]
        lib.dg_rmat_edges.restype = ctypes.c_int64
        lib.dg_rmat_fill.argtypes = [P, vp, vp]
        lib.dg_validate.argtypes = [P]
        lib.dg_num_threads.restype = ctypes.c_int
        lib.dg_set_threads.argtypes = [ctypes.c_int]
        omp = os.environ.get("DIGEN_THREADS")
        if omp:
            lib.dg_set_threads(int(omp))
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Problem:
    """One synthetic instance of X = P X + B (CSC, column j = out-edges of j)."""
    name: str
    n: int
    col_ptr: np.ndarray            # int64[n+1]
    row_idx: np.ndarray            # int32[nnz]
    values: np.ndarray | None      # float64[nnz] (signed mode) or None (PageRank)
    b: np.ndarray | None           # float64[n] or None (PageRank default (1-d)/n)
    d: float
    stop: float                    # metric residual target |F|_1 < stop (BASELINE.json)
    parity_stop: float             # tighter residual target for parity

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def b_vector(self) -> np.ndarray:
        if self.b is not None:
            return self.b
        return np.full(self.n, (1.0 - self.d) / self.n)

    def stats(self) -> dict:
        deg = np.diff(self.col_ptr)
        return {"n": self.n, "edges": self.nnz, "avg_degree": self.nnz / self.n,
                "dangling": int((deg == 0).sum()), "dangling_pct": float((deg == 0).mean() * 100),
                "max_deg": int(deg.max()) if self.n else 0}


def _csc(p: _Params, with_vals: bool):
    lib = _L()
    n = p.n
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    rc = lib.dg_csc_count(ctypes.byref(p), _ptr(col_ptr))
    if rc:
        raise ValueError(f"dg_csc_count failed rc={rc}")
    nnz = int(col_ptr[-1])
    row_idx = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64) if with_vals else None
    rc = lib.dg_csc_fill(ctypes.byref(p), _ptr(col_ptr), _ptr(row_idx), _ptr(vals))
    if rc:
        raise ValueError(f"dg_csc_fill failed rc={rc}")
    return col_ptr, row_idx, vals


def uniform_graph(n: int = 1000, seed: int = 1, deg_lo: int = 1, deg_hi: int = 10):
    """configs[0]: out-degree U{deg_lo..deg_hi}, distinct uniform destinations, no self-loops."""
    p = _Params(kind=DG_UNIFORM, n=n, seed=seed, deg_lo=deg_lo, deg_hi=min(deg_hi, n - 1))
    return _csc(p, False)[:2]


# x_min of the Pareto-floor degree law, chosen by running this generator at full N
# so that post-dedup L matches BASELINE.json: ~7.0e6 at N=1e6, ~1.6e9 at N=1e8
# (x_min=1.48 gave 7.12e6, x_min=3.53 gave 1.627e9 with seed 1).
XMIN_C2 = 1.455
XMIN_C4 = 3.47


def web_graph(n: int, seed: int = 1, x_min: float = XMIN_C2, p_dangling: float = 0.15,
              p_local: float = 0.7, window: int = 1000, max_deg: int = 5000):
    """configs[1]/[3]: Zipf-tailed out-degree, 15% dangling, 70% local / 30% Zipf-over-id."""
    p = _Params(kind=DG_WEB, n=n, seed=seed, x_min=x_min, p_dangling=p_dangling,
                p_local=p_local, window=window, max_deg=min(max_deg, n - 1))
    return _csc(p, False)[:2]


def rmat_coo(scale: int, seed: int = 1, edge_factor: int = 16, a=0.57, b=0.19, c=0.19):
    """configs[2]: raw R-MAT COO samples (src -> dst), ids permuted, duplicates kept."""
    lib = _L()
    p = _Params(kind=DG_RMAT, n=1 << scale, seed=seed, scale=scale, edge_factor=edge_factor,
                a=a, b=b, c=c)
    m = lib.dg_rmat_edges(ctypes.byref(p))
    if m < 0:
        raise ValueError("bad rmat params")
    src = np.empty(m, dtype=np.int32)
    dst = np.empty(m, dtype=np.int32)
    rc = lib.dg_rmat_fill(ctypes.byref(p), _ptr(src), _ptr(dst))
    if rc:
        raise ValueError(f"dg_rmat_fill rc={rc}")
    return src, dst


def signed_system(n: int, seed: int = 1, nnz_per_col: int = 20, col_abs_sum: float = 0.9):
    """configs[4]: 20 distinct uniform rows per column, U[-1,1] values scaled to |col|_1 = 0.9, B ~ U[-1,1]."""
    lib = _L()
    p = _Params(kind=DG_SIGNED, n=n, seed=seed, nnz_per_col=min(nnz_per_col, n),
                col_abs_sum=col_abs_sum)
    col_ptr, row_idx, vals = _csc(p, True)
    b = np.empty(n, dtype=np.float64)
    rc = lib.dg_b_signed(ctypes.byref(p), _ptr(b))
    if rc:
        raise ValueError(f"dg_b_signed rc={rc}")
    return col_ptr, row_idx, vals, b


def num_threads() -> int:
    return int(_L().dg_num_threads())


# ------------------------------------------------------------------ configs --
# BASELINE.json configs[0..4] -> C1..C5.  The metric stop targets are the ones
# BASELINE.json states; the parity stops are SURVEY §8c-Q1's readings.

def config(name: str, seed: int = 1, n: int | None = None, scale: int | None = None) -> Problem:
    """Build config C1..C5 (optionally shrunk: n= for C1/C2/C4/C5, scale= for C3).

    C3 is returned with col_ptr/row_idx = None; its CSC must be built from the
    COO (method side) -- use rmat_coo() and a CSC builder.
    """
    d = 0.85
    if name == "C1":
        n = n or 1000
        cp, ri = uniform_graph(n, seed)
        return Problem("C1", n, cp, ri, None, None, d, 1e-12, 1e-12)
    if name == "C2":
        n = n or 1_000_000
        cp, ri = web_graph(n, seed, XMIN_C2)
        return Problem("C2", n, cp, ri, None, None, d, 1e-9, 1e-9 * (1 - d))
    if name == "C4":
        n = n or 100_000_000
        cp, ri = web_graph(n, seed, XMIN_C4)
        return Problem("C4", n, cp, ri, None, None, d, 1e-9, 1e-9 * (1 - d))
    if name == "C5":
        n = n or 1_000_000
        cp, ri, v, b = signed_system(n, seed)
        bn = float(np.abs(b).sum())
        return Problem("C5", n, cp, ri, v, b, 0.9, 1e-9 * bn, 5e-10 * bn)
    if name == "C3":
        scale = scale or 24
        return Problem("C3", 1 << scale, None, None, None, None, d, 1e-9, 1e-9 * (1 - d))
    raise KeyError(name)

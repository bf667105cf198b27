"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration.

configs[3] (C4: N=1e8, 1.6e9 edges) and configs[2] (C3: R-MAT scale 24) are too
large for the oracle's fixed point, so parity is proven through properties that
hold at any size (SURVEY §8c "what pins each part"):

* the exact identity F = B - (I-P)H (App. A.1) checked element by element on a
  sample of rows (random rows, the Zipf-hot prefix, the last rows) by an
  independent numpy in-edge sum over the whole CSC -- with the contraction
  bound it gives ||X - H||_1 <= |F|_1/(1-d), so r < target is parity;
* conservation |F|_1 + (1-d)|H|_1 + d sum_dangling H = |B|_1 (App. A.2);
* |F|_1 from di_get_residual equals the host sum of F; F, H >= 0; the logged
  r_p are non-increasing; the edge total equals the sum of the logged E_p;
* the first passes' frontier sizes against the oracle run on the same input,
  pass by pass (exact up to the first near-tie with T_p, reading R8).
"""
import numpy as np
import pytest

import diter_inputs as gen
import oracle
import paper_1202_6168_b200 as di

pytestmark = pytest.mark.gpu


import bench                 # bench.SCHEDULES: the launch configuration bench.py times


def _bench_opts(cfg):
    # bench.py's launch configuration (profile=1: per-kernel CUDA events in the graph)
    pol, alpha, frac, key = bench.SCHEDULES[cfg]
    return di.default_options(policy=pol, profile=1, alpha=alpha, hybrid_frac=frac, select_key=key)


def _sampled_identity(n, cp, ri, H, F, b, d, rows):
    """max over sampled rows j of |F_j - (B_j - H_j + sum_{i -> j} (d/#out_i) H_i)| / scale_j."""
    lut = np.zeros(n, dtype=bool)
    lut[rows] = True
    deg = np.diff(cp)
    w = np.where(deg > 0, d / np.maximum(deg, 1), 0.0)
    acc = np.zeros(n)
    acc_abs = np.zeros(n)
    nnz = int(cp[-1])
    chunk = 1 << 26
    for e0 in range(0, nnz, chunk):
        r = ri[e0:min(nnz, e0 + chunk)]
        m = np.flatnonzero(lut[r])
        if m.size == 0:
            continue
        col = np.searchsorted(cp, m + e0, side="right") - 1      # column (source) of each edge
        v = w[col] * H[col]
        np.add.at(acc, r[m], v)
        np.add.at(acc_abs, r[m], np.abs(v))
    pred = b[rows] - H[rows] + acc[rows]
    scale = np.abs(b[rows]) + np.abs(H[rows]) + acc_abs[rows]
    return float(np.max(np.abs(F[rows] - pred) / scale))


def _full_scale_case(p, cfg, n_oracle_passes):
    n, cp, ri = p.n, p.col_ptr, p.row_idx
    policy, ALPHA, FRAC, key = bench.SCHEDULES[cfg]
    ctx = di.di_create(n, cp, ri, None, None, p.d, _bench_opts(cfg))
    di.di_run(ctx, p.stop)                         # metric target (bench)
    r_metric = di.di_get_residual(ctx)
    di.di_run(ctx, p.parity_stop)                  # resumed to the parity target (reading R1)
    H = di.di_get_history(ctx)
    F = di.di_get_fluid(ctx)
    r = di.di_get_residual(ctx)
    log = di.di_get_pass_log(ctx)
    stats = di.di_get_stats(ctx)
    di.di_destroy(ctx)
    b = np.full(n, (1.0 - p.d) / n)
    bn = 1.0 - p.d
    assert r_metric < p.stop and r < p.parity_stop
    assert r == pytest.approx(np.abs(F).sum(), rel=1e-12)
    assert F.min() >= 0.0 and H.min() >= 0.0
    assert np.all(np.diff(log["r"]) <= 1e-15)
    assert stats["edges"] == int(log["edges"].sum())
    deg = np.diff(cp)
    cons = np.abs(F).sum() + (1 - p.d) * H.sum() + p.d * H[deg == 0].sum()
    assert abs(cons - bn) <= 1e-12 * bn, cons - bn                 # App. A.2
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([rng.integers(0, n, 20000), np.arange(64),
                                     np.arange(n - 64, n), np.argsort(H)[-64:]]))
    ident = _sampled_identity(n, cp, ri, H, F, b, p.d, rows)
    assert ident <= 1e-12, ident                                    # App. A.1, per element
    # bound: ||X - H||_1 <= r / (1 - d) <= 1e-8 |B|_1 (north_star tolerance)
    assert r / (1 - p.d) <= 1e-8 * bn
    # first passes against the oracle on the same input (tie-aware, reading R8)
    P = oracle.Problem(n, cp, ri, None, None, p.d, key=key)
    st = P.init(ALPHA)
    near = []
    for _ in range(n_oracle_passes):
        T = st.T
        a = np.abs(st.F)
        near.append(int((np.abs(a - T) <= 1e-12 * T).sum()))
        P.snapshot(st, p.stop, policy, ALPHA, FRAC, max_passes=1)
    k = n_oracle_passes
    first_tie = next((q for q in range(k) if near[q] > 0), k)
    o = np.array([l[3] for l in st.log[:k]])
    np.testing.assert_array_equal(log["frontier"][:first_tie], o[:first_tie])
    np.testing.assert_array_equal(log["T"][:k], [l[1] for l in st.log[:k]])
    assert np.all(np.abs(log["frontier"][:k] - o) <= 0.05 * o + 2)


def test_c4_full_scale_parity():
    """configs[3]: N=1e8 web-like PageRank, bench's schedule (HYBRID, per-edge key)."""
    p = gen.config("C4", 1)
    _full_scale_case(p, "C4", 3)


def test_c3_full_scale_parity():
    """configs[2]: R-MAT scale 24, CSC built on the GPU (K8), bench's schedule."""
    p = gen.config("C3", 1)
    src, dst = gen.rmat_coo(24, 1)
    p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
    del src, dst
    _full_scale_case(p, "C3", 3)


def test_more_than_2_31_edges():
    """Maximum-size edge case: a web-like graph with nnz > 2^31 (64-bit edge offsets
    through create/validation, hot-window sampling, scatter and hub chunks), in C4's
    launch configuration; the same properties as above (oracle first passes too)."""
    n = 55_000_000
    cp, ri = gen.web_graph(n, 2, 10.0)
    assert cp[-1] > 2 ** 31, cp[-1]
    p = gen.config("C4", 2, n=1000)               # for d, stop, parity_stop only
    p.n, p.col_ptr, p.row_idx = n, cp, ri
    _full_scale_case(p, "C4", 2)


def test_max_nodes_cycle_closed_form():
    """Maximum-size edge case for node ids: n = 2^31 - 1 (the ABI's limit) on the
    directed N-cycle, whose fixed point is X_i = 1/N.  Every pass
    diffuses every node (uniform F), so the solve also streams ~17 GB of F per pass.
    Checks |X - H|_1 <= |F|_1 / (1 - d) against the closed form and that |F|_1 is exact."""
    n = 2 ** 31 - 1
    cp = np.arange(n + 1, dtype=np.int64)
    ri = np.arange(1, n + 1, dtype=np.int64)
    ri[-1] = 0
    ri = ri.astype(np.int32)
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(policy=di.DI_POLICY_GEOM))
    del cp, ri
    target = 1e-6
    di.di_run(ctx, target)
    r = di.di_get_residual(ctx)
    H = di.di_get_history(ctx)
    st = di.di_get_stats(ctx)
    di.di_destroy(ctx)
    assert r < target and st["passes"] > 50
    err = float(np.abs(H - 1.0 / n).sum())
    assert err <= r / 0.15 * (1 + 1e-9), (err, r / 0.15)
    assert H.min() > 0.0 and abs(float(H.sum()) - (1.0 - r / 0.15)) <= 1e-9

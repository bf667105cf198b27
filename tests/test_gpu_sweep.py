"""One-kernel asynchronous sweeps (options.sweep = 1) against the CPU oracle.

A sweep takes and diffuses every node above T_p at once (the paper's cyclic scan
with immediate diffusion), so the pass log is not the
snapshot oracle's; the limit is the same X.  Bars: H within 1e-8 |B|_1
of the oracle's X, the identity F = B - (I-P)H on every row (App. A.1), |F|_1
below the target; on every config kind (web-like with and without the key, R-MAT
with hub columns, signed P, uniform).
"""
import numpy as np
import pytest

import diter_inputs as gen
import paper_1202_6168_b200 as di

from test_gpu_parity import TOL, _check_state, _gpu, _xref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", [0, 1, 2])
@pytest.mark.parametrize("policy", [di.DI_POLICY_GEOM, di.DI_POLICY_HYBRID])
def test_sweep_web(key, policy):
    n = 150_001
    cp, ri = gen.web_graph(n, 2, gen.XMIN_C4)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, sweep=1, select_key=key, policy=policy, alpha=2.0,
                            hybrid_frac=0.5)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)
    assert st["edges"] == log["edges"].sum() and st["passes"] == len(log)


def test_sweep_rmat_hubs():
    """R-MAT scale 16 (columns > 8192 edges go through the hub kernel after the sweep)."""
    src, dst = gen.rmat_coo(16, 1)
    n = 1 << 16
    cp, ri = di.di_csc_from_coo(n, src, dst)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, sweep=1, select_key=1)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)


def _hub_graph(n, seed, hubs):
    """Uniform graph (out-degree 1..10) whose columns `hubs` (col -> #out) are replaced by
    hub columns of distinct random rows: every hub is pushed in 2048-edge chunks, the
    last chunk ragged, some hubs adjacent to each other."""
    cp, ri = gen.uniform_graph(n, seed)
    rng = np.random.default_rng(seed)
    cols = [ri[cp[i]:cp[i + 1]] for i in range(n)]
    for c, deg in hubs.items():
        cols[c] = np.sort(rng.choice(n, size=deg, replace=False)).astype(np.int32)
    lens = np.array([len(x) for x in cols], dtype=np.int64)
    cp2 = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=cp2[1:])
    return cp2, np.concatenate(cols).astype(np.int32)


@pytest.mark.parametrize("signed", [False, True])
def test_sweep_hub_chunks_in_kernel(signed):
    """Hub columns (> 8192 edges) selected in a sweep: their chunks are listed and pushed
    inside the sweep kernel by warps whose spans are done.  Many hubs of ragged chunk counts,
    three solves on one context (di_reset between: the chunk table must come back empty),
    PageRank and signed P; H vs the oracle's X and the identity on every row each time."""
    n = 40_000
    hubs = {0: 30_000, 1: 8_193, 2: 12_288, 5_000: 20_481, 5_001: 9_000, 39_999: 16_384, 20_000: 24_576}
    cp, ri = _hub_graph(n, 11, hubs)
    vals = b = None
    d = 0.85
    if signed:
        rng = np.random.default_rng(5)
        vals = rng.uniform(-1.0, 1.0, size=len(ri))
        deg = np.diff(cp)
        colsum = np.add.reduceat(np.abs(vals), cp[:-1][deg > 0])
        scale = np.zeros(n)
        scale[deg > 0] = 0.9 / colsum
        vals *= np.repeat(scale, deg)
        b = rng.uniform(-1.0, 1.0, size=n)
        d = 0.9
    X, P, bn = _xref(n, cp, ri, vals, b, d)
    target = (5e-10 if signed else 1e-9) * bn
    ctx = di.di_create(n, cp, ri, vals, b, d, di.default_options(sweep=1, policy=di.DI_POLICY_GEOM))
    try:
        for _ in range(3):
            di.di_reset(ctx)
            di.di_run(ctx, target)
            H = di.di_get_history(ctx)
            F = di.di_get_fluid(ctx)
            r = di.di_get_residual(ctx)
            assert di.di_get_pass_log(ctx)["bin_hub"].sum() >= len(hubs)     # every hub diffused
            assert np.abs(H - X).sum() <= TOL * bn
            _check_state(n, cp, ri, vals, b, d, H, F, r, target)
    finally:
        di.di_destroy(ctx)


def test_sweep_signed_and_small():
    n = 30_000
    cp, ri, v, b = gen.signed_system(n, 2)
    X, P, bn = _xref(n, cp, ri, v, b, 0.9)
    target = 5e-10 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, vals=v, b=b, d=0.9, sweep=1)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, v, b, 0.9, H, F, r, target)
    for n in (1, 33, 257, 1000):
        cp, ri = gen.uniform_graph(max(n, 2), 3)
        n = max(n, 2)
        X, P, bn = _xref(n, cp, ri)
        H, F, log, r, st = _gpu(n, cp, ri, 1e-12, sweep=1)
        assert np.abs(H - X).sum() <= TOL * bn
        _check_state(n, cp, ri, None, None, 0.85, H, F, r, 1e-12)


def test_sweep_resume_reset_state():
    n = 60_000
    cp, ri = gen.web_graph(n, 4, gen.XMIN_C4)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(sweep=1, select_key=1))
    di.di_run(ctx, 1e-6)
    _check_state(n, cp, ri, None, None, 0.85, di.di_get_history(ctx), di.di_get_fluid(ctx),
                 di.di_get_residual(ctx), 1e-6)
    di.di_run(ctx, target)
    H1 = di.di_get_history(ctx)
    di.di_reset(ctx)
    di.di_run(ctx, target)
    H2, F2, r2 = di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_residual(ctx)
    di.di_destroy(ctx)
    for H in (H1, H2):
        assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H2, F2, r2, target)


def test_sweep_max_passes_and_checkpoint():
    """max_passes stops a sweep run with a consistent state (NOT_CONVERGED, identity on
    every row); di_set_state resumes from a checkpoint to the same X; any
    check_interval (passes per captured graph) gives the same answer."""
    n = 80_000
    cp, ri = gen.web_graph(n, 6, gen.XMIN_C4)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(sweep=1, select_key=1, max_passes=5,
                                                                       check_interval=3))
    s = di.di_run(ctx, target, raise_on_not_converged=False)
    assert s == di.DI_ERR_NOT_CONVERGED
    H, F = di.di_get_history(ctx), di.di_get_fluid(ctx)
    r = di.di_get_residual(ctx)
    assert di.di_get_stats(ctx)["passes"] == 5
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, float("inf"))
    di.di_destroy(ctx)
    for ci in (1, 7, 16):
        ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(sweep=1, select_key=1, check_interval=ci))
        di.di_set_state(ctx, F, H)                     # resume from the checkpoint
        di.di_run(ctx, target)
        H2, F2, r2 = di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_residual(ctx)
        di.di_destroy(ctx)
        assert np.abs(H2 - X).sum() <= TOL * bn
        _check_state(n, cp, ri, None, None, 0.85, H2, F2, r2, target)


def test_sweep_degenerate_graphs():
    """The degenerate cases of the method under sweeps: one node with a self-loop (its own
    push lands in the F_i it just took: X = b / (1 - d)), one dangling node,
    P = 0 (every column dangling: X = B exactly after one sweep), a graph of isolated
    self-loops, and a target already met (no sweep runs)."""
    cp = np.array([0, 1], np.int64)
    ri = np.array([0], np.int32)
    H, F, log, r, _ = _gpu(1, cp, ri, 1e-14, sweep=1)
    assert abs(H[0] - 1.0) <= 1e-14 / 0.15 + 1e-15 and r < 1e-14
    H0, F0, log0, r0, _ = _gpu(1, np.array([0, 0], np.int64), np.zeros(0, np.int32), 1e-30, sweep=1)
    assert H0[0] == pytest.approx(0.15, rel=1e-15) and F0[0] == 0.0 and len(log0) == 1
    n = 1000
    b = np.linspace(0, 1, n)
    H, F, log, r, _ = _gpu(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), 1e-300, b=b, sweep=1)
    np.testing.assert_array_equal(H, b)
    assert r == 0.0 and not F.any()
    n = 777
    cp = np.arange(n + 1, dtype=np.int64)
    ri = np.arange(n, dtype=np.int32)
    H, F, log, r, _ = _gpu(n, cp, ri, 1e-13, sweep=1, select_key=1)
    np.testing.assert_allclose(H, np.full(n, 0.15 / n / 0.15), rtol=1e-10)      # b_i / (1 - d)
    H, F, log, r, st = _gpu(n, cp, ri, 1.0, sweep=1)                          # |B|_1 = 0.15 < 1
    assert st["passes"] == 0 and not H.any() and r == pytest.approx(0.15, rel=1e-12)


@pytest.mark.parametrize("n", [31, 127, 129, 4099, 1_000_003])
def test_sweep_ragged_sizes(n):
    """Sizes around the sweep's 128-node span and 32-node item, and one that spans many
    ticket stripes with a ragged last span, with the bench's stripe / run settings."""
    cp, ri = gen.web_graph(n, 11, window=min(1000, n // 2 or 1), max_deg=min(5000, n - 1))
    X, P, bn = _xref(n, cp, ri)
    H, F, log, r, _ = _gpu(n, cp, ri, 1e-9 * bn, sweep=1, select_key=1, scatter_run=6, scatter_stripes=4)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, 1e-9 * bn)


@pytest.mark.parametrize("c", [0, 8, 64])
def test_sweep_key_offset(c):
    """options.key_offset (reading R27): the sweep's derived per-edge key |F_i| / (#out_i + c).
    Any c is another selection order of the same method: same X, exact identity;
    c = 0 is the default c = 1; a negative value is rejected."""
    n = 150_001
    cp, ri = gen.web_graph(n, 3, gen.XMIN_C4)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, sweep=1, select_key=1, alpha=2.0, hybrid_frac=0.55, key_offset=c)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)
    if c == 0:
        H1, F1, log1, r1, st1 = _gpu(n, cp, ri, target, sweep=1, select_key=1, alpha=2.0, hybrid_frac=0.55, key_offset=1)
        assert abs(st1["passes"] - st["passes"]) <= 3       # asynchronous sweeps: not deterministic
        with pytest.raises(di.DiError):
            di.di_create(n, cp, ri, None, None, 0.85, di.default_options(sweep=1, key_offset=-1))

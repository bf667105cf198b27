"""Far-edge deferral (options.far_defer, defer.cu) against the CPU oracle.

The deferral pushes a column's far edges (|row - src| > 2048) as increments
(H_i - H_old_i) p_ji every far_defer passes -- the paper's increment push,
PAPER.md:227-250 -- so the pass schedule is not the snapshot oracle's and the
frontier logs are not compared (they are, with deferral off, in
test_gpu_parity.py).  What must hold (App. A.1):
H within 1e-8 |B|_1 of the oracle's X, the identity F = B - (I-P)H on every
row after every di_run (nothing left pending), |F|_1 below the target.  The
number of deferred edges is an integer, checked against a numpy count.
"""
import numpy as np
import pytest

import diter_inputs as gen
import paper_1202_6168_b200 as di

from test_gpu_parity import TOL, _check_state, _gpu, _xref

pytestmark = pytest.mark.gpu

NEAR = 2048          # kNear


def _far_count(n, cp, ri):
    """Edges deferred by a context whose F has no L2 persisting window (n < 2^23):
    |row - src| > 2048 and row outside the 2048-row shared-memory hot window, which
    starts at a 1024-aligned row the library picks -- returns the count for every
    candidate start (the test checks membership)."""
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    far = np.abs(ri.astype(np.int64) - src) > NEAR
    rows = ri[far].astype(np.int64)
    tot = int(far.sum())
    blk = np.bincount(rows >> 10, minlength=(n >> 10) + 2)
    starts = range(0, max(1, n - 2048 + 1), 1024)
    return {tot - int(blk[h >> 10] + blk[(h >> 10) + 1]) for h in starts} | (
        {tot - int(((rows >= n - 2048)).sum())} if n > 2048 else {0})


def _web(n, seed=1):
    return gen.web_graph(n, seed, gen.XMIN_C4)


@pytest.mark.parametrize("m", [1, 3, 8, 16])
@pytest.mark.parametrize("key", [0, 1])
def test_defer_matches_oracle(m, key):
    n = 120_000
    cp, ri = _web(n, seed=m)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, far_defer=m, select_key=key, alpha=2.0, hybrid_frac=0.5)
    assert st["far_edges"] in _far_count(n, cp, ri) and st["far_edges"] > 0
    assert st["far_flushes"] >= 1
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)


def test_defer_large_graph_and_default_off():
    """A C4-shaped graph of 2^22 nodes with deferral on; the default leaves it off."""
    n = 1 << 22
    cp, ri = _web(n, seed=5)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, far_defer=4, select_key=1, alpha=2.0, hybrid_frac=0.5)
    assert st["far_edges"] in _far_count(n, cp, ri)
    assert st["far_flushes"] >= 1
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options())
    assert di.di_get_stats(ctx)["far_edges"] == 0
    di.di_destroy(ctx)


def test_defer_resume_reset_state():
    n = 50_000
    cp, ri = _web(n, seed=4)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(far_defer=4))
    di.di_run(ctx, 1e-6)
    # between runs nothing is pending: the identity holds exactly
    _check_state(n, cp, ri, None, None, 0.85, di.di_get_history(ctx), di.di_get_fluid(ctx),
                 di.di_get_residual(ctx), 1e-6)
    di.di_run(ctx, target)
    H1 = di.di_get_history(ctx)
    F1 = di.di_get_fluid(ctx)
    di.di_reset(ctx)
    assert di.di_get_stats(ctx)["far_flushes"] == 0
    di.di_run(ctx, target)
    H2 = di.di_get_history(ctx)
    for H in (H1, H2):
        assert np.abs(H - X).sum() <= TOL * bn
    # checkpoint / resume from the first run's state: H_old restarts at H
    di.di_set_state(ctx, F1, H1)
    di.di_run(ctx, target * 0.1)
    H3, F3, r3 = di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_residual(ctx)
    di.di_destroy(ctx)
    _check_state(n, cp, ri, None, None, 0.85, H3, F3, r3, target * 0.1)


def test_defer_max_passes_keeps_identity():
    """A max_passes stop delivers what is pending before returning NOT_CONVERGED."""
    n = 40_000
    cp, ri = _web(n, seed=6)
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(far_defer=5, max_passes=7,
                                                                       check_interval=4))
    s = di.di_run(ctx, 1e-14, raise_on_not_converged=False)
    assert s == di.DI_ERR_NOT_CONVERGED
    H, F = di.di_get_history(ctx), di.di_get_fluid(ctx)
    r = di.di_get_residual(ctx)
    di.di_destroy(ctx)
    b = np.full(n, 0.15 / n)
    from test_gpu_parity import _pmat
    assert np.abs(F - (b - H + _pmat(n, cp, ri) @ H)).sum() <= 1e-12 * 0.15
    assert r > 1e-14


def test_defer_edge_cases():
    """Every edge far (random rows), dangling columns, duplicates, self-loops."""
    rng = np.random.default_rng(3)
    n = 9000
    cols = []
    for i in range(n):
        if i % 9 == 0:
            cols.append(np.zeros(0, np.int32))
            continue
        c = rng.integers(0, n, size=int(rng.integers(1, 12))).astype(np.int32)
        if i % 4 == 0:
            c = np.concatenate([c, c[:2], [i]]).astype(np.int32)
        cols.append(c)
    deg = np.array([len(c) for c in cols])
    cp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ri = np.concatenate(cols).astype(np.int32)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    for m in (2, 7):
        H, F, log, r, st = _gpu(n, cp, ri, target, far_defer=m)
        assert st["far_edges"] in _far_count(n, cp, ri)
        assert np.abs(H - X).sum() <= TOL * bn
        _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)


def test_defer_off_paths():
    """Signed P, the fused persistent kernel and far_defer = -1 never defer."""
    n = 20_000
    cp, ri, v, b = gen.signed_system(n, 1)
    ctx = di.di_create(n, cp, ri, v, b, 0.9, di.default_options(far_defer=4))
    assert di.di_get_stats(ctx)["far_edges"] == 0
    di.di_destroy(ctx)
    cp, ri = _web(n)
    for o in (dict(far_defer=4, pass_kernel=2), dict(far_defer=-1)):
        ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(**o))
        assert di.di_get_stats(ctx)["far_edges"] == 0
        di.di_destroy(ctx)

"""Near-edge pull (options.near_pull, pull.cu) against the CPU oracle.

A pull pass is the same block pass as a push pass: every edge
of every taken node adds p_ji s_i once; only the summation order changes (reading
R8).  So the bars are the ones of test_gpu_parity.py: H within 1e-8 |B|_1 of the
oracle's X, the identity F = B - (I-P)H on every row, and the pass log equal to
the oracle's at a fixed schedule up to SURVEY §8c-Q8 ties.  The near in-edge
table's size is an integer, checked exactly against a numpy count.
"""
import numpy as np
import pytest

import diter_inputs as gen
import oracle
import paper_1202_6168_b200 as di

from test_gpu_parity import TOL, _check_state, _compare_logs_q8, _gpu, _oracle_passes_with_ties, _xref

pytestmark = pytest.mark.gpu

W = 1024            # kPullW: near iff |row - src| <= W (and #out_src <= 65535)


def _near_count(n, cp, ri):
    deg = np.diff(cp)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    near = np.abs(ri.astype(np.int64) - src) <= W
    near &= np.repeat(deg <= 65535, deg)
    return int(near.sum())


def _web(n, seed=1):
    cp, ri = gen.web_graph(n, seed, gen.XMIN_C4)
    return cp, ri


@pytest.mark.parametrize("n", [40_000, 150_001])
def test_pull_every_pass_matches_oracle(n):
    """Pull forced on every pass (pull_permille = 1): H, identity, table size."""
    cp, ri = _web(n)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    H, F, log, r, st = _gpu(n, cp, ri, target, near_pull=1, pull_permille=1, select_key=1,
                            alpha=2.0, hybrid_frac=0.5)
    assert st["pull_near_edges"] == _near_count(n, cp, ri)
    assert st["pull_passes"] >= len(log) - 3      # the first passes' estimate may be below 1 permille
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)


def test_pull_off_and_auto_agree():
    """near_pull = -1 (push only), auto, and forced: same X, tables only when on."""
    n = 60_000
    cp, ri = _web(n, seed=2)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    for np_opt in (-1, 0, 1):
        H, F, log, r, st = _gpu(n, cp, ri, target, near_pull=np_opt, select_key=1, alpha=2.0, hybrid_frac=0.5)
        assert np.abs(H - X).sum() <= TOL * bn
        _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)
        if np_opt < 0:
            assert st["pull_near_edges"] == 0 and st["pull_passes"] == 0
        else:
            assert st["pull_near_edges"] == _near_count(n, cp, ri)


def test_pull_log_matches_oracle_geom():
    """Fixed schedule (GEOM): frontier sizes pass for pass as the oracle (Q8 ties aside)."""
    n = 50_000
    cp, ri = _web(n, seed=3)
    P = oracle.Problem(n, cp, ri)
    target = 1e-9 * 0.15
    st, near = _oracle_passes_with_ties(P, target, oracle.GEOM)
    H, F, log, r, stats = _gpu(n, cp, ri, target, policy=di.DI_POLICY_GEOM, near_pull=1, pull_permille=1)
    assert stats["pull_passes"] > 0
    _compare_logs_q8(log, st, near)


def test_pull_edge_cases():
    """Ragged last tile, window clipping at both ends, self-loops, duplicates, a column
    of > 65535 edges (kept on the push path), dangling columns."""
    rng = np.random.default_rng(7)
    n = 3 * 2048 + 77
    cols = []
    for i in range(n):
        if i % 11 == 0:
            cols.append(np.zeros(0, np.int32))                      # dangling
            continue
        k = int(rng.integers(1, 24))
        loc = (i + rng.integers(-1100, 1101, size=k)) % n          # near, wrapped near, just-far
        glob = rng.integers(0, n, size=int(rng.integers(0, 4)))
        c = np.concatenate([loc, glob, [i]] if i % 5 == 0 else [loc, glob]).astype(np.int32)
        if i % 7 == 0:
            c = np.concatenate([c, c[:3]])                          # duplicates add
        cols.append(c)
    cols[5] = rng.integers(0, n, size=70_000).astype(np.int32)      # > 65535 edges: never near
    cols[n - 3] = np.arange(n - 40, n, dtype=np.int32)               # window clipped at the top
    cols[2] = np.arange(0, 30, dtype=np.int32)                       # ... and at the bottom
    deg = np.array([len(c) for c in cols])
    cp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ri = np.concatenate(cols).astype(np.int32)
    X, P, bn = _xref(n, cp, ri)
    target = 1e-9 * bn
    for key in (0, 1):
        H, F, log, r, st = _gpu(n, cp, ri, target, near_pull=1, pull_permille=1, select_key=key)
        assert st["pull_near_edges"] == _near_count(n, cp, ri)
        assert st["pull_passes"] > 0
        assert np.abs(H - X).sum() <= TOL * bn
        _check_state(n, cp, ri, None, None, 0.85, H, F, r, target)


def test_pull_resume_and_reset():
    """di_run resumable and di_reset restarting with pull on: same answers."""
    n = 30_000
    cp, ri = _web(n, seed=4)
    X, P, bn = _xref(n, cp, ri)
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(near_pull=1, pull_permille=1))
    di.di_run(ctx, 1e-6)
    di.di_run(ctx, 1e-9 * bn)
    H1 = di.di_get_history(ctx)
    di.di_reset(ctx)
    assert di.di_get_stats(ctx)["pull_passes"] == 0
    di.di_run(ctx, 1e-9 * bn)
    H2 = di.di_get_history(ctx)
    F = di.di_get_fluid(ctx)
    r = di.di_get_residual(ctx)
    di.di_destroy(ctx)
    for H in (H1, H2):
        assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H2, F, r, 1e-9 * bn)


def test_pull_signed_and_fused_stay_push():
    """Signed P and the fused persistent kernel never build the table."""
    n = 20_000
    cp, ri, v, b = gen.signed_system(n, 1)
    ctx = di.di_create(n, cp, ri, v, b, 0.9, di.default_options(near_pull=1))
    assert di.di_get_stats(ctx)["pull_near_edges"] == 0
    di.di_destroy(ctx)
    cp, ri = _web(n)
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(near_pull=1, pass_kernel=2))
    assert di.di_get_stats(ctx)["pull_near_edges"] == 0
    di.di_destroy(ctx)

"""Distributed path on ONE GPU: K ranks as K host threads of one process, each
with its own context and stream, over the in-process loopback fabric of
libditer (csrc/dist.cu).  No kernel waits on another rank -- all waiting is
host-side -- so this is safe on a single GPU (B200_PROFILING.md).  The same
kernels, outbox compaction, exchange rounds, merge and termination run as with
NCCL; only the transport differs.
"""
import threading

import numpy as np
import pytest

import diter_inputs as gen
import oracle
import paper_1202_6168_b200 as di
from paper_1202_6168_b200 import dist

pytestmark = pytest.mark.gpu


def run_ranks(K, n, cp, ri, vals, b, d, target, bounds, mode, key, **opts):
    cid = dist.loopback_comm_id(key)
    out = [None] * K
    err = [None] * K

    def worker(r):
        try:
            lcp, lri, lv, lb = dist.shard_csc(cp, ri, vals, b, bounds, r)
            o = di.default_options(exchange_mode=mode, **opts)
            ctx = di.di_create_dist(r, K, cid, bounds, n, lcp, lri, lv, lb, d, o)
            di.di_run(ctx, target)
            out[r] = (di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_pass_log(ctx),
                      di.di_get_stats(ctx), di.di_get_residual(ctx),
                      di.di_get_pagerank(ctx) if vals is None and b is None else None)
            di.di_destroy(ctx)
        except Exception as e:          # surfaced below
            err[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)             # a failed rank aborts the loopback group: peers return
        assert not t.is_alive(), f"rank thread hung; errors: {err}"
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    H = np.concatenate([o[0] for o in out])
    F = np.concatenate([o[1] for o in out])
    return H, F, out


@pytest.mark.parametrize("K,key,remote", [(2, di.DI_KEY_RAW, 0), (4, di.DI_KEY_RAW, 0), (3, di.DI_KEY_EDGE, 0),
                                          (2, di.DI_KEY_RAW, 1), (3, di.DI_KEY_EDGE, 1),
                                          (2, di.DI_KEY_RAW, 2), (4, di.DI_KEY_EDGE, 2),
                                          (3, di.DI_KEY_PAPER, 0), (2, di.DI_KEY_PAPER, 1)])
def test_sync_matches_single_gpu_passes(K, key, remote):
    """SYNC mode is the single-GPU snapshot pass: same per-pass frontier sizes,
    edges and thresholds (random B: no exact-arithmetic ties), same fixed point --
    with the raw and the per-edge selection key (per-edge weights need only local
    out-degrees) and the paper key (global in-degrees by a reduce-scatter at create),
    and with remote edges pushed per diffusion, as H increments at
    each exchange (NEXT f2) or applied by the receivers from the
    shipped increments (NEXT f3): the same fluid reaches the same
    rows before the next selection."""
    n = 200_000
    cp, ri = gen.web_graph(n, 5)
    rng = np.random.default_rng(3)
    b = rng.random(n) + 0.5
    b *= 0.15 / b.sum()
    target = 1e-9 * 0.15
    H1, _, log1 = di.solve(n, cp, ri, target, b=b, select_key=key)
    bounds = dist.partition_bounds(cp, K)
    H, F, outs = run_ranks(K, n, cp, ri, None, b, 0.85, target, bounds, di.DI_EXCHANGE_SYNC,
                           f"sync{K}k{key}r{remote}", select_key=key, remote_push=remote)
    for o in outs:        # every rank logs the same global pass records
        lg = o[2]
        np.testing.assert_array_equal(lg["frontier"], log1["frontier"])
        np.testing.assert_array_equal(lg["edges"], log1["edges"])
        np.testing.assert_array_equal(lg["T"], log1["T"])
        assert o[3]["exchanges"] > 0 and o[3]["exchanged_bytes"] > 0
    X = oracle.Problem(n, cp, ri, None, b).solve(1e-12 * 0.15 * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * 0.15
    assert np.abs(F).sum() < target


@pytest.mark.parametrize("K,cost", [(2, "out"), (3, "inout"), (4, "out"), (8, "inout")])
def test_async_parity(K, cost):
    """ASYNC mode (send when s_k > r_k/K, rounds every check_interval passes):
    parity with the oracle and a closed mass ledger."""
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost=cost, row_idx=p.row_idx)
    H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds,
                           di.DI_EXCHANGE_ASYNC, f"async{K}{cost}", check_interval=4)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn          # no mass lost or duplicated in flight
    assert all(o[4] < p.parity_stop for o in outs)  # global residual on every rank
    Xp = np.concatenate([o[5] for o in outs])       # completed PageRank, global |H|_1 (f4)
    assert abs(Xp.sum() - 1.0) <= 1e-12
    assert np.abs(Xp - X / X.sum()).sum() <= 2e-8


@pytest.mark.parametrize("K", [2, 4])
def test_async_remote_increments(K):
    """NEXT f2: remote edges pushed from H - H_old at exchange
    rounds instead of at every diffusion.  Parity with the oracle, a closed ledger,
    the completed PageRank, and fewer pushes into the outbox than per-diffusion
    pushing on the same problem (nodes re-diffuse between rounds)."""
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost="inout", row_idx=p.row_idx)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    deg = np.diff(p.col_ptr)
    pushes = {}
    for remote in (di.DI_REMOTE_PER_DIFFUSION, di.DI_REMOTE_INCREMENT):
        H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds,
                               di.DI_EXCHANGE_ASYNC, f"incr{K}r{remote}", check_interval=8, remote_push=remote)
        assert np.abs(H - X).sum() <= 1e-8 * bn
        ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
        assert abs(ledger - bn) <= 1e-12 * bn
        assert all(o[4] < p.parity_stop for o in outs)
        pushes[remote] = sum(o[3]["remote_pushes"] for o in outs)
    assert 0 < pushes[di.DI_REMOTE_INCREMENT] < pushes[di.DI_REMOTE_PER_DIFFUSION]


@pytest.mark.parametrize("K,cost", [(2, "out"), (4, "inout")])
def test_async_receiver_computes(K, cost):
    """NEXT f3: senders ship (column, H increment) once per peer
    owning rows of the column; receivers apply their stored in-edges.  Parity, a
    closed ledger, the completed PageRank; the receivers do the remote pushes."""
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost=cost, row_idx=p.row_idx)
    H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds,
                           di.DI_EXCHANGE_ASYNC, f"recv{K}{cost}", check_interval=4, remote_push=di.DI_REMOTE_RECEIVER)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    assert all(o[4] < p.parity_stop for o in outs)
    Xp = np.concatenate([o[5] for o in outs])
    assert np.abs(Xp - X / X.sum()).sum() <= 2e-8
    assert sum(o[3]["remote_pushes"] for o in outs) > 0 and all(o[3]["exchanged_bytes"] > 0 for o in outs)


def test_async_receiver_computes_signed_unsorted_rows():
    """Signed P with each column's rows in reverse (unsorted) order: the create-time
    partition groups remote rows by peer, so receiver-computes stays exact."""
    n = 60_000
    cp, ri, v, b = gen.signed_system(n, 4)
    ri2, v2 = ri.copy(), v.copy()
    for j in range(n):
        a, z = cp[j], cp[j + 1]
        ri2[a:z] = ri[a:z][::-1]
        v2[a:z] = v[a:z][::-1]
    bn = np.abs(b).sum()
    bounds = dist.partition_bounds(cp, 3)
    H, F, outs = run_ranks(3, n, cp, ri2, v2, b, 0.9, 5e-10 * bn, bounds, di.DI_EXCHANGE_ASYNC, "recvsigned",
                           remote_push=di.DI_REMOTE_RECEIVER)
    X, _ = oracle.Problem(n, cp, ri, v, b, 0.9).jacobi(1e-13 * bn)
    assert np.abs(H - X).sum() <= 1e-8 * bn


def test_async_remote_increments_signed():
    n = 100_000
    cp, ri, v, b = gen.signed_system(n, 3)
    bn = np.abs(b).sum()
    bounds = dist.partition_bounds(cp, 3)
    H, F, outs = run_ranks(3, n, cp, ri, v, b, 0.9, 5e-10 * bn, bounds, di.DI_EXCHANGE_ASYNC, "signedincr",
                           remote_push=di.DI_REMOTE_INCREMENT)
    X, _ = oracle.Problem(n, cp, ri, v, b, 0.9).jacobi(1e-13 * bn)
    assert np.abs(H - X).sum() <= 1e-8 * bn


def _run_ranks_fn(K, key, fn):
    """K loopback ranks, each running fn(rank, comm_id) in its own thread."""
    cid = dist.loopback_comm_id(key)
    out, err = [None] * K, [None] * K

    def worker(r):
        try:
            out[r] = fn(r, cid)
        except Exception as e:
            err[r] = e
    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)             # a failed rank aborts the loopback group: peers return
        assert not t.is_alive(), f"rank thread hung; errors: {err}"
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("remote,l2", [(0, 0), (1, 0), (2, 0), (1, 1)])
def test_rebalance_moves_state_and_keeps_parity(remote, l2):
    """NEXT f4: di_rebalance ships columns, F, H (and B) of moved
    nodes mid-solve; the run resumes on the new ranges and reaches the same X with a
    closed ledger.  Random positive B exercises the B transfer (di_reset after it).
    l2 = 1: every rank forces a 1 MB L2 persisting window, which the rebuilt context
    re-applies on the stream it inherits."""
    K = 3
    p = gen.config("C2", 2, n=200_000)
    rng = np.random.default_rng(2)
    b = rng.random(p.n) + 0.5
    b *= 0.15 / b.sum()
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K)
    nb = bounds.copy()
    nb[1] = int(bounds[1] * 0.8)                   # rank 0 gives nodes to rank 1
    nb[2] = int(bounds[2] + (p.n - bounds[2]) * 0.25)   # rank 1 takes nodes from rank 2

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, b, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_ASYNC, check_interval=4, remote_push=remote,
                               l2_persist=1 if l2 else 0)
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
        if l2:
            assert di.di_get_stats(ctx)["l2_window_bytes"] > 0
        di.di_run(ctx, 1e-4)
        h0 = di.di_get_history(ctx).sum()
        di.di_rebalance(ctx, nb)
        if l2:
            assert di.di_get_stats(ctx)["l2_window_bytes"] > 0
        got = di.di_get_bounds(ctx)
        res = (list(got), ctx.n_local, h0)
        di.di_run(ctx, p.parity_stop)
        H, F, st = di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_stats(ctx)
        di.di_reset(ctx)                           # F = B over the new range
        Fr = di.di_get_fluid(ctx)
        di.di_destroy(ctx)
        return res, H, F, st, Fr
    outs = _run_ranks_fn(K, f"rebal{remote}{l2}", fn)
    for r, o in enumerate(outs):
        assert o[0][0] == list(nb) and o[0][1] == nb[r + 1] - nb[r]
        assert o[3]["rebalances"] == 1
    H = np.concatenate([o[1] for o in outs])
    F = np.concatenate([o[2] for o in outs])
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx, None, b).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    np.testing.assert_array_equal(np.concatenate([o[4] for o in outs]), b)


def test_adaptation_moves_boundaries_on_skewed_partition():
    """options.adapt_rounds: on the out-edge-balanced partition of a Zipf-over-id
    graph rank 0 holds most of the residual and work, so the rule moves omega_1
    down; the solve stays exact."""
    K = 2
    p = gen.config("C2", 1, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost="out")

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_ASYNC, check_interval=4, adapt_rounds=1,
                               remote_push=di.DI_REMOTE_INCREMENT)
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
        di.di_run(ctx, p.parity_stop)
        out = (di.di_get_bounds(ctx), ctx.n_local, di.di_get_history(ctx), di.di_get_fluid(ctx), di.di_get_stats(ctx))
        di.di_destroy(ctx)
        return out
    outs = _run_ranks_fn(K, "adapt", fn)
    nb = outs[0][0]
    assert list(nb) == list(outs[1][0])
    assert outs[0][4]["rebalances"] > 0 and nb[1] < bounds[1]
    H = np.concatenate([o[2] for o in outs])
    F = np.concatenate([o[3] for o in outs])
    assert len(H) == p.n
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn


def test_async_signed():
    n = 100_000
    cp, ri, v, b = gen.signed_system(n, 3)
    bn = np.abs(b).sum()
    bounds = dist.partition_bounds(cp, 2)
    H, F, outs = run_ranks(2, n, cp, ri, v, b, 0.9, 5e-10 * bn, bounds, di.DI_EXCHANGE_ASYNC, "signed")
    X, _ = oracle.Problem(n, cp, ri, v, b, 0.9).jacobi(1e-13 * bn)
    assert np.abs(H - X).sum() <= 1e-8 * bn


def test_rebalance_rejects_bad_bounds_and_keeps_state():
    """Invalid new bounds are rejected on every rank before any collective step; the
    contexts stay usable and still reach parity."""
    K = 2
    p = gen.config("C2", 3, n=100_000)
    bounds = dist.partition_bounds(p.col_ptr, K)

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d,
                                di.default_options(exchange_mode=di.DI_EXCHANGE_ASYNC))
        bad = []
        for nb in ([0, bounds[1], p.n - 1], [0, 0, p.n], [0, p.n, p.n]):
            try:
                di.di_rebalance(ctx, nb)
            except di.DiError as e:
                bad.append(e.status)
        di.di_run(ctx, p.parity_stop)
        out = (bad, di.di_get_history(ctx), di.di_get_bounds(ctx))
        di.di_destroy(ctx)
        return out
    outs = _run_ranks_fn(K, "badbounds", fn)
    for o in outs:
        assert o[0] == [di.DI_ERR_INVALID_ARG] * 3
        np.testing.assert_array_equal(o[2], bounds)
    H = np.concatenate([o[1] for o in outs])
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * 0.15 * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * 0.15


@pytest.mark.parametrize("mode", [di.DI_EXCHANGE_SYNC, di.DI_EXCHANGE_ASYNC])
def test_dist_profile_kernel_times(mode):
    """profile=1 on distributed contexts: events around each local pass's select and
    scatter, read back at the round's host sync (bench.py's roofline at N > 1)."""
    p = gen.config("C2", 1, n=200_000)
    bounds = dist.partition_bounds(p.col_ptr, 2)
    _, _, out = run_ranks(2, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.stop, bounds, mode,
                          "prof%d" % mode, profile=1)
    for o in out:
        s = o[3]
        assert s["kt_scatter_ms"] > 0 and s["kt_select_ms"] > 0
        assert s["kt_passes"] == s["passes"]


# ---------------------------------------------------------------- P2P exchange --
# DI_EXCHANGE_P2P (csrc/p2p.cu): the paper's send rule with records written straight
# into the receiver's inbox ring (here: contexts of one process map each other's
# windows by pointer), merges at the start of each round, and a board-triggered
# quiesce-then-reduce confirmation as the only collectives of a run.

def _p2p_opts(**kw):
    return dict(check_interval=4, remote_push=di.DI_REMOTE_INCREMENT, **kw)


@pytest.mark.parametrize("K,cost", [(2, "out"), (3, "inout"), (4, "out"), (8, "out")])
def test_p2p_parity_ledger_and_no_collective_per_round(K, cost):
    """Parity with the oracle's fixed point, a closed mass ledger (nothing lost or
    duplicated in flight), the global residual on every rank -- and the collective
    count of the run: one all-reduce at its start plus four per confirmation, however
    many rounds ran (the bulk ASYNC rounds need >= 3 per round)."""
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost=cost, row_idx=p.row_idx)

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, **_p2p_opts())
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
        c0 = di.di_get_stats(ctx)["collectives"]
        di.di_run(ctx, p.parity_stop)
        st = di.di_get_stats(ctx)
        out = (di.di_get_history(ctx), di.di_get_fluid(ctx), st, st["collectives"] - c0,
               di.di_get_residual(ctx), di.di_get_pagerank(ctx))
        di.di_destroy(ctx)
        return out
    outs = _run_ranks_fn(K, f"p2p{K}{cost}", fn)
    H = np.concatenate([o[0] for o in outs])
    F = np.concatenate([o[1] for o in outs])
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    for o in outs:
        st, run_coll = o[2], o[3]
        assert o[4] < p.parity_stop
        rounds = st["passes"] // 4
        assert st["confirms"] >= 1 and rounds > 3 * st["confirms"], (rounds, st["confirms"])
        assert run_coll == 1 + 4 * st["confirms"], (run_coll, st["confirms"])
        assert st["exchanges"] > 0 and st["exchanged_bytes"] > 0
    Xp = np.concatenate([o[5] for o in outs])
    assert abs(Xp.sum() - 1.0) <= 1e-12


def test_p2p_memory_scales_with_ranks():
    """Per-rank exchange memory: the compact outbox and inbox rings of P2P stay below the
    bulk mode's dense outbox of N doubles on every rank, and their mean per rank falls
    as K grows.  (The owner of the Zipf-over-id head receives from
    every peer, so the largest rank's inbox does not shrink with K.)"""
    p = gen.config("C2", 1, n=400_000)
    per = {}
    for mode in (di.DI_EXCHANGE_ASYNC, di.DI_EXCHANGE_P2P):
        for K in (2, 4, 8):
            bounds = dist.partition_bounds(p.col_ptr, K)

            def fn(r, cid):
                lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
                o = di.default_options(exchange_mode=mode, **_p2p_opts())
                ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
                b = di.di_get_stats(ctx)["exchange_bytes_resident"]
                di.di_destroy(ctx)
                return b
            per[(mode, K)] = _run_ranks_fn(K, f"mem{mode}{K}", fn)
    mean = {K: np.mean(per[(di.DI_EXCHANGE_P2P, K)]) for K in (2, 4, 8)}
    for K in (2, 4, 8):
        assert max(per[(di.DI_EXCHANGE_P2P, K)]) < min(per[(di.DI_EXCHANGE_ASYNC, K)]) / 2
    assert mean[8] < mean[4] < mean[2], mean


def test_p2p_signed_reset_rerun_and_limits():
    """Signed P (C5-like) over 3 ranks against the oracle's Jacobi fixed point; a
    di_reset + second run reproduces the parity; rebalance is refused (slots fixed at
    create); P2P without remote increments is refused at create on every rank."""
    n, K = 60_000, 3
    cp, ri, v, b = gen.signed_system(n, 2)
    bn = float(np.abs(b).sum())
    bounds = dist.partition_bounds(cp, K)
    X, _ = oracle.Problem(n, cp, ri, v, b, 0.9).jacobi(1e-13 * bn)

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(cp, ri, v, b, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, **_p2p_opts())
        ctx = di.di_create_dist(r, K, cid, bounds, n, lcp, lri, lv, lb, 0.9, o)
        di.di_run(ctx, 5e-10 * bn)
        H1 = di.di_get_history(ctx)
        di.di_reset(ctx)
        di.di_run(ctx, 5e-10 * bn)
        H2 = di.di_get_history(ctx)
        try:
            di.di_rebalance(ctx, bounds)
            rb = None
        except di.DiError as e:
            rb = e.status
        di.di_destroy(ctx)
        return H1, H2, rb
    outs = _run_ranks_fn(K, "p2psigned", fn)
    for j in (0, 1):
        H = np.concatenate([o[j] for o in outs])
        assert np.abs(H - X).sum() <= 1e-8 * bn
    assert all(o[2] == di.DI_ERR_UNSUPPORTED for o in outs)

    def bad(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(cp, ri, v, b, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, remote_push=di.DI_REMOTE_PER_DIFFUSION)
        try:
            di.di_create_dist(r, K, cid, bounds, n, lcp, lri, lv, lb, 0.9, o)
        except di.DiError as e:
            return e.status
        return None
    assert _run_ranks_fn(K, "p2pbad", bad) == [di.DI_ERR_INVALID_ARG] * K


def test_create_failure_on_one_rank_fails_every_rank():
    """One rank's input fails validation (a row index out of range): every rank's
    di_create_dist fails -- that rank with DI_ERR_INVALID_ARG, its peers with
    DI_ERR_STATE after the agreement -- and none waits forever in a later collective."""
    K = 3
    p = gen.config("C2", 1, n=30_000)
    bounds = dist.partition_bounds(p.col_ptr, K)

    def fn(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        if r == 1:
            lri = lri.copy()
            lri[len(lri) // 2] = p.n + 5
        for mode in (di.DI_EXCHANGE_ASYNC,):
            try:
                ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d,
                                        di.default_options(exchange_mode=mode, select_key=di.DI_KEY_PAPER))
                di.di_destroy(ctx)
            except di.DiError as e:
                return e.status
        return None
    st = _run_ranks_fn(K, "createfail", fn)
    assert st[1] == di.DI_ERR_INVALID_ARG
    assert st[0] == st[2] == di.DI_ERR_STATE


def test_p2p_checkpoint_resume():
    """di_set_state on distributed P2P contexts: a run stopped by max_passes on K = 2
    loopback ranks, each rank's (F, H) loaded into a new pair of contexts, continues to
    the oracle's fixed point with a closed ledger."""
    K = 2
    p = gen.config("C2", 2, n=200_000)
    bounds = dist.partition_bounds(p.col_ptr, K)

    def first(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, max_passes=12, **_p2p_opts())
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
        st = di.di_run(ctx, p.parity_stop, raise_on_not_converged=False)
        out = (st, di.di_get_fluid(ctx), di.di_get_history(ctx))
        di.di_destroy(ctx)
        return out
    a = _run_ranks_fn(K, "ckpt1", first)
    assert all(o[0] == di.DI_ERR_NOT_CONVERGED for o in a)

    def second(r, cid):
        lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
        o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, **_p2p_opts())
        ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
        di.di_set_state(ctx, a[r][1], a[r][2])
        di.di_run(ctx, p.parity_stop)
        out = (di.di_get_history(ctx), di.di_get_fluid(ctx))
        di.di_destroy(ctx)
        return out
    b = _run_ranks_fn(K, "ckpt2", second)
    H = np.concatenate([o[0] for o in b])
    F = np.concatenate([o[1] for o in b])
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * 0.15 * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * 0.15
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - 0.15) <= 1e-12 * 0.15


@pytest.mark.parametrize("mode,K,remote", [(di.DI_EXCHANGE_ASYNC, 2, di.DI_REMOTE_PER_DIFFUSION),
                                           (di.DI_EXCHANGE_ASYNC, 4, di.DI_REMOTE_INCREMENT),
                                           (di.DI_EXCHANGE_ASYNC, 3, di.DI_REMOTE_RECEIVER),
                                           (di.DI_EXCHANGE_P2P, 2, di.DI_REMOTE_INCREMENT),
                                           (di.DI_EXCHANGE_P2P, 4, di.DI_REMOTE_INCREMENT),
                                           (di.DI_EXCHANGE_P2P, 8, di.DI_REMOTE_INCREMENT)])
def test_sweeps_on_ranks(mode, K, remote):
    """Distributed ranks running their local passes as asynchronous sweeps (options.sweep,
    reading R26): parity with the oracle, a closed mass ledger, the global residual on
    every rank; with the per-edge key (f1)."""
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost="out", row_idx=p.row_idx)
    H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds, mode,
                           f"sweep{mode}{K}{remote}", check_interval=4, remote_push=remote, sweep=1,
                           select_key=di.DI_KEY_EDGE)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    assert all(o[4] < p.parity_stop for o in outs)


def test_pilot_rebalanced_ranges_keep_parity_and_level_the_work():
    """Ranges re-balanced by a pilot solve's measured work (dist.partition_bounds_measured,
    bench --pilot-solves): the second solve, on the new ranges, still matches the oracle
    with a closed ledger, and the ranks' performed pushes are closer to level than on the
    out-edge partition (the Zipf head makes rank 0 the busiest there)."""
    K = 4
    p = gen.config("C2", 2, n=400_000)
    bn = 0.15
    opts = dict(check_interval=2, remote_push=di.DI_REMOTE_INCREMENT, sweep=1, select_key=di.DI_KEY_EDGE)

    def solve(bounds, tag):
        H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds,
                               di.DI_EXCHANGE_P2P, tag, **opts)
        work = []
        for r, o in enumerate(outs):
            lri = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)[1]
            rho = dist.remote_fraction(lri, int(bounds[r]), int(bounds[r + 1]))
            work.append(dist.pushes_performed(o[3], rho, 1))
        return H, F, np.asarray(work)

    b0 = dist.partition_bounds(p.col_ptr, K, cost="out")
    _, _, w0 = solve(b0, "pilot0")
    b1 = dist.partition_bounds_measured(p.col_ptr, K, b0, w0)
    assert b1[0] == 0 and b1[-1] == p.n and np.all(np.diff(b1) > 0)
    H, F, w1 = solve(b1, "pilot1")
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    assert b1[1] < b0[1]                                   # the head rank gave columns away
    assert w1.max() / w1.mean() < w0.max() / w0.mean(), (w0, w1)


@pytest.mark.parametrize("sleep", [-1, 0, 60])
def test_p2p_sleep_modes_keep_parity(sleep):
    """P2P sleep: off, the absolute rule r_k < target / K, and the relative
    rule (asleep below 60 % of the rank's even share of the fluid on the board).  Sleeping ranks
    keep merging and sending, so every mode ends at the oracle's X with a closed ledger; the
    relative rule does put ranks to sleep on a Zipf-head graph."""
    K = 3
    p = gen.config("C2", 2, n=300_000)
    bn = 0.15
    bounds = dist.partition_bounds(p.col_ptr, K, cost="out")
    H, F, outs = run_ranks(K, p.n, p.col_ptr, p.row_idx, None, None, 0.85, p.parity_stop, bounds,
                           di.DI_EXCHANGE_P2P, f"sleep{sleep}", check_interval=2,
                           remote_push=di.DI_REMOTE_INCREMENT, sweep=1, select_key=di.DI_KEY_EDGE, p2p_sleep=sleep)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * bn * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * bn
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - bn) <= 1e-12 * bn
    assert all(o[4] < p.parity_stop for o in outs)
    slept = sum(o[3]["sleep_rounds"] for o in outs)
    if sleep < 0:
        assert slept == 0
    if sleep == 60:
        assert slept > 0

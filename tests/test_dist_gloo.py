"""Multi-rank host logic on CPU: world_size 2 over torch.distributed 'gloo'
(127.0.0.1).  Covers what the N>1 bench path does on the host -- partition
bounds, CSC sharding, the NCCL unique-id broadcast -- and checks the exchange
protocol of csrc/dist.cu (SYNC and ASYNC rounds, send rule, termination with
in-flight mass) with the numpy model in tests/dist_model.py against the oracle.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _host_logic(rank, world, port):
    _init(rank, world, port)
    try:
        import diter_inputs as gen
        from paper_1202_6168_b200 import dist as dd
        cp, ri = gen.web_graph(50_000, 4)
        for cost in ("out", "inout"):
            bounds = dd.partition_bounds(cp, world, cost=cost, row_idx=ri)
            allb = [None] * world
            dist.all_gather_object(allb, bounds.tolist())
            assert all(x == allb[0] for x in allb)            # every rank, same ranges
            shard = dd.shard_csc(cp, ri, None, None, bounds, rank)
            shards = [None] * world
            dist.all_gather_object(shards, (shard[0].tolist(), shard[1].tolist()))
            # the shards reassemble the global CSC exactly
            cps = [np.asarray(s[0]) for s in shards]
            re_cp = np.concatenate([cps[0]] + [c[1:] + sum(x[-1] for x in cps[:k]) for k, c in enumerate(cps) if k > 0])
            np.testing.assert_array_equal(re_cp, cp)
            np.testing.assert_array_equal(np.concatenate([np.asarray(s[1]) for s in shards]), ri)
        # pilot re-balancing (bench --pilot-solves): every rank gathers the same work numbers and
        # derives the same new ranges; the rank with twice the work density gives columns away
        bounds = dd.partition_bounds(cp, world)
        shard = dd.shard_csc(cp, ri, None, None, bounds, rank)
        rho = dd.remote_fraction(shard[1], int(bounds[rank]), int(bounds[rank + 1]))
        ri_np = np.asarray(shard[1])
        assert rho == np.mean((ri_np < bounds[rank]) | (ri_np >= bounds[rank + 1]))
        stats = {"edges": int(shard[0][-1]) * (2 if rank == 0 else 1), "remote_pushes": 0}
        work = [None] * world
        dist.all_gather_object(work, dd.pushes_performed(stats, 0.0, 1))
        nb = dd.partition_bounds_measured(cp, world, bounds, work)
        allb = [None] * world
        dist.all_gather_object(allb, nb.tolist())
        assert all(x == allb[0] for x in allb)
        assert nb[0] == 0 and nb[-1] == len(cp) - 1 and np.all(np.diff(nb) > 0)
        assert nb[1] < bounds[1]
        # rank 0's new share of the measured work is 1 / world (within one column's cost)
        dens = np.where(np.arange(len(cp) - 1) < bounds[1], 2.0, 1.0)
        wcum = np.concatenate([[0.0], np.cumsum(np.diff(cp) * dens)])
        assert abs(wcum[nb[1]] / wcum[-1] - 1.0 / world) < 1e-3
        cid = dd.nccl_comm_id()                               # rank 0 creates, broadcast over gloo
        ids = [None] * world
        dist.all_gather_object(ids, cid)
        assert len(cid) == 128 and all(x == ids[0] for x in ids)
        lid = dd.loopback_comm_id("k")
        assert lid[:8] == b"DILOOP01" and len(lid) == 128
    finally:
        dist.destroy_process_group()


def _protocol(rank, world, port, mode):
    _init(rank, world, port)
    try:
        import diter_inputs as gen
        import oracle
        from dist_model import RankModel
        from paper_1202_6168_b200 import dist as dd
        n = 4000
        cp, ri = gen.web_graph(n, 6, window=100, max_deg=300)
        rng = np.random.default_rng(1)
        b = rng.random(n) + 0.5
        b *= 0.15 / b.sum()
        bounds = dd.partition_bounds(cp, world)
        lcp, lri, _, lb = dd.shard_csc(cp, ri, None, b, bounds, rank)
        m = RankModel(rank, world, bounds, lcp, lri, lb, n)
        target = 1e-10 * 0.15
        R = m.run_sync(target) if mode == "sync" else m.run_async(target)
        Hs = [None] * world
        dist.all_gather_object(Hs, (m.H.tolist(), m.F.tolist(), m.log, m.exchanged))
        H = np.concatenate([np.asarray(h[0]) for h in Hs])
        F = np.concatenate([np.asarray(h[1]) for h in Hs])
        P = oracle.Problem(n, cp, ri, None, b)
        X = P.solve(1e-14 * 0.15).H
        assert np.abs(H - X).sum() <= 1e-8 * 0.15
        deg = np.diff(cp)
        ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
        assert abs(ledger - 0.15) <= 1e-13                    # nothing lost in flight
        assert np.abs(F).sum() < target and R < target
        assert sum(h[3] for h in Hs) > 0                      # fluid did cross ranks
        if mode == "sync":
            st = P.init()
            P.snapshot(st, target, oracle.HYBRID)
            assert [(l[1], l[3]) for l in st.log] == [tuple(x) for x in Hs[0][2]]
    finally:
        dist.destroy_process_group()


def _p2p_protocol(rank, world, port, key):
    _init(rank, world, port)
    try:
        import diter_inputs as gen
        import oracle
        from dist_model import P2PRank
        from paper_1202_6168_b200 import dist as dd
        n = 4000
        cp, ri = gen.web_graph(n, 6, window=100, max_deg=300)
        rng = np.random.default_rng(1)
        b = rng.random(n) + 0.5
        b *= 0.15 / b.sum()
        bounds = dd.partition_bounds(cp, world)
        lcp, lri, _, lb = dd.shard_csc(cp, ri, None, b, bounds, rank)
        m = P2PRank(rank, world, bounds, lcp, lri, lb, n, key)
        target = 1e-10 * 0.15
        # rank 1 runs its rounds slower: the ranks drift apart, messages arrive late
        delay = (lambda r: 0.002 * ((r * 7919) % 3)) if rank == 1 else None
        try:
            R = m.run_p2p(target, delay=delay)
        finally:
            m.close()
        out = [None] * world
        dist.all_gather_object(out, (m.H.tolist(), m.F.tolist(), m.exchanged, m.collectives, m.confirms,
                                     len(m.log)))
        H = np.concatenate([np.asarray(h[0]) for h in out])
        F = np.concatenate([np.asarray(h[1]) for h in out])
        X = oracle.Problem(n, cp, ri, None, b).solve(1e-14 * 0.15).H
        assert np.abs(H - X).sum() <= 1e-8 * 0.15
        deg = np.diff(cp)
        ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
        assert abs(ledger - 0.15) <= 1e-13                    # nothing lost or duplicated in flight
        assert R < target and np.abs(F).sum() < target
        assert sum(h[2] for h in out) > 0
        for h in out:
            # one all-reduce to start the run + four per confirmation, none per round
            assert h[3] == 1 + 4 * h[4] and h[4] >= 1
            assert h[5] // 4 > 3 * h[4]                       # rounds >> confirmations
    finally:
        dist.destroy_process_group()


def test_p2p_protocol_two_ranks():
    """The barrier-free exchange (DI_EXCHANGE_P2P) as a protocol: shared-memory windows
    with inbox rings and published heads, ranks drifting apart, board-triggered
    quiesce-then-reduce termination -- parity, closed ledger, collectives only in the
    confirmations."""
    key = f"dip2p{os.getpid()}"
    mp.spawn(_p2p_protocol, args=(2, _free_port(), key), nprocs=2, join=True)


def test_host_logic_two_ranks():
    mp.spawn(_host_logic, args=(2, _free_port()), nprocs=2, join=True)


@pytest.mark.parametrize("mode", ["sync", "async"])
def test_exchange_protocol_two_ranks(mode):
    mp.spawn(_protocol, args=(2, _free_port(), mode), nprocs=2, join=True)

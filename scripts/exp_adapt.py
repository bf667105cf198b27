"""Partition adaptation (NEXT f4) on K loopback ranks: per-rank diffusion work
(edges) max / mean with and without options.adapt_rounds, on the out-edge and the
in+out-edge balanced contiguous partitions.  Experiment."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di
from paper_1202_6168_b200 import dist

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
p = gen.config("C4", 1, n=n)
for K in (2, 4, 8):
    for cost in ("out", "inout"):
        bounds = dist.partition_bounds(p.col_ptr, K, cost=cost, row_idx=p.row_idx)
        for adapt in (0, 1, 2):
            st, nbs = [None] * K, [None] * K
            cid = dist.loopback_comm_id(f"a{K}{cost}{adapt}")

            def w(r):
                lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
                o = di.default_options(exchange_mode=di.DI_EXCHANGE_ASYNC, check_interval=4, adapt_rounds=adapt,
                                       remote_push=1, select_key=1, alpha=2.0, hybrid_frac=0.5)
                ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
                di.di_run(ctx, p.stop)
                st[r] = di.di_get_stats(ctx)
                nbs[r] = di.di_get_bounds(ctx)
                di.di_destroy(ctx)
            th = [threading.Thread(target=w, args=(r,)) for r in range(K)]
            [t.start() for t in th]
            [t.join() for t in th]
            e = np.array([s["edges"] for s in st], dtype=float)
            print(f"K={K} {cost:5s} adapt={adapt}: work max/mean={e.max() / e.mean():.3f} total={e.sum():.3e} "
                  f"rebalances={st[0]['rebalances']} passes(max)={max(s['passes'] for s in st)} "
                  f"bounds0={list(bounds)} -> {list(nbs[0])}", flush=True)

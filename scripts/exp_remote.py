"""Remote-push modes on K loopback ranks (one GPU): outbox pushes, exchanged bytes,
passes -- per-diffusion, H increments (NEXT f2), receiver computes (NEXT f3).  Experiment."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di
from paper_1202_6168_b200 import dist

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
p = gen.config("C2", 1, n=n)
for K in (2, 4, 8):
    bounds = dist.partition_bounds(p.col_ptr, K, cost="inout", row_idx=p.row_idx)
    for remote in (0, 1, 2):
        for ci, rr in ((4, 1),):
            st = [None] * K
            cid = dist.loopback_comm_id(f"x{K}{remote}{ci}{rr}")

            def w(r):
                lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, r)
                o = di.default_options(exchange_mode=di.DI_EXCHANGE_ASYNC, check_interval=ci, remote_push=remote,
                                       select_key=1, alpha=2.0, hybrid_frac=0.3, receive_rescale=rr)
                ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
                di.di_run(ctx, p.stop)
                st[r] = di.di_get_stats(ctx)
                di.di_destroy(ctx)
            th = [threading.Thread(target=w, args=(r,)) for r in range(K)]
            [t.start() for t in th]
            [t.join() for t in th]
            print(f"K={K} remote={['diff', 'incr', 'recv'][remote]} ci={ci} rescale={rr}: outbox pushes={sum(s['remote_pushes'] for s in st):.4e} "
                  f"exchanged={sum(s['exchanged_bytes'] for s in st) / 1e6:.1f} MB edges={sum(s['edges'] for s in st):.4e} "
                  f"passes(max)={max(s['passes'] for s in st)}", flush=True)

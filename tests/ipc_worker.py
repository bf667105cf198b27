"""One rank of a DI_EXCHANGE_P2P run in its own process (tests/test_gpu_ipc.py):
the shared-memory fabric for the collectives, the peers' windows mapped with
cudaIpcOpenMemHandle.  argv: rank world name n out.npz"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import diter_inputs as gen                      # noqa: E402
import paper_1202_6168_b200 as di               # noqa: E402
from paper_1202_6168_b200 import dist           # noqa: E402

rank, world, name, n, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5]
p = gen.config("C2", 2, n=n)
bounds = dist.partition_bounds(p.col_ptr, world)
lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, None, None, bounds, rank)
o = di.default_options(exchange_mode=di.DI_EXCHANGE_P2P, remote_push=di.DI_REMOTE_INCREMENT, check_interval=4,
                       device=0)
ctx = di.di_create_dist(rank, world, dist.shm_comm_id(name), bounds, p.n, lcp, lri, lv, lb, p.d, o)
c0 = di.di_get_stats(ctx)["collectives"]
di.di_run(ctx, p.parity_stop)
st = di.di_get_stats(ctx)
H, F = di.di_get_history(ctx), di.di_get_fluid(ctx)
r = di.di_get_residual(ctx)
di.di_destroy(ctx)
np.savez(out, H=H, F=F, r=r, run_coll=st["collectives"] - c0, confirms=st["confirms"], passes=st["passes"],
         exchanged=st["exchanged_bytes"])

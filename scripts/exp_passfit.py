"""Per-pass select / scatter device times (options.profile = 1) of one solve, and a
least-squares fit  t_scatter = a + b * nodes + c * edges  over the passes:
    python scripts/exp_passfit.py C4 [near_pull] [extra key=value options ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import diter_inputs as gen  # noqa: E402
import paper_1202_6168_b200 as di  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
npull = int(sys.argv[2]) if len(sys.argv) > 2 else -1
extra = dict(kv.split("=") for kv in sys.argv[3:])
pol, alpha, frac, key = bench.SCHEDULES[cfg]
if cfg == "C3":
    p = gen.config(cfg, 1)
    src, dst = gen.rmat_coo(24, 1)
    p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
    del src, dst
else:
    p = gen.config(cfg, 1)
opts = di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key,
                          scatter_run=bench.SCATTER_RUN.get(cfg, 0), far_defer=npull,
                          **{k: int(v) for k, v in extra.items()})
ctx = di.di_create(p.n, p.col_ptr, p.row_idx, None, None, 0.85, opts)
for _ in range(2):
    di.di_reset(ctx)
    di.di_run(ctx, p.stop)
di.di_reset(ctx)
di.di_set_profile(ctx, 1)
di.di_run(ctx, p.stop)
log = di.di_get_pass_log(ctx)
st = di.di_get_stats(ctx)
nodes = (log["frontier"] - log["dangling"]).astype(float)
edges = log["edges"].astype(float)
tsc = log["t_scatter_us"]
tsel = log["t_select_us"]
print(f"{cfg}: passes {len(log)} select {tsel.sum() / 1e3:.2f} ms scatter {tsc.sum() / 1e3:.2f} ms "
      f"(profiled run {st['run_ms']:.2f} ms)")
for k in range(len(log)):
    print(f"  pass {k:3d} nodes {nodes[k] / 1e6:7.2f}M edges {edges[k] / 1e6:8.2f}M sel {tsel[k]:8.1f} us "
          f"scatter {tsc[k]:8.1f} us")
m = nodes > 0
A = np.stack([np.ones(m.sum()), nodes[m] / 1e6, edges[m] / 1e6], 1)
coef, *_ = np.linalg.lstsq(A, tsc[m], rcond=None)
print(f"fit: scatter_us = {coef[0]:.1f} + {coef[1]:.2f} us/M nodes + {coef[2]:.3f} us/M edges")
print(f"  totals: fixed {coef[0] * m.sum() / 1e3:.1f} ms, nodes {coef[1] * nodes.sum() / 1e9:.1f} ms, "
      f"edges {coef[2] * edges.sum() / 1e9:.1f} ms")
di.di_destroy(ctx)

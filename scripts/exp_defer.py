"""A/B of the far-edge deferral on one generated graph (GPU):
    python scripts/exp_pull.py C4 "-1:0 1:0 1:60 1:200" [steps]
Each variant far_defer:unused gets a fresh context (create time printed),
2 warm-up solves, then `steps` timed solves (di_run device time, stats.run_ms)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import diter_inputs as gen  # noqa: E402
import paper_1202_6168_b200 as di  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
variants = (sys.argv[2] if len(sys.argv) > 2 else "-1:0 1:0").split()
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
pol, alpha, frac, key = bench.SCHEDULES[cfg]
t = time.perf_counter()
p = gen.config(cfg, 1)
print(f"generated {cfg} n={p.n} nnz={p.nnz} in {time.perf_counter() - t:.1f}s", flush=True)
for v in variants:
    npull, pm = (int(x) for x in v.split(":"))
    opts = di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key,
                              scatter_run=bench.SCATTER_RUN.get(cfg, 0), far_defer=npull, reserved1=pm)
    t = time.perf_counter()
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, None, None, 0.85, opts)
    t_create = time.perf_counter() - t
    ms = []
    warm = int(os.environ.get("EXP_WARM", "2"))
    for k in range(warm + steps):
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
        if k >= warm:
            ms.append(di.di_get_stats(ctx)["run_ms"])
    st = di.di_get_stats(ctx)
    print(f"{cfg} far_defer={npull:2d}: {np.median(ms):8.2f} ms/solve (min {min(ms):.2f}) "
          f"passes {st['passes']} flushes {st['far_flushes']} edges {st['edges']:.4e} "
          f"far_edges {st['far_edges']} create {t_create:.2f}s", flush=True)
    di.di_destroy(ctx)

"""Phase times of the e2e step (di_create from pinned host buffers, di_run,
di_get_history, di_destroy) on C4 in bench's launch configuration.  Experiment."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = gen.config(cfg, 1)
pol, alpha, frac, key = bench.SCHEDULES[cfg]
o = di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key)
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (p.col_ptr, p.row_idx)]
H = torch.empty(p.n, dtype=torch.float64).pin_memory()
for rep in range(int(os.environ.get("REPS", "4"))):
    t = [time.perf_counter()]
    ctx = di.di_create(p.n, pin[0], pin[1], None, None, p.d, o)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    di.di_run(ctx, p.stop)
    t.append(time.perf_counter())
    di.di_get_history(ctx, H)
    t.append(time.perf_counter())
    di.di_destroy(ctx)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: create {d[0]:.1f} ms  run {d[1]:.1f}  get_history {d[2]:.1f}  destroy {d[3]:.1f}  total {sum(d):.1f}", flush=True)

# first vs repeated solves on one context, profile 0 / 1
for prof in (0, 1):
    o.profile = prof
    ctx = di.di_create(p.n, pin[0], pin[1], None, None, p.d, o)
    for k in range(3):
        di.di_reset(ctx)
        t = time.perf_counter()
        di.di_run(ctx, p.stop)
        s = di.di_get_stats(ctx)
        print(f"profile={prof} solve {k}: wall {1e3 * (time.perf_counter() - t):.1f} ms device {s['run_ms']:.1f} ms "
              f"passes {s['passes']} graph launches {s['graph_launches']}", flush=True)
    di.di_destroy(ctx)

"""Print a per-pass breakdown (frontier, edges, phase times) of one solve in the
bench's launch configuration (bench.SCHEDULES), plus the unprofiled solve time."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2"); ap.add_argument("--n", type=int, default=None)
ap.add_argument("--pass-kernel", type=int, default=0)
ap.add_argument("--every", type=int, default=8)
ap.add_argument("--hot", type=int, default=0)
a = ap.parse_args()
p = gen.config(a.config, 1, n=a.n)
pol, alpha, frac, key = bench.SCHEDULES[a.config]


def solve(profile):
    o = di.default_options(profile=profile, pass_kernel=a.pass_kernel, hot_window=a.hot, policy=pol,
                           alpha=alpha, hybrid_frac=frac, select_key=key,
                           scatter_run=bench.SCATTER_RUN.get(a.config, 0))
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, o)
    for _ in range(3):
        di.di_reset(ctx); di.di_run(ctx, p.stop)
    s = di.di_get_stats(ctx)
    lg = di.di_get_pass_log(ctx) if profile else None
    di.di_destroy(ctx)
    return s, lg


s0, _ = solve(0)
s, lg = solve(1)
print(f"{a.config} passes={s['passes']} run_ms={s0['run_ms']:.3f} (profiled {s['run_ms']:.3f}) edges={s['edges']} "
      f"sel_ms={s['kt_select_ms']:.3f} sc_ms={s['kt_scatter_ms']:.3f} fin_ms={s['kt_finalize_ms']:.3f}")
for r in lg[::a.every]:
    print(f"p={r['pass']:4d} S={r['frontier']:10d} E={r['edges']:11d} sel={r['t_select_us']:8.1f}us sc={r['t_scatter_us']:8.1f}us")

"""Small driver for ncu captures: build config, one solve (or max_passes passes)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--max-passes", type=int, default=40)
ap.add_argument("--policy", default="hybrid")
ap.add_argument("--opt", action="append", default=[])
a = ap.parse_args()
p = gen.config(a.config, 1, n=a.n)
kw = {k: int(v) for k, v in (o.split("=") for o in a.opt)}
opts = di.default_options(max_passes=a.max_passes, check_interval=8, pass_kernel=1, **kw,
                          policy=di.DI_POLICY_GEOM if a.policy == "geom" else di.DI_POLICY_HYBRID)
ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, opts)
t = time.perf_counter()
st = di.di_run(ctx, p.stop, raise_on_not_converged=False)
print("status", st, "passes", di.di_get_stats(ctx)["passes"], "s", time.perf_counter() - t)
di.di_destroy(ctx)

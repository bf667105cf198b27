"""Small driver for ncu captures: build a config, one solve (or max_passes passes)
in bench.py's launch configuration (bench.SCHEDULES), extra options via --opt k=v."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench
if os.environ.get("DITER_LIB"):
    di.LIB_PATH = os.environ["DITER_LIB"]   # experiment: another build of the library

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--max-passes", type=int, default=40)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--pass-csv", default=None, help="write the solve's pass log (frontier, edges, dangling)")
a = ap.parse_args()
p = gen.config(a.config, 1, n=a.n)
if a.config == "C3":
    src, dst = gen.rmat_coo(24, 1)
    p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
    del src, dst
pol, alpha, frac, key = bench.SCHEDULES[a.config]
kw = dict(policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key, check_interval=8, pass_kernel=1,
          max_passes=a.max_passes, scatter_run=bench.SCATTER_RUN.get(a.config, 0),
          sweep=bench.SWEEP.get(a.config, 0), scatter_stripes=bench.SCATTER_STRIPES.get(a.config, 0),
          key_offset=bench.KEY_OFFSET.get(a.config, 0))
kw.update({k: int(v) for k, v in (o.split("=") for o in a.opt)})
ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, di.default_options(**kw))
t = time.perf_counter()
st = di.di_run(ctx, p.stop, raise_on_not_converged=False)
print("status", st, "passes", di.di_get_stats(ctx)["passes"], "s", time.perf_counter() - t)
if a.pass_csv:
    lg = di.di_get_pass_log(ctx)
    with open(a.pass_csv, "w") as f:
        f.write(",".join(lg.dtype.names) + "\n")
        for row in lg:
            f.write(",".join(str(x) for x in row) + "\n")
di.di_destroy(ctx)

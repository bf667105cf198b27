"""Compare option variants on one generated config (experiment driver, not a bench).

    python scripts/sweep.py --config C4 --variants "scatter_kernel=0;scatter_kernel=1"

For each variant: median device time of `--reps` solves (di_reset + di_run, CUDA
events inside the library), passes, edges, then one profiled solve for the
select / scatter split.
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di
if os.environ.get("DITER_LIB"):
    di.LIB_PATH = os.environ["DITER_LIB"]   # experiment: another build of the library

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variants", default="")
ap.add_argument("--policy", default="bench")
a = ap.parse_args()
p = gen.config(a.config, 1, n=a.n)
if a.config == "C3":
    src, dst = gen.rmat_coo(24, 1)
    p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
    del src, dst
for v in [x for x in a.variants.split(";")] or [""]:
    kw = {}
    for item in filter(None, v.split(",")):
        k, val = item.split("=")
        kw[k.strip()] = float(val) if "." in val else int(val)
    if a.policy == "bench":      # the bench's launch configuration
        import bench
        pol, alpha, frac, key = bench.SCHEDULES[a.config]
        for k_, v_ in (("policy", pol), ("alpha", alpha), ("hybrid_frac", frac), ("select_key", key),
                       ("scatter_run", bench.SCATTER_RUN.get(a.config, 0)),
                       ("key_offset", bench.KEY_OFFSET.get(a.config, 0))):
            kw.setdefault(k_, v_)
    kw.setdefault("policy", di.DI_POLICY_GEOM if a.policy == "geom" else di.DI_POLICY_HYBRID)
    kw["policy"] = int(kw["policy"])
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, di.default_options(**kw))
    ts = []
    for _ in range(a.reps + 1):
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
        ts.append(di.di_get_stats(ctx)["run_ms"])
    s = di.di_get_stats(ctx)
    di.di_destroy(ctx)
    kw["profile"] = 1
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, di.default_options(**kw))
    di.di_reset(ctx)
    di.di_run(ctx, p.stop)
    sp = di.di_get_stats(ctx)
    di.di_destroy(ctx)
    print(f"{a.config} [{v}] ms={np.median(ts[1:]):.3f} (min {min(ts[1:]):.3f}) passes={s['passes']} "
          f"edges={s['edges']:.4e} | profiled: sel={sp['kt_select_ms']:.2f} sc={sp['kt_scatter_ms']:.2f} ms",
          flush=True)

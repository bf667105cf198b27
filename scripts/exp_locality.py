"""Experiment: scatter throughput vs destination locality on web-like graphs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
for p_local, window in [(0.7, 1000), (1.0, 1000), (0.0, 1000), (1.0, 100000)]:
    cp, ri = gen.web_graph(n, 1, gen.XMIN_C4, p_local=p_local, window=window)
    for pol in (di.DI_POLICY_GEOM,):
        ctx = di.di_create(n, cp, ri, options=di.default_options(profile=1, policy=pol, max_passes=12))
        di.di_run(ctx, 1e-9, raise_on_not_converged=False)
        s = di.di_get_stats(ctx)
        print(json.dumps({"p_local": p_local, "window": window, "nnz": int(cp[-1]), "passes": s["passes"],
                          "scatter_Gedges_s": s["edges"] / s["kt_scatter_ms"] / 1e6,
                          "select_ms_per_pass": s["kt_select_ms"] / s["kt_passes"],
                          "scatter_ms_per_pass": s["kt_scatter_ms"] / s["kt_passes"]}), flush=True)
        di.di_destroy(ctx)

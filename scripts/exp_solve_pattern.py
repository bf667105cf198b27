"""Whole keyed solves (bench C4 schedule) on N=1e8 graphs with different local /
Zipf-over-id mixes: scatter G edges/s over the solve.  Experiment."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench
n = 100_000_000
pol, alpha, frac, key = bench.SCHEDULES["C4"]
for pl in (1.0, 0.7):
    cp, ri = gen.web_graph(n, 1, gen.XMIN_C4, p_local=pl)
    ctx = di.di_create(n, cp, ri, options=di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac,
                                                             select_key=key, profile=1))
    for _ in range(2):
        di.di_reset(ctx)
        di.di_run(ctx, 1e-9)
    s = di.di_get_stats(ctx)
    lg = di.di_get_pass_log(ctx)
    print(f"p_local={pl}: solve {s['run_ms']:.1f} ms passes {s['passes']} edges {s['edges']:.3e} nodes {s['nodes']:.3e} "
          f"scatter {s['kt_scatter_ms']:.1f} ms -> {s['edges'] / s['kt_scatter_ms'] * 1e-6:.1f} G edges/s, "
          f"select {s['kt_select_ms']:.1f} ms; edges/node {s['edges'] / s['nodes']:.2f}", flush=True)
    di.di_destroy(ctx)
    del cp, ri

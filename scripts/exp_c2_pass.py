"""C2 per-pass kernel times (profile=1 events in the graph) in bench's schedule."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench
p = gen.config("C2", 1)
pol, alpha, frac, key = bench.SCHEDULES["C2"]
for ci in (16, 64):
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, options=di.default_options(
        policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key, profile=1, check_interval=ci))
    for _ in range(3):
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
    s = di.di_get_stats(ctx)
    lg = di.di_get_pass_log(ctx)
    print(f"ci={ci}: solve {s['run_ms']:.3f} ms passes {s['passes']} sel {s['kt_select_ms']:.3f} sc {s['kt_scatter_ms']:.3f} "
          f"fin {s['kt_finalize_ms']:.3f} graph launches {s['graph_launches']}")
    sel, sc = lg["t_select_us"], lg["t_scatter_us"]
    print(f"  per pass select median {np.median(sel):.1f} us, scatter median {np.median(sc):.1f} us; "
          f"frontier median {np.median(lg['frontier']):.0f}, edges median {np.median(lg['edges']):.0f}")
    di.di_destroy(ctx)

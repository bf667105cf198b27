"""Scatter cost by push pattern: pass-0 (every node selected) scatter time on
N=1e8 web-like graphs with different local / Zipf-over-id mixes (experiment)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
for pl in [0.7, 0.0]:
    cp, ri = gen.web_graph(n, 1, gen.XMIN_C4, p_local=pl)
    for far in [-1, 1]:
        ctx = di.di_create(n, cp, ri, options=di.default_options(profile=1, max_passes=1, far_push=far))
        ts = []
        for _ in range(3):
            di.di_reset(ctx)
            di.di_run(ctx, 0.0, raise_on_not_converged=False)
            lg = di.di_get_pass_log(ctx)
            ts.append((lg["t_select_us"][0], lg["t_scatter_us"][0]))
        di.di_destroy(ctx)
        e = int(cp[-1])
        sel, sc = min(ts, key=lambda t: t[1])
        print(f"p_local={pl} far={far} edges={e:.3e} select={sel:.0f}us scatter={sc:.0f}us "
              f"-> {e / sc * 1e-3:.1f} G edges/s", flush=True)
    del cp, ri

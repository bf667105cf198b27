"""C3 (permuted R-MAT): the same keyed solve on the graph as generated vs with node
ids relabelled by descending in-degree (a host-side permutation, CSC rebuilt on
the GPU by di_csc_from_coo).  Experiment."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import diter_inputs as gen
import paper_1202_6168_b200 as di
import bench
p = gen.config("C3", 1)
src, dst = gen.rmat_coo(24, 1)
cp, ri = di.di_csc_from_coo(p.n, src, dst)
del src, dst
pol, alpha, frac, key = bench.SCHEDULES["C3"]
indeg = np.bincount(ri, minlength=p.n)
order = np.argsort(-indeg, kind="stable")          # new id k = old node order[k]
perm = np.empty(p.n, dtype=np.int32)
perm[order] = np.arange(p.n, dtype=np.int32)        # old -> new
s_old = np.repeat(np.arange(p.n, dtype=np.int32), np.diff(cp))
cp2, ri2 = di.di_csc_from_coo(p.n, perm[s_old], perm[ri])
del s_old
top = np.sort(indeg)[::-1]
print(f"in-degree share of the top 2048 rows {top[:2048].sum() / top.sum():.3f}, top 1M {top[:1 << 20].sum() / top.sum():.3f}")
for name, (c, r) in (("generated", (cp, ri)), ("relabelled", (cp2, ri2))):
    ctx = di.di_create(p.n, c, r, options=di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac,
                                                             select_key=key, profile=1))
    for _ in range(2):
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
    s = di.di_get_stats(ctx)
    print(f"{name}: solve {s['run_ms']:.1f} ms passes {s['passes']} edges {s['edges']:.3e} scatter {s['kt_scatter_ms']:.1f} "
          f"select {s['kt_select_ms']:.1f}", flush=True)
    di.di_destroy(ctx)

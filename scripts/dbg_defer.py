import numpy as np, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1202_6168_b200 as di
from test_gpu_parity import _pmat
rng = np.random.default_rng(1)
n = 6000
cols = [np.unique(rng.integers(0, n, size=int(rng.integers(1, 8)))).astype(np.int32) for i in range(n)]
deg = np.array([len(c) for c in cols]); cp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64); ri = np.concatenate(cols).astype(np.int32)
src = np.repeat(np.arange(n), deg); print("far edges", (np.abs(ri - src) > 2048).sum(), "of", len(ri))
Pm = _pmat(n, cp, ri); b = np.full(n, 0.15 / n)
for m in (-1, 1, 3):
    ctx = di.di_create(n, cp, ri, None, None, 0.85, di.default_options(far_defer=m, max_passes=1, check_interval=1))
    print("m", m, "stats far_edges", di.di_get_stats(ctx)["far_edges"])
    for k in range(6):
        s = di.di_run(ctx, 1e-15, raise_on_not_converged=False)
        H, F = di.di_get_history(ctx), di.di_get_fluid(ctx)
        st = di.di_get_stats(ctx)
        ident = np.abs(F - (b - H + Pm @ H)).sum()
        print(f"  run {k} s={s} passes {st['passes']} flushes {st['far_flushes']} |F| {np.abs(F).sum():.6e} |H| {H.sum():.6e} ident {ident:.3e}")
    di.di_destroy(ctx)

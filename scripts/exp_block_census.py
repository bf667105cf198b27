"""Per-pass census of 32-node blocks (CPU oracle, the bench schedules): how many blocks
hold no fluid at all (what a non-zero-block bitmap would let k_select skip) and how
many hold at least one node above T_p (what it must read).  C4-like = the C4 generator
and schedule at N = 1e6."""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, diter_inputs as gen, oracle, bench
for cfg, n in (("C4", 1_000_000), ("C2", None)):
    p = gen.config(cfg if cfg != "C4" else "C2", 1, n=n)
    pol, a, f, key = bench.SCHEDULES[cfg]
    P = oracle.Problem(p.n, p.col_ptr, p.row_idx, key=key)
    st = P.init(a)
    zs = []; sel = []
    while True:
        F = st.F
        nb = len(F)//32
        blk = np.abs(F[:nb*32]).reshape(nb,32).max(1)
        zs.append(float((blk == 0).mean()))
        T = st.T
        kw = P.kw.astype(np.float64) if P.kw is not None else 1.0
        key_ = np.abs(F)*kw
        bs = (key_[:nb*32].reshape(nb,32) > T).any(1)
        sel.append(float(bs.mean()))
        rc = P.snapshot(st, p.stop, pol, a, f, max_passes=1)
        if rc == oracle.OK: break
    print(cfg, "schedule", (pol,a,f,key), "passes", len(zs), "zero-block frac: mean %.4f max %.4f" % (np.mean(zs), np.max(zs)),
          "blocks with a selected node: mean %.3f min %.3f" % (np.mean(sel), np.min(sel)))

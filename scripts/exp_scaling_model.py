"""Multi-GPU model from K loopback ranks on ONE GPU (experiment; no multi-GPU box here).

Runs the bench's N > 1 configuration (ASYNC, rounds every 4 passes, remote edges as H
increments, in+out-balanced ranges, the config's schedule) as K in-process ranks on one
GPU and records what each rank would do on its own GPU: passes, scanned nodes, edges,
remote pushes, exchange rounds and bytes.  The ranks share the GPU here, so their times
mean nothing; the work split and the traffic do.  Model of the K-GPU time:

    T_K = T_1 * max_k [ s * (passes_k n_k) / (passes_1 N) + (1 - s) * (E_k + R_k) / E_1 ]
          + rounds * (max_k bytes_k per round / B_link + t_round)

with T_1, s (select share) and E_1 from the 1-GPU bench line, B_link = 450 GB/s (half the
900 GB/s per direction of NVLink 5 through NVSwitch, for an all-to-all-v) and t_round =
40 us (a grouped ncclSend/Recv, two all-reduces and the host sync of a round).

    python scripts/exp_scaling_model.py C4 248.7 0.224 2.6595e10 [out|inout]

With sweeps (MODEL_SWEEP, default bench.SWEEP[cfg]) there is no select kernel: s is
the scan's share of the sweep's algorithmic bytes (8 N of 8 N + 40 |S| + 20 E).

MODEL_MODE=p2p models DI_EXCHANGE_P2P instead: no round barrier, so each rank runs
at its own pace and the job ends at the last confirmation:

    T_K = max_k [ T_1 * compute_k + rounds_k * t_round + bytes_k / B_p2p ] + confirms * t_confirm

with B_p2p = 900 GB/s (NVLink 5 per direction; the records are stores into the
receiver's memory), t_round = 40 us (the round's host sync and small kernels) and
t_confirm = 150 us (four collectives and three merges).
"""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import diter_inputs as gen
import paper_1202_6168_b200 as di
from paper_1202_6168_b200 import dist
import bench
if os.environ.get("DITER_LIB"):
    di.LIB_PATH = os.environ["DITER_LIB"]   # experiment: another build of the library

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
T1 = float(sys.argv[2]) if len(sys.argv) > 2 else 248.7
s_sel = float(sys.argv[3]) if len(sys.argv) > 3 else 0.224
E1 = float(sys.argv[4]) if len(sys.argv) > 4 else 2.6595e10
COST = sys.argv[5] if len(sys.argv) > 5 else "inout"     # partition cost: "out" or "inout"
B_LINK, T_ROUND = 450e9, 40e-6
KS = [int(k) for k in os.environ.get("MODEL_K", "2,4,8").split(",")]
ROUND = int(os.environ.get("MODEL_ROUND_PASSES", "4"))      # bench --round-passes
REMOTE = int(os.environ.get("MODEL_REMOTE_PUSH", "1"))      # bench --remote-push
RESCALE = int(os.environ.get("MODEL_RESCALE", "1"))          # options.receive_rescale
SLEEP = int(os.environ.get("MODEL_SLEEP", "0"))              # options.p2p_sleep (0 on, -1 off)
ADAPT = int(os.environ.get("MODEL_ADAPT", "0"))              # options.adapt_rounds (ASYNC; 0 off)
P2P = os.environ.get("MODEL_MODE", "async") == "p2p"
MODE = di.DI_EXCHANGE_P2P if P2P else di.DI_EXCHANGE_ASYNC   # SYNC's di_stats.edges are global totals
B_P2P, T_CONFIRM = 900e9, 150e-6

p = gen.config(cfg, 1)
if cfg == "C3":
    src, dst = gen.rmat_coo(24, 1)
    p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
    del src, dst
pol, alpha, frac, key = bench.SCHEDULES[cfg]
alpha_k = float(os.environ.get("MODEL_ALPHA", alpha))        # schedule of the K ranks (default: 1 GPU's)
frac_k = float(os.environ.get("MODEL_FRAC", frac))
SWEEP = int(os.environ.get("MODEL_SWEEP", bench.SWEEP.get(cfg, 0)))     # options.sweep (R26) on every rank
RUN = bench.SCATTER_RUN.get(cfg, 0)
# passes of the 1-GPU solve (scan term of the model)
o1 = di.default_options(policy=pol, alpha=alpha, hybrid_frac=frac, select_key=key, sweep=SWEEP, scatter_run=RUN,
                        scatter_stripes=bench.SCATTER_STRIPES.get(cfg, 0), key_offset=bench.KEY_OFFSET.get(cfg, 0))
c1 = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, o1)
di.di_run(c1, p.stop)
P1 = di.di_get_stats(c1)["passes"]
di.di_destroy(c1)
out = {"mode": "p2p" if P2P else "async", "sweep": SWEEP, "config": cfg, "partition": COST, "round_passes": ROUND, "remote_push": REMOTE, "T1_ms": T1, "select_share": s_sel, "E1": E1, "passes_1": P1, "K": {}}
PILOT = int(os.environ.get("MODEL_PILOT", "0"))               # pilot solves whose measured work re-balances the ranges
for K, pilot in [(K, it) for K in KS for it in range(PILOT + 1)]:
    if pilot == 0:
        bounds = dist.partition_bounds(p.col_ptr, K, cost=COST, row_idx=p.row_idx)
    else:
        bounds = dist.partition_bounds_measured(p.col_ptr, K, bounds, [dist.pushes_performed(s, rh, REMOTE) for s, rh in zip(st, rho)])
        print(f"K={K} pilot {pilot}: bounds {[int(b) for b in bounds]}", flush=True)
    st = [None] * K
    err = [None] * K
    rho = [0.0] * K
    cid = dist.loopback_comm_id(f"model{cfg}{K}p{pilot}")

    def w(r):
        try:
            lcp, lri, lv, lb = dist.shard_csc(p.col_ptr, p.row_idx, p.values, p.b, bounds, r)
            rho[r] = dist.remote_fraction(lri, int(bounds[r]), int(bounds[r + 1]))
            o = di.default_options(policy=pol, alpha=alpha_k, hybrid_frac=frac_k, select_key=key,
                                   exchange_mode=MODE, check_interval=ROUND, remote_push=REMOTE,
                                   receive_rescale=RESCALE, p2p_sleep=SLEEP, sweep=SWEEP, scatter_run=RUN,
                                   adapt_rounds=ADAPT, key_offset=bench.KEY_OFFSET.get(cfg, 0))
            ctx = di.di_create_dist(r, K, cid, bounds, p.n, lcp, lri, lv, lb, p.d, o)
            di.di_run(ctx, p.stop)
            st[r] = di.di_get_stats(ctx)
            di.di_destroy(ctx)
        except Exception as e:
            err[r] = e
    t = time.perf_counter()
    th = [threading.Thread(target=w, args=(r,)) for r in range(K)]
    [x.start() for x in th]
    [x.join() for x in th]
    for e in err:
        if e is not None:
            raise e
    wall = time.perf_counter() - t
    rounds = max(s["exchanges"] for s in st)
    # conservative work term (rounds 1-2 of this model): every edge of a diffused node plus
    # every increment push, i.e. remote edges counted twice in DI_REMOTE_INCREMENT mode
    comps_cons = [s_sel * (s["passes"] * s["n_local"]) / (P1 * p.n) + (1 - s_sel) * (s["edges"] + s["remote_pushes"]) / E1
                  for s in st]
    # pushes actually performed (dist.pushes_performed): MODEL_WORK=performed (default) / conservative
    # + the increment kernel's scan of the rank's nodes at every round (col_ptr, nloc, H, H_old:
    # 28 B per node at the measured HBM copy rate), which the edge term does not hold
    inc_scan = [(s["passes"] / ROUND) * s["n_local"] * 28.0 / 6.5e12 / (T1 * 1e-3) if REMOTE else 0.0 for s in st]
    comps_perf = [s_sel * (s["passes"] * s["n_local"]) / (P1 * p.n) + (1 - s_sel) * dist.pushes_performed(s, rh, REMOTE) / E1 + x
                  for s, rh, x in zip(st, rho, inc_scan)]
    comps = comps_cons if os.environ.get("MODEL_WORK", "performed") == "conservative" else comps_perf
    comp = max(comps)
    per_round = max(s["exchanged_bytes"] for s in st) / max(1, rounds)
    if P2P:
        # ranks do not wait for each other between confirmations
        TK = max(T1 * 1e-3 * c + (s["passes"] / ROUND) * T_ROUND + s["exchanged_bytes"] / B_P2P
                 for c, s in zip(comps, st)) + max(s["confirms"] for s in st) * T_CONFIRM
    else:
        TK = T1 * 1e-3 * comp + rounds * (per_round / B_LINK + T_ROUND)
    eff = T1 * 1e-3 / (K * TK)
    out["K"][K if pilot == 0 else f"{K} pilot {pilot}"] = {"bounds": [int(b) for b in bounds], "passes": [s["passes"] for s in st], "n_local": [s["n_local"] for s in st],
                   "edges": [s["edges"] for s in st], "remote_pushes": [s["remote_pushes"] for s in st],
                   "rounds": rounds, "bytes_per_round_max": per_round,
                   "exchanged_bytes_total": sum(s["exchanged_bytes"] for s in st),
                   "compute_fraction_of_T1": comp, "compute_per_rank": comps,
                   "compute_per_rank_conservative": comps_cons, "remote_edge_share": rho,
                   "efficiency_model_conservative": T1 * 1e-3 / (K * (max(T1 * 1e-3 * c + (s["passes"] / ROUND) * T_ROUND + s["exchanged_bytes"] / B_P2P for c, s in zip(comps_cons, st)) + max(s["confirms"] for s in st) * T_CONFIRM)) if P2P else None, "T_K_model_ms": TK * 1e3,
                   "efficiency_model": eff, "confirms": [s["confirms"] for s in st],
                   "collectives": [s["collectives"] for s in st],
                   "exchange_bytes_resident": [s["exchange_bytes_resident"] for s in st],
                   "loopback_wall_s": wall, "passes_per_rank": [s["passes"] for s in st],
                   "sleep_rounds": [s["sleep_rounds"] for s in st]}
    print(f"K={K}: rounds={rounds} max bytes/round={per_round / 1e6:.1f} MB  edges sum={sum(s['edges'] for s in st):.4e} "
          f"(1 GPU {E1:.4e})  compute max/T1={comp:.3f}  T_K model={TK * 1e3:.1f} ms  efficiency={eff:.2f}", flush=True)
print(json.dumps(out))

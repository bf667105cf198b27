#!/usr/bin/env python
"""bench.py -- D-iteration diffusion sweep (arXiv 1202.6168) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A "step" is one whole solve of the hot path: di_reset (F = B, H = 0) then
di_run until |F|_1 < the config's metric target (BASELINE.json), on the
synthetic input already resident in HBM.  value = edges diffused per second
(sum of E_p over the solve / device time of di_run, CUDA events on the
library's stream), max over ranks for N > 1.

One JSON line on rank 0:
  roofline      -- the dominant kernel (k_scatter): algorithmic bytes 20 E per
                   launch / its average launch time, events recorded inside the
                   captured graph during the timed region; peak = measured HBM
                   copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  -- the CPU oracle (1 core) on a bounded sample of the same solve
  e2e           -- same metric through the public C ABI with host buffers:
                   di_create (H2D of the graph from pinned host memory) + di_run +
                   di_get_history (D2H) + di_destroy per step
  clocks        -- nvidia-smi samples taken during the timed region
--impl reference runs the oracle arm (the reference of this tier) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges diffused/s and time to |F|_1<1e-9 at 1/2/4/8 B200; % HBM roofline"

WORKLOADS = {
    "C1": "configs[0]: uniform out-degree 1..10 PageRank, N=1e3, stop |F|_1<1e-12",
    "C2": "configs[1]: web-like PageRank N=1e6 (~7.0e6 edges, 15% dangling), stop |F|_1<1e-9",
    "C3": "configs[2]: R-MAT scale 24 PageRank (ids permuted, dedup), stop |F|_1<1e-9",
    "C4": "configs[3]: web-like PageRank N=1e8 (~1.6e9 edges, 15% dangling), stop |F|_1<1e-9",
    "C5": "configs[4]: signed sparse N=1e6, 20 nnz/col, |col|_1=0.9, stop |F|_1<1e-9|B|_1",
}
L2_BYTES = 126 * 2 ** 20

# Launch configuration per workload: (policy, alpha, hybrid_frac, select_key) with
# policy 0 = GEOM / 1 = HYBRID (reading R4) and key 0 = raw |F_i|, 1 = per-edge
# |F_i|/(#out_i+1).  Tuned on B200 within the paper's
# alpha range [1.2, 2]; DESIGN.md §7 has the sweep.  Every choice is
# the same method (any order converges to the same X).
SCHEDULES = {
    "C1": (1, 1.5, 0.05, 0),
    "C2": (1, 2.0, 0.30, 1),
    "C3": (1, 1.5, 0.50, 1),
    "C4": (1, 2.0, 0.60, 1),
    "C5": (1, 2.0, 0.15, 0),
}

# options.sweep of the launch configuration: 1 = one-kernel asynchronous sweeps (the
# paper's cyclic scan with immediate diffusion, reading R26) on the large graphs --
# C4 248.7 -> 193 ms, C3 181 -> 138 ms; the small L2-resident ones keep snapshot
# passes (C2 3.7 vs 5.5 ms, C5 2.7 vs 3.8 ms).
SWEEP = {"C3": 1, "C4": 1}

# The snapshot-pass configuration of the sweep configs (select, then scatter; the
# schedule the bit-exact frontier tests pin), reported beside the headline as
# `snapshot`.
SNAPSHOT_SCHEDULES = {"C3": (1, 1.5, 0.05, 1), "C4": (1, 2.0, 0.50, 1)}

# Frontier groups (snapshot) / node spans (sweep) per dynamic grab (options.scatter_run;
# library default 2): snapshot C4 3 (248.7 vs 250.1 ms), C3 1 (181.3 vs 183.3 ms); sweeps
# C4 6 (spans after the first of a grab are prefetched: 182.2 vs 185.1 ms at 3), C3 1.
SCATTER_RUN = {"C3": 1, "C4": 6}
SNAPSHOT_SCATTER_RUN = {"C3": 1, "C4": 3}
# Ticket stripes (options.scatter_stripes; default 8): C4 sweeps 4 (193.1 vs 193.8 ms).
SCATTER_STRIPES = {"C4": 4}
# options.key_offset: under sweeps the derived per-edge key is |F_i| / (#out_i + c) (reading R27).
# Measured on C4: c = 8 with f = 0.55 reaches the target in 172.7 ms instead of 176.1 (59 sweeps,
# 2.22e10 edges) but diffuses fewer edges per second (1.285e11 vs 1.309e11) at a lower k_sweep
# fraction (0.528 vs 0.551): the headline metric is edges/s and the roofline fraction, so the
# bench keeps the paper-style key c = 1 (profiles/r04_sweep_variants.md, r04_bench_c4_key_offset8.json).
KEY_OFFSET = {}

# The raw key |F_i| > T_p (north_star's literal selection) on C4, reported beside the
# headline as `raw_key`: HYBRID alpha = 2, f = 0.15 (its best schedule).
RAW_KEY_SCHEDULE = (1, 2.0, 0.15, 0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default=None, choices=[None, "geom", "hybrid"])
    # threshold schedule T_k <- T_k / alpha (alpha in [1.2, 2], results "not
    # sensitive"); HYBRID lowers T only when |S_p| <= f N (reading R4); see SCHEDULES
    ap.add_argument("--alpha", type=float, default=None, help="default: SCHEDULES[config]")
    ap.add_argument("--hybrid-frac", type=float, default=None, help="default: SCHEDULES[config]")
    ap.add_argument("--key", type=int, default=None, choices=[0, 1, 2],
                    help="selection key 0 raw / 1 per-edge / 2 paper; default: SCHEDULES[config]")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="bound on the oracle sample for cpu_baseline / reference steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-raw-key", action="store_true",
                    help="skip the extra raw-key (|F_i| > T, north_star's literal key) C4 solve")
    ap.add_argument("--scale", type=int, default=None, help="C3 scale override (tests)")
    ap.add_argument("--n", type=int, default=None, help="node-count override (tests)")
    ap.add_argument("--pass-csv", default=None, help="write the last solve's per-pass log here")
    ap.add_argument("--dist-path", action="store_true",
                    help="tests: run the N > 1 code path (di_create_dist over NCCL) even with one rank")
    ap.add_argument("--sweep", type=int, default=None, choices=[0, 1],
                    help="options.sweep: 1 one-kernel async sweeps, 0 snapshot passes; default: SWEEP[config]")
    ap.add_argument("--no-snapshot", action="store_true",
                    help="skip the extra snapshot-pass solve reported as `snapshot` (sweep configs)")
    ap.add_argument("--far-defer", type=int, default=0,
                    help="options.far_defer (one GPU): 0 auto, -1 off, > 0 passes between far-edge flushes")
    ap.add_argument("--l2-persist", type=int, default=0,
                    help="options.l2_persist: 0 auto, -1 off, > 0 window MB (experiments)")
    ap.add_argument("--exchange", default="p2p", choices=["sync", "async", "p2p"],
                    help="multi-GPU exchange mode (DESIGN.md §6): sync = per-pass rounds, async = the paper's "
                         "send rule in bulk rounds every rank joins, p2p = the paper's send rule with records "
                         "written into the receivers' inbox rings (no collective per round; default)")
    ap.add_argument("--round-passes", type=int, default=None,
                    help="N > 1: local passes per round (default: 2 for p2p, 4 for async; DESIGN.md §6 model)")
    ap.add_argument("--remote-push", type=int, default=1, choices=[0, 1],
                    help="N > 1: 0 per diffusion, 1 H increments at rounds (NEXT f2)")
    ap.add_argument("--partition", default="out", choices=["out", "inout", "inhalf"],
                    help="edge-balanced contiguous ranges by out-edges (default: with remote edges "
                         "pushed by the senders as H increments, receiving is a cheap merge; "
                         "scripts/exp_scaling_model.py) or by in+out edges")
    ap.add_argument("--pilot-solves", type=int, default=None,
                    help="N > 1 (default 1; 0 with --dist-path on one GPU): untimed pilot solves before the warm-up; after each, the ranges are "
                         "re-balanced by the ranks' measured diffusion work (dist.partition_bounds_measured, "
                         "the paper's adaptation of the sets Omega_k applied between solves) and the "
                         "contexts are rebuilt on the new ranges")
    a = ap.parse_args()
    if a.round_passes is None:
        a.round_passes = 2 if a.exchange == "p2p" else 4
    if a.pilot_solves is None:
        # one pilot: C4 K = 8 modeled 0.56 -> 0.71 (profiles/r04_sweep_variants.md); a second does not
        # improve on it.  Both arms resolve it here, so their `config` strings agree.
        a.pilot_solves = 1 if max(a.gpus, int(os.environ.get("WORLD_SIZE", "1"))) > 1 else 0
    return a


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ inputs --

def load_problem(args):
    """Seeded synthetic input of the config (host arrays); every rank builds the
    same graph (deterministic counter-based generator), then keeps its shard."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and "DIGEN_THREADS" not in os.environ:
        os.environ["DIGEN_THREADS"] = str(max(1, (os.cpu_count() or 1) // world))
    import diter_inputs as gen
    t = time.perf_counter()
    p = gen.config(args.config, args.seed, n=args.n, scale=args.scale)
    if args.config == "C3":
        # configs[2]: CSC built from the raw R-MAT COO on the GPU (K8, di_csc_from_coo)
        import paper_1202_6168_b200 as di
        src, dst = gen.rmat_coo(args.scale or 24, args.seed)
        p.col_ptr, p.row_idx = di.di_csc_from_coo(p.n, src, dst)
        del src, dst
    log(f"[bench] generated {args.config}: n={p.n} nnz={p.nnz} in {time.perf_counter() - t:.1f}s")
    return p


def graph_residency(p, world=1):
    """(bytes resident per GPU -- graph + F + H, split over `world` ranks -- and whether
    bench flushes L2 between steps: when that is under 4x the L2)."""
    graph_bytes = 8 * (p.n + 1) + 4 * p.nnz + (8 * p.nnz if p.values is not None else 0)
    resident = (graph_bytes + 16 * p.n) / world
    return resident, resident < 4 * L2_BYTES


def bench_config(args, p, pol, world, resident, flushed):
    """The workload description both arms print (the reference arm times the oracle on
    this same configuration)."""
    par = "dp1" if world == 1 else (f"node-partition x{world} ({args.partition}-balanced ranges"
                                    f"{', re-balanced by %d pilot solves' % args.pilot_solves if args.pilot_solves else ''}, {args.exchange} exchange, "
                                    f"rounds every {args.round_passes} passes, remote edges "
                                    f"{'as H increments' if args.remote_push else 'per diffusion'})")
    return {"workload": WORKLOADS[args.config], "n": p.n, "nnz": p.nnz,
            "stop": p.stop, "policy": "geom" if pol == 0 else "hybrid", "seed": args.seed,
            "alpha": args.alpha, "hybrid_frac": args.hybrid_frac,
            "select_key": ["raw", "per-edge", "paper"][args.key],
            "scatter_run": SCATTER_RUN.get(args.config, 2),
            "scatter_stripes": SCATTER_STRIPES.get(args.config, 8),
            "key_offset": KEY_OFFSET.get(args.config, 1) if args.sweep and args.key == 1 else 1,
            "passes": ("one-kernel asynchronous sweeps (options.sweep = 1, reading R26)"
                       if args.sweep and (world == 1 or args.exchange != "sync")
                       else "snapshot passes (select, then scatter)"),
            "parallelism": par,
            "l2": ("flushed between steps (252 MB write)" if flushed else
                   f"inputs ({resident / 1e9:.1f} GB resident per GPU) larger than L2 (126 MB)")}


def policy_of(args):
    """Fill args.alpha / hybrid_frac / key from SCHEDULES where not given; return the policy."""
    pol, alpha, frac, key = SCHEDULES[args.config]
    if args.sweep is None:
        args.sweep = SWEEP.get(args.config, 0)
    if args.alpha is None:
        args.alpha = alpha
    if args.hybrid_frac is None:
        args.hybrid_frac = frac
    if args.key is None:
        args.key = key
    if args.policy == "geom":
        return 0
    if args.policy == "hybrid":
        return 1
    return pol


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first sample so
            # that a short timed region (C2: ~20 ms) is not left without one
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ cpu baseline --

_ORACLE_PROBLEM = {}
ORACLE_CORE = 0     # the oracle's one pinned host core


def oracle_sample(p, policy_geom: bool, seconds: float, state=None, alpha=1.5, hybrid_frac=0.05, key=0):
    """Time the CPU oracle (as it stands, 1 thread) on snapshot passes of the same
    solve until `seconds` elapse; returns (edges, secs, passes, state)."""
    import oracle
    if key not in _ORACLE_PROBLEM:        # key weights are setup, not timed (like di_create)
        _ORACLE_PROBLEM[key] = oracle.Problem(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, key=key)
    P = _ORACLE_PROBLEM[key]
    st = state or P.init(alpha)
    pol = oracle.GEOM if policy_geom else oracle.HYBRID
    e0, p0 = st.edges, st.passes
    edges = passes = 0
    # one core, like `taskset -c <core>`: pid 0 = this thread
    old_aff = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {ORACLE_CORE if ORACLE_CORE in old_aff else min(old_aff)})
    try:
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            rc = P.snapshot(st, p.stop, pol, alpha, hybrid_frac, max_passes=1)
            if rc == oracle.OK:
                # the solve is done (small configs finish within one sample): start the
                # same solve again from F = B so that the sample keeps doing real passes
                edges += st.edges - e0
                passes += st.passes - p0
                st = P.init(alpha)
                e0, p0 = 0, 0
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old_aff)
    return edges + st.edges - e0, dt, passes + st.passes - p0, st


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_cpu():
    """CPU model and logical core count of the host the oracle runs on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model}, nproc {os.cpu_count()}"


def ncu_traffic(config, kernel="k_scatter"):
    """(DRAM bytes read + written per launch of `kernel`, source): the mean over every
    launch of one solve of this config, measured by ncu (scripts/ncu_traffic.py ->
    profiles/ncu_traffic.json; cold-cache serialised replays).  (None, why) if the
    config has no capture of that kernel."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)[config]
        if d.get("kernel", "k_scatter") != kernel:
            return None, f"no ncu capture of {kernel} on this config"
        return float(d["mean_dram_bytes_per_launch"]), (
            f"ncu dram__bytes_read.sum + dram__bytes_write.sum, mean over the {d['launches']} {kernel} "
            f"launches of one {config} solve (profiles/ncu_traffic.json; cold-cache replays)")
    except Exception:
        return None, "no ncu capture of this config"


# -------------------------------------------------------------- reference arm --

def run_reference(args, rank, world):
    """The oracle arm (this tier's reference): rank 0 only, each step one bounded
    sample of the same solve on the host cores."""
    if rank != 0:
        return
    p = load_problem(args)
    geom = policy_of(args) == 0
    per = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    st = None
    for _ in range(args.warmup):
        _, _, _, st = oracle_sample(p, geom, per, st, args.alpha, args.hybrid_frac, args.key)
    edges, secs, passes = 0, 0.0, 0
    for _ in range(args.steps):
        e, dt, np_, st = oracle_sample(p, geom, per, st, args.alpha, args.hybrid_frac, args.key)
        edges += e
        secs += dt
        passes += np_
    v = edges / secs if secs > 0 else 0.0
    sample = (f"{passes} snapshot passes of the {args.config} solve (continued across steps, restarted "
              f"from F = B when it converges; ~{per:.1f}s per step), full graph")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": bench_config(args, p, policy_of(args), world, *graph_residency(p, world)),
           "cpu_baseline": {"value": v, "unit": "edges/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
                            "pinned_core": ORACLE_CORE, "sample": sample},
           "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ our arm --

def make_ctx(args, p, opts, di, rank, world, comm_id, bounds, host=None):
    """One GPU: di_create; N ranks: di_create_dist on this rank's shard (NCCL)."""
    cp, ri, vv, bb = host if host is not None else (p.col_ptr, p.row_idx, p.values, p.b)
    if world == 1 and not args.dist_path:
        return di.di_create(p.n, cp, ri, vv, bb, p.d, opts)
    return di.di_create_dist(rank, world, comm_id, bounds, p.n, cp, ri, vv, bb, p.d, opts)


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1202_6168_b200 as di
    from paper_1202_6168_b200 import dist as dd

    torch.cuda.set_device(local_rank)
    dist = world > 1 or args.dist_path
    if dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                                             rank=rank, world_size=world)
    p = load_problem(args)
    pol = policy_of(args)
    mode = {"sync": di.DI_EXCHANGE_SYNC, "async": di.DI_EXCHANGE_ASYNC, "p2p": di.DI_EXCHANGE_P2P}[args.exchange]
    # N > 1 (ASYNC): exchange rounds every 4 passes, remote edges pushed as H
    # increments at the rounds (NEXT f2), receive-side T rescale --
    # DESIGN.md §6 "Multi-GPU" has the loopback measurements behind these choices
    dist_kw = dict(check_interval=args.round_passes, remote_push=args.remote_push) if dist else {}
    opts = di.default_options(policy=pol, device=local_rank, profile=0, exchange_mode=mode,
                              alpha=args.alpha, hybrid_frac=args.hybrid_frac, select_key=args.key,
                              scatter_run=SCATTER_RUN.get(args.config, 0), l2_persist=args.l2_persist,
                              far_defer=args.far_defer, sweep=args.sweep,
                              scatter_stripes=SCATTER_STRIPES.get(args.config, 0),
                              key_offset=KEY_OFFSET.get(args.config, 0), **dist_kw)
    comm_id, bounds, shard = None, None, None
    if dist:
        bounds = dd.partition_bounds(p.col_ptr, world, cost=args.partition, row_idx=p.row_idx)
        comm_id = dd.nccl_comm_id()
        shard = dd.shard_csc(p.col_ptr, p.row_idx, p.values, p.b, bounds, rank)
    t = time.perf_counter()
    ctx = make_ctx(args, p, opts, di, rank, world, comm_id, bounds, shard)
    log(f"[bench] rank {rank} create {time.perf_counter() - t:.2f}s")
    for it in range(args.pilot_solves if dist else 0):
        # pilot solve on the current ranges; every rank derives the same new bounds from
        # the gathered work (pushes performed: dist.pushes_performed)
        torch.distributed.barrier()
        di.di_run(ctx, p.stop)
        s = di.di_get_stats(ctx)
        rho = dd.remote_fraction(shard[1], int(bounds[rank]), int(bounds[rank + 1]))
        mine = torch.tensor([dd.pushes_performed(s, rho, args.remote_push)], dtype=torch.float64, device="cuda")
        works = [torch.zeros_like(mine) for _ in range(world)]
        torch.distributed.all_gather(works, mine)
        di.di_destroy(ctx)
        bounds = dd.partition_bounds_measured(p.col_ptr, world, bounds, [float(w.item()) for w in works])
        comm_id = dd.nccl_comm_id()
        shard = dd.shard_csc(p.col_ptr, p.row_idx, p.values, p.b, bounds, rank)
        ctx = make_ctx(args, p, opts, di, rank, world, comm_id, bounds, shard)
        log(f"[bench] rank {rank} pilot {it + 1}: bounds {[int(b) for b in bounds]}")
    resident, flushed = graph_residency(p, world)
    flush = None
    if flushed:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")

    def step():
        if flush is not None:
            flush.fill_(1.0)                     # evict L2 between timed solves
            torch.cuda.synchronize()
        di.di_reset(ctx)
        if dist:
            torch.distributed.barrier()
        di.di_run(ctx, p.stop)
        return di.di_get_stats(ctx)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    # di_stats counters run since create (di_reset restarts the solve counters); the
    # launch count is per di_run (run_kernel_launches), summed over the timed steps
    tot = {"run_ms": 0.0, "edges": 0, "passes": 0, "kt_scatter_ms": 0.0, "kt_select_ms": 0.0,
           "kt_finalize_ms": 0.0, "scatter_bytes": 0, "alg_bytes": 0, "run_kernel_launches": 0,
           "nodes": 0, "dangling": 0, "exchanged_bytes": 0, "exchanges": 0}
    coll0 = di.di_get_stats(ctx)
    wall0 = time.perf_counter()
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            s = step()
            for k in tot:
                tot[k] += s[k]
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    coll1 = di.di_get_stats(ctx)
    # Kernel durations for the roofline: the same K steps again with CUDA events
    # between the pass kernels (di_set_profile).  The events split the captured pass
    # graph and cost ~25 us of device time per pass, so `value` is timed without them.
    di.di_set_profile(ctx, True)
    if dist:
        torch.distributed.barrier()
    prof = {k: 0 for k in ("run_ms", "kt_scatter_ms", "kt_select_ms", "kt_finalize_ms", "scatter_bytes",
                           "passes", "edges", "alg_bytes", "nodes", "dangling")}
    for _ in range(args.steps):
        s = step()
        for k in prof:
            prof[k] += s[k]
    torch.cuda.synchronize()
    di.di_set_profile(ctx, False)
    if args.pass_csv and rank == 0:
        lg = di.di_get_pass_log(ctx)
        with open(args.pass_csv, "w") as fcsv:
            fcsv.write(",".join(lg.dtype.names) + "\n")
            for row in lg:
                fcsv.write(",".join(str(x) for x in row) + "\n")
    r_final = di.di_get_residual(ctx)
    assert r_final < p.stop, r_final
    run_ms_rank = tot["run_ms"]
    edges_all = tot["edges"]
    if dist:   # max time over ranks, work summed over ranks
        t_ = torch.tensor([run_ms_rank], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t_, op=torch.distributed.ReduceOp.MAX)
        e_ = torch.tensor([float(tot["edges"]), float(tot["exchanged_bytes"])], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(e_)
        tot["run_ms"] = float(t_.item())
        # di_stats.edges is the rank's own count under ASYNC but the global count under
        # SYNC (pass totals are all-reduced every pass): sum only the former
        edges_all = int(e_[0].item()) if mode != di.DI_EXCHANGE_SYNC else int(tot["edges"])
        xbytes_all = int(e_[1].item())
    run_s = tot["run_ms"] / 1e3
    value = edges_all / run_s
    peak, peak_kind = measured_peaks()
    sweep = bool(args.sweep) and (not dist or mode != di.DI_EXCHANGE_SYNC)
    # Dominant kernel: k_scatter (snapshot passes: algorithmic bytes 20 E + 16 per
    # non-dangling diffused node, di_stats.scatter_bytes) or k_sweep (async sweeps: the
    # whole pass, SURVEY §8d's B_p = 8 N + 40 |S_p| + 20 E_p, di_stats.alg_bytes);
    # the "scatter" span of the profile events covers it (+ k_scatter_hubs if any).
    kbytes = prof["alg_bytes"] if sweep else prof["scatter_bytes"]
    kname = "k_sweep" if sweep else "k_scatter"
    scat_gbs = kbytes / (prof["kt_scatter_ms"] / 1e3) / 1e9
    n_launch = prof["passes"]                      # executed k_scatter / k_sweep launches
    traffic, traffic_src = ncu_traffic(args.config, kname)
    kt_sum = prof["kt_scatter_ms"] + prof["kt_select_ms"] + prof["kt_finalize_ms"]
    shares = ({"k_sweep": prof["kt_scatter_ms"] / kt_sum, "k_finalize": (prof["kt_finalize_ms"] + prof["kt_select_ms"]) / kt_sum}
              if sweep else
              {"k_select": prof["kt_select_ms"] / kt_sum, "k_scatter": prof["kt_scatter_ms"] / kt_sum,
               "k_finalize": prof["kt_finalize_ms"] / kt_sum})
    roofline = {"bound": "hbm", "achieved": scat_gbs, "peak": peak, "unit": "GB/s",
                "frac": scat_gbs / peak, "frac_of_nominal_8TBps": scat_gbs / 8000.0, "traffic": traffic,
                "traffic_source": traffic_src,
                "kernel": kname, "peak_kind": peak_kind,
                "bytes_per_launch": kbytes / max(1, n_launch),
                "bytes_model": ("8 N + 40 |S_p| + 20 E_p per sweep (SURVEY §8d B_p; F scan, diffused node, edge)"
                                if sweep else "20 E_p + 16 (|S_p| - dangling) per scatter (row idx + F RMW, col_ptr pair)"),
                "avg_launch_ms": prof["kt_scatter_ms"] / max(1, n_launch),
                "share_of_step": prof["kt_scatter_ms"] / max(1e-9, run_ms_rank),
                "kernel_shares": shares,
                "timing": f"CUDA events between the pass kernels on the library stream over {args.steps} "
                          f"more steps right after the timed region (rank {rank}); their ms_per_step "
                          f"{prof['run_ms'] / args.steps:.3f} includes the events' own cost",
                "path_alg_GBps": tot["alg_bytes"] / (run_ms_rank / 1e3) / 1e9}
    # ---- the snapshot-pass configuration on the same graph (extra key, sweep configs)
    snapshot = None
    if sweep and not args.no_snapshot and args.config in SNAPSHOT_SCHEDULES:
        snapshot = run_snapshot(args, p, opts, di)
    # ---- the raw key on the same graph (extra key; the headline keeps the per-edge key)
    raw = None
    if not dist and args.config == "C4" and args.key != 0 and not args.no_raw_key:
        raw = run_raw_key(args, p, opts, di, torch)
    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, p, opts, di, torch, rank, world, comm_id, bounds, shard, dist)
    # ---- cpu baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        e, dt, npass, st = oracle_sample(p, pol == di.DI_POLICY_GEOM, args.cpu_seconds, None,
                                         args.alpha, args.hybrid_frac, args.key)
        rate = e / dt if dt > 0 else None
        cpu = {"value": rate, "unit": "edges/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
               "pinned_core": ORACLE_CORE,
               "sample": f"first {npass} snapshot passes ({e} edges) of the same {args.config} solve "
                         f"on the full graph, {dt:.1f}s on 1 pinned host core",
               # the whole solve at the sampled rate (the first passes are the densest)
               "time_to_target_s_est": (edges_all / args.steps) / rate if rate else None}
    clocks = clk.summary()
    st_last = di.di_get_stats(ctx)
    l2_window = (f"{st_last['l2_window_bytes'] / 2**20:.0f} MB persisting over F rows from "
                 f"{st_last['l2_window_row']} (options.l2_persist auto)") if st_last["l2_window_bytes"] else "none"
    # Second roof of the scatter: every edge is one fp64 RED (or shared-memory ATOMS)
    # lane, and the SM issues at most one such lane per ~1.29 cycles (B300_MICROARCH
    # "REDG spread"; 229 G lanes/s measured on this B200, profiles/r01_red_microbench.txt),
    # whatever the target -- so edges/s inside k_scatter against that issue rate.
    sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    red_peak = n_sm * sm_mhz * 1e6 / 1.29
    red_ach = prof["edges"] / (prof["kt_scatter_ms"] / 1e3)
    roofline["atomic_issue"] = {"bound": "lsu_atomic", "achieved": red_ach / 1e9, "peak": red_peak / 1e9,
                                "unit": "G lanes/s", "frac": red_ach / red_peak,
                                "peak_source": f"{n_sm} SMs x {sm_mhz:.0f} MHz / 1.29 cycles per RED lane"}
    di.di_destroy(ctx)
    out = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot["run_ms"] / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": bench_config(args, p, pol, world, resident, flush is not None),
           "l2_window": l2_window,
           "time_to_target_ms": tot["run_ms"] / args.steps,
           "passes_per_solve": tot["passes"] / args.steps,
           "normalized_iterations": edges_all / args.steps / p.nnz,
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "raw_key": raw, "snapshot": snapshot,
           # our kernels in the timed steps: di_run's (graph nodes counted) + di_reset's k_init_state
           "gpu_launches": int(tot["run_kernel_launches"]) + args.steps,
           "clocks": clocks,
           "nvlink_bytes_per_round": (xbytes_all / max(1, tot["exchanges"])) if dist else 0,
           "nvlink_bytes_per_solve": (xbytes_all / args.steps) if dist else 0,
           # fabric collectives (all-reduce, all-to-all) and P2P confirmations per timed solve, rank 0
           "collectives_per_solve": (coll1["collectives"] - coll0["collectives"]) / args.steps if dist else 0,
           "confirms_per_solve": (coll1["confirms"] - coll0["confirms"]) / args.steps if dist else 0,
           # untimed pilot solves whose measured work re-balanced the ranges before the warm-up
           "pilot_solves": args.pilot_solves if dist else 0,
           "exchange_bytes_resident": coll1["exchange_bytes_resident"] if dist else 0,
           "wall_s_timed": wall}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def run_snapshot(args, p, opts, di):
    """The sweep config in snapshot passes (select, then scatter): its own context and
    schedule (SNAPSHOT_SCHEDULES), 1 warm-up + min(steps, 3) timed solves, same timing."""
    import copy
    pol, alpha, frac, key = SNAPSHOT_SCHEDULES[args.config]
    o = copy.copy(opts)
    o.policy, o.alpha, o.hybrid_frac, o.select_key, o.profile, o.sweep = pol, alpha, frac, key, 0, 0
    o.scatter_run, o.scatter_stripes = SNAPSHOT_SCATTER_RUN.get(args.config, 0), 0
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, o)
    try:
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
        steps = max(1, min(args.steps, 3))
        ms = edges = passes = sb = 0
        for _ in range(steps):
            di.di_reset(ctx)
            di.di_run(ctx, p.stop)
            st = di.di_get_stats(ctx)
            ms += st["run_ms"]
            edges += st["edges"]
            passes += st["passes"]
    finally:
        di.di_destroy(ctx)
    return {"passes": "snapshot (select, then scatter)", "policy": "hybrid", "alpha": alpha,
            "hybrid_frac": frac, "select_key": ["raw", "per-edge", "paper"][key], "steps": steps,
            "time_to_target_ms": ms / steps, "edges_per_s": edges / (ms / 1e3),
            "passes_per_solve": passes / steps, "normalized_iterations": edges / steps / p.nnz}


def run_raw_key(args, p, opts, di, torch):
    """C4 with the raw key |F_i| > T_p: its own context (key weights are create-time),
    1 warm-up + min(steps, 3) timed solves, same timing as the headline."""
    import copy
    pol, alpha, frac, key = RAW_KEY_SCHEDULE
    o = copy.copy(opts)
    o.policy, o.alpha, o.hybrid_frac, o.select_key, o.profile = pol, alpha, frac, key, 0
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, p.values, p.b, p.d, o)
    try:
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
        steps = max(1, min(args.steps, 3))
        ms = edges = passes = 0
        for _ in range(steps):
            di.di_reset(ctx)
            di.di_run(ctx, p.stop)
            st = di.di_get_stats(ctx)
            ms += st["run_ms"]
            edges += st["edges"]
            passes += st["passes"]
    finally:
        di.di_destroy(ctx)
    return {"select_key": "raw", "policy": "hybrid", "alpha": alpha, "hybrid_frac": frac, "steps": steps,
            "time_to_target_ms": ms / steps, "edges_per_s": edges / (ms / 1e3),
            "passes_per_solve": passes / steps, "normalized_iterations": edges / steps / p.nnz}


def run_e2e(args, p, opts, di, torch, rank=0, world=1, comm_id=None, bounds=None, shard=None, dist=False):
    """Same metric through di_create/di_run/di_get_history with pinned host buffers."""
    src = shard if shard is not None else (p.col_ptr, p.row_idx, p.values, p.b)
    pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() if a is not None else None for a in src]
    n_loc = int(len(src[0]) - 1)
    H = torch.empty(n_loc, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in pin if t is not None)
    d2h = n_loc * 8
    import copy
    o2 = copy.copy(opts)
    o2.profile = 0

    def one():
        # an ncclUniqueId initialises one communicator only: every distributed
        # context gets a fresh one (collective over the torch process group)
        cid = comm_id
        if dist:
            from paper_1202_6168_b200 import dist as dd
            cid = dd.nccl_comm_id()
        ctx = make_ctx(args, p, o2, di, rank, world, cid, bounds, pin)
        di.di_run(ctx, p.stop)
        di.di_get_history(ctx, H)
        e = di.di_get_stats(ctx)["edges"]
        di.di_destroy(ctx)
        return e

    one()                                          # warm (allocator, module load)
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    edges = 0
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        edges += one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if dist:
        t_ = torch.tensor([dt, float(edges)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t_[:1], op=torch.distributed.ReduceOp.MAX)
        e_ = t_[1:].clone()
        if opts.exchange_mode != di.DI_EXCHANGE_SYNC:      # SYNC edge counts are global already
            torch.distributed.all_reduce(e_)
        dt, edges = float(t_[0].item()), float(e_[0].item())
    return {"value": edges / dt, "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "ms_per_step": dt * 1e3 / steps}


def launch_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-exec this command under
    torch.distributed.run with N ranks on this node (one per GPU), or fail loudly
    when the node has fewer than N GPUs -- never a 1-rank run labelled N."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"[bench] --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {have}")
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("[bench] " + " ".join(cmd))
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            log(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}")
            sys.exit(2)
    else:
        world = 1
    if args.impl == "reference":
        # the oracle arm runs on rank 0's host cores only; without torchrun it still
        # reports the job's N
        run_reference(args, rank, max(world, args.gpus))
        return
    if args.gpus > 1 and world == 1:
        launch_ranks(args)
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

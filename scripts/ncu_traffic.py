"""DRAM traffic of every k_scatter launch of one solve, from an ncu metrics CSV.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:k_scatter --clock-control none --csv --log-file L.csv \
        python scripts/profile_run.py --config C4 --max-passes 1000 --pass-csv P.csv
    python scripts/ncu_traffic.py --config C4 --launches L.csv --passes P.csv

Writes profiles/ncu_traffic.json[config]: per-launch DRAM bytes (read + write) of
the first `passes` k_scatter launches (the ones that did work; graph passes after
convergence exit at once), their algorithmic bytes 20 E_p + 16 (|S_p| - dangling_p)
(+ 8 E_p signed), and the means bench.py reports as roofline.traffic.
ncu replays each kernel with a cold L2 and serialised, so the means are an upper
bound on what the live solve moves.
"""
import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--launches", required=True)
ap.add_argument("--passes", required=True)
ap.add_argument("--signed", action="store_true")
ap.add_argument("--kernel", default="k_scatter", choices=["k_scatter", "k_sweep"])
ap.add_argument("--n", type=int, default=None, help="nodes (k_sweep: 8 N scan bytes per launch)")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
ap.add_argument("--source", default="")
a = ap.parse_args()

# ncu --csv: one row per (kernel launch, metric); the header row starts with "ID"
launches = {}
order = []
with open(a.launches) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if a.kernel not in r["Kernel Name"] or "hubs" in r["Kernel Name"]:
        continue
    k = r["ID"]
    if k not in launches:
        launches[k] = {}
        order.append(k)
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
             "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
    launches[k][r["Metric Name"]] = v * scale

with open(a.passes) as f:
    passes = list(csv.DictReader(f))
n = len(passes)
rows = [launches[k] for k in order[:n]]
if len(rows) < n:
    raise SystemExit(f"{len(rows)} {a.kernel} launches in the CSV, {n} passes in the log")
per_edge = 28 if a.signed else 20
dram, alg, dur = [], [], []
for p, r in zip(passes, rows):
    E, S, D = int(p["edges"]), int(p["frontier"]), int(p["dangling"])
    # k_sweep: the whole pass, SURVEY §8d B_p = 8 N + 40 |S_p| + 20 E_p (+ 8 E_p signed)
    alg.append(8 * a.n + 40 * S + per_edge * E if a.kernel == "k_sweep" else per_edge * E + 16 * (S - D))
    dram.append(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"])
    dur.append(r.get("gpu__time_duration.sum", 0.0))
out = {}
if os.path.exists(a.out):
    with open(a.out) as f:
        out = json.load(f)
out[a.config] = {
    "kernel": a.kernel,
    "_source": a.source or f"ncu metrics of every {a.kernel} launch of one {a.config} solve "
                            "(scripts/profile_run.py, bench launch configuration), cold-cache replays",
    "launches": n,
    "mean_dram_bytes_per_launch": sum(dram) / n,
    "mean_alg_bytes_per_launch": sum(alg) / n,
    "traffic_over_algorithmic": sum(dram) / sum(alg),
    "ncu_scatter_ms_per_solve": sum(dur) * 1e3,
    "per_launch": [{"pass": int(p["pass"]), "alg_bytes": x, "dram_bytes": y, "us": t * 1e6}
                   for p, x, y, t in zip(passes, alg, dram, dur)],
}
with open(a.out, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out[a.config].items() if k != "per_launch"}, indent=1))

"""bench.py's JSON line on a GPU (short C2 run): every key of the contract the driver
reads, with sane values -- a guard against breaking it while changing the bench."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C2", "--steps", "2",
                          "--warmup", "3", "--cpu-seconds", "2"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "traffic_source"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] == 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 8 * d["config"]["n"]
    # launches of the timed steps only: per solve at least select + scatter + finalize per
    # pass, at most one captured graph (16 passes) of overrun plus the per-run kernels
    per = d["gpu_launches"] / d["steps"]
    assert 3 * d["passes_per_solve"] <= per <= 3 * (d["passes_per_solve"] + 16) + 16, (per, d["passes_per_solve"])
    assert c["pinned_core"] >= 0 and "l2_window" in d
    assert set(("sm_mhz", "sm_max_mhz", "reasons")) <= set(d["clocks"])


@pytest.mark.parametrize("exchange", ["p2p", "async"])
def test_bench_distributed_path_one_rank(exchange):
    """bench.py's N > 1 code path on one GPU (--dist-path: di_create_dist over a real
    one-rank NCCL communicator made through torch.distributed): the NCCL fabric's
    collectives run, the exchange mode's stats reach the line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C2", "--steps", "2",
                          "--warmup", "3", "--cpu-seconds", "1", "--dist-path", "--exchange", exchange,
                          "--no-cpu-baseline"] + (["--pilot-solves", "1"] if exchange == "p2p" else []),
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["collectives_per_solve"] > 0 and d["exchange_bytes_resident"] > 0
    if exchange == "p2p":
        # the pilot solve's re-balancing ran (one rank: the range stays [0, n)) and is reported
        assert "pilot 1: bounds [0, 1000000]" in out.stderr and d["pilot_solves"] == 1
        assert d["confirms_per_solve"] >= 1
        assert d["collectives_per_solve"] == 1 + 4 * d["confirms_per_solve"]
    assert d["e2e"]["value"] > 0


def test_bench_line_sweep_config():
    """The sweep launch configuration (C4 shape, shrunk): k_sweep is the roofline kernel,
    its bytes follow SURVEY §8d's B_p, launches are one sweep + one finalize per pass, and
    the snapshot-pass solve is reported beside it."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C4", "--n", "4000000",
                          "--steps", "2", "--warmup", "3", "--cpu-seconds", "1", "--no-raw-key"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    r = d["roofline"]
    assert r["kernel"] == "k_sweep" and "k_sweep" in r["kernel_shares"] and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert "sweeps" in d["config"]["passes"]
    per = d["gpu_launches"] / d["steps"]
    assert 2 * d["passes_per_solve"] <= per <= 2 * (d["passes_per_solve"] + 16) + 16, (per, d["passes_per_solve"])
    s = d["snapshot"]
    assert s["time_to_target_ms"] > 0 and s["passes_per_solve"] > 0

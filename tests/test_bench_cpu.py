"""bench.py's host-side pieces on CPU: the reference arm (the oracle, this tier's
reference) prints one contract line and keeps doing real passes on a config whose
solve ends inside one sample; helper outputs are well formed."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_line_on_small_config():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "3", "--cpu-seconds", "5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    # C1's whole solve takes milliseconds: the sample restarts it instead of timing nothing
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert "nproc" in d["cpu_baseline"]["host"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_helpers():
    import bench
    peak, kind = bench.measured_peaks()
    assert peak > 1000 and kind in ("measured", "fallback")
    assert "nproc" in bench.host_cpu()
    # measured per-launch DRAM bytes of a committed ncu capture, or None with a reason
    t, src = bench.ncu_traffic("C4")
    assert (t is None and src) or (1e8 < t < 3e10 and "ncu" in src)
    t, src = bench.ncu_traffic("no-such-config")
    assert t is None and src


def test_gpus_flag_fails_loudly_without_gpus():
    """--gpus N > 1 outside torchrun re-executes under torch.distributed.run with N ranks,
    or exits non-zero when the node has fewer GPUs: never a 1-rank line labelled N."""
    import torch
    if torch.cuda.device_count() >= 2:
        return
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "needs 2 GPUs" in out.stderr
    assert out.stdout.strip() == ""


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in out.stderr

"""The C boundary used from C: tests/c/abi_consumer.c compiled with gcc against
include/diter.h and linked to the in-tree libditer.so (CPU: it builds and links;
GPU: it runs and meets the cycle's closed form and the error bound's equality)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1202_6168_b200")
SRC = os.path.join(ROOT, "tests", "c", "abi_consumer.c")


def _build(tmp_path):
    exe = str(tmp_path / "abi_consumer")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-lditer", f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_consumer_builds_and_links(tmp_path):
    exe = _build(tmp_path)
    # every symbol it uses resolves against the in-tree library
    out = subprocess.run(["ldd", exe], capture_output=True, text=True)
    assert "libditer.so" in out.stdout and "not found" not in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1000, 1_000_003])
def test_c_consumer_runs(tmp_path, n):
    exe = _build(tmp_path)
    out = subprocess.run([exe, str(n)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok=1" in out.stdout

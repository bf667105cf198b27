"""DI_EXCHANGE_P2P across PROCESSES on one GPU: each rank a separate process, the
collectives over the shared-memory fabric, every peer window mapped with
cudaIpcOpenMemHandle -- the code path of an 8-GPU box minus NVLink itself (NCCL
refuses two ranks on one device).  No kernel waits on another rank; the ranks'
kernels just time-share the GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

import diter_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_across_processes_ipc(tmp_path, world):
    n = 200_000
    name = f"ipc{os.getpid()}w{world}"
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), str(r), str(world),
                               name, str(n), str(tmp_path / f"r{r}.npz")],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(world)]
    errs = []
    for pr in procs:
        try:
            _, e = pr.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            pr.kill()
            _, e = pr.communicate()
        errs.append((pr.returncode, e[-2000:]))
    assert all(rc == 0 for rc, _ in errs), errs
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    H = np.concatenate([o["H"] for o in outs])
    F = np.concatenate([o["F"] for o in outs])
    p = gen.config("C2", 2, n=n)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * 0.15 * 0.15).H
    assert np.abs(H - X).sum() <= 1e-8 * 0.15
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(ledger - 0.15) <= 1e-12 * 0.15
    for o in outs:
        assert float(o["r"]) < p.parity_stop
        assert int(o["run_coll"]) == 1 + 4 * int(o["confirms"]) and int(o["confirms"]) >= 1
        assert int(o["exchanged"]) > 0

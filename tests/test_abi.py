"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/diter.h declares, fills default options, and its host-side helper
di_partition_cb matches the oracle bit for bit."""
import os
import re

import numpy as np
import pytest

import diter_inputs as gen
import oracle
import paper_1202_6168_b200 as di

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "diter.h")).read()
    return sorted(set(re.findall(r"DI_API\s+[\w\s\*]*?\b(di_\w+)\s*\(", hdr)))


def test_header_declares_binding_exports():
    assert declared_symbols() == sorted(di.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = di.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_default_options():
    o = di.default_options()
    assert o.policy == di.DI_POLICY_HYBRID and o.alpha == 1.5 and o.hybrid_frac == 0.05
    assert o.check_interval == 16 and o.max_passes == 1_000_000 and o.device == -1


def test_struct_sizes_match_header():
    """The ctypes layouts equal the structs compiled into libditer.so (no GPU needed)."""
    import ctypes
    lib = di.load_library()
    assert ctypes.sizeof(di.di_options) == lib.di_struct_size(0)
    assert ctypes.sizeof(di.di_stats) == lib.di_struct_size(1)
    assert ctypes.sizeof(di.di_pass_log) == lib.di_struct_size(2) == 88
    assert lib.di_struct_size(3) == 0


@pytest.mark.parametrize("K", [1, 2, 3, 4, 8])
def test_partition_cb_matches_oracle(K):
    cp, _ = gen.web_graph(100_000, 3)
    for cost in (cp, cp + np.arange(len(cp), dtype=np.int64)):
        np.testing.assert_array_equal(di.di_partition_cb(cost, K), oracle.partition_cb(cost, K))


def test_partition_cb_edge_cases():
    # all-zero cost: ranges forced non-empty
    cost = np.zeros(9, dtype=np.int64)
    np.testing.assert_array_equal(di.di_partition_cb(cost, 4), oracle.partition_cb(cost, 4))
    # one huge node
    cost = np.concatenate([[0], np.cumsum([1000, 1, 1, 1, 1])]).astype(np.int64)
    np.testing.assert_array_equal(di.di_partition_cb(cost, 3), oracle.partition_cb(cost, 3))
    np.testing.assert_array_equal(di.di_partition_cb(cost, 5), [0, 1, 2, 3, 4, 5])
    with pytest.raises(di.DiError):
        di.di_partition_cb(cost, 6)


def test_library_then_torch_import_order():
    """libditer links the NCCL torch loads (rpath to the nvidia-nccl wheel): loading
    libditer first must not break a later `import torch` (an older system libnccl
    loaded first left libtorch_cuda without ncclDevCommCreate)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1202_6168_b200 as di; "
            "di.load_library(); import torch; print('ok')") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


def test_partition_bounds_measured():
    """Pilot re-balancing of the ranges (dist.partition_bounds_measured): equal work per
    stored edge reproduces the Cost-Balanced split; a rank with k times the work per edge
    keeps 1/K of the measured work; K may differ from the pilot's; bad input is rejected."""
    from paper_1202_6168_b200 import dist as dd
    rng = np.random.default_rng(5)
    deg = rng.integers(0, 30, 20_000)
    cp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    b = dd.partition_bounds(cp, 4)
    stored = np.diff(cp[b]).astype(float)
    np.testing.assert_array_equal(dd.partition_bounds_measured(cp, 4, b, stored), b)
    np.testing.assert_array_equal(dd.partition_bounds_measured(cp, 4, b, 3.5 * stored), b)
    work = stored * np.array([3.0, 1.0, 1.0, 2.0])
    nb = dd.partition_bounds_measured(cp, 4, b, work)
    dens = np.repeat(np.array([3.0, 1.0, 1.0, 2.0]), np.diff(b))
    wcum = np.concatenate([[0.0], np.cumsum(deg * dens)])
    for k in range(1, 4):
        assert abs(wcum[nb[k]] / wcum[-1] - k / 4) < 2e-3
    nb2 = dd.partition_bounds_measured(cp, 2, b, work)         # pilot on 4 ranks, 2 new ranges
    assert abs(wcum[nb2[1]] / wcum[-1] - 0.5) < 2e-3
    for bad in ([1.0, 1.0], [0.0, 0.0, 0.0, 0.0], [1.0, -1.0, 1.0, 1.0]):
        with pytest.raises(ValueError):
            dd.partition_bounds_measured(cp, 4, b, bad)
    st = {"edges": 1000, "remote_pushes": 50}
    assert dd.pushes_performed(st, 0.25, 1) == 800.0 and dd.pushes_performed(st, 0.25, 0) == 1000.0
    ri = np.array([0, 5, 9, 10, 19, 3], dtype=np.int32)
    assert dd.remote_fraction(ri, 5, 10) == 4 / 6 and dd.remote_fraction(ri[:0], 0, 1) == 0.0

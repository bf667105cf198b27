"""Generator determinism and recipe checks (diter_inputs; CPU only)."""
import numpy as np

import diter_inputs as gen


def test_deterministic_and_seeded():
    a = gen.web_graph(20000, 5)
    b = gen.web_graph(20000, 5)
    c = gen.web_graph(20000, 6)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])


def test_uniform_recipe():
    """configs[0]: outdeg in [1,10], distinct destinations, no self-loops, no dangling."""
    cp, ri = gen.uniform_graph(1000, 1)
    deg = np.diff(cp)
    assert deg.min() >= 1 and deg.max() <= 10 and abs(deg.mean() - 5.5) < 0.5
    for j in range(1000):
        col = ri[cp[j]:cp[j + 1]]
        assert np.all(np.diff(col) > 0) and not np.any(col == j)
        assert col.min() >= 0 and col.max() < 1000


def test_web_recipe():
    """configs[1]: ~15% dangling, Zipf-tailed degree <= 5000, 70% local within +-1000."""
    n = 200_000
    cp, ri = gen.web_graph(n, 1)
    deg = np.diff(cp)
    assert abs((deg == 0).mean() - 0.15) < 0.01
    assert deg.max() <= 5000
    src = np.repeat(np.arange(n), deg)
    assert not np.any(src == ri)
    off = (ri.astype(np.int64) - src) % n
    off = np.minimum(off, n - off)
    local = (off <= 1000).mean()
    assert 0.68 < local < 0.80        # 70% local + the global draws that land nearby
    # sorted unique rows per column
    same = src[1:] == src[:-1]
    assert np.all(np.diff(ri.astype(np.int64))[same] > 0)
    # Zipf over id: low ids receive far more global edges than high ids
    assert (ri < n // 100).mean() > 0.1


def test_signed_recipe():
    cp, ri, v, b = gen.signed_system(5000, 2)
    deg = np.diff(cp)
    assert np.all(deg == 20)
    colsum = np.add.reduceat(np.abs(v), cp[:-1])
    np.testing.assert_allclose(colsum, 0.9, rtol=1e-14)
    assert v.min() < 0 < v.max() and b.min() < 0 < b.max()
    assert np.all(np.abs(b) <= 1)


def test_rmat_recipe():
    src, dst = gen.rmat_coo(12, 1)
    assert len(src) == 16 << 12
    assert src.min() >= 0 and src.max() < 4096
    d = np.bincount(src, minlength=4096)
    assert d.max() > 20 * d.mean()        # skewed

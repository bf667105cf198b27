"""Pins of the CPU oracle against things other than itself (CPU only).

Each test pins an oracle function to a closed form, a worked example from
SPEC.md (tests/golden/spec_examples.json, cited), a library routine (LAPACK
via numpy.linalg.solve, scipy.sparse), brute force on tiny inputs, or an
invariant the paper states or that follows from its
definitions.  A plausible slip in the oracle (dropped term,
wrong sign/index, transposed operand, wrong weight, wrong threshold
direction) fails at least one of these.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp

import diter_inputs as gen
import oracle

D = 0.85


def csc_from_edges(n, edges):
    """Map-of-sets CSC (test-side, SPEC.md:83 style): column j = sorted children of j."""
    cols = {j: set() for j in range(n)}
    for (j, i) in edges:
        cols[j].add(i)
    col_ptr = [0]
    rows = []
    for j in range(n):
        rows.extend(sorted(cols[j]))
        col_ptr.append(len(rows))
    return np.array(col_ptr, np.int64), np.array(rows, np.int32)


def p_matrix(n, col_ptr, row_idx, values=None, d=D):
    """scipy P with p_ij = weight of edge j -> i."""
    deg = np.diff(col_ptr)
    if values is None:
        w = np.repeat(np.where(deg > 0, d / np.maximum(deg, 1), 0.0), deg)
    else:
        w = values
    return sp.csc_matrix((w, row_idx, col_ptr), shape=(n, n))


def lapack_solve(n, col_ptr, row_idx, values=None, b=None, d=D):
    P = p_matrix(n, col_ptr, row_idx, values, d).toarray()
    if b is None:
        b = np.full(n, (1 - d) / n)
    return np.linalg.solve(np.eye(n) - P, b)


def run(n, col_ptr, row_idx, target, values=None, b=None, d=D, policy=oracle.HYBRID, **kw):
    P = oracle.Problem(n, col_ptr, row_idx, values, b, d)
    st = P.init(kw.pop("alpha", 1.5))
    rc = P.snapshot(st, target, policy, **kw)
    return P, st, rc


# ----------------------------------------------------------- closed forms ---

@pytest.mark.parametrize("n", [2, 3, 7, 50])
@pytest.mark.parametrize("policy", [oracle.GEOM, oracle.HYBRID])
def test_cycle_uniform_closed_form(n, policy):
    """Directed N-cycle, B_i = (1-d)/N: X_i = 1/N (App. A.3)."""
    cp, ri = csc_from_edges(n, [(j, (j + 1) % n) for j in range(n)])
    P, st, rc = run(n, cp, ri, 1e-15, policy=policy)
    assert rc == oracle.OK
    np.testing.assert_allclose(st.H, 1.0 / n, rtol=0, atol=1e-14)
    np.testing.assert_allclose(P.dense_solve(), 1.0 / n, rtol=1e-14)


@pytest.mark.parametrize("n", [3, 7, 20])
def test_complete_digraph_closed_form(n):
    cp, ri = csc_from_edges(n, [(j, i) for j in range(n) for i in range(n) if i != j])
    P, st, rc = run(n, cp, ri, 1e-15)
    np.testing.assert_allclose(st.H, 1.0 / n, atol=1e-14)
    np.testing.assert_allclose(P.dense_solve(), 1.0 / n, rtol=1e-13)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_cycle_point_source(n):
    """N-cycle with B = (1-d) e_0: x_k = (1-d) d^k / (1-d^N) (App. A.3)."""
    cp, ri = csc_from_edges(n, [(j, (j + 1) % n) for j in range(n)])
    b = np.zeros(n)
    b[0] = 1 - D
    x = np.array([(1 - D) * D ** k / (1 - D ** n) for k in range(n)])
    P, st, rc = run(n, cp, ri, 1e-16, b=b)
    np.testing.assert_allclose(st.H, x, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(P.dense_solve(), x, rtol=1e-13)


@pytest.mark.parametrize("n", [4, 8])
def test_complete_digraph_point_source(n):
    cp, ri = csc_from_edges(n, [(j, i) for j in range(n) for i in range(n) if i != j])
    b = np.zeros(n)
    b[0] = 1 - D
    y = D * (1 - D) / ((n - 1) - D * (n - 2) - D ** 2)
    x = np.full(n, y)
    x[0] = (1 - D) + D * y
    P, st, rc = run(n, cp, ri, 1e-16, b=b)
    np.testing.assert_allclose(st.H, x, rtol=1e-12)
    np.testing.assert_allclose(P.dense_solve(), x, rtol=1e-13)


@pytest.mark.parametrize("m", [1, 2, 5, 12])
def test_chain_with_dangling_end(m):
    """Chain 0->1->...->m-1, last node dangling (fluid leaves): x_k = b(1-d^(k+1))/(1-d)."""
    cp, ri = csc_from_edges(m, [(k, k + 1) for k in range(m - 1)])
    b = np.full(m, 0.05)
    x = 0.05 * (1 - D ** (np.arange(m) + 1)) / (1 - D)
    P, st, rc = run(m, cp, ri, 1e-16, b=b, policy=oracle.GEOM)
    np.testing.assert_allclose(st.H, x, rtol=1e-13)
    np.testing.assert_allclose(P.dense_solve(), x, rtol=1e-13)


def test_single_node_self_loop():
    """N=1 self-loop: x = b/(1-d); with b = 1-d, x = 1."""
    cp, ri = csc_from_edges(1, [(0, 0)])
    P, st, rc = run(1, cp, ri, 1e-13)
    assert abs(st.H[0] - 1.0) <= 1e-13 / (1 - D) + 1e-15
    assert abs(P.dense_solve()[0] - 1.0) < 1e-14


def test_no_edges_gives_b():
    """P = 0 (or d -> 0): X = B (App. A.3)."""
    n = 5
    cp, ri = csc_from_edges(n, [])
    b = np.array([0.1, 0.2, 0.3, 0.0, 0.4])
    P, st, rc = run(n, cp, ri, 1e-300, b=b)
    np.testing.assert_array_equal(st.H, b)
    np.testing.assert_array_equal(st.F, 0.0)
    # d -> 0 with edges present: X -> B
    cp2, ri2 = csc_from_edges(n, [(0, 1), (1, 2), (2, 0), (3, 4)])
    P2 = oracle.Problem(n, cp2, ri2, None, b, 1e-12)
    np.testing.assert_allclose(P2.dense_solve(), b, atol=1e-12)


# ------------------------------------------------------- library routines ---

@pytest.mark.parametrize("seed", [1, 2, 3])
def test_dense_solve_matches_lapack(seed):
    cp, ri = gen.web_graph(300, seed, window=20, max_deg=50)
    P = oracle.Problem(300, cp, ri)
    np.testing.assert_allclose(P.dense_solve(), lapack_solve(300, cp, ri), rtol=1e-12, atol=1e-16)
    cps, ris, v, b = gen.signed_system(200, seed, nnz_per_col=7)
    Ps = oracle.Problem(200, cps, ris, v, b, 0.9)
    np.testing.assert_allclose(Ps.dense_solve(), lapack_solve(200, cps, ris, v, b, 0.9),
                               rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1_matches_lapack_and_bound_equality(seed):
    """configs[0] (C1): H vs LAPACK; dangling-free PageRank gives |X-H|_1 = r/(1-d) exactly
    because 1^T (I-P)^-1 = 1^T/(1-d) (App. A.1)."""
    cp, ri = gen.uniform_graph(1000, seed)
    X = lapack_solve(1000, cp, ri)
    for target in (1e-6, 1e-9, 1e-12):
        P, st, rc = run(1000, cp, ri, target)
        r = float(np.abs(st.F).sum())
        err = float(np.abs(X - st.H).sum())
        assert r < target
        assert err <= r / (1 - D) * (1 + 1e-9) + 1e-15
        assert abs(err - r / (1 - D)) <= 1e-12 * max(r / (1 - D), 1e-3) + 5e-15
        assert np.all(st.H <= X + 1e-15)                     # H increases to X


def test_jacobi_matches_lapack_signed():
    cp, ri, v, b = gen.signed_system(400, 4, nnz_per_col=20)
    P = oracle.Problem(400, cp, ri, v, b, 0.9)
    X, it = P.jacobi(1e-14 * np.abs(b).sum())
    np.testing.assert_allclose(X, lapack_solve(400, cp, ri, v, b, 0.9), rtol=1e-9, atol=1e-12)
    st = P.solve(1e-13 * np.abs(b).sum())
    assert np.abs(st.H - X).sum() <= 1e-13 * np.abs(b).sum() / (1 - 0.9) * 1.01 + 1e-12


# ------------------------------------------------------------- invariants ---

def _identity_residual(n, cp, ri, v, b, d, st):
    """|F - (B - (I-P) H)|_1 by an independent scipy SpMV (App. A.1)."""
    Pm = p_matrix(n, cp, ri, v, d)
    return float(np.abs(st.F - (b - st.H + Pm @ st.H)).sum())


@pytest.mark.parametrize("policy", [oracle.GEOM, oracle.HYBRID])
def test_identity_conservation_monotonicity_pagerank(policy):
    """Per pass: F = B - (I-P)H; |F| + (1-d)|H| + d sum_dangling H = |B| (App. A.2; BASELINE
    north_star conservation 'with dangling columns ... replaced by a bound'); H non-decreasing;
    |F|_1 non-increasing."""
    n = 3000
    cp, ri = gen.web_graph(n, 7, window=50, max_deg=200)
    deg = np.diff(cp)
    assert (deg == 0).sum() > 100
    b = np.full(n, (1 - D) / n)
    P = oracle.Problem(n, cp, ri)
    st = P.init()
    Hprev = st.H.copy()
    rprev = np.abs(st.F).sum()
    for k in range(40):
        P.snapshot(st, 0.0, policy, max_passes=1)
        assert _identity_residual(n, cp, ri, None, b, D, st) <= 1e-15
        lhs = np.abs(st.F).sum() + (1 - D) * st.H.sum() + D * st.H[deg == 0].sum()
        assert abs(lhs - 0.15) <= 1e-15
        assert lhs <= 0.15 + 1e-15 and np.abs(st.F).sum() + (1 - D) * st.H.sum() <= 0.15 + 1e-15
        assert np.all(st.H >= Hprev)
        r = np.abs(st.F).sum()
        assert r <= rprev + 1e-18
        Hprev, rprev = st.H.copy(), r
    assert st.passes == 40 and len(st.log) == 40


def test_identity_and_monotone_residual_signed():
    cp, ri, v, b = gen.signed_system(2000, 5, nnz_per_col=20)
    P = oracle.Problem(2000, cp, ri, v, b, 0.9)
    st = P.init()
    rprev = np.abs(st.F).sum()
    for k in range(25):
        P.snapshot(st, 0.0, oracle.HYBRID, max_passes=1)
        assert _identity_residual(2000, cp, ri, v, b, 0.9, st) <= 1e-11
        r = np.abs(st.F).sum()
        assert r <= rprev * (1 + 1e-14)           # A.2: |F| drops by >= (1-d)|s| per take
        rprev = r


def test_log_matches_state():
    """The log's r_p is |F|_1 before pass p; E_p = sum of out-degrees over S_p."""
    n = 500
    cp, ri = gen.web_graph(n, 3, window=30, max_deg=40)
    P = oracle.Problem(n, cp, ri)
    st = P.init()
    deg = np.diff(cp)
    for p in range(12):
        F_before = st.F.copy()
        T = st.T
        P.snapshot(st, 0.0, oracle.GEOM, max_passes=1)
        _, T_log, r_log, cnt, E, dang = st.log[-1]
        S = np.abs(F_before) > T                   # brute-force recount on the same bytes
        assert T_log == T
        assert r_log == pytest.approx(np.abs(F_before).sum(), rel=1e-15)
        assert cnt == S.sum() and E == deg[S].sum() and dang == (deg[S] == 0).sum()
    # GEOM: T_p = T_0 / alpha^p by repeated division
    Ts = [l[1] for l in st.log]
    for a, b_ in zip(Ts, Ts[1:]):
        assert b_ == a / 1.5


def test_first_pass_selects_all_uniform_b():
    """T_0 = max|B|/alpha (reading R5) with strict '>' selects every node in pass 0."""
    cp, ri = gen.uniform_graph(200, 9)
    P, st, rc = run(200, cp, ri, 0.0, max_passes=1)
    assert st.log[0][3] == 200 and st.log[0][1] == ((1 - D) / 200) / 1.5


def test_hybrid_threshold_rule():
    """HYBRID: T drops by alpha iff |S_p| <= f N, else stays (reading R4)."""
    cp, ri = gen.web_graph(2000, 2, window=40, max_deg=100)
    P, st, rc = run(2000, cp, ri, 1e-12, policy=oracle.HYBRID, hybrid_frac=0.05)
    log = st.log
    for cur, nxt in zip(log, log[1:]):
        if cur[3] <= 0.05 * 2000:
            assert nxt[1] == cur[1] / 1.5
        else:
            assert nxt[1] == cur[1]


# ---------------------------------------------------------- worked examples ---

def test_spec_init_example(golden):
    g = golden["init_uniform_n4"]
    cp, ri = csc_from_edges(4, [(0, 1)])
    P = oracle.Problem(4, cp, ri, None, None, g["d"])
    st = P.init()
    np.testing.assert_allclose(st.F, g["F"], rtol=1e-15)
    assert oracle.l1(st.F) == pytest.approx(g["residual"], rel=1e-15)
    assert g["residual"] / (1 - g["d"]) == pytest.approx(golden["error_bound"]["bound"])


def test_spec_two_cycle_diffuse(golden):
    g = golden["two_cycle_diffuse"]
    cp, ri = csc_from_edges(2, [(0, 1), (1, 0)])
    P = oracle.Problem(2, cp, ri, None, None, g["d"])
    st = P.init()
    st.F[:] = g["F0"]
    P.diffuse_node(st, g["node"])
    np.testing.assert_allclose(st.F, g["F1"], rtol=1e-15)
    np.testing.assert_allclose(st.H, g["H1"], rtol=1e-15)
    assert oracle.l1(st.F) == pytest.approx(g["residual"], rel=1e-15)


def test_spec_star_and_outgoing(golden):
    g = golden["star5_diffuse"]
    cp, ri = csc_from_edges(6, [(0, k) for k in range(1, 6)])
    P = oracle.Problem(6, cp, ri, None, None, g["d"])
    st = P.init()
    st.F[:] = 0
    st.F[0] = 2.0
    assert P.diffuse_node(st, 0) == 5
    np.testing.assert_allclose(st.F[1:], g["gain_per_unit"] * 2.0, rtol=1e-15)
    o = golden["compute_outgoing"]
    cp, ri = csc_from_edges(3, [(0, 1), (0, 2)])
    P = oracle.Problem(3, cp, ri, None, None, o["d"])
    st = P.init()
    st.F[:] = [o["sent"], 0, 0]
    P.diffuse_node(st, 0)
    np.testing.assert_allclose(st.F[1:], o["per_child"], rtol=1e-15)


def test_hand_traced_chain(golden):
    g = golden["chain3_geom_trace"]
    cp, ri = csc_from_edges(g["n"], g["edges"])
    b = np.full(g["n"], g["b"])
    P, st, rc = run(g["n"], cp, ri, 1e-300, b=b, d=g["d"], policy=oracle.GEOM, alpha=g["alpha"])
    assert rc == oracle.OK
    assert [l[3] for l in st.log] == g["frontier"]
    assert [l[4] for l in st.log] == g["edges_per_pass"]
    assert [l[5] for l in st.log] == g["dangling_per_pass"]
    np.testing.assert_allclose([l[2] for l in st.log], g["r"], rtol=1e-14)
    np.testing.assert_allclose(st.H, g["H_final"], rtol=1e-14)


# ---------------------------------------------------- order independence ---

@pytest.mark.parametrize("seed", [1, 2])
def test_sequential_and_snapshot_same_limit(seed):
    """Any admissible sequence reaches the same X."""
    cp, ri = gen.web_graph(800, seed, window=25, max_deg=60)
    X = lapack_solve(800, cp, ri)
    P = oracle.Problem(800, cp, ri)
    st_seq = P.init()
    assert P.sequential(st_seq, 1e-13) == oracle.OK
    st_snap = P.solve(1e-13, oracle.GEOM)
    for st in (st_seq, st_snap):
        assert np.abs(st.H - X).sum() <= 1e-13 / (1 - D) * 1.01 + 1e-15
    cps, ris, v, b = gen.signed_system(300, seed, nnz_per_col=10)
    Ps = oracle.Problem(300, cps, ris, v, b, 0.9)
    Xs = lapack_solve(300, cps, ris, v, b, 0.9)
    s1 = Ps.init()
    assert Ps.sequential(s1, 1e-12) == oracle.OK
    assert np.abs(s1.H - Xs).sum() <= 1e-12 / 0.1 * 1.01


# -------------------------------------------------------------- CSC / partition ---

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_csc_from_coo_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n, m = 37, 400
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    cp, ri = oracle.csc_from_coo(n, src, dst)
    cp2, ri2 = csc_from_edges(n, list(zip(src.tolist(), dst.tolist())))
    np.testing.assert_array_equal(cp, cp2)
    np.testing.assert_array_equal(ri, ri2)
    # scipy's COO->CSC (sum duplicates) has the same structure
    A = sp.coo_matrix((np.ones(m), (dst, src)), shape=(n, n)).tocsc()
    A.sum_duplicates()
    A.sort_indices()
    np.testing.assert_array_equal(cp, A.indptr)
    np.testing.assert_array_equal(ri, A.indices)


def test_csc_from_coo_rmat_small():
    src, dst = gen.rmat_coo(10, 3)
    cp, ri = oracle.csc_from_coo(1 << 10, src, dst)
    A = sp.coo_matrix((np.ones(len(src)), (dst, src)), shape=(1024, 1024)).tocsc()
    A.sum_duplicates()
    A.sort_indices()
    np.testing.assert_array_equal(cp, A.indptr)
    np.testing.assert_array_equal(ri, A.indices)
    assert cp[-1] < len(src)           # R-MAT at scale 10 has duplicates to drop


def test_partition_examples(golden):
    g = golden["cb_partition_example"]
    cost = np.concatenate([[0], np.cumsum(g["outdeg"])])
    np.testing.assert_array_equal(oracle.partition_cb(cost, g["K"]), g["bounds"])
    for n, K, b in golden["uniform_partition_examples"]["cases"]:
        np.testing.assert_array_equal(oracle.partition_uniform(n, K), b)


@pytest.mark.parametrize("seed", range(6))
def test_partition_cb_bruteforce(seed):
    """Brute force over all contiguous K-splits: the CB rule returns the split whose k-th
    boundary is the first index where the prefix cost reaches ceil(kL/K) -- check by
    enumerating all splits and also the balance bound max part <= L/K + max single cost."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 11))
    deg = rng.integers(0, 9, n)
    cost = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    L = int(cost[-1])
    for K in range(1, min(n, 4) + 1):
        b = oracle.partition_cb(cost, K)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 1)
        splits = [s for s in itertools.combinations(range(1, n), K - 1)]
        assert tuple(b[1:-1]) in splits
        parts = [cost[b[k + 1]] - cost[b[k]] for k in range(K)]
        assert max(parts) <= -(-L // K) + deg.max()
        if L > 0 and np.all(deg > 0):
            # every boundary is the earliest index reaching its quota (unless clamped)
            for k in range(1, K):
                goal = -(-k * L // K)
                first = int(np.argmax(cost >= goal))
                assert b[k] == max(first, b[k - 1] + 1) or b[k] == n - (K - k)


def test_partition_equal_degrees_is_uniform():
    """All degrees equal -> CB = uniform."""
    for n, K in [(12, 3), (100, 4), (64, 8)]:
        cost = np.arange(n + 1, dtype=np.int64) * 5
        np.testing.assert_array_equal(oracle.partition_cb(cost, K), oracle.partition_uniform(n, K))


# ----------------------------------------------------- selection key (f1) ---
# i_n = argmax F_i / ((#in_i + 1)(#out_i + 1)), approximated by a
# threshold; per-edge variant 1/(#out_i + 1).

KEY_GRAPH = (3, [(0, 1), (0, 2), (1, 2), (2, 0)])   # edges j -> i; #out = 2,1,1; #in = 1,1,2


def test_key_weights_hand():
    """Hand values: #out = (2,1,1), #in = (1,1,2) -> per-edge 1/3, 1/2, 1/2;
    paper 1/(2*3), 1/(2*2), 1/(3*2); each rounded once to fp32 (reading R20)."""
    n, edges = KEY_GRAPH
    cp, ri = csc_from_edges(n, edges)
    np.testing.assert_array_equal(oracle.key_weights(n, cp, ri, oracle.KEY_RAW), np.ones(3, np.float32))
    np.testing.assert_array_equal(oracle.key_weights(n, cp, ri, oracle.KEY_EDGE),
                                  np.array([1 / 3, 1 / 2, 1 / 2], np.float32))
    np.testing.assert_array_equal(oracle.key_weights(n, cp, ri, oracle.KEY_PAPER),
                                  np.array([1 / 6, 1 / 4, 1 / 6], np.float32))


@pytest.mark.parametrize("key,expect", [(oracle.KEY_RAW, 3), (oracle.KEY_EDGE, 2), (oracle.KEY_PAPER, 1)])
def test_key_first_pass_hand(key, expect):
    """Uniform B = b, alpha = 1.2.  raw: T0 = b/1.2 < b = every key -> 3 nodes.
    per-edge: keys b/3, b/2, b/2, T0 = (b/2)/1.2 = b/2.4 -> nodes 1, 2.
    paper: keys b/6, b/4, b/6, T0 = (b/4)/1.2 = b/4.8 -> node 1 only."""
    n, edges = KEY_GRAPH
    cp, ri = csc_from_edges(n, edges)
    P = oracle.Problem(n, cp, ri, key=key)
    st = P.init(1.2)
    P.snapshot(st, 0.0, oracle.GEOM, 1.2, max_passes=1)
    assert st.log[0][3] == expect
    sel = np.flatnonzero(st.H > 0)
    assert list(sel) == {3: [0, 1, 2], 2: [1, 2], 1: [1]}[expect]


@pytest.mark.parametrize("key", [oracle.KEY_EDGE, oracle.KEY_PAPER])
@pytest.mark.parametrize("policy", [oracle.GEOM, oracle.HYBRID])
def test_key_same_fixed_point(key, policy):
    """Any selection order converges to the same X: the keyed run
    reaches LAPACK's solution on a random graph with dangling nodes."""
    n = 300
    cp, ri = gen.web_graph(n, 5, window=50, max_deg=40)
    X = np.linalg.solve(np.eye(n) - p_matrix(n, cp, ri).toarray(), np.full(n, (1 - D) / n))
    P = oracle.Problem(n, cp, ri, key=key)
    st = P.init()
    assert P.snapshot(st, 1e-15, policy) == oracle.OK
    assert np.abs(st.H - X).sum() <= 1e-13


@pytest.mark.parametrize("key,wv", [(oracle.KEY_EDGE, 0.5), (oracle.KEY_PAPER, 0.25)])
def test_key_on_cycle_equals_raw(key, wv):
    """Directed cycle: #in = #out = 1, so w = 1/2 (per-edge) or 1/4 (paper) on every
    node, exact in fp32: keyed selection is the raw selection with T scaled by w,
    so the logs (frontier, edges) coincide pass for pass."""
    n = 50
    cp, ri = csc_from_edges(n, [(j, (j + 1) % n) for j in range(n)])
    rng = np.random.default_rng(3)
    b = rng.random(n) * 0.15 / n
    np.testing.assert_array_equal(oracle.key_weights(n, cp, ri, key), np.full(n, wv, np.float32))
    logs = []
    for k in (oracle.KEY_RAW, key):
        P = oracle.Problem(n, cp, ri, b=b, key=k)
        st = P.init()
        P.snapshot(st, 1e-12, oracle.HYBRID)
        logs.append([(l[3], l[4]) for l in st.log])
    assert logs[0] == logs[1]


def test_key_reduces_work_weblike():
    """The degree-weighted key is the paper's heuristic for cheaper convergence
    (P:208-212); on a web-like graph (N = 2e5, HYBRID) the per-edge and paper keys
    need fewer elementary diffusions than the raw key (18.9 ->
    13.9 / 12.7 normalized iterations)."""
    p = gen.config("C2", 1, n=200_000)
    work = {}
    for k in (oracle.KEY_RAW, oracle.KEY_EDGE, oracle.KEY_PAPER):
        P = oracle.Problem(p.n, p.col_ptr, p.row_idx, key=k)
        st = P.init()
        assert P.snapshot(st, 1e-9 * 0.15, oracle.HYBRID) == oracle.OK
        work[k] = st.edges / p.nnz
    assert work[oracle.KEY_EDGE] < 0.9 * work[oracle.KEY_RAW]
    assert work[oracle.KEY_PAPER] < 0.9 * work[oracle.KEY_RAW]


# ------------------------------------------- completed PageRank (f4, App. A.4) ---

def test_completed_pagerank_two_nodes_closed_form():
    """0 -> 1, node 1 dangling.  Completed Q' = [[0, 1/2], [1, 1/2]]; with x0 + x1 = 1,
    x0 = d x1 / 2 + (1-d)/2  =>  x0 = 1/(2+d), x1 = (1+d)/(2+d)."""
    cp, ri = csc_from_edges(2, [(0, 1)])
    X = oracle.Problem(2, cp, ri).completed_pagerank_dense()
    np.testing.assert_allclose(X, [1 / (2 + D), (1 + D) / (2 + D)], rtol=1e-15)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_completed_pagerank_is_normalised_fluid_leaves_solution(seed):
    """App. A.4: the completed solution sums to 1 (Q' stochastic) and equals X/|X|_1 of
    the fluid-leaves system, here from LAPACK; and power iteration on the completed
    Google matrix (an independent route) converges to it."""
    n = 400
    cp, ri = gen.web_graph(n, seed, window=30, max_deg=60)
    assert (np.diff(cp) == 0).sum() > 20
    Xc = oracle.Problem(n, cp, ri).completed_pagerank_dense()
    assert abs(Xc.sum() - 1.0) <= 1e-13
    X = lapack_solve(n, cp, ri)
    np.testing.assert_allclose(Xc, X / X.sum(), rtol=1e-11, atol=1e-16)
    deg = np.diff(cp)
    G = p_matrix(n, cp, ri, d=1.0).toarray()
    G[:, deg == 0] = 1.0 / n
    x = np.full(n, 1.0 / n)
    for _ in range(400):
        x = D * G @ x + (1 - D) / n
    np.testing.assert_allclose(Xc, x, rtol=1e-12, atol=1e-16)


def test_identity_check_helper_catches_a_misrouted_push():
    """tests/identity_check.py (the every-row check the full-scale GPU tests use) is ~0
    on the oracle's state after real passes, and flags one push sent to the wrong row
    (mass-conserving, so global checks miss it) at both rows it touched."""
    import identity_check as ic
    n = 3000
    cp, ri = gen.web_graph(n, 4)
    P = oracle.Problem(n, cp, ri)
    st = P.init(1.5)
    P.snapshot(st, 1e-30, oracle.HYBRID, 1.5, 0.05, max_passes=12)
    b = np.full(n, 0.15 / n)
    e, _ = ic.identity_residual(n, cp, ri, st.H, st.F, b, 0.85)
    assert e <= 1e-13, e
    F = st.F.copy()
    j = int(np.argmax(st.F))
    v = 0.5 * F[j]
    F[j] -= v
    F[(j + 17) % n] += v
    e, row = ic.identity_residual(n, cp, ri, st.H, F, b, 0.85)
    assert e > 1e-3 and row in (j, (j + 17) % n)

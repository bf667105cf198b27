"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): ||H_gpu - X||_1 <= 1e-8 |B|_1 with X the
oracle's fixed point on the same seeded inputs; integer outputs bit-exact
(CSC construction, per-pass frontier sizes at the same threshold schedule).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import diter_inputs as gen
import oracle
import paper_1202_6168_b200 as di

pytestmark = pytest.mark.gpu

TOL = 1e-8          # ||H - X||_1 <= TOL |B|_1  (north_star)


def _xref(n, cp, ri, vals=None, b=None, d=0.85):
    """Oracle fixed point: snapshot run to r <= 1e-12 |B|_1."""
    P = oracle.Problem(n, cp, ri, vals, b, d)
    bn = float(np.abs(P.b).sum())
    st = P.solve(1e-12 * bn * (1 - d))
    return st.H, P, bn


def _pmat(n, cp, ri, vals=None, d=0.85):
    deg = np.diff(cp)
    w = vals if vals is not None else np.repeat(np.where(deg > 0, d / np.maximum(deg, 1), 0.0), deg)
    return sp.csc_matrix((w, ri, cp), shape=(n, n))


def _gpu(n, cp, ri, target, vals=None, b=None, d=0.85, **opts):
    ctx = di.di_create(n, cp, ri, vals, b, d, di.default_options(**opts))
    di.di_run(ctx, target)
    H = di.di_get_history(ctx)
    F = di.di_get_fluid(ctx)
    log = di.di_get_pass_log(ctx)
    r = di.di_get_residual(ctx)
    stats = di.di_get_stats(ctx)
    di.di_destroy(ctx)
    return H, F, log, r, stats


def _check_state(n, cp, ri, vals, b, d, H, F, r, target):
    """Exact identity F = B - (I-P)H by an independent SpMV, and r = |F|_1 < target."""
    if b is None:
        b = np.full(n, (1 - d) / n)
    bn = np.abs(b).sum()
    Pm = _pmat(n, cp, ri, vals, d)
    ident = np.abs(F - (b - H + Pm @ H)).sum()
    assert ident <= 1e-12 * bn, ident
    assert r == pytest.approx(np.abs(F).sum(), rel=1e-12, abs=1e-300)
    assert r < target


def _oracle_passes_with_ties(P, target, policy, rel=1e-12):
    """Oracle run one pass at a time, recording per pass the number of nodes whose
    |F_i| is within `rel` of T_p (ties in exact arithmetic that rounding order may
    break either way -- reading R8 / SURVEY §8c-Q8)."""
    st = P.init()
    near = []
    while True:
        T = st.T
        a = np.abs(st.F)
        near_p = int((np.abs(a - T) <= rel * T).sum())
        rc = P.snapshot(st, target, policy, max_passes=1)
        if len(st.log) == len(near):
            break
        near.append(near_p)
        if rc == oracle.OK:
            break
    return st, near


def _compare_logs_q8(glog, st, near):
    """Frontier sizes equal pass for pass until the first pass where the oracle's F
    holds a near-tie; after it the runs may drift by the tie, so only the size of
    the drift is bounded.  A mismatch with no earlier tie fails."""
    olog = st.log
    k = min(len(glog), len(olog))
    g = glog["frontier"][:k]
    o = np.array([l[3] for l in olog[:k]])
    first_tie = next((p for p in range(k) if near[p] > 0), k)
    np.testing.assert_array_equal(g[:first_tie], o[:first_tie])
    if first_tie < k:
        assert np.all(np.abs(g[first_tie:] - o[first_tie:]) <= 0.05 * o[first_tie:] + 2)
        ge, oe = glog["edges"][:k].sum(), sum(l[4] for l in olog[:k])
        assert abs(ge - oe) <= 0.01 * oe
    return first_tie


def _compare_logs(glog, olog, n_cmp=None):
    k = min(len(glog), len(olog)) if n_cmp is None else n_cmp
    assert k > 0
    g_front = glog["frontier"][:k]
    o_front = np.array([l[3] for l in olog[:k]])
    g_T = glog["T"][:k]
    o_T = np.array([l[1] for l in olog[:k]])
    np.testing.assert_array_equal(g_T, o_T)            # same schedule, bit for bit
    np.testing.assert_array_equal(g_front, o_front)    # Q8: exact on these inputs
    np.testing.assert_array_equal(glog["edges"][:k], [l[4] for l in olog[:k]])
    np.testing.assert_array_equal(glog["dangling"][:k], [l[5] for l in olog[:k]])


# ------------------------------------------------------------------ configs ---

@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("policy", [di.DI_POLICY_GEOM, di.DI_POLICY_HYBRID])
def test_c1_parity_dense(seed, policy):
    """configs[0]: N=1000, stop |F|_1 < 1e-12, dense solve."""
    cp, ri = gen.uniform_graph(1000, seed)
    X = oracle.Problem(1000, cp, ri).dense_solve()
    H, F, log, r, stats = _gpu(1000, cp, ri, 1e-12, policy=policy)
    assert np.abs(H - X).sum() <= TOL * 0.15
    # dangling-free PageRank: |X - H|_1 = r/(1-d) exactly (App. A.1)
    assert np.abs(X - H).sum() == pytest.approx(r / 0.15, rel=1e-6, abs=1e-15)
    _check_state(1000, cp, ri, None, None, 0.85, H, F, r, 1e-12)
    P = oracle.Problem(1000, cp, ri)
    st = P.init()
    P.snapshot(st, 1e-12, policy)
    _compare_logs(log, st.log)
    _same_stop_pass(log, st, 1e-12)


def _same_stop_pass(log, st, target):
    """The run stops after the same pass as the oracle, unless the residual at the
    boundary pass sits within rounding of the target (a tie decided by summation
    order, reading R8 applied to the stop test): then one pass more or fewer."""
    if len(log) == st.passes:
        return
    assert abs(len(log) - st.passes) == 1, (len(log), st.passes)
    r_edge = log["r"][st.passes] if len(log) > st.passes else st.log[len(log)][2]
    assert abs(r_edge / target - 1.0) < 1e-9, r_edge


@pytest.mark.parametrize("seed", [1, 2])
def test_c2_full_parity(seed):
    """configs[1] at full size (N=1e6, ~7M edges): parity stop 1e-9|B|_1 (reading R1)."""
    p = gen.config("C2", seed)
    X, P, bn = _xref(p.n, p.col_ptr, p.row_idx)
    H, F, log, r, stats = _gpu(p.n, p.col_ptr, p.row_idx, p.parity_stop)
    err = np.abs(H - X).sum()
    assert err <= TOL * bn, err / bn
    assert np.all(H <= X + 1e-15)                               # H increases to X
    _check_state(p.n, p.col_ptr, p.row_idx, None, None, 0.85, H, F, r, p.parity_stop)
    deg = np.diff(p.col_ptr)
    cons = np.abs(F).sum() + 0.15 * H.sum() + 0.85 * H[deg == 0].sum()
    assert abs(cons - bn) <= 1e-12 * bn                         # App. A.2
    st, near = _oracle_passes_with_ties(P, p.parity_stop, oracle.HYBRID)
    _compare_logs_q8(log, st, near)
    assert abs(stats["passes"] - st.passes) <= 2


_ORACLE_CACHE = {}


def _c2_random_b_oracle(policy, key=0):
    """Oracle run (memoised per policy and key) on the configs[1] graph with a random B."""
    if (policy, key) not in _ORACLE_CACHE:
        p = gen.config("C2", 3)
        rng = np.random.default_rng(7)
        b = rng.random(p.n) + 0.5
        b *= 0.15 / b.sum()
        target = 1e-9 * 0.15
        P = oracle.Problem(p.n, p.col_ptr, p.row_idx, None, b, key=key)
        st, near = _oracle_passes_with_ties(P, target, policy)
        _ORACLE_CACHE[(policy, key)] = (p, b, target, st, near)
    return _ORACLE_CACHE[(policy, key)]


VARIANTS = {
    "default": {},
    "fused": {"pass_kernel": 2},                       # cooperative persistent pass kernel
    "runs": {"scatter_run": 7, "scatter_stripes": 3},  # other grab run / stripe counts
    "nohot": {"hot_window": -1},                       # every push an L2 RED
    "far": {"far_push": 1, "far_warm_log2": 16},       # far-push bins forced on (auto: off)
    "key_edge": {"select_key": di.DI_KEY_EDGE},        # per-edge key 1/(#out+1)
    "key_paper": {"select_key": di.DI_KEY_PAPER},      # paper key 1/((#in+1)(#out+1))
    "key_paper_fused": {"select_key": di.DI_KEY_PAPER, "pass_kernel": 2},
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("policy", [di.DI_POLICY_GEOM, di.DI_POLICY_HYBRID])
def test_c2_graph_random_b_logs_exact(policy, variant):
    """configs[1] graph with a seeded random positive B: no exact-arithmetic ties with
    T_p, so frontier sizes, edges and dangling counts match the oracle pass for pass --
    for every pass-kernel / scatter-schedule option."""
    p, b, target, st, near = _c2_random_b_oracle(policy, VARIANTS[variant].get("select_key", 0))
    H, F, log, r, stats = _gpu(p.n, p.col_ptr, p.row_idx, target, b=b, policy=policy, **VARIANTS[variant])
    assert sum(near) == 0
    _compare_logs(log, st.log)
    assert len(log) == st.passes and stats["edges"] == st.edges
    # bins partition the frontier
    np.testing.assert_array_equal(log["bin_low"] + log["bin_mid"] + log["bin_hub"] + log["dangling"],
                                  log["frontier"])
    _check_state(p.n, p.col_ptr, p.row_idx, None, b, 0.85, H, F, r, target)


@pytest.mark.parametrize("n", [100_000, 1_000_000])
def test_c5_signed_parity(n):
    """configs[4]: signed P, |col|_1 = 0.9, stop 1e-9|B|_1 (parity stop 5e-10|B|_1), Jacobi."""
    cp, ri, v, b = gen.signed_system(n, 1)
    bn = np.abs(b).sum()
    X, P, _ = _xref(n, cp, ri, v, b, 0.9)
    Xj, it = P.jacobi(1e-13 * bn)
    assert np.abs(X - Xj).sum() <= 1e-10 * bn
    H, F, log, r, stats = _gpu(n, cp, ri, 5e-10 * bn, v, b, 0.9)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, v, b, 0.9, H, F, r, 5e-10 * bn)
    assert np.all(np.diff(log["r"]) <= 1e-12 * bn)              # |F|_1 non-increasing (A.2)


def test_c3_small_csc_and_parity():
    """configs[2] shape at scale 18: GPU COO->CSC bit-exact vs the oracle builder; parity
    (max out-degree ~1.6e4 > kMidMax, so the hub path runs)."""
    src, dst = gen.rmat_coo(18, 1)
    n = 1 << 18
    cp_o, ri_o = oracle.csc_from_coo(n, src, dst)
    cp_g, ri_g = di.di_csc_from_coo(n, src, dst)
    np.testing.assert_array_equal(cp_g, cp_o)
    np.testing.assert_array_equal(ri_g, ri_o)
    X, P, bn = _xref(n, cp_o, ri_o)
    H, F, log, r, stats = _gpu(n, cp_g, ri_g, 1e-9 * bn, policy=di.DI_POLICY_GEOM)
    assert np.abs(H - X).sum() <= TOL * bn
    assert log["bin_hub"].max() > 0                             # hubs exercised
    st, near = _oracle_passes_with_ties(P, 1e-9 * bn, oracle.GEOM)
    _compare_logs_q8(log, st, near)


def test_c3_full_scale_csc_bitexact():
    """configs[2] at full size (scale 24, 2.7e8 samples): CSC bit-exact vs the oracle."""
    src, dst = gen.rmat_coo(24, 1)
    n = 1 << 24
    cp_g, ri_g = di.di_csc_from_coo(n, src, dst)
    cp_o, ri_o = oracle.csc_from_coo(n, src, dst)
    np.testing.assert_array_equal(cp_g, cp_o)
    np.testing.assert_array_equal(ri_g, ri_o)


# -------------------------------------------------------------- edge cases ---

def test_single_node_self_loop_and_dangling():
    cp = np.array([0, 1], np.int64)
    ri = np.array([0], np.int32)
    H, F, log, r, _ = _gpu(1, cp, ri, 1e-14)
    assert abs(H[0] - 1.0) <= 1e-14 / 0.15 + 1e-15
    cp0 = np.array([0, 0], np.int64)
    H0, F0, log0, r0, _ = _gpu(1, cp0, np.zeros(0, np.int32), 1e-30)
    assert H0[0] == pytest.approx(0.15, rel=1e-15) and F0[0] == 0.0 and len(log0) == 1


def test_all_dangling_and_empty_edges():
    n = 1000
    cp = np.zeros(n + 1, np.int64)
    b = np.linspace(0, 1, n)
    H, F, log, r, _ = _gpu(n, cp, np.zeros(0, np.int32), 1e-300, b=b)
    np.testing.assert_array_equal(H, b)                         # X = B when P = 0
    assert r == 0.0


@pytest.mark.parametrize("n", [31, 33, 257, 4099, 1_000_003])
def test_ragged_sizes(n):
    cp, ri = gen.web_graph(n, 11, window=min(1000, n // 2 or 1), max_deg=min(5000, n - 1))
    X, P, bn = _xref(n, cp, ri)
    H, F, log, r, _ = _gpu(n, cp, ri, 1e-9 * bn)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, 1e-9 * bn)


def test_hub_chunks_and_duplicates():
    """A node with 20000 out-edges (10 chunks) and duplicate rows (they add)."""
    rng = np.random.default_rng(5)
    n = 30000
    cols = [np.sort(rng.integers(0, n, 20000)).astype(np.int32)]      # duplicates kept
    for j in range(1, n):
        k = int(rng.integers(0, 40))
        cols.append(np.sort(rng.choice(n, k, replace=False)).astype(np.int32))
    cp = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    ri = np.concatenate(cols)
    X, P, bn = _xref(n, cp, ri)
    H, F, log, r, _ = _gpu(n, cp, ri, 1e-10 * bn, policy=di.DI_POLICY_GEOM)
    assert log["bin_hub"].sum() > 0 and log["bin_mid"].sum() > 0 and log["bin_low"].sum() > 0
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, None, None, 0.85, H, F, r, 1e-10 * bn)


def test_select_exact_on_dumped_fluid():
    """K1 frontier count equals a CPU recount on the same F bytes."""
    p = gen.config("C2", 2, n=200_000)
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, options=di.default_options(max_passes=7,
                                                                              check_interval=1))
    assert di.di_run(ctx, 1e-300, raise_on_not_converged=False) == di.DI_ERR_NOT_CONVERGED
    F = di.di_get_fluid(ctx)
    stats = di.di_get_stats(ctx)
    assert stats["passes"] == 7
    T = stats["threshold"]
    di.di_run(ctx, 1e-300, raise_on_not_converged=False)       # resumable: 7 more passes
    log = di.di_get_pass_log(ctx)
    assert len(log) == 14 and log["T"][7] == T
    assert log["frontier"][7] == int((np.abs(F) > T).sum())
    assert log["r"][7] == pytest.approx(np.abs(F).sum(), rel=1e-13)
    di.di_destroy(ctx)


def test_target_already_met_and_resume():
    cp, ri = gen.uniform_graph(1000, 4)
    ctx = di.di_create(1000, cp, ri)
    di.di_run(ctx, 1.0)                                          # |B|_1 = 0.15 < 1: no pass
    assert di.di_get_stats(ctx)["passes"] == 0
    di.di_run(ctx, 1e-6)
    p1 = di.di_get_stats(ctx)["passes"]
    di.di_run(ctx, 1e-12)
    s = di.di_get_stats(ctx)
    assert s["passes"] > p1 and di.di_get_residual(ctx) < 1e-12
    X = oracle.Problem(1000, cp, ri).dense_solve()
    assert np.abs(di.di_get_history(ctx) - X).sum() <= TOL * 0.15
    di.di_destroy(ctx)


def test_invalid_inputs_rejected():
    cp = np.array([0, 2, 1, 3], np.int64)
    ri = np.array([0, 1, 2], np.int32)
    with pytest.raises(di.DiError) as e:
        di.di_create(3, cp, ri)
    assert e.value.status == di.DI_ERR_INVALID_ARG
    cp = np.array([0, 1, 2, 3], np.int64)
    with pytest.raises(di.DiError) as e:
        di.di_create(3, cp, np.array([0, 5, 1], np.int32))
    assert e.value.status == di.DI_ERR_INVALID_ARG
    with pytest.raises(di.DiError) as e:
        di.di_create(3, cp, np.array([0, 1, 2], np.int32), d=1.0)
    assert e.value.status == di.DI_ERR_INVALID_ARG
    with pytest.raises(di.DiError) as e:
        di.di_create(3, cp, np.array([0, 1, 2], np.int32), values=np.array([0.5, 0.95, -0.2]), d=0.9)
    assert e.value.status == di.DI_ERR_CONTRACTION


def test_device_getters():
    import torch
    cp, ri = gen.uniform_graph(1000, 2)
    ctx = di.di_create(1000, cp, ri)
    di.di_run(ctx, 1e-10)
    h = torch.empty(1000, dtype=torch.float64, device="cuda")
    di.di_get_history_device(ctx, h)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(h.cpu().numpy(), di.di_get_history(ctx))
    di.di_destroy(ctx)


@pytest.mark.parametrize("seed", [1, 2])
def test_completed_pagerank_output(seed):
    """NEXT f4 (completed PageRank): di_get_pagerank = H/|H|_1 against the
    oracle's dense completed system (N = 1500 web-like graph with dangling nodes), and
    the device variant byte-for-byte."""
    import torch
    n = 1500
    cp, ri = gen.web_graph(n, seed, window=100, max_deg=200)
    assert (np.diff(cp) == 0).sum() > 50
    Xc = oracle.Problem(n, cp, ri).completed_pagerank_dense()
    ctx = di.di_create(n, cp, ri)
    di.di_run(ctx, 1e-14)
    x = di.di_get_pagerank(ctx)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    di.di_get_pagerank_device(ctx, d)
    torch.cuda.synchronize()
    di.di_destroy(ctx)
    assert abs(x.sum() - 1.0) <= 1e-12
    assert np.abs(x - Xc).sum() <= 1e-11
    np.testing.assert_array_equal(d.cpu().numpy(), x)


def test_completed_pagerank_needs_default_pagerank_context():
    """H/|H|_1 is the completed PageRank only for P = dQ with B = (1-d)/N (App. A.4): a
    personalised B or a signed P makes di_get_pagerank return DI_ERR_STATE."""
    n = 2000
    cp, ri = gen.web_graph(n, 3, window=100, max_deg=200)
    b = np.random.default_rng(0).random(n)
    b *= 0.15 / b.sum()
    for kw in ({"b": b}, {"values": np.full(len(ri), 0.5 / np.maximum(1, np.diff(cp)).repeat(np.diff(cp)))}):
        ctx = di.di_create(n, cp, ri, kw.get("values"), kw.get("b"), 0.85)
        di.di_run(ctx, 1e-10)
        with pytest.raises(di.DiError) as e:
            di.di_get_pagerank(ctx)
        assert e.value.status == di.DI_ERR_STATE
        di.di_destroy(ctx)


@pytest.mark.parametrize("opts", [{"far_push": 1, "far_warm_log2": 12}, {"pass_kernel": 2},
                                  {"select_key": di.DI_KEY_EDGE}])
def test_signed_variants(opts):
    """configs[4] shape (signed P) through the far-push bins, the fused persistent
    kernel and the per-edge key: parity with the Jacobi fixed point and the exact
    identity F = B - (I-P)H."""
    n = 200_000
    cp, ri, v, b = gen.signed_system(n, 2)
    bn = np.abs(b).sum()
    X, _ = oracle.Problem(n, cp, ri, v, b, 0.9).jacobi(1e-13 * bn)
    H, F, log, r, stats = _gpu(n, cp, ri, 5e-10 * bn, v, b, 0.9, **opts)
    assert np.abs(H - X).sum() <= TOL * bn
    _check_state(n, cp, ri, v, b, 0.9, H, F, r, 5e-10 * bn)


def test_bounds_and_rebalance_on_one_gpu():
    """A single-GPU context owns [0, n); di_rebalance needs a distributed context."""
    cp, ri = gen.uniform_graph(1000, 3)
    ctx = di.di_create(1000, cp, ri)
    np.testing.assert_array_equal(di.di_get_bounds(ctx), [0, 1000])
    with pytest.raises(di.DiError) as e:
        di.di_rebalance(ctx, [0, 500, 1000])
    assert e.value.status == di.DI_ERR_INVALID_ARG
    di.di_run(ctx, 1e-12)                     # the context is still usable
    assert di.di_get_residual(ctx) < 1e-12
    di.di_destroy(ctx)


def test_set_profile_same_solve_and_kernel_times():
    """di_set_profile re-captures the pass graph with events between the kernels:
    the solve is the same up to the order of the fp64 REDs (which differs between
    any two runs) and the kernel times fill."""
    p = gen.config("C2", 1)
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, None, None, 0.85, di.default_options())
    out = []
    for on in (False, True, False):
        di.di_set_profile(ctx, on)
        di.di_reset(ctx)
        di.di_run(ctx, p.stop)
        s = di.di_get_stats(ctx)
        out.append((di.di_get_history(ctx), s))
        if on:
            assert s["kt_scatter_ms"] > 0 and s["kt_select_ms"] > 0 and s["kt_passes"] == s["passes"]
            lg = di.di_get_pass_log(ctx)
            assert np.all(lg["t_scatter_us"] > 0)
        else:
            assert s["kt_scatter_ms"] == 0
    di.di_destroy(ctx)
    # two stopped solves agree to the sum of their bounds r/(1-d), not better:
    # the RED order moves ties at a threshold and with them the stopping state
    for k in (1, 2):
        assert np.abs(out[k][0] - out[0][0]).sum() <= 2 * p.stop / 0.15
        assert abs(out[k][1]["passes"] - out[0][1]["passes"]) <= 1


def test_far_push_large_segment_prefix():
    """Far-push bins on a 4e6-node web-like graph: the staged far scatter's static (45 KB)
    plus dynamic (segment prefix, ~9.5 KB) shared memory exceeds the default 48 KB and
    runs on the opt-in.  Same solution as the plain scatter, exact identity F = B - (I-P)H."""
    p = gen.config("C2", 3, n=4_000_000)
    H0, F0, _, r0, s0 = _gpu(p.n, p.col_ptr, p.row_idx, p.stop)
    H1, F1, _, r1, s1 = _gpu(p.n, p.col_ptr, p.row_idx, p.stop, far_push=1, far_warm_log2=16)
    bn = 0.15                                      # |B|_1 = (1 - d)
    _check_state(p.n, p.col_ptr, p.row_idx, None, None, 0.85, H1, F1, r1, p.stop)
    assert np.abs(H1 - H0).sum() <= 2 * p.stop / 0.15 + 1e-12 * bn
    assert abs(s1["passes"] - s0["passes"]) <= 1


@pytest.mark.parametrize("opts", [{"l2_persist": 4}, {"l2_persist": 64}, {"l2_persist": 8, "hot_window": -1}])
def test_l2_persist_window_forced(opts):
    """options.l2_persist > 0 forces a persisting L2 window over F's most-pushed rows (a
    cache hint only; without the in-degree sample -- hot window off -- it starts at row
    0): the solve is unchanged -- exact identity, same passes as without."""
    p = gen.config("C2", 2)
    H0, F0, _, r0, s0 = _gpu(p.n, p.col_ptr, p.row_idx, p.stop, l2_persist=-1,
                             hot_window=opts.get("hot_window", 0))
    H1, F1, _, r1, s1 = _gpu(p.n, p.col_ptr, p.row_idx, p.stop, **opts)
    _check_state(p.n, p.col_ptr, p.row_idx, None, None, 0.85, H1, F1, r1, p.stop)
    assert np.abs(H1 - H0).sum() <= 2 * p.stop / 0.15
    assert abs(s1["passes"] - s0["passes"]) <= 1


def test_checkpoint_resume_set_state():
    """di_set_state (checkpoint / resume): a solve stopped by max_passes, its (F, H)
    loaded into a fresh context, continues to the same fixed point; the
    restarted schedule begins at T = max |F_i| w_i / alpha, and F = B - (I-P)H holds."""
    p = gen.config("C2", 3, n=200_000)
    o = di.default_options(select_key=di.DI_KEY_EDGE, alpha=2.0, hybrid_frac=0.3, max_passes=25)
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, None, None, p.d, o)
    assert di.di_run(ctx, p.parity_stop, raise_on_not_converged=False) == di.DI_ERR_NOT_CONVERGED
    F, H = di.di_get_fluid(ctx), di.di_get_history(ctx)
    di.di_destroy(ctx)
    o2 = di.default_options(select_key=di.DI_KEY_EDGE, alpha=2.0, hybrid_frac=0.3)
    ctx = di.di_create(p.n, p.col_ptr, p.row_idx, None, None, p.d, o2)
    di.di_set_state(ctx, F, H)
    w = oracle.key_weights(p.n, p.col_ptr, p.row_idx, oracle.KEY_EDGE).astype(np.float64)
    assert di.di_get_stats(ctx)["threshold"] == pytest.approx(float(np.max(np.abs(F) * w)) / 2.0, rel=1e-15)
    di.di_run(ctx, p.parity_stop)
    H2, F2 = di.di_get_history(ctx), di.di_get_fluid(ctx)
    di.di_destroy(ctx)
    X = oracle.Problem(p.n, p.col_ptr, p.row_idx).solve(1e-12 * 0.15 * 0.15).H
    assert np.abs(H2 - X).sum() <= 1e-8 * 0.15
    assert np.all(H2 >= H)                          # the resumed history only grows
    deg = np.diff(p.col_ptr)
    ledger = np.abs(F2).sum() + 0.15 * H2.sum() + 0.85 * H2[deg == 0].sum()
    assert abs(ledger - 0.15) <= 1e-12 * 0.15

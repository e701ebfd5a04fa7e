"""Pins for the CPU oracle (oracle/rsi_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself:

* values PRINTED in the paper's worked example on the
  reconstructed §VI graph (tests/golden/worked_example.txt);
* closed forms (entropy of a uniform / one-community row; complete graphs with
  c equal communities, derivation in DESIGN.md §3);
* special cases (k = 2, one community, stars, degree < 2);
* an independent O(n^3) brute force (tests/bruteforce.py) on random planted
  partitions (SPEC S:542 recipe);
* invariances (vertex relabeling, target order, community relabeling);
* a second implementation's values (SURVEY Appendix A.2 karate partitions).
"""
import math

import numpy as np
import pytest

import gen
import oracle
from bruteforce import brute, select_targets as bf_select


def fx(name):
    g, meta = gen.load_fixture(name)
    return g, meta


# ---------------------------------------------------------------- worked example
def test_worked_example_printed_values():
    g, meta = fx("worked_example")
    targets = [int(x) for x in meta["targets"]]
    r = oracle.run(g, targets=targets, K=10)
    # P:196 border set
    assert list(np.nonzero(r.border)[0]) == [int(x) for x in meta["expect_border"]]
    # P:491 u's histogram (C1, C2, C3, C4) and T
    assert list(r.f[0]) == [int(x) for x in meta["expect_u_counts"]]
    assert r.T[0] == int(meta["expect_u_T"][0])
    # P:491 H(L1) = 1, omega'_u(C1) = 2  (|L| = L_all - 1 = 2)
    L_all = int(np.count_nonzero(r.f[0]))
    assert r.omega[0, 0] / (L_all - 1) == pytest.approx(float(meta["expect_u_H_C1"][0]), abs=1e-15)
    assert r.omega[0, 0] == pytest.approx(float(meta["expect_u_omega_C1"][0]), abs=1e-15)
    # P:491 omega_max = 4.754 and 2/4.754 = 0.42
    v, tol = map(float, meta["expect_omega_max"])
    assert v <= r.omega_max < v + tol          # printed value is truncated
    v, tol = map(float, meta["expect_u_norm_C1"])
    assert abs(r.omega[0, 0] / r.omega_max - v) <= tol
    # P:506 printed normalized weights (2 decimals)
    cidx = {t: i for i, t in enumerate(targets)}
    for tok in meta["expect_norm"]:
        vc, val = tok.split("=")
        vert, comm = map(int, vc.split(":"))
        assert round(r.omega[vert, cidx[comm]] / r.omega_max, 2) == pytest.approx(float(val))
    # P:506 triads: two Type-I, one Type-II at u
    assert (r.nI[0], r.nII[0]) == tuple(int(x) for x in meta["expect_u_triads"])
    # P:506 R(u) = 0.422, printed truncated to 3 decimals
    v, tol = map(float, meta["expect_R_u"])
    assert v <= r.R[0] < v + tol
    # ... and inside the interval the 2-decimal rounding of P:506's weights allows
    def eq4(d):
        a, b, c, e = 0.95 + d, 0.96 + d, 0.86 + d, 0.42 + d
        return ((a * b * c) ** (1 / 3) + (a * a * e) ** (1 / 3) + (c * c * a) ** (1 / 3)) / 6
    assert eq4(-0.005) <= r.R[0] <= eq4(0.005)


def test_worked_example_printed_arithmetic():
    """P:506's own arithmetic with its 2-decimal weights gives 0.422."""
    s = ((0.95 * 0.96 * 0.86) ** (1 / 3) + (0.95 * 0.95 * 0.42) ** (1 / 3) + (0.86 * 0.86 * 0.95) ** (1 / 3)) / 6
    g, meta = fx("worked_example")
    r = oracle.run(g, targets=[1, 2, 3, 4], K=3)
    assert abs(s - 0.422) <= 0.0005
    assert abs(r.R[0] - s) <= 0.001


# ---------------------------------------------------------------- weights (Eq.3/5)
def _w(rows):
    return oracle.weights(np.array(rows, dtype=np.int32))


def test_entropy_special_cases():
    # all neighbours in one community -> H = 0 (north_star invariant), row zero
    assert np.all(_w([[5, 0, 0]]) == 0.0)
    assert np.all(_w([[0, 0, 7, 0]]) == 0.0)
    # uniform over m other communities -> H = log2(m); |L| = L_all - 1
    for m in range(2, 9):
        row = [0] + [3] * m
        w = _w([row])[0]
        assert w[0] == pytest.approx(math.log2(m) * (m - 1), rel=1e-15)
        # own column removed: uniform over m-1 -> log2(m-1) * (m-1)
        assert w[1] == pytest.approx(math.log2(m - 1) * (m - 1), rel=1e-15, abs=0)
    # SPEC S:172-174 examples: [1,1,1] -> 2 ; [2,1,1] col0 -> 2 ; [5,0,0] -> 0
    assert _w([[1, 1, 1]])[0, 0] == pytest.approx(2.0, abs=1e-15)
    assert _w([[2, 1, 1]])[0, 0] == pytest.approx(2.0, abs=1e-15)
    # two-point distribution: H = h2(p) binary entropy
    w = _w([[0, 1, 3]])[0]
    h2 = -(0.25 * math.log2(0.25) + 0.75 * math.log2(0.75))
    assert w[0] == pytest.approx(h2 * 1, rel=1e-15)
    assert w[1] == 0.0 and w[2] == 0.0  # one remaining community -> H = 0


def test_closed_form_matches_direct():
    """Eq. H_optimal == Eq.3 direct within 1e-10 relative for counts <= 1e5
    (SPEC S:541 with the bound relaxed per SURVEY finding 8)."""
    rng = np.random.default_rng(7)
    f = rng.integers(0, 100_000, size=(4000, 6)).astype(np.int32)
    f[rng.random(f.shape) < 0.3] = 0
    a = oracle.weights(f)
    b = oracle.weights(f, closed_form=True)
    nz = a > 0
    assert np.all((a == 0) == (np.abs(b) < 1e-9))
    assert np.max(np.abs(a[nz] - b[nz]) / a[nz]) < 1e-10


# ---------------------------------------------------------------- closed forms
def kn_closed_form(c, m):
    """Complete graph K_{cm}, c communities of m vertices, targets = all
    (derivation in DESIGN.md §3.3)."""
    if c == 2:   # one other community: H = 0, but Type-II triads still exist (counted, C-23)
        return 0.0, 0, (c - 1) * m * (m - 1)
    if m == 1:
        return math.log2(c - 2) / math.log2(c - 1), (c - 1) * (c - 2), 0
    Y = (c - 1) * m - 1
    Hf = -(((m - 1) / Y) * math.log2((m - 1) / Y) + (c - 2) * (m / Y) * math.log2(m / Y))
    h = Hf / math.log2(c - 1)
    R = ((c - 1) * (c - 2) * m * m * h + (m - 1) * (c - 1) * m * h ** (2 / 3)) / ((c * m - 1) * (c * m - 2))
    return R, (c - 1) * (c - 2) * m * m, (c - 1) * m * (m - 1)


@pytest.mark.parametrize("c,m", [(2, 3), (3, 1), (3, 3), (3, 5), (4, 1), (4, 2), (5, 1), (5, 3), (6, 4), (7, 2)])
def test_complete_graph_closed_form(c, m):
    n = c * m
    comm = [i // m for i in range(n)]
    g = gen.from_adjacency(np.ones((n, n), dtype=bool), comm)
    r = oracle.run(g, targets=list(range(c)), K=n)
    R, nI, nII = kn_closed_form(c, m)
    assert np.allclose(r.R, R, rtol=1e-13, atol=0)
    assert np.all(r.nI == nI) and np.all(r.nII == nII)
    if c >= 3 and m >= 2:
        assert r.omega_max == pytest.approx((c - 1) * math.log2(c - 1), rel=1e-15)


# ---------------------------------------------------------------- degenerate cases
def test_single_community_all_zero():
    g = gen.planted_partition(30, 1, 0.3, 0.3, seed=1)
    r = oracle.run(g, k=1, K=5)
    assert not r.border.any() and np.all(r.R == 0) and r.omega_max == 0
    assert r.pred.size == 0 and list(r.top_ids) == [0, 1, 2, 3, 4]


def test_k2_all_zero_and_karate():
    g, meta = fx("karate")
    assert g.m == 78
    r = oracle.run(g, k=2, K=5)
    assert r.omega_max == 0.0 and np.all(r.R == 0)
    assert list(r.top_ids) == [int(x) for x in meta["expect_top5"]]


def test_star_and_degree_one():
    # star: centre in community 0, leaves in 1 -> no two predecessors of any head share... leaves d=1
    n = 8
    edges = [(0, i) for i in range(1, n)]
    g = gen.from_edges(n, edges, [0] + [1] * (n - 1))
    r = oracle.run(g, targets=[0, 1], K=3)
    assert np.all(r.R == 0)
    # degree-1 heads score 0 and count no triads (C-22)
    assert np.all(r.nI[1:] == 0) and np.all(r.nII[1:] == 0)


def test_triangle_three_communities():
    g = gen.from_edges(3, [(0, 1), (1, 2), (0, 2)], [0, 1, 2])
    r = oracle.run(g, targets=[0, 1, 2], K=3)
    assert np.all(r.R == 0) and np.all(r.nI == 2) and np.all(r.nII == 0)


# ---------------------------------------------------------------- brute force
PP_CASES = [(int(n), int(c), seed) for seed, (n, c) in enumerate(
    zip(np.random.default_rng(2024).integers(20, 201, 40), np.random.default_rng(99).integers(3, 7, 40)))]


@pytest.mark.parametrize("n,c,seed", PP_CASES)
def test_oracle_vs_bruteforce(n, c, seed):
    rng = np.random.default_rng(seed + 1000)
    g = gen.planted_partition(n, c, p_in=float(rng.uniform(0.1, 0.4)), p_out=float(rng.uniform(0.02, 0.12)),
                              seed=seed)
    k = int(min(len(np.unique(g.comm)), rng.integers(2, c + 1)))
    t_or = oracle.select_targets(g.comm, k)
    assert list(t_or) == list(bf_select(g.comm, k))
    r = oracle.run(g, targets=t_or, K=g.n)
    b = brute(g, t_or)
    assert np.array_equal(r.border.astype(bool), b["border"])
    assert np.array_equal(r.f, b["f"]) and np.array_equal(r.T, b["f"].sum(1))
    np.testing.assert_allclose(r.omega, b["omega"], rtol=1e-13, atol=1e-15)
    assert r.omega_max == pytest.approx(b["omega_max"], rel=1e-13)
    assert np.array_equal(r.nI, b["nI"]) and np.array_equal(r.nII, b["nII"])
    np.testing.assert_allclose(r.R, b["R"], rtol=1e-12, atol=0)
    # top-k ids: exact unless an adjacent pair is a near tie (C-13)
    R = b["R"]
    near = any(abs(R[b["order"][i]] - R[b["order"][i + 1]]) <= 1e-12 * max(R[b["order"][i]], 1e-300)
               and R[b["order"][i]] != R[b["order"][i + 1]] for i in range(g.n - 1))
    if not near:
        assert list(r.top_ids) == b["order"]
    # G' predecessor lists
    for u in range(g.n):
        nb = g.col[g.rowptr[u]:g.rowptr[u + 1]]
        want = [int(x) for x in nb if g.comm[x] != g.comm[u]]
        assert list(r.pred[r.pred_off[u]:r.pred_off[u + 1]]) == want


# ---------------------------------------------------------------- invariances
def test_vertex_relabel_and_target_order_invariance():
    g = gen.planted_partition(90, 5, 0.25, 0.06, seed=5)
    t = oracle.select_targets(g.comm, 4)
    r = oracle.run(g, targets=t, K=10)
    # vertex permutation: scores permute
    perm = np.random.default_rng(3).permutation(g.n)
    inv = np.argsort(perm)
    A = np.zeros((g.n, g.n), dtype=bool)
    for u in range(g.n):
        A[perm[u], perm[g.col[g.rowptr[u]:g.rowptr[u + 1]]]] = True
    comm2 = np.empty_like(g.comm)
    comm2[perm] = g.comm
    r2 = oracle.run(gen.from_adjacency(A, comm2), targets=t, K=10)
    np.testing.assert_array_equal(r2.R[perm], r.R)   # bit-exact: exact fixed-point sums
    # target column order: same scores up to the entropy's summation order
    r3 = oracle.run(g, targets=t[::-1].copy(), K=10)
    np.testing.assert_allclose(r3.R, r.R, rtol=1e-14, atol=0)
    # community relabel (injective map, targets mapped along)
    relabel = {int(c): 1000 - 7 * int(c) for c in np.unique(g.comm)}
    g4 = gen.Graph(g.rowptr, g.col, np.array([relabel[int(c)] for c in g.comm], dtype=np.int32))
    r4 = oracle.run(g4, targets=[relabel[int(x)] for x in t], K=10)
    np.testing.assert_array_equal(r4.R, r.R)


# ---------------------------------------------------------------- second implementation (karate)
@pytest.mark.parametrize("name", ["karate_greedy3", "karate_louvain4"])
def test_karate_partitions(name):
    g, meta = fx(name)
    k = len(np.unique(g.comm))
    r = oracle.run(g, k=k, K=5)
    assert r.omega_max == pytest.approx(float(meta["expect_omega_max"][0]), rel=1e-15)
    assert int(r.border.sum()) == int(meta["expect_n_border"][0])
    assert int(r.nI.sum()) == int(meta["expect_sum_nI"][0])
    assert int(r.nII.sum()) == int(meta["expect_sum_nII"][0])
    for i, tok in enumerate(meta["expect_top5"]):
        vid, val = tok.split(":")
        assert r.top_ids[i] == int(vid)
        assert r.top_scores[i] == pytest.approx(float(val), abs=1e-11)
    counts_s, om_s = meta["expect_row0"]
    cols = [int(np.nonzero(r.targets == c)[0][0]) for c in range(k)]   # row in community-id order
    assert [int(r.f[0, cc]) for cc in cols] == [int(x) for x in counts_s.split(":")]
    np.testing.assert_allclose([r.omega[0, cc] for cc in cols], [float(x) for x in om_s.split(":")], atol=1e-6)
    if "expect_tie" in meta:
        ties = [int(x) for x in meta["expect_tie"]]
        assert len({r.R[t] for t in ties}) == 1            # bitwise-equal scores
        assert r.R[ties[0]].hex() == "0x1.3f72284032fc4p+0"


# ---------------------------------------------------------------- top-k and targets
def test_topk_rules():
    ids, sc = oracle.topk(np.array([0.5, 0.2, 0.9]), 2)
    assert list(ids) == [2, 0] and list(sc) == [0.9, 0.5]
    ids, _ = oracle.topk(np.zeros(5), 3)                           # S:298 ties by id
    assert list(ids) == [0, 1, 2]
    ids, _ = oracle.topk(np.array([1.0, 2.0]), 10)                 # S:299 clamp
    assert list(ids) == [1, 0]


def test_select_targets_ties():
    comm = np.array([5, 5, 3, 3, 9, 9, 1, 7, 7, 7])
    assert list(oracle.select_targets(comm, 3)) == [7, 3, 5]        # size desc, id asc
    with pytest.raises(ValueError):
        oracle.select_targets(comm, 6)


# ---------------------------------------------------------------- all communities (NEXT-2)
def test_all_communities_singletons_closed_form():
    """K_c with c singleton communities, targets = all (k = c > 254 possible):
    every vertex sees c-1 communities once; its own column is absent (f = 0), so
    omega_u(own) = H(uniform over c-1) (L_all - 1) = (c-2) log2(c-1) -- the
    maximum cell, which only an omega_max over ALL cells (C-7) finds -- and
    every present column has omega = (c-2) log2(c-2).  Each vertex closes
    (c-1)(c-2) Type-I triads with term (h^3)^(1/3) = h, h = log2(c-2)/log2(c-1),
    so R = h (m = 1)."""
    c = 300
    g = gen.from_adjacency(np.ones((c, c), dtype=bool), list(range(c)))
    r = oracle.run(g, k=c, K=5)
    assert r.omega_max == pytest.approx((c - 2) * math.log2(c - 1), rel=1e-14)
    own = r.omega[np.arange(c), [list(r.targets).index(v) for v in range(c)]]
    np.testing.assert_allclose(own, (c - 2) * math.log2(c - 1), rtol=1e-14)
    np.testing.assert_allclose(r.R, math.log2(c - 2) / math.log2(c - 1), rtol=1e-13)
    assert np.all(r.nI == (c - 1) * (c - 2)) and np.all(r.nII == 0)
    assert list(r.targets) == list(range(c))          # equal sizes: ascending id (C-15)


@pytest.mark.parametrize("n,c,seed", [(60, 20, 1), (120, 50, 2), (200, 100, 3), (150, 150, 4)])
def test_all_communities_vs_bruteforce(n, c, seed):
    """Many small communities, targets = all: most columns of a row have f = 0."""
    rng = np.random.default_rng(seed + 3000)
    g = gen.planted_partition(n, c, p_in=float(rng.uniform(0.3, 0.8)), p_out=float(rng.uniform(0.03, 0.1)),
                              seed=seed + 3100)
    k = len(np.unique(g.comm))
    t_or = oracle.select_targets(g.comm, k)
    assert list(t_or) == list(bf_select(g.comm, k))
    r = oracle.run(g, targets=t_or, K=g.n)
    b = brute(g, t_or)
    assert np.array_equal(r.f, b["f"])
    np.testing.assert_allclose(r.omega, b["omega"], rtol=1e-13, atol=1e-15)
    assert r.omega_max == pytest.approx(b["omega_max"], rel=1e-13)
    assert np.array_equal(r.nI, b["nI"]) and np.array_equal(r.nII, b["nII"])
    np.testing.assert_allclose(r.R, b["R"], rtol=1e-12, atol=0)


def _dense_from_tables(tab, n):
    k = tab.targets.size
    f = np.zeros((n, k), dtype=np.int32)
    w = np.repeat(tab.omega_abs[:, None], k, axis=1)
    rows = np.repeat(np.arange(n), np.diff(tab.off))
    f[rows, tab.cols] = tab.cnt
    w[rows, tab.cols] = tab.omega
    return f, w


@pytest.mark.parametrize("n,c,seed", [(60, 20, 1), (120, 50, 2), (200, 100, 3), (150, 150, 4), (300, 6, 5)])
def test_tables_all_vs_dense_and_bruteforce(n, c, seed):
    """oracle_tables_all / oracle_rsi_all (row tables, targets = all) against the
    dense oracle (identical bits: same sums in the same order) and the brute force."""
    rng = np.random.default_rng(seed + 4000)
    g = gen.planted_partition(n, c, p_in=float(rng.uniform(0.3, 0.8)), p_out=float(rng.uniform(0.03, 0.1)),
                              seed=seed + 4100)
    tab = oracle.tables_all(g)
    k = tab.targets.size
    r = oracle.run(g, k=k, K=5)
    assert np.array_equal(tab.targets, r.targets)
    f, w = _dense_from_tables(tab, g.n)
    assert np.array_equal(f, r.f)
    assert np.array_equal(w, r.omega)
    assert tab.omega_max == r.omega_max
    R, nI, nII = oracle.rsi_all(g, tab, np.arange(g.n))
    assert np.array_equal(R, r.R) and np.array_equal(nI, r.nI) and np.array_equal(nII, r.nII)
    b = brute(g, r.targets)
    np.testing.assert_allclose(R, b["R"], rtol=1e-12, atol=0)
    assert np.array_equal(nI, b["nI"]) and np.array_equal(nII, b["nII"])


def test_tables_all_singletons():
    c = 300
    g = gen.from_adjacency(np.ones((c, c), dtype=bool), list(range(c)))
    tab = oracle.tables_all(g)
    assert tab.omega_max == pytest.approx((c - 2) * math.log2(c - 1), rel=1e-14)
    np.testing.assert_allclose(tab.omega_abs, (c - 2) * math.log2(c - 1), rtol=1e-14)
    np.testing.assert_allclose(tab.omega, (c - 2) * math.log2(c - 2), rtol=1e-14)
    R, nI, nII = oracle.rsi_all(g, tab, np.arange(0, c, 37))
    np.testing.assert_allclose(R, math.log2(c - 2) / math.log2(c - 1), rtol=1e-13)

"""Pins of the NEXT-3 literal variants in the oracle (SURVEY §8(c) C-3, C-4,
C-7; DESIGN reading C-30): the literal Eq. 2 |L(u,v)|, Algorithm 1's
|L| > 1 gate and omega_max over Algorithm 1's E_b, against the
complete-graph closed forms, a hand-computed star, and a brute force that runs
Algorithm 1's Step 2 loops literally (every pair of border vertices)."""
import math

import numpy as np
import pytest

import gen
import oracle


def complete_singletons(c):
    return gen.from_edges(c, [(i, j) for i in range(c) for j in range(i + 1, c)], np.arange(c, dtype=np.int32))


@pytest.mark.parametrize("c", [4, 5, 6, 8])
def test_complete_graph_literal_closed_form(c):
    """K_c, one community per vertex, all targets: Algorithm 2 gives
    log2(c-2)/log2(c-1); the literal |L| (own column: L_all = c-1) gives
    (c-2) log2(c-2) / ((c-1) log2(c-1)) (0.5944 for c = 5)"""
    g = complete_singletons(c)
    r0 = oracle.run_variant(g, c, 0)
    r1 = oracle.run_variant(g, c, oracle.LITERAL_L)
    assert r0.R == pytest.approx(np.full(c, math.log2(c - 2) / math.log2(c - 1)), rel=1e-14)
    assert r1.R == pytest.approx(np.full(c, (c - 2) * math.log2(c - 2) / ((c - 1) * math.log2(c - 1))), rel=1e-14)
    if c == 5:
        assert round(float(r1.R[0]), 4) == 0.5944


def test_star_gate_by_hand():
    """centre v (community 0) with leaves in communities 1 and 2, all targets:
    column 0 has f = 0 and the other two communities once each: H = 1;
    Algorithm 2's |L| = L_all - 1 = 1 -> 1, gated -> 0, literal |L| = 2 -> 2"""
    g = gen.from_edges(3, [(0, 1), (0, 2)], np.array([0, 1, 2], np.int32))
    targets = np.array([0, 1, 2], np.int32)
    f, _ = oracle.counts(g, targets)
    assert f[0].tolist() == [0, 1, 1]
    assert oracle.weights_variant(f, 0)[0, 0] == 1.0
    assert oracle.weights_variant(f, oracle.GATE_L)[0, 0] == 0.0
    assert oracle.weights_variant(f, oracle.LITERAL_L)[0, 0] == 2.0
    assert oracle.weights_variant(f, oracle.LITERAL_L | oracle.GATE_L)[0, 0] == 2.0
    # columns 1, 2: one remaining community, H = 0 under every variant
    for fl in range(4):
        assert oracle.weights_variant(f, fl)[0, 1:].tolist() == [0.0, 0.0]


def brute_weights(g, targets, literal, gate):
    """Eq. 2/3/5 per (v, C_i) from the definitions: L = target communities of
    N(v) other than C_i with their frequencies, p = f / sum f, H = -sum p log2 p"""
    k = len(targets)
    w = np.zeros((g.n, k))
    for v in range(g.n):
        nb = [int(g.comm[x]) for x in g.col[g.rowptr[v]:g.rowptr[v + 1]]]
        for i, ci in enumerate(targets):
            freq = {}
            for c in nb:
                if c in targets:
                    freq[c] = freq.get(c, 0) + 1
            L_all = len(freq)
            others = {c: fr for c, fr in freq.items() if c != ci}
            tot = sum(others.values())
            H = -math.fsum(fr / tot * math.log2(fr / tot) for fr in others.values()) if tot else 0.0
            L = len(others) if literal else L_all - 1
            w[v, i] = 0.0 if (L <= 0 or (gate and L <= 1)) else H * L
    return w


def brute_wmax_eb(g, targets, w, literal):
    """Algorithm 1 Step 2 literally: u, v over V_b, C(u) = C(v) or
    v in N(u), |L(u,v)| > 1 -> edge (v -> u) of weight omega_v(C(u))"""
    border = [v for v in range(g.n)
              if any(g.comm[x] != g.comm[v] for x in g.col[g.rowptr[v]:g.rowptr[v + 1]])]
    col_of = {int(t): i for i, t in enumerate(targets)}
    m = 0.0
    for u in border:
        cu = int(g.comm[u])
        if cu not in col_of:
            continue
        i = col_of[cu]
        nu = set(int(x) for x in g.col[g.rowptr[u]:g.rowptr[u + 1]])
        for v in border:
            if g.comm[v] != cu and v not in nu:
                continue
            nb = [int(g.comm[x]) for x in g.col[g.rowptr[v]:g.rowptr[v + 1]]]
            present = set(c for c in nb if c in col_of)
            L = len(present - {cu}) if literal else len(present) - 1
            if L > 1:
                m = max(m, w[v, i])
    return m


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("flags", [0, 1, 2, 3])
def test_variants_against_brute_force(seed, flags):
    g = gen.planted_partition(60, 5, 0.25, 0.06, 300 + seed)
    k = 4
    targets = oracle.select_targets(g.comm, k)
    f, _ = oracle.counts(g, targets)
    w = oracle.weights_variant(f, flags)
    wb = brute_weights(g, [int(t) for t in targets], bool(flags & 1), bool(flags & 2))
    assert np.allclose(w, wb, rtol=1e-13, atol=0.0)
    assert oracle.omega_max_eb(g, targets, f, w, flags) == pytest.approx(
        brute_wmax_eb(g, targets, w, bool(flags & 1)), rel=1e-15)
    if flags == 0:
        assert np.array_equal(w, oracle.weights(f))          # the adopted reading is variant 0


def test_wmax_eb_excludes_cells_without_edges():
    """a vertex whose largest weight is toward a target community it has no
    neighbour in: that cell is not an E_b edge, so the E_b maximum
    is smaller than the all-cells maximum (C-7)"""
    # v = 0 (community 0, not a target) with neighbours in communities 1, 2, 3;
    # target 4 has no neighbour of v: omega_0(4) = log2(3) * 2 is the largest
    # cell, while v's E_b cells (columns 1-3) weigh 1 * 2
    edges = [(0, 1), (0, 2), (0, 3), (4, 5), (4, 1)]
    comm = np.array([0, 1, 2, 3, 4, 4], np.int32)
    g = gen.from_edges(6, edges, comm)
    targets = np.array([1, 2, 3, 4], np.int32)
    f, _ = oracle.counts(g, targets)
    w = oracle.weights_variant(f, 0)
    assert w[0, 3] == pytest.approx(2 * math.log2(3), rel=1e-15)
    assert oracle.omega_max(w) == w[0, 3]
    eb = oracle.omega_max_eb(g, targets, f, w, 0)
    assert eb == 2.0
    assert eb == pytest.approx(brute_wmax_eb(g, targets, w, False), rel=1e-15)


def test_lemma4_border_probability_bounds():
    """Lemma 4: on planted partitions with
    inter-community probability p, the border fraction lies within
    [1 - e^{-(|V| - n_L) p}, 1 - e^{-(|V| - n_S) p}] +- 3 standard errors"""
    n, c, p = 400, 8, 0.004
    fr, lo, hi = [], [], []
    for s in range(30):
        g = gen.planted_partition(n, c, 0.05, p, 7000 + s)
        sizes = np.bincount(g.comm, minlength=c)
        fr.append(oracle.border(g).sum() / n)                 # border mask
        lo.append(1 - math.exp(-(n - sizes.max()) * p))
        hi.append(1 - math.exp(-(n - sizes.min()) * p))
    fr = np.array(fr)
    se = fr.std(ddof=1) / math.sqrt(fr.size)
    assert np.mean(lo) - 3 * se <= fr.mean() <= np.mean(hi) + 3 * se
    assert 0.6 < fr.mean() < 0.9                              # not a degenerate instance
    # the closed form itself (SPEC S:452 example)
    assert (1 - math.exp(-0.5), 1 - math.exp(-0.9)) == pytest.approx((0.39347, 0.59343), abs=1e-5)

"""Pins of the NEXT-1 oracle (absolute AWCC under cumulative random removal,
PAPER §VII.B; DESIGN readings C-28, C-29) against
things other than itself: SPEC's worked values, the plain definition of AWCC
re-derived with Python sets, closed forms of the number of survivors on
complete graphs with one community per vertex, nestedness of the removal sets,
an explicit sort-and-remove brute force, the SplitMix64 reference outputs of
the key generator, and a binomial check that removal is uniform."""
import numpy as np
import pytest

import gen
import oracle

M64 = (1 << 64) - 1
GOLDEN_RATIO = 0x9E3779B97F4A7C15


def complete_graph(n):
    edges = [(u, v) for u in range(n) for v in range(u + 1, n)]
    return gen.from_edges(n, edges, np.arange(n, dtype=np.int32), f"K{n}")


def plain_awcc(g, S):
    """(1/|S|) sum |zeta(v)|/d(v), zeta(v) = communities of v's neighbours"""
    tot = 0.0
    for v in S:
        nb = g.col[g.rowptr[v]:g.rowptr[v + 1]]
        d = nb.size
        if d:
            tot += len(set(int(g.comm[x]) for x in nb)) / d
    return tot / len(S)


def test_key_generator_is_splitmix64():
    # SplitMix64 from state 0: outputs mix(k * golden) for k = 1, 2 (reference values)
    assert oracle.mix64(GOLDEN_RATIO) == 0xE220A8397B1DCDAF
    assert oracle.mix64((2 * GOLDEN_RATIO) & M64) == 0x6E789E6AA1B965F4


def test_spec_examples():
    # S={v}, 4 neighbours over 2 communities -> 0.5
    g = gen.from_edges(5, [(0, 1), (0, 2), (0, 3), (0, 4)], np.array([0, 1, 1, 2, 2], np.int32))
    _, mean = oracle.awcc_removal(g, [0], "edge", 5, 75, 1, 3)
    assert mean[0] == 0.5
    # a singleton zeta with d = 1 -> 1.0; two vertices 0.5 and 1.0 -> 0.75
    _, mean = oracle.awcc_removal(g, [1], "edge", 5, 75, 1, 3)
    assert mean[0] == 1.0
    _, mean = oracle.awcc_removal(g, [0, 1], "edge", 5, 75, 1, 3)
    assert mean[0] == 0.75


@pytest.mark.parametrize("name,scale", [("karate", None), ("dblp", 0.01)])
def test_step0_is_plain_awcc(name, scale):
    g = gen.load_fixture(name)[0] if scale is None else gen.config_graph(name, scale)
    rng = np.random.default_rng(5)
    S = rng.choice(g.n, size=min(25, g.n), replace=False).astype(np.int32)
    for mode in ("edge", "node"):
        zeta, mean = oracle.awcc_removal(g, S, mode, 5, 75, 2, 11)
        assert mean[0] == pytest.approx(plain_awcc(g, S), rel=1e-15)
        for s, v in enumerate(S):
            nb = g.col[g.rowptr[v]:g.rowptr[v + 1]]
            assert zeta[0, 0, s] == len(set(int(g.comm[x]) for x in nb))


@pytest.mark.parametrize("n,step", [(12, 5), (30, 5), (9, 25)])
def test_closed_form_survivors_complete_graph(n, step):
    """K_n with one community per vertex: zeta(v) = v's surviving neighbours, so
    sum_v zeta = 2 (m - r_j) (edges) and (n - r_j)(n - r_j - 1) (nodes),
    r_j = floor(j * step * M / 100)."""
    g = complete_graph(n)
    m = n * (n - 1) // 2
    S = np.arange(n, dtype=np.int32)
    J1 = 100 // step + 1
    ze, _ = oracle.awcc_removal(g, S, "edge", step, 100, 3, 99)
    zn, _ = oracle.awcc_removal(g, S, "node", step, 100, 3, 99)
    for t in range(3):
        for j in range(J1):
            re, rn = (j * step * m) // 100, (j * step * n) // 100
            assert ze[t, j].sum() == 2 * (m - re)
            assert zn[t, j].sum() == (n - rn) * (n - rn - 1)
    assert (ze[:, -1] == 0).all() and (zn[:, -1] == 0).all()      # 100 %: nothing survives


def test_removal_sets_are_nested():
    g = gen.config_graph("dblp", 0.02)
    S = np.argsort(-np.diff(g.rowptr))[:25].astype(np.int32)
    for mode in ("edge", "node"):
        zeta, mean = oracle.awcc_removal(g, S, mode, 5, 75, 4, 1234)
        assert (np.diff(zeta, axis=1) <= 0).all()                 # per trial, per vertex
        assert (np.diff(mean) <= 0).all()


def _keys(st, ids):
    return [oracle.mix64(st ^ i) for i in ids]


@pytest.mark.parametrize("mode", ["edge", "node"])
def test_bruteforce_sort_and_remove(mode):
    """explicit sort of the keys, removal of the r_j smallest, zeta by Python sets"""
    g = gen.config_graph("dblp", 0.003)
    S = np.arange(0, g.n, 7)[:20].astype(np.int32)
    seed, trials, step = 42, 2, 10
    zeta, _ = oracle.awcc_removal(g, S, mode, step, 60, trials, seed)
    md = 0 if mode == "edge" else 1
    edges = [(u, int(v)) for u in range(g.n) for v in g.col[g.rowptr[u]:g.rowptr[u + 1]] if v > u]
    for t in range(trials):
        st = oracle.mix64((seed + (2 * t + md) * GOLDEN_RATIO) & M64)
        items = [(u << 32) | v for u, v in edges] if mode == "edge" else list(range(g.n))
        order = np.argsort(np.array(_keys(st, items), dtype=np.uint64), kind="stable")
        for j in range(60 // step + 1):
            r = (j * step * len(items)) // 100
            gone = set(items[i] for i in order[:r])
            for s, v in enumerate(S):
                v = int(v)
                if mode == "node" and v in gone:
                    want = 0
                else:
                    comms = set()
                    for x in g.col[g.rowptr[v]:g.rowptr[v + 1]]:
                        x = int(x)
                        key = (min(v, x) << 32) | max(v, x) if mode == "edge" else x
                        if key not in gone:
                            comms.add(int(g.comm[x]))
                    want = len(comms)
                assert zeta[t, j, s] == want, (t, j, v)


def test_removal_is_uniform():
    """each edge of a 10x10 grid is removed at 50 % in about half of 400 trials"""
    n = 100
    edges = [(i * 10 + j, i * 10 + j + 1) for i in range(10) for j in range(9)] + \
            [(i * 10 + j, (i + 1) * 10 + j) for i in range(9) for j in range(10)]
    g = gen.from_edges(n, edges, np.arange(n, dtype=np.int32))
    S = np.arange(n, dtype=np.int32)
    zeta, _ = oracle.awcc_removal(g, S, "edge", 50, 50, 400, 2024)
    deg = np.diff(g.rowptr)
    frac_kept = zeta[:, 1, :].sum(axis=0) / (400.0 * deg)   # per vertex: kept incident edges
    # binomial: 400 * d(v) draws at p = 1/2 -> sd <= 0.025; a 6-sd band
    assert np.all(np.abs(frac_kept - 0.5) < 0.15)
    assert abs(frac_kept.mean() - 0.5) < 0.02

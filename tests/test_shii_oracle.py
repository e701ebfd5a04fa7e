"""Pins of the NEXT-4 oracle (SHII under IC / LT diffusion, PAPER §VII.A
P:602-605; DESIGN reading C-31) against things other than
itself: SPEC's worked star, the p = 0 and p = 1 limits (the seed alone; its
connected component, from scipy), independent Python re-runs of the two
diffusion models (IC as live-edge reachability, LT as an incremental threshold
process, whose fixpoint is unique), and monotonicity in p."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

import gen
import oracle

M64 = (1 << 64) - 1
SALT = 0xD1B54A32D192ED03


def run_salt(seed, r, model):
    return oracle.mix64((seed + (2 * r + model + 1) * SALT) & M64)


def py_ic(g, u0, sr, p):
    thr = int(p * 2.0 ** 64) if p < 1 else None
    act = {u0}
    stack = [u0]
    while stack:
        a = stack.pop()
        for b in g.col[g.rowptr[a]:g.rowptr[a + 1]]:
            b = int(b)
            if b in act:
                continue
            if thr is None or oracle.mix64(sr ^ ((a << 32) | b)) < thr:
                act.add(b)
                stack.append(b)
    return act


def py_lt(g, u0, sr):
    """incremental: counters of active neighbours, activation when the count
    reaches ceil(theta * d) (and >= 1)"""
    d = np.diff(g.rowptr)
    need = {}
    for v in range(g.n):
        key = oracle.mix64(sr ^ v)
        need[v] = max(1, -(-(key * int(d[v])) // (1 << 64)))   # ceil(key d / 2^64), exact
    cnt = [0] * g.n
    act = {u0}
    frontier = [u0]
    while frontier:
        nxt = []
        for a in frontier:
            for b in g.col[g.rowptr[a]:g.rowptr[a + 1]]:
                b = int(b)
                if b in act:
                    continue
                cnt[b] += 1
                if cnt[b] >= need[b]:
                    act.add(b)
                    nxt.append(b)
        frontier = nxt
    return act


def test_spec_star_example():
    """IC with p = 1, star centre seed in C1 with neighbours {C2, C2, C1}:
    4 influenced, 2 outside C1 -> 0.5"""
    g = gen.from_edges(4, [(0, 1), (0, 2), (0, 3)], np.array([1, 2, 2, 1], np.int32))
    out, per, m = oracle.shii(g, [0], "ic", 1.0, 3, 5)
    assert out[0, :, 0].tolist() == [4, 4, 4] and out[0, :, 1].tolist() == [2, 2, 2]
    assert per[0] == 0.5 and m == 0.5


def test_ic_limits():
    g = gen.config_graph("dblp", 0.01)
    S = np.array([0, 5, 17, 123], np.int32)
    out, per, _ = oracle.shii(g, S, "ic", 0.0, 4, 9)
    assert (out[:, :, 0] == 1).all() and (out[:, :, 1] == 0).all() and (per == 0).all()
    A = csr_matrix((np.ones(g.col.size), g.col, g.rowptr), shape=(g.n, g.n))
    _, lab = connected_components(A, directed=False)
    out, per, _ = oracle.shii(g, S, "ic", 1.0, 2, 9)
    for s, u in enumerate(S):
        comp = np.nonzero(lab == lab[u])[0]
        assert out[s, 0, 0] == comp.size
        assert out[s, 0, 1] == int((g.comm[comp] != g.comm[u]).sum())
        assert per[s] == out[s, 0, 1] / comp.size


@pytest.mark.parametrize("model", ["ic", "lt"])
def test_models_against_python_reruns(model):
    g = gen.config_graph("dblp", 0.01)
    rng = np.random.default_rng(3)
    S = rng.choice(g.n, size=6, replace=False).astype(np.int32)
    p, runs, seed = 0.2, 4, 77
    out, per, mean = oracle.shii(g, S, model, p, runs, seed)
    md = 0 if model == "ic" else 1
    for s, u in enumerate(S):
        vals = []
        for r in range(runs):
            sr = run_salt(seed, r, md)
            act = py_ic(g, int(u), sr, p) if model == "ic" else py_lt(g, int(u), sr)
            outc = sum(1 for v in act if g.comm[v] != g.comm[u])
            assert out[s, r, 0] == len(act) and out[s, r, 1] == outc, (s, r)
            vals.append(outc / len(act))
        assert per[s] == pytest.approx(sum(vals) / runs, rel=1e-15)
    assert mean == pytest.approx(per.mean(), rel=1e-15)


def test_ic_monotone_in_p():
    """the same coins: a larger p keeps every live edge live"""
    g = gen.config_graph("dblp", 0.01)
    S = np.array([3, 30, 300], np.int32)
    a, _, _ = oracle.shii(g, S, "ic", 0.05, 5, 11)
    b, _, _ = oracle.shii(g, S, "ic", 0.15, 5, 11)
    assert (a[:, :, 0] <= b[:, :, 0]).all()


def test_lt_fixpoint_conditions():
    """every inactive vertex is below its threshold at the end"""
    g = gen.config_graph("dblp", 0.01)
    u0, seed = 42, 5
    sr = run_salt(seed, 0, 1)
    act = py_lt(g, u0, sr)
    out, _, _ = oracle.shii(g, [u0], "lt", 0.1, 1, seed)
    assert out[0, 0, 0] == len(act)
    d = np.diff(g.rowptr)
    for v in range(g.n):
        if v in act:
            continue
        a = sum(1 for x in g.col[g.rowptr[v]:g.rowptr[v + 1]] if int(x) in act)
        assert a == 0 or a * (1 << 64) < oracle.mix64(sr ^ v) * int(d[v])

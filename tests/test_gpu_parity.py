"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs -- bit-exact on counts, border sets, G' lists, triad counts
and top-k ids; fp64 scores within 1e-9 relative (BASELINE north_star)."""
import numpy as np
import pytest

import gen
import oracle
from rsgpu import assert_scores_close, assert_topk, compare_full, run_gpu

pytestmark = pytest.mark.gpu

rsb = pytest.importorskip("paper_2508_01485_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rsb.load_library()


def full(g, k=None, targets=None, K=None, exact_topk=False):
    K = K or g.n
    r_or = oracle.run(g, k=k, targets=targets, K=K)
    r_gpu = run_gpu(g, k=k, targets=r_or.targets, K=K)
    compare_full(g, r_or, r_gpu, exact_topk=exact_topk)
    return r_or, r_gpu


# ---------------------------------------------------------------- fixtures
def test_worked_example():
    g, meta = gen.load_fixture("worked_example")
    r_or, r_gpu = full(g, targets=[int(x) for x in meta["targets"]], exact_topk=True)
    assert 0.422 <= r_gpu["R"][0] < 0.423
    assert (r_gpu["nI"][0], r_gpu["nII"][0]) == (2, 1)


@pytest.mark.parametrize("name,k", [("karate", 2), ("karate_greedy3", 3), ("karate_louvain4", 4)])
def test_karate(name, k):
    g, meta = gen.load_fixture(name)
    r_or, r_gpu = full(g, k=k, exact_topk=True)
    if "expect_tie" in meta:
        ties = [int(x) for x in meta["expect_tie"]]
        assert len({r_gpu["R"][t] for t in ties}) == 1          # exact fixed-point ties
        assert list(r_gpu["top_ids"][:3]) == ties


@pytest.mark.parametrize("c,m", [(3, 1), (3, 3), (4, 2), (5, 3), (6, 4), (2, 5)])
def test_complete_graphs(c, m):
    n = c * m
    g = gen.from_adjacency(np.ones((n, n), dtype=bool), [i // m for i in range(n)])
    full(g, targets=list(range(c)), exact_topk=True)


def test_degenerate_cases():
    # star: centre in one community, leaves in another
    g = gen.from_edges(9, [(0, i) for i in range(1, 9)], [0] + [1] * 8)
    r_or, r_gpu = full(g, targets=[0, 1], exact_topk=True)
    assert np.all(r_gpu["R"] == 0)
    # triangle over three communities: counted, zero weight
    g = gen.from_edges(3, [(0, 1), (1, 2), (0, 2)], [0, 1, 2])
    r_or, r_gpu = full(g, targets=[0, 1, 2], exact_topk=True)
    assert np.all(r_gpu["nI"] == 2)
    # isolated vertices and a single edge
    g = gen.from_edges(6, [(0, 1)], [0, 1, 0, 1, 2, 2])
    full(g, k=2, exact_topk=True)


# ---------------------------------------------------------------- random graphs vs oracle
PP = [(int(n), int(c), s) for s, (n, c) in enumerate(
    zip(np.random.default_rng(11).integers(20, 400, 24), np.random.default_rng(12).integers(3, 9, 24)))]


@pytest.mark.parametrize("n,c,seed", PP)
def test_planted_partitions(n, c, seed):
    rng = np.random.default_rng(seed + 77)
    g = gen.planted_partition(n, c, float(rng.uniform(0.05, 0.4)), float(rng.uniform(0.01, 0.1)), seed=seed + 500)
    k = int(min(len(np.unique(g.comm)), rng.integers(2, c + 1)))
    full(g, k=k)


def test_many_columns_smem_path():
    """k > 8 takes the shared-memory histogram / B-table path."""
    g = gen.planted_partition(600, 14, 0.12, 0.03, seed=3)
    full(g, k=12)


def test_uncoded_communities_full_id_compare():
    """More than 255 communities: the smaller ones share the 0xFF code and the
    border / P-list tests fall back to the full int32 ids."""
    rng = np.random.default_rng(5)
    n = 3000
    g = gen.planted_partition(n, 1, 0.004, 0.004, seed=9)
    comm = rng.integers(0, 700, size=n).astype(np.int32)
    comm[: n // 2] = rng.integers(0, 4, size=n // 2)      # four big communities
    g = gen.Graph(g.rowptr, g.col, comm)
    full(g, k=4)


@pytest.mark.parametrize("name,scale", [("dblp", 0.05), ("lj", 0.004), ("orkut", 0.003), ("orkut", 0.01)])
def test_rsgen_scaled(name, scale):
    g = gen.config_graph(name, scale=scale)
    full(g, k=5, K=200)


def test_dblp_full_size():
    g = gen.config_graph("dblp")
    full(g, k=5, K=25)


# ---------------------------------------------------------------- API behaviour
def test_determinism_and_reuse():
    g = gen.config_graph("orkut", scale=0.003)
    s = rsb.Scorer(0)
    a = run_gpu(g, k=5, scorer=s)
    b = run_gpu(g, k=5, scorer=s)
    assert np.array_equal(a["R"].view(np.uint64), b["R"].view(np.uint64))
    assert np.array_equal(a["top_ids"], b["top_ids"])
    s.close()


@pytest.mark.parametrize("shares", [2, 3, 8])
def test_phase_e_rank_split_emulated(shares):
    """The multi-GPU split of Phase E by middle vertex (items strided over the
    ranks, light warp tasks likewise) run as sequential shares on one GPU: every
    triangle is found exactly once, so scores and Type-I counts are bit-identical
    to the unsplit run (the rank sum itself is an exact u64 allreduce)."""
    g = gen.config_graph("orkut", scale=0.003)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, 5)
    R1 = np.empty(g.n)
    st1 = rsb.rs_score(s.ctx, R1, True, 0)
    t1a, _ = s.triad_counts()
    R2 = np.empty(g.n)
    st2 = rsb.rs_score(s.ctx, R2, True, rsb.RS_E_SHARES(shares))
    t1b, _ = s.triad_counts()
    s.close()
    assert np.array_equal(R1.view(np.uint64), R2.view(np.uint64))
    assert np.array_equal(t1a, t1b)
    assert st1["n_triangles"] == st2["n_triangles"] and st1["n_probes"] == st2["n_probes"]


def test_triad_counts_right_after_score():
    """rs_get_triad_counts straight after rs_score, with no other getter before it,
    on a fresh context and again after switching to other communities (and another
    k): n_I and n_II (the removal sets, C-1) must be the oracle's both times
    (regression: n_II once read a count table only the counts getter filled)."""
    g = gen.config_graph("orkut", scale=0.003)
    rng = np.random.default_rng(31)
    comm2 = rng.permutation(np.max(g.comm) + 1).astype(np.int32)[g.comm]   # relabelled communities
    comm2[rng.integers(0, g.n, g.n // 5)] = 7                               # and a different partition
    g2 = gen.Graph(g.rowptr, g.col, comm2)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    for gg, k in ((g, 5), (g2, 4), (g, 6)):
        s.set_communities(gg.comm, k)
        s.score()
        t1, t2 = s.triad_counts()
        r_or = oracle.run(gg, k=k, K=10)
        np.testing.assert_array_equal(r_or.nI, t1)
        np.testing.assert_array_equal(r_or.nII, t2)
    s.close()


def test_topk_edges_and_device_outputs():
    import torch
    g, _ = gen.load_fixture("karate_greedy3")
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col, validate=True)
    s.set_communities(g.comm, 3)
    s.score()
    ids, sc = s.topk(1000)                 # K > n clamps
    assert len(ids) == g.n
    r_or = oracle.run(g, k=3, K=g.n)
    assert list(ids) == list(r_or.top_ids)
    ids1, _ = s.topk(1)
    assert list(ids1) == [12]
    d_ids = torch.empty(5, dtype=torch.int32, device="cuda")
    d_sc = torch.empty(5, dtype=torch.float64, device="cuda")
    cnt = s.topk(5, d_ids, d_sc)
    torch.cuda.synchronize()
    assert cnt == 5 and d_ids.cpu().tolist() == list(r_or.top_ids[:5])
    # device-resident inputs
    s2 = rsb.Scorer(0)
    s2.load_csr(torch.from_numpy(g.rowptr).cuda(), torch.from_numpy(g.col).cuda())
    s2.set_communities(torch.from_numpy(g.comm).cuda(), 3)
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    s2.score(scores_out=out)
    torch.cuda.synchronize()
    assert_scores_close(r_or.R, out.cpu().numpy())
    s.close()
    s2.close()


def test_user_targets_and_errors():
    g, _ = gen.load_fixture("karate_louvain4")
    r_or = oracle.run(g, targets=[3, 0, 2], K=10)
    r_gpu = run_gpu(g, targets=[3, 0, 2], K=10)
    compare_full(g, r_or, r_gpu, exact_topk=True)
    s = rsb.Scorer(0)
    with pytest.raises(rsb.RsError) as e:
        s.score()
    assert e.value.status == rsb.RS_ESTATE
    # asymmetric CSR
    rp = np.array([0, 1, 1], dtype=np.int64)
    with pytest.raises(rsb.RsError) as e:
        s.load_csr(rp, np.array([1], dtype=np.int32), validate=True)
    assert e.value.status == rsb.RS_EINVAL and "symmetric" in str(e.value)
    # unsorted row
    rp = np.array([0, 2, 3, 4], dtype=np.int64)
    with pytest.raises(rsb.RsError) as e:
        s.load_csr(rp, np.array([2, 1, 0, 0], dtype=np.int32), validate=True)
    assert "ascending" in str(e.value)
    s.load_csr(g.rowptr, g.col, validate=True)
    with pytest.raises(rsb.RsError):
        s.set_communities(g.comm, 5)           # only 4 communities
    with pytest.raises(rsb.RsError):
        s.set_communities(g.comm, 2, targets=[0, 0])
    with pytest.raises(rsb.RsError):
        s.set_communities(-g.comm - 1, 2)
    s.close()


# ---------------------------------------------------------------- NEXT-1: robustness evaluation
@pytest.mark.parametrize("name,scale", [("karate", None), ("dblp", 0.02), ("orkut", 0.003), ("lj", 0.002)])
@pytest.mark.parametrize("mode", ["edge", "node"])
def test_awcc_removal_parity(name, scale, mode):
    """|zeta_j(v)| bit-exact and the mean AWCC per step bit-identical to the
    oracle (DESIGN C-28, C-29), S = the GPU's top-25 plus a random set."""
    g = gen.load_fixture(name)[0] if scale is None else gen.config_graph(name, scale)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    k = 2 if name == "karate" else 5
    s.set_communities(g.comm, k)
    s.score()
    top, _ = s.topk(min(25, g.n))
    rng = np.random.default_rng(17)
    S = np.concatenate([top, rng.choice(g.n, size=min(10, g.n), replace=False)]).astype(np.int32)
    zg, mg = s.awcc_removal(S, mode, 5, 75, 3, 0xA11CE)
    s.close()
    zo, mo = oracle.awcc_removal(g, S, mode, 5, 75, 3, 0xA11CE)
    assert np.array_equal(zg, zo)
    assert np.array_equal(mg.view(np.uint64), mo.view(np.uint64))


def test_awcc_removal_full_orkut_edges():
    """full-size Orkut shape (117 M edges), one trial, 10 % steps to 100 %"""
    g = gen.config_graph("orkut")
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, 5)
    s.score()
    top, _ = s.topk(25)
    zg, mg = s.awcc_removal(top, "edge", 10, 100, 1, 7)
    s.close()
    zo, mo = oracle.awcc_removal(g, top, "edge", 10, 100, 1, 7)
    assert np.array_equal(zg, zo)
    assert np.array_equal(mg, mo)
    assert (zg[0, -1] == 0).all()


def test_awcc_removal_errors():
    g, _ = gen.load_fixture("karate")
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    with pytest.raises(rsb.RsError):
        s.awcc_removal([0, 1])                      # communities not set
    s.set_communities(g.comm, 2)
    for bad in [dict(S=[]), dict(S=[99]), dict(S=[0], step_pct=0), dict(S=[0], max_pct=101),
                dict(S=[0], trials=0)]:
        with pytest.raises((rsb.RsError, ValueError)):
            s.awcc_removal(**bad)
    s.close()


# ---------------------------------------------------------------- NEXT-3: literal variants
@pytest.mark.parametrize("vflags", [1, 2, 3, 4, 7])
@pytest.mark.parametrize("name,scale,k", [("karate", None, 2), ("dblp", 0.02, 5), ("orkut", 0.003, 5),
                                          ("lj", 0.002, 7)])
def test_literal_variants_parity(vflags, name, scale, k):
    """the literal Eq. 2 |L| (1), Algorithm 1's gate (2) and omega_max over E_b (4):
    weights, omega_max, scores, triad counts and top-k against oracle.run_variant
    (rs_score flags = oracle flags << 16: RS_LITERAL_L, RS_GATE_L, RS_WMAX_EB)"""
    g = gen.load_fixture(name)[0] if scale is None else gen.config_graph(name, scale)
    r_or = oracle.run_variant(g, k, vflags, K=g.n)
    r_gpu = run_gpu(g, k=k, targets=r_or.targets, K=g.n, flags=vflags << 16)
    compare_full(g, r_or, r_gpu)


# ---------------------------------------------------------------- NEXT-4: SHII
@pytest.mark.parametrize("model,p", [("ic", 0.05), ("ic", 0.2), ("ic", 1.0), ("lt", 0.0)])
@pytest.mark.parametrize("name,scale", [("karate", None), ("dblp", 0.02), ("orkut", 0.003)])
def test_shii_parity(model, p, name, scale):
    """influenced counts per (seed, run) exact and the SHII means bit-identical to
    the oracle (DESIGN C-31), S = the GPU's top-10 plus random seeds"""
    g = gen.load_fixture(name)[0] if scale is None else gen.config_graph(name, scale)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, 2 if name == "karate" else 5)
    s.score()
    top, _ = s.topk(min(10, g.n))
    rng = np.random.default_rng(23)
    S = np.concatenate([top, rng.choice(g.n, size=min(5, g.n), replace=False)]).astype(np.int32)
    og, pg, mg = s.shii(S, model, p, 3, 0x5111)
    s.close()
    oo, po, mo = oracle.shii(g, S, model, p, 3, 0x5111)
    assert np.array_equal(og, oo)
    assert np.array_equal(pg.view(np.uint64), po.view(np.uint64))
    assert mg == mo


@pytest.mark.parametrize("model,p", [("ic", 0.1), ("ic", 1.0), ("lt", 0.0)])
def test_shii_parity_many_diffusions(model, p):
    """more (seed, run) diffusions than one IC batch holds (64): 29 seeds x 3 runs
    = 87, the second batch starting inside seed 21's runs; counts per (seed, run)
    exact, means bitwise the oracle's (DESIGN C-31)"""
    g = gen.config_graph("orkut", 0.003)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, 5)
    rng = np.random.default_rng(29)
    S = rng.choice(g.n, size=29, replace=False).astype(np.int32)
    S[7] = S[3]                                    # a repeated seed
    og, pg, mg = s.shii(S, model, p, 3, 0xC0FFEE)
    s.close()
    oo, po, mo = oracle.shii(g, S, model, p, 3, 0xC0FFEE)
    assert np.array_equal(og, oo)
    assert np.array_equal(pg.view(np.uint64), po.view(np.uint64))
    assert mg == mo


def test_shii_errors():
    g, _ = gen.load_fixture("karate")
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, 2)
    for bad in [dict(S=[]), dict(S=[40]), dict(S=[0], p=1.5), dict(S=[0], runs=0)]:
        with pytest.raises((rsb.RsError, ValueError)):
            s.shii(**bad)
    s.close()


@pytest.mark.parametrize("log2", [4, 7, 12])
def test_pipelined_load_chunks(log2):
    """rs_load_csr from host arrays with the col_idx copy cut into chunks of
    2^log2 entries (rows relabelled and sorted as each chunk arrives, rows of
    every length class incl. >= 512 and >= 8192): scores and every artefact
    bitwise identical to the one-piece load."""
    g = gen.config_graph("orkut", scale=0.004)
    n = g.n
    # a hub row of >= 8192 entries so that every sort path runs
    extra = np.arange(1, min(n, 9000), dtype=np.int64)
    adj_rows = [set(g.col[g.rowptr[u]:g.rowptr[u + 1]].tolist()) for u in range(n)]
    for v in extra:
        adj_rows[0].add(int(v)); adj_rows[int(v)].add(0)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum([len(r) for r in adj_rows])
    col = np.concatenate([np.array(sorted(r), dtype=np.int32) for r in adj_rows])
    out = []
    for flags in (0, rsb.RS_LOAD_CHUNK_LOG2(log2)):
        s = rsb.Scorer(0)
        s.load_csr(rowptr, col, flags=flags)
        s.set_communities(g.comm, 5)
        R = np.empty(n)
        s.score(scores_out=R)
        off, pl = s.pred()
        t1, t2 = s.triad_counts()
        out.append((R, off, pl, t1, t2, s.topk(25)[0]))
        s.close()
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))

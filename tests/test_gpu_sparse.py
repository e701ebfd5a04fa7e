"""GPU parity of the all-communities mode (NEXT-2): every
community is a target (rs_set_communities k = RS_ALL_COMMUNITIES), the GPU keeps
sparse per-vertex community tables; the oracle computes the plain definition
with targets = all communities (dense tables, O0-O8).  Bit-exact on counts,
borders, G' lists, triad counts and top-k ids; weights 1e-10, scores 1e-9."""
import math

import numpy as np
import pytest

import gen
import oracle
from rsgpu import assert_scores_close, compare_full, run_gpu

pytestmark = pytest.mark.gpu

rsb = pytest.importorskip("paper_2508_01485_b200")
ALL = -1   # RS_ALL_COMMUNITIES


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rsb.load_library()


def full_all(g, K=None, exact_topk=False):
    K = K or g.n
    nc = len(np.unique(g.comm))
    r_or = oracle.run(g, k=nc, K=K)            # targets = all, size desc / id asc
    r_gpu = run_gpu(g, k=ALL, K=K)
    assert len(r_gpu["targets"]) == nc
    compare_full(g, r_or, r_gpu, exact_topk=exact_topk)
    return r_or, r_gpu


def test_worked_example_all():
    g, _ = gen.load_fixture("worked_example")
    r_or, r_gpu = full_all(g, exact_topk=True)
    assert 0.422 <= r_gpu["R"][0] < 0.423                       # P:506 (targets = C1..C4 = all)
    assert (r_gpu["nI"][0], r_gpu["nII"][0]) == (2, 1)


@pytest.mark.parametrize("name", ["karate", "karate_greedy3", "karate_louvain4"])
def test_karate_all(name):
    g, meta = gen.load_fixture(name)
    r_or, r_gpu = full_all(g, exact_topk=True)
    if "expect_tie" in meta:
        ties = [int(x) for x in meta["expect_tie"]]
        assert len({r_gpu["R"][t] for t in ties}) == 1
        assert list(r_gpu["top_ids"][:3]) == ties


@pytest.mark.parametrize("c,m", [(3, 1), (3, 3), (5, 3), (6, 4), (2, 5)])
def test_complete_graphs_all(c, m):
    n = c * m
    g = gen.from_adjacency(np.ones((n, n), dtype=bool), [i // m for i in range(n)])
    full_all(g, exact_topk=True)


def test_complete_graph_many_singletons():
    """K_300 with 300 singleton communities (k = 300 > 254): every R equals the
    closed form log2(c-2)/log2(c-1) (m = 1)."""
    c = 300
    g = gen.from_adjacency(np.ones((c, c), dtype=bool), list(range(c)))
    r_or, r_gpu = full_all(g, K=10)
    want = math.log2(c - 2) / math.log2(c - 1)
    np.testing.assert_allclose(r_gpu["R"], want, rtol=1e-12)
    assert np.all(r_gpu["nI"] == (c - 1) * (c - 2)) and np.all(r_gpu["nII"] == 0)


PP = [(int(n), int(c), s) for s, (n, c) in enumerate(
    zip(np.random.default_rng(21).integers(20, 400, 12), np.random.default_rng(22).integers(2, 40, 12)))]


@pytest.mark.parametrize("n,c,seed", PP)
def test_planted_partitions_all(n, c, seed):
    rng = np.random.default_rng(seed + 91)
    g = gen.planted_partition(n, c, float(rng.uniform(0.05, 0.4)), float(rng.uniform(0.01, 0.1)), seed=seed + 900)
    if len(np.unique(g.comm)) < 2:
        pytest.skip("one community")
    full_all(g, K=25)


@pytest.mark.parametrize("name,scale,n_comm", [("dblp", 0.02, 64), ("lj", 0.003, 600), ("orkut", 0.004, 300),
                                               ("lj", 0.002, 1200), ("dblp", 0.02, 1000)])
def test_rsgen_many_communities(name, scale, n_comm):
    g = gen.config_graph(name, scale=scale, n_comm=n_comm, zipf_s=0.8)
    full_all(g, K=25)


def test_sparse_matches_dense_mode():
    """k <= 254 communities: the all-communities mode and explicit targets = all
    compute the same scores (weights may differ by rounding of X's sum order)."""
    g = gen.config_graph("orkut", scale=0.003, n_comm=40)
    nc = len(np.unique(g.comm))
    tg = oracle.select_targets(g.comm, nc)
    r_dense = run_gpu(g, targets=tg, K=50)
    r_sp = run_gpu(g, k=ALL, K=50)
    assert np.array_equal(r_dense["targets"], r_sp["targets"])
    assert np.array_equal(r_dense["f"], r_sp["f"])
    np.testing.assert_array_equal(r_dense["nI"], r_sp["nI"])
    np.testing.assert_array_equal(r_dense["nII"], r_sp["nII"])
    np.testing.assert_allclose(r_sp["R"], r_dense["R"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("shares", [2, 5])
def test_sparse_rank_split_emulated(shares):
    g = gen.config_graph("orkut", scale=0.004, n_comm=500, zipf_s=0.8)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, ALL)
    R1 = np.empty(g.n)
    s.score(scores_out=R1)
    t1a, _ = s.triad_counts()
    R2 = np.empty(g.n)
    s.score(scores_out=R2, flags=rsb.RS_E_SHARES(shares))
    t1b, _ = s.triad_counts()
    assert np.array_equal(R1.view(np.uint64), R2.view(np.uint64))
    assert np.array_equal(t1a, t1b)
    s.close()


def test_sparse_errors_and_switching():
    g = gen.config_graph("dblp", scale=0.01, n_comm=100)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    with pytest.raises(rsb.RsError) as e:
        rsb.rs_set_communities(s.ctx, g.comm, ALL, np.array([0, 1], dtype=np.int32))
    assert e.value.status == rsb.RS_EINVAL
    with pytest.raises(rsb.RsError) as e:
        s.set_communities(np.zeros(g.n, dtype=np.int32), ALL)   # one community
    assert e.value.status == rsb.RS_EINVAL
    s.set_communities(g.comm, ALL)
    with pytest.raises(rsb.RsError) as e:
        s.score(flags=rsb.RS_LITERAL_L)
    assert e.value.status == rsb.RS_EINVAL
    # all -> explicit k -> all on one context
    R_all = np.empty(g.n)
    s.score(scores_out=R_all)
    s.set_communities(g.comm, 5)
    R5 = np.empty(g.n)
    s.score(scores_out=R5)
    r5 = oracle.run(g, k=5, K=10)
    np.testing.assert_allclose(R5, r5.R, rtol=1e-9)
    s.set_communities(g.comm, ALL)
    R_all2 = np.empty(g.n)
    s.score(scores_out=R_all2)
    assert np.array_equal(R_all.view(np.uint64), R_all2.view(np.uint64))
    s.close()


def test_sparse_hub_rows_and_repeatability():
    """Rows of every length class incl. >= 8192 (CUB segmented sort of the
    neighbour columns) and 2048..8192 (CTA tables): full parity, and repeated
    rs_score calls bitwise identical (the row sort is ordered before the forked
    table bins)."""
    n, c = 9000, 300
    rng = np.random.default_rng(5)
    comm = rng.integers(0, c, n).astype(np.int32)
    adj = np.zeros((n, n), dtype=bool)
    adj[0, :] = True                                  # degree n-1 >= 8192
    adj[1:4] |= rng.random((3, n)) < 0.4              # ~3600: CTA class
    m = 60000
    a_, b_ = rng.integers(0, n, m), rng.integers(0, n, m)
    adj[a_, b_] = True
    adj |= adj.T
    g = gen.from_adjacency(adj, comm)
    assert np.diff(g.rowptr).max() >= 8192
    full_all(g, K=25)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, ALL)
    R = [np.empty(g.n) for _ in range(3)]
    for r in R:
        s.score(scores_out=r)
    _, w1 = s.weights()
    assert all(np.array_equal(R[0].view(np.uint64), r.view(np.uint64)) for r in R[1:])
    s.close()


def _check_tables(s, tab):
    """The GPU's sparse rows against oracle.tables_all: columns and counts
    bit-exact for every vertex, weights (present and absent) within 1e-10."""
    off, cols, cnt, om, oa = s.comm_tables()
    assert np.array_equal(off, tab.off)
    assert np.array_equal(cols, tab.cols) and np.array_equal(cnt, tab.cnt)
    for got, want in ((om, tab.omega), (oa, tab.omega_abs)):
        nz = want != 0
        assert np.array_equal(got != 0, nz)
        if nz.any():
            assert np.max(np.abs(got[nz] - want[nz]) / want[nz]) <= 1e-10


@pytest.mark.parametrize("name,scale,n_comm", [("lj", 0.003, 600), ("orkut", 0.004, 2000)])
def test_comm_tables_getter(name, scale, n_comm):
    g = gen.config_graph(name, scale=scale, n_comm=n_comm, zipf_s=0.8)
    tab = oracle.tables_all(g)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, ALL)
    assert np.array_equal(s.targets(), tab.targets)
    R = np.empty(g.n)
    st = s.score(scores_out=R, stats=True)
    assert abs(st["omega_max"] - tab.omega_max) <= 1e-10 * tab.omega_max
    _check_tables(s, tab)
    heads = np.arange(g.n)
    Ro, nI, nII = oracle.rsi_all(g, tab, heads)
    assert_scores_close(Ro, R)
    t1, t2 = s.triad_counts()
    assert np.array_equal(nI, t1) and np.array_equal(nII, t2)
    s.close()


def test_full_size_all_communities_sampled():
    """The bench's NEXT-2 workload (bench.SPARSE_CFG: LiveJournal shape, 10 000
    communities) in its launch configuration: every vertex's sparse row (columns,
    counts, weights), omega_max and borders against the oracle, scores and triad
    counts on sampled heads (random + the GPU's top-25 + the highest degrees),
    and the top-K property on the sample."""
    from bench import SPARSE_CFG
    g = gen.config_graph(SPARSE_CFG["base"], n_comm=SPARSE_CFG["n_comm"], zipf_s=SPARSE_CFG["zipf_s"])
    tab = oracle.tables_all(g)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, ALL)
    assert np.array_equal(s.targets(), tab.targets)
    R = np.empty(g.n)
    st = s.score(scores_out=R, stats=True)
    assert abs(st["omega_max"] - tab.omega_max) <= 1e-10 * tab.omega_max
    _check_tables(s, tab)
    assert np.array_equal(np.nonzero(oracle.border(g))[0].astype(np.int32), s.border())
    top_ids, top_sc = s.topk(25)
    t1, t2 = s.triad_counts()
    rng = np.random.default_rng(7)
    deg = np.diff(g.rowptr)
    heads = np.unique(np.concatenate([rng.integers(0, g.n, 400), top_ids.astype(np.int64), np.argsort(deg)[-20:]]))
    Ro, nI, nII = oracle.rsi_all(g, tab, heads)
    assert_scores_close(Ro, R[heads])
    assert np.array_equal(nI, t1[heads]) and np.array_equal(nII, t2[heads])
    assert np.all(Ro[~np.isin(heads, top_ids)] <= top_sc[-1] * (1 + 1e-9))
    s.close()

"""The multi-GPU path on one GPU: `world` emulated
ranks (rs_create_emulated -- host threads, one context each, collectives as
host barriers + device-to-device copies) each run their whole pipeline: the
Phase A shard of their own vertex range, the exchange of Phase A's outputs,
their share of the Type-I middle vertices with the limb sum over the ranks,
the Type-II pull and finalize of their own heads, and rs_topk's filtered
local select + all-gather + merge. The merged world must give bitwise the
single-GPU scores, top-K ids and scores, and the exact artefacts."""
import threading

import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

rsb = pytest.importorskip("paper_2508_01485_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rsb.load_library()


def one_rank(s, g, k, K, flags=0):
    s.load_csr(g.rowptr, g.col)
    s.set_communities(g.comm, k)
    R = np.empty(g.n)
    st = s.score(scores_out=R, stats=True, gather=True, flags=flags)
    ids, sc = s.topk(K)
    t1, t2 = s.triad_counts()
    f, T = s.counts()
    w, wmax = s.weights()
    return dict(R=R, ids=ids, sc=sc, t1=t1, t2=t2, f=f, T=T, w=w, wmax=wmax, bv=s.border(),
                tri=st["n_triangles"], probes=st["n_probes"], omega_max=st["omega_max"])


def run_world(g, k, K, world, flags=0):
    import torch
    W = rsb.EmuWorld(world)
    out, err = [None] * world, []

    def main(r):
        try:
            stream = torch.cuda.Stream(device=0)
            s = rsb.Scorer(0, stream.cuda_stream, rank=r, world=world, emu=W)
            out[r] = one_rank(s, g, k, K, flags)
            s.close()
        except Exception as e:  # reported by the main thread
            err.append(f"rank {r}: {e!r}")

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    W.close()
    assert not err, err
    assert all(o is not None for o in out), "a rank did not finish"
    return out


CASES = [("orkut", 0.01, 5), ("lj", 0.004, 5), ("dblp", 0.05, 7)]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,scale,k", CASES)
def test_emulated_world_matches_single_gpu(name, scale, k, world, flags=0):
    g = gen.config_graph(name, scale=scale)
    K = 50
    s = rsb.Scorer(0)
    ref = one_rank(s, g, k, K)
    s.close()
    out = run_world(g, k, K, world, flags)
    np.testing.assert_array_equal(sum(o["t2"] for o in out), ref["t2"])
    for r, o in enumerate(out):
        np.testing.assert_array_equal(o["t1"], ref["t1"])
        assert o["omega_max"] == ref["omega_max"] and o["tri"] == ref["tri"] and o["probes"] == ref["probes"]
        bad = np.nonzero(o["R"].view(np.uint64) != ref["R"].view(np.uint64))[0]
        assert bad.size == 0, (f"rank {r}: {bad.size} scores differ, e.g. {bad[:8].tolist()} "
                               f"{o['R'][bad[:4]].tolist()} vs {ref['R'][bad[:4]].tolist()}")
        assert np.array_equal(o["ids"], ref["ids"]) and np.array_equal(o["sc"].view(np.uint64), ref["sc"].view(np.uint64))
        assert o["omega_max"] == ref["omega_max"] and o["tri"] == ref["tri"] and o["probes"] == ref["probes"]
        np.testing.assert_array_equal(o["t1"], ref["t1"])            # n_I: summed over the ranks
        assert np.array_equal(o["f"], ref["f"]) and np.array_equal(o["T"], ref["T"])
        assert np.array_equal(o["w"].view(np.uint64), ref["w"].view(np.uint64)) and o["wmax"] == ref["wmax"]
        assert np.array_equal(o["bv"], ref["bv"])
    # n_II: each rank reports its own heads (zeros elsewhere)
    np.testing.assert_array_equal(sum(o["t2"] for o in out), ref["t2"])
    # the GPU's filtered local select + merge equals the host protocol's merge of
    # every rank's candidates (rs_local_candidates over the gathered scores)
    n = g.n
    ck, ci = rsb.rs_local_candidates(ref["R"], np.arange(n, dtype=np.int32), K)
    mi, ms = rsb.rs_merge_candidates(ck, ci, min(K, n))
    assert np.array_equal(mi, ref["ids"])


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("name,scale,k", CASES[:2])
def test_emulated_world_replicated_phase_a(name, scale, k, world):
    """RS_REPLICATE_A (the north_star's replicated CSR + labels): every rank runs
    Phase A over all vertices, no Phase A exchange; bitwise the single GPU's
    results, and the only exchanged bytes are the limb reduce-scatter (+ the
    counters and the optional score gather)"""
    test_emulated_world_matches_single_gpu(name, scale, k, world, flags=rsb.RS_REPLICATE_A)
    g = gen.config_graph(name, scale=scale)
    import torch
    W = rsb.EmuWorld(world)
    xb, err = [None] * world, []

    def main(r):
        try:
            s = rsb.Scorer(0, torch.cuda.Stream(device=0).cuda_stream, rank=r, world=world, emu=W)
            s.load_csr(g.rowptr, g.col)
            s.set_communities(g.comm, k)
            st = s.score(stats=True, flags=rsb.RS_REPLICATE_A)
            xb[r] = (st["xchg_allreduce_bytes"], st["xchg_allgather_bytes"], st["xchg_reduce_scatter_bytes"])
            s.close()
        except Exception as e:
            err.append(repr(e))

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    W.close()
    assert not err, err
    for ar, ag, rsc in xb:
        assert ag == 0 and ar == 16 and rsc == 24 * g.n


def test_emulated_world_tiny_and_errors():
    """karate with 8 ranks (ranges of a few vertices, some heads-free) and the
    multi-GPU restrictions (k <= 8 explicit targets)."""
    g, _ = gen.load_fixture("karate")
    s = rsb.Scorer(0)
    ref = one_rank(s, g, 2, 34)
    s.close()
    for o in run_world(g, 2, 34, 8):
        assert np.array_equal(o["R"].view(np.uint64), ref["R"].view(np.uint64))
        assert np.array_equal(o["ids"], ref["ids"])
    W = rsb.EmuWorld(1)
    s = rsb.Scorer(0, rank=0, world=1, emu=W)        # a world of one is the single-GPU path
    o = one_rank(s, g, 2, 34)
    s.close()
    W.close()
    assert np.array_equal(o["R"].view(np.uint64), ref["R"].view(np.uint64))
    with pytest.raises(rsb.RsError):
        rsb.EmuWorld(0)


def test_emulated_world_serial_mode_repeats():
    """serial mode (the multi-GPU model of bench.py): ranks take turns inside
    rs_score, several calls in a row, same bits as the concurrent world"""
    import torch
    g = gen.config_graph("orkut", scale=0.004)
    s = rsb.Scorer(0)
    ref = one_rank(s, g, 5, 25)
    s.close()
    world = 4
    W = rsb.EmuWorld(world)
    W.serial(True)
    out, err = [None] * world, []

    def main(r):
        try:
            stream = torch.cuda.Stream(device=0)
            sc = rsb.Scorer(0, stream.cuda_stream, rank=r, world=world, emu=W)
            sc.load_csr(g.rowptr, g.col)
            sc.set_communities(g.comm, 5)
            for _ in range(3):
                R = np.empty(g.n)
                st = sc.score(scores_out=R, stats=True, gather=True)
            out[r] = (R, st["ms_phase"])
            sc.close()
        except Exception as e:
            err.append(repr(e))

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    W.close()
    assert not err and all(o is not None for o in out), err
    for R, ph in out:
        assert np.array_equal(R.view(np.uint64), ref["R"].view(np.uint64))
        assert ph[0] > 0 and ph[2] > 0


@pytest.mark.parametrize("nbytes", [64, 8 << 20])
def test_nccl_transport_world1(nbytes):
    """The NCCL transport of rs_create_dist on real hardware: a one-rank
    communicator (only one GPU is available to these tests) runs every
    collective the exchange uses -- all-reduce sum / max, all-gather, the
    grouped-broadcast all-gather of segments, the grouped-reduce reduce-scatter
    of segments -- through NCCL's kernels on a torch stream; librs checks each
    result bit for bit (a world of one leaves / copies its input)."""
    import torch
    s = torch.cuda.Stream()
    rsb.rs_nccl_selftest(torch.cuda.current_device(), s.cuda_stream, nbytes)
    rsb.rs_nccl_selftest(torch.cuda.current_device(), None, nbytes)   # a stream of its own
    with pytest.raises(rsb.RsError):
        rsb.rs_nccl_selftest(torch.cuda.current_device(), None, 12)

"""Memory hygiene of librs without compute-sanitizer (closed on this pool,
profiles/r02_compute_sanitizer_closed.txt): a read of device memory that no
kernel wrote, or of a table left over from an earlier call, changes results.

* poison: every device allocation filled with 0x00, 0xFF or 0xA5 before use
  (rs_debug_poison) -> every output of the pipeline and every getter bitwise
  identical across the three bytes (the initcheck stand-in);
* reuse: a context that scored other communities (another k, another mode)
  first gives bitwise the outputs of a fresh context (stale-table reads).
"""
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
    yield
    rsb.rs_debug_poison(-1)


def everything(s, g, k, K=50, flags=0):
    """every output of one step and of every getter, as raw bytes"""
    s.set_communities(g.comm, k)
    R = np.empty(g.n)
    st = s.score(scores_out=R, stats=True, flags=flags)
    ids, sc = s.topk(K)
    out = {"R": R, "ids": ids, "sc": sc, "wmax": np.array([st["omega_max"]]),
           "tri": np.array([st["n_triangles"], st["n_probes"], st["n_border"], st["n_pred_entries"]])}
    t1, t2 = s.triad_counts()
    out.update(nI=t1, nII=t2)
    if k != rsb.RS_ALL_COMMUNITIES:
        f, T = s.counts()
        w, _ = s.weights()
        out.update(f=f, T=T, w=w)
    else:
        out.update(zip(("off", "cols", "cnt", "om", "oa"), s.comm_tables()))
    out["bv"] = s.border()
    out["off_p"], out["pred"] = s.pred()
    return {a: np.ascontiguousarray(b).view(np.uint8) for a, b in out.items()}


def same(a, b):
    assert a.keys() == b.keys()
    for key in a:
        assert np.array_equal(a[key], b[key]), key


CASES = [("orkut", 0.004, 5), ("lj", 0.003, 7), ("dblp", 0.03, 12), ("orkut", 0.003, rsb.RS_ALL_COMMUNITIES)]


@pytest.mark.parametrize("name,scale,k", CASES)
def test_poisoned_allocations_do_not_change_results(name, scale, k):
    g = gen.config_graph(name, scale=scale)
    outs = []
    for byte in (0x00, 0xFF, 0xA5):
        rsb.rs_debug_poison(byte)
        s = rsb.Scorer(0)
        s.load_csr(g.rowptr, g.col)
        outs.append(everything(s, g, k))
        s.close()
    rsb.rs_debug_poison(-1)
    same(outs[0], outs[1])
    same(outs[0], outs[2])


def test_reused_context_equals_fresh():
    g = gen.config_graph("orkut", scale=0.004)
    rng = np.random.default_rng(3)
    other = gen.Graph(g.rowptr, g.col, rng.permutation(g.comm.max() + 1).astype(np.int32)[g.comm])
    rsb.rs_debug_poison(0x5A)
    s = rsb.Scorer(0)
    s.load_csr(g.rowptr, g.col)
    everything(s, other, 7)                             # another partition, another k
    everything(s, other, rsb.RS_ALL_COMMUNITIES)        # the sparse mode in between
    everything(s, g, 5, flags=rsb.RS_LITERAL_L | rsb.RS_WMAX_EB)   # a variant
    reused = everything(s, g, 5)
    s.close()
    rsb.rs_debug_poison(0xC3)
    f = rsb.Scorer(0)
    f.load_csr(g.rowptr, g.col)
    fresh = everything(f, g, 5)
    f.close()
    rsb.rs_debug_poison(-1)
    same(reused, fresh)

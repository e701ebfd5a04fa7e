"""Full-size parity (BASELINE configs[2..4] shapes, the bench's launch
configuration): the CUDA path through the C-ABI against the UNCHANGED oracle
over EVERY head (oracle/parallel.py splits the heads over the host cores;
each head is still one single-threaded oracle_rsi evaluation).

* LJ and Orkut shapes: every count, weight (1e-10), border flag and G' list
  bit-exact / in tolerance, every score within 1e-9 relative, every n_I / n_II
  bit-exact, and the top-25 ids exactly the oracle's (a swap is tolerated only
  between oracle scores within 1e-12 relative, reading C-13, and reported).
* Friendster shape (1.8 G edges): against tests/golden/friendster_top25.txt,
  written from oracle/ only by tools/oracle_golden.py (all 65.6 M heads).
"""
import math
import os

import numpy as np
import pytest

import gen
import oracle
from oracle.parallel import rsi_all_heads
from rsgpu import SCORE_RTOL, WEIGHT_RTOL, assert_scores_close, assert_topk, run_gpu

pytestmark = pytest.mark.gpu

rsb = pytest.importorskip("paper_2508_01485_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rsb.load_library()


@pytest.mark.parametrize("name", ["lj", "orkut"])
def test_full_size_exact(name):
    g = gen.config_graph(name)
    r_gpu = run_gpu(g, k=5, K=25, validate=False)
    t = oracle.select_targets(g.comm, 5)
    assert np.array_equal(t, r_gpu["targets"])
    f, T = oracle.counts(g, t)
    assert np.array_equal(f, r_gpu["f"]) and np.array_equal(T, r_gpu["T"])
    w = oracle.weights(f)
    del f, T
    wmax = oracle.omega_max(w)
    nz = w != 0
    assert np.array_equal(nz, r_gpu["omega"] != 0)
    assert np.max(np.abs(r_gpu["omega"][nz] - w[nz]) / w[nz]) <= WEIGHT_RTOL
    assert abs(r_gpu["omega_max"] - wmax) <= WEIGHT_RTOL * wmax
    del nz
    assert np.array_equal(np.nonzero(oracle.border(g))[0].astype(np.int32), r_gpu["border"])
    off, pl = oracle.pred(g)
    np.testing.assert_array_equal(off, r_gpu["pred_off"])
    np.testing.assert_array_equal(pl, r_gpu["pred"])
    del off, pl
    R, nI, nII, info = rsi_all_heads(g, t, w, wmax)
    assert_scores_close(R, r_gpu["R"])
    np.testing.assert_array_equal(nI, r_gpu["nI"])
    np.testing.assert_array_equal(nII, r_gpu["nII"])
    ids, sc = oracle.topk(R, 25)
    assert_topk(ids, r_gpu["top_ids"], lambda v: R[v])
    np.testing.assert_allclose(r_gpu["top_scores"], sc, rtol=SCORE_RTOL, atol=0)
    print(f"{name}: oracle over {g.n} heads in {info['wall_s']:.0f}s on {info['procs']} processes "
          f"(single-thread sum {info['cpu_s']:.0f}s)")


def _golden(path):
    meta, top, nxt, sample = {}, [], [], []
    with open(path) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            key, *rest = line.split()
            if key == "top":
                top.append((int(rest[1]), float(rest[2]), int(rest[3]), int(rest[4])))
            elif key == "next":
                nxt.append((int(rest[1]), float(rest[2]), int(rest[3]), int(rest[4])))
            elif key == "sample":
                sample.append((int(rest[0]), float(rest[1]), int(rest[2]), int(rest[3])))
            else:
                meta[key] = rest
    return meta, top, nxt, sample


GOLDEN_FR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "friendster_top25.txt")


@pytest.mark.skipif(not os.path.exists(GOLDEN_FR), reason="tools/oracle_golden.py friendster not run")
def test_friendster_top25_golden():
    """BASELINE configs[4] (north_star's target): librs's top-25 on the
    1.8 G-edge Friendster shape equals the oracle's (all heads scored by the
    oracle offline, tests/golden/friendster_top25.txt), plus every score and
    triad count of a seeded head sample, omega_max and whole-graph sums."""
    import torch
    meta, top, nxt, sample = _golden(GOLDEN_FR)
    g = gen.config_graph("friendster")
    assert (g.n, g.m) == (int(meta["n"][0]), int(meta["m"][0]))
    dev = torch.device("cuda", 0)
    s = rsb.Scorer(0)
    rp = torch.from_numpy(g.rowptr).to(dev)
    cl = torch.from_numpy(g.col).to(dev)
    s.load_csr(rp, cl)
    del rp, cl
    torch.cuda.empty_cache()
    s.set_communities(g.comm, int(meta["k"][0]))
    R = np.empty(g.n)
    st = s.score(scores_out=R, stats=True)
    ids, sc = s.topk(int(meta["K"][0]))
    t1, t2 = s.triad_counts()
    targets = s.targets()
    s.close()
    assert list(map(int, targets)) == [int(x) for x in meta["targets"]]
    wm = float(meta["omega_max"][0])
    assert abs(st["omega_max"] - wm) <= WEIGHT_RTOL * wm
    ref = {v: r for v, r, _, _ in top + nxt}
    assert_topk([v for v, _, _, _ in top], ids, lambda v: ref.get(int(v), -1.0))
    for (v, r, a, b), got in zip(top, sc):
        assert abs(got - r) <= SCORE_RTOL * r
        assert (t1[v], t2[v]) == (a, b)
    sv = np.array([x[0] for x in sample], dtype=np.int64)
    assert_scores_close(np.array([x[1] for x in sample]), R[sv])
    np.testing.assert_array_equal(np.array([x[2] for x in sample]), t1[sv])
    np.testing.assert_array_equal(np.array([x[3] for x in sample]), t2[sv])
    assert int(np.count_nonzero(R)) == int(meta["nonzero_R"][0])
    assert abs(math.fsum(R.tolist()) - float(meta["sum_R"][0])) <= SCORE_RTOL * float(meta["sum_R"][0])
    assert int(t1.sum()) == int(meta["sum_nI"][0]) and int(t2.sum()) == int(meta["sum_nII"][0])

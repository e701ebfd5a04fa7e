"""World-size-2 tests of the multi-GPU host protocol on CPU with
torch.distributed over gloo. Every rank computes the head-range split with
librs's exported protocol function (the same code the GPU kernel k_split runs)
and the ranks must agree; each rank then takes the top-K of its own range,
the candidates are all-gathered across processes (the exchange rs_topk does
with ncclAllGather) and merged with rs_merge_candidates, which must give the
oracle's global top-K (ties by ascending id; C-14) on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
INT32_MAX = 2**31 - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(rank, world, port, case, args, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        q.put((rank, "ok", case(rank, world, *args)))
    except Exception as e:  # report, the parent asserts
        q.put((rank, "err", repr(e)))
    finally:
        dist.destroy_process_group()


def _run(case, *args, world=WORLD):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_entry, args=(r, world, port, case, args, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in ps:
        r, status, res = q.get(timeout=240)
        assert status == "ok", res
        out[r] = res
    for p in ps:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _gather(arr):
    """all_gather of an equal-length 1-D int64 array across the ranks."""
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return np.concatenate([p.numpy() for p in parts])


# ---------------------------------------------------------------- cases (run in the ranks)
def case_split(rank, world, n, seed):
    import paper_2508_01485_b200 as rsb
    rng = np.random.default_rng(seed)
    work = rng.pareto(1.2, n).astype(np.int64) + 1          # heavy-tailed d(u) + 1
    incl = np.cumsum(work)
    b = rsb.rs_split_ranges(incl, world)
    allb = _gather(b).reshape(world, world + 1)
    assert (allb == allb[0]).all(), "ranks disagree on the split"
    assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
    total = int(incl[-1])
    part = [int(work[b[r]:b[r + 1]].sum()) for r in range(world)]
    assert sum(part) == total
    # each range reaches its share, overshooting by at most one vertex
    assert max(part) <= -(-total // world) + int(work.max())
    return b.tolist()


def _local_candidates(scores, ids, K):
    """rank-local Step-4 candidates through librs's exported protocol function
    (rs_local_candidates: key desc, id asc, padded (0, INT32_MAX)), the order
    the GPU's filtered local select produces (checked against it by
    tests/test_gpu_multirank.py)."""
    import paper_2508_01485_b200 as rsb
    ck, ci = rsb.rs_local_candidates(scores, ids, K)
    return ck, ci.astype(np.int64)


def case_merge(rank, world, scores, K):
    import paper_2508_01485_b200 as rsb
    n = scores.shape[0]
    b = rsb.rs_split_ranges(np.arange(1, n + 1, dtype=np.int64), world)
    ids = np.arange(b[rank], b[rank + 1], dtype=np.int64)
    ck, ci = _local_candidates(scores[b[rank]:b[rank + 1]], ids, K)
    gk = _gather(ck.view(np.int64)).view(np.uint64)
    gi = _gather(ci).astype(np.int32)
    mi, ms = rsb.rs_merge_candidates(gk, gi, min(K, n))
    return mi.tolist(), ms.tolist()


# ---------------------------------------------------------------- tests
def test_split_ranges_agree_and_balance():
    res = _run(case_split, 10_000, 7)
    assert res[0] == res[1]


def test_split_ranges_edge_cases():
    import paper_2508_01485_b200 as rsb
    assert rsb.rs_split_ranges(np.zeros(0, np.int64), 3).tolist() == [0, 0, 0, 0]
    assert rsb.rs_split_ranges(np.array([5], np.int64), 4).tolist()[-1] == 1
    b = rsb.rs_split_ranges(np.cumsum(np.ones(8, np.int64)), 4)
    assert b.tolist() == [0, 2, 4, 6, 8]
    with pytest.raises(rsb.RsError):
        rsb.rs_split_ranges(np.ones(3, np.int64), 0)


def test_topk_merge_matches_oracle_scores():
    import gen
    import oracle
    g = gen.config_graph("dblp", 0.01)
    res = oracle.run(g, k=5, K=25)
    out = _run(case_merge, np.asarray(res.R, dtype=np.float64), 25)
    for ids, sc in out:                       # identical on every rank
        assert ids == list(res.top_ids)
        assert np.array_equal(np.array(sc), np.asarray(res.top_scores))


def test_topk_merge_ties_across_ranks():
    """many equal scores straddling the range boundary: ties resolved by id."""
    import oracle
    rng = np.random.default_rng(11)
    scores = rng.choice(np.array([0.0, 0.25, 0.5, 0.75]), size=997)
    scores[::7] = 0.75
    ids_o, sc_o = oracle.topk(scores, 60)
    out = _run(case_merge, scores, 60)
    for ids, sc in out:
        assert ids == list(ids_o)
        assert np.array_equal(np.array(sc), np.asarray(sc_o))


def test_local_candidates_order_and_padding():
    import paper_2508_01485_b200 as rsb
    ck, ci = rsb.rs_local_candidates(np.array([0.5, -0.0, 0.5, 0.25]), np.array([9, 3, 4, 1], np.int32), 6)
    assert ci.tolist() == [4, 9, 1, 3, INT32_MAX, INT32_MAX]
    assert ck.tolist()[:4] == rsb.score_keys(np.array([0.5, 0.5, 0.25, 0.0])).tolist() and ck.tolist()[4:] == [0, 0]


def test_topk_merge_K_larger_than_candidates():
    import paper_2508_01485_b200 as rsb
    keys = rsb.score_keys(np.array([0.5, 0.0, 0.5, -0.0]))
    ids, sc = rsb.rs_merge_candidates(keys, np.array([9, 3, 4, 1], np.int32), 10)
    assert ids.tolist() == [4, 9, 1, 3] and sc.tolist() == [0.5, 0.5, 0.0, 0.0]

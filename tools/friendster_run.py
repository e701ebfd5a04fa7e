"""BASELINE configs[4] shape on ONE B200: the Friendster-shape DC-SBM (65.6 M
vertices, ~1.8 G edges) scored end to end through the C-ABI,
timed like bench.py (CUDA events, L2 flushed between steps), then checked
against the CPU oracle: target columns, every vertex's counts, border flags,
every weight (1e-10) and omega_max exactly as in the full-size parity tests,
and scores / triad counts one by one on a head sample (random + the GPU's
top-25 + the highest-degree heads) plus the top-K property on the sample.

Runs on the GPU box (about 10 minutes, ~60 GB host RAM, ~150 GB HBM):
    python tools/friendster_run.py > gpurun_out/friendster.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2508_01485_b200 as rsb  # noqa: E402


def main():
    import torch
    dev = torch.device("cuda", 0)
    out = {"workload": "friendster-shape DC-SBM (SURVEY §8(d), BASELINE configs[4]) on 1 B200", "k": 5, "K": 25}
    t0 = time.time()
    g = gen.config_graph("friendster")
    out.update(n=g.n, m=g.m, nnz=g.nnz, gen_s=round(time.time() - t0, 1), d_max=int(np.diff(g.rowptr).max()))
    print(json.dumps({"generated": out}), file=sys.stderr, flush=True)

    stream = torch.cuda.Stream(dev)
    s = rsb.Scorer(0, stream.cuda_stream)
    rp = torch.from_numpy(g.rowptr).to(dev)
    cl = torch.from_numpy(g.col).to(dev)
    cm = torch.from_numpy(g.comm).to(dev)
    t1 = time.time()
    s.load_csr(rp, cl)
    torch.cuda.synchronize(dev)
    out["load_s"] = round(time.time() - t1, 2)
    del rp, cl
    torch.cuda.empty_cache()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ids = torch.empty(25, dtype=torch.int32, device=dev)
    sco = torch.empty(25, dtype=torch.float64, device=dev)
    ms = []
    for i in range(2 + 5):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.set_communities(cm, 5)
        s.score()
        s.topk(25, ids, sco)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    st = s.score(stats=True)
    step = float(np.median(ms))
    out.update(ms_per_step=round(step, 3), GTEPS=round(g.m / (step * 1e-3) / 1e9, 3),
               step_ms_all=[round(x, 3) for x in ms], phase_ms=[round(x, 3) for x in st["ms_phase"][:4]],
               n_border=st["n_border"], pred_entries=st["n_pred_entries"], triangles=st["n_triangles"],
               probes=st["n_probes"], omega_max=st["omega_max"],
               hbm_used_gb=round(torch.cuda.mem_get_info(dev)[1] / 1e9 - torch.cuda.mem_get_info(dev)[0] / 1e9, 1))
    print(json.dumps({"gpu": out}), file=sys.stderr, flush=True)

    # GPU artefacts to the host
    R_gpu = np.empty(g.n)
    s.score(scores_out=R_gpu)
    top_ids, top_sc = s.topk(25)
    f_gpu, T_gpu = s.counts()
    w_gpu, wmax_gpu = s.weights()
    bv_gpu = s.border()
    t1_gpu, t2_gpu = s.triad_counts()
    tg = s.targets()
    s.close()
    del cm, flush
    torch.cuda.empty_cache()

    # oracle (single-threaded C), same checks as tests/test_gpu_parity.py::test_full_size_sampled
    par = {}
    t2 = time.time()
    t = oracle.select_targets(g.comm, 5)
    par["targets"] = bool(np.array_equal(t, tg))
    f, T = oracle.counts(g, t)
    par["counts_bitexact"] = bool(np.array_equal(f, f_gpu) and np.array_equal(T, T_gpu))
    del f_gpu
    w = oracle.weights(f)
    wmax = oracle.omega_max(w)
    nz = w != 0
    par["weight_zero_pattern"] = bool(np.array_equal(nz, w_gpu != 0))
    par["weight_max_rel_err"] = float(np.max(np.abs(w_gpu[nz] - w[nz]) / w[nz])) if nz.any() else 0.0
    par["omega_max_rel_err"] = abs(wmax_gpu - wmax) / wmax if wmax > 0 else abs(wmax_gpu)
    del w_gpu
    par["border_bitexact"] = bool(np.array_equal(np.nonzero(oracle.border(g))[0].astype(np.int32), bv_gpu))
    rng = np.random.default_rng(4)
    deg = np.diff(g.rowptr)
    heads = np.unique(np.concatenate([rng.integers(0, g.n, 300), top_ids.astype(np.int64), np.argsort(deg)[-10:]]))
    R, nI, nII = oracle.rsi(g, t, w, wmax, heads)
    zo, zg = R == 0, R_gpu[heads] == 0
    rel = np.abs(R_gpu[heads][~zo] - R[~zo]) / R[~zo] if (~zo).any() else np.zeros(1)
    par["sampled_heads"] = int(heads.size)
    par["score_zero_pattern"] = bool(np.array_equal(zo, zg))
    par["score_max_rel_err"] = float(rel.max())
    par["triad_counts_bitexact"] = bool(np.array_equal(nI, t1_gpu[heads]) and np.array_equal(nII, t2_gpu[heads]))
    kth = top_sc[-1]
    par["topk_property_on_sample"] = bool(np.all(R[~np.isin(heads, top_ids)] <= kth * (1 + 1e-9)))
    par["oracle_s"] = round(time.time() - t2, 1)
    par["pass"] = bool(par["targets"] and par["counts_bitexact"] and par["weight_zero_pattern"]
                       and par["weight_max_rel_err"] <= 1e-10 and par["omega_max_rel_err"] <= 1e-10
                       and par["border_bitexact"] and par["score_zero_pattern"] and par["score_max_rel_err"] <= 1e-9
                       and par["triad_counts_bitexact"] and par["topk_property_on_sample"])
    out["parity"] = par
    out["top5"] = [[int(a), float(b)] for a, b in zip(top_ids[:5], top_sc[:5])]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

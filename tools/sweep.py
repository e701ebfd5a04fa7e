"""SURVEY §8(d) sweeps on the LiveJournal shape: mixing mu in {0.1, 0.2, 0.3,
0.5} (k = 5) and target count k in {4, 5, 6, 7} (mu = 0.2), plus the other
configs (DBLP, LJ, Orkut) at k = 5. Device step time (rs_set_communities +
rs_score + rs_topk(25), CUDA events, L2 flushed, median of 5 after 3 warm-ups),
GTEPS and the per-phase split. One JSON line per case.
    python tools/sweep.py > gpurun_out/sweep.jsonl
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2508_01485_b200 as rsb  # noqa: E402


def run(name, g, k, stream, dev, flush):
    import torch
    s = rsb.Scorer(0, stream.cuda_stream)
    rp = torch.from_numpy(g.rowptr).to(dev)
    cl = torch.from_numpy(g.col).to(dev)
    cm = torch.from_numpy(g.comm).to(dev)
    s.load_csr(rp, cl)
    ids = torch.empty(25, dtype=torch.int32, device=dev)
    sco = torch.empty(25, dtype=torch.float64, device=dev)
    ms = []
    for i in range(3 + 5):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.set_communities(cm, k)
        s.score()
        s.topk(25, ids, sco)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= 3:
            ms.append(e0.elapsed_time(e1))
    st = s.score(stats=True)
    s.close()
    step = float(np.median(ms))
    return {"case": name, "n": g.n, "m": g.m, "k": k, "ms_per_step": round(step, 4),
            "GTEPS": round(g.m / (step * 1e-3) / 1e9, 3),
            "phase_ms": {"A": round(st["ms_phase"][0], 4), "ED": round(st["ms_phase"][2], 4),
                         "F": round(st["ms_phase"][3], 4)},
            "n_border": st["n_border"], "pred_entries": st["n_pred_entries"], "triangles": st["n_triangles"],
            "probes": st["n_probes"]}


def main():
    import torch
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    cases = [("lj mu=%g" % mu, "lj", dict(mu=mu), 5) for mu in (0.1, 0.2, 0.3, 0.5)]
    cases += [("lj k=%d" % k, "lj", {}, k) for k in (4, 6, 7)]
    cases += [("dblp k=5", "dblp", {}, 5), ("orkut k=5", "orkut", {}, 5)]
    for name, cfg, over, k in cases:
        t = time.time()
        g = gen.config_graph(cfg, **over)
        r = run(name, g, k, stream, dev, flush)
        r["gen_s"] = round(time.time() - t, 1)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

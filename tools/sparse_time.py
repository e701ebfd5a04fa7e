"""Time the all-communities mode (NEXT-2) on an LFR-style graph (many
communities) with per-phase stats. usage: python tools/sparse_time.py [cfg] [n_comm]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
import paper_2508_01485_b200 as rsb

cfg = sys.argv[1] if len(sys.argv) > 1 else "lj"
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
t = time.time()
g = gen.config_graph(cfg, n_comm=nc, zipf_s=0.8)
print(f"gen {time.time()-t:.1f}s n={g.n} m={g.m} comms={len(np.unique(g.comm))}", flush=True)
s = rsb.Scorer(0)
s.load_csr(g.rowptr, g.col)
for mode in ["all", 64]:
    s.set_communities(g.comm, rsb.RS_ALL_COMMUNITIES if mode == "all" else mode)
    for i in range(3):
        s.score()
    torch.cuda.synchronize()
    ts = []
    for i in range(5):
        st = s.score(stats=True)
        ts.append(st)
    ms = [sum(x["ms_phase"][:4]) for x in ts]
    print(mode, "k=", s.k, "ms", [round(x, 3) for x in ms], "phases", [round(x, 3) for x in ts[-1]["ms_phase"][:4]],
          "GTEPS", round(g.m / (np.median(ms) * 1e6), 2), "pred", ts[-1]["n_pred_entries"], "tri", ts[-1]["n_triangles"],
          "wmax", ts[-1]["omega_max"], flush=True)
s.close()

"""debug: emulated world vs single GPU, per-rank breakdown of n_II / scores by internal id"""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import gen
import paper_2508_01485_b200 as rsb
from test_gpu_multirank import one_rank, run_world

g = gen.config_graph("orkut", scale=0.01)
s = rsb.Scorer(0)
ref = one_rank(s, g, 5, 50)
s.close()
world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = run_world(g, 5, 50, world)
deg = np.diff(g.rowptr)
order = np.lexsort((np.arange(g.n), -deg))        # internal id -> original (degree desc, stable)
inv = np.empty(g.n, np.int64); inv[order] = np.arange(g.n)
cuts = np.linspace(0, g.n, 9).astype(int)
for r, o in enumerate(out):
    nz = np.nonzero(o["t2"])[0]
    print("rank", r, "nonzero t2 internal id range", inv[nz].min() if nz.size else None, inv[nz].max() if nz.size else None)
t2 = sum(o["t2"] for o in out)
bad = np.nonzero(t2 != ref["t2"])[0]
print("t2 bad", bad.size, "internal ids hist", np.histogram(inv[bad], bins=cuts)[0].tolist())
print("t2 examples", [(int(v), int(inv[v]), int(t2[v]), int(ref["t2"][v]), int(deg[v])) for v in bad[:10]])
for r, o in enumerate(out):
    b1 = np.nonzero(o["t1"] != ref["t1"])[0]
    bR = np.nonzero(o["R"] != ref["R"])[0]
    print("rank", r, "t1 bad", b1.size, "R bad", bR.size, np.histogram(inv[bR], bins=cuts)[0].tolist(),
          "f ok", np.array_equal(o["f"], ref["f"]), "w ok", np.array_equal(o["w"], ref["w"]), "bv ok", np.array_equal(o["bv"], ref["bv"]),
          "tri", o["tri"], ref["tri"], "probes", o["probes"], ref["probes"], "wmax", o["omega_max"], ref["omega_max"])

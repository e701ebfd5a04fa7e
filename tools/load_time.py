"""rs_load_csr timing: device-resident input and host (pinned) input, per config.
    python tools/load_time.py orkut [friendster]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2508_01485_b200 as rsb  # noqa: E402
import torch  # noqa: E402

for name in sys.argv[1:] or ["orkut"]:
    g = gen.config_graph(name)
    dev = torch.device("cuda", 0)
    s = rsb.Scorer(0)
    rp, cl = torch.from_numpy(g.rowptr).to(dev), torch.from_numpy(g.col).to(dev)
    for _ in range(2):
        s.load_csr(rp, cl)
    torch.cuda.synchronize()
    t = time.perf_counter(); s.load_csr(rp, cl); torch.cuda.synchronize(); dt_dev = time.perf_counter() - t
    del rp, cl
    rph, clh = torch.from_numpy(g.rowptr).pin_memory(), torch.from_numpy(g.col).pin_memory()
    s.load_csr(rph, clh)
    torch.cuda.synchronize()
    t = time.perf_counter(); s.load_csr(rph, clh); torch.cuda.synchronize(); dt_host = time.perf_counter() - t
    print(f"{name}: nnz={g.nnz} load from device {dt_dev*1e3:.2f} ms, from pinned host {dt_host*1e3:.2f} ms "
          f"(H2D {g.col.nbytes/1e9:.2f} GB)", flush=True)
    s.close()

"""One bench step (rs_set_communities + rs_score + rs_topk, the bench's device-
resident inputs) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off`: the capture holds exactly one step's kernels.
    python tools/ncu_step.py [--config orkut] [--warmup 2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2508_01485_b200 as rsb  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="orkut")
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--k", type=int, default=5)
    a = p.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    g = gen.config_graph(a.config)
    stream = torch.cuda.Stream(dev)
    s = rsb.Scorer(0, stream.cuda_stream)
    rp, cl, cm = (torch.from_numpy(x).to(dev) for x in (g.rowptr, g.col, g.comm))
    s.load_csr(rp, cl)
    ids = torch.empty(25, dtype=torch.int32, device=dev)
    sc = torch.empty(25, dtype=torch.float64, device=dev)

    def step():
        s.set_communities(cm, a.k)
        s.score()
        s.topk(25, ids, sc)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize(dev)
    torch.cuda.profiler.stop()
    print("one step captured", a.config, g.n, g.m)


if __name__ == "__main__":
    main()

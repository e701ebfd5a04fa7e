"""One rs_score of every rank of an emulated world (serial mode: the ranks take
turns between collectives, so their kernels never overlap) bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off --metrics
gpu__time_duration.sum`: the launch list says where a rank's time goes at N
ranks (kernels whose work does not shrink with N).
    python tools/ncu_world.py [--config orkut] [--world 8]"""
import argparse
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2508_01485_b200 as rsb  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="orkut")
    p.add_argument("--world", type=int, default=8)
    p.add_argument("--k", type=int, default=5)
    p.add_argument("--replicated", action="store_true", help="RS_REPLICATE_A (Phase A on every rank)")
    a = p.parse_args()
    import torch
    g = gen.config_graph(a.config)
    N = a.world
    fl = rsb.RS_REPLICATE_A if a.replicated else 0
    W = rsb.EmuWorld(N)
    W.serial(True)
    bar = threading.Barrier(N)
    err, out = [], [None] * N

    def rank(r):
        try:
            stream = torch.cuda.Stream(device=0)
            s = rsb.Scorer(0, stream.cuda_stream, rank=r, world=N, emu=W)
            s.load_csr(g.rowptr, g.col)
            s.set_communities(g.comm, a.k)
            for _ in range(2):
                s.score(flags=fl)
            torch.cuda.synchronize()
            bar.wait()
            if r == 0:
                torch.cuda.profiler.start()
            bar.wait()
            st = s.score(stats=True, flags=fl)
            torch.cuda.synchronize()
            bar.wait()
            if r == 0:
                torch.cuda.profiler.stop()
            own = [round(x - w, 4) for x, w in zip(st["ms_phase"][:6], st["ms_xwait"][:6])]
            out[r] = own
            print(f"rank {r} own kernel ms per phase {own}", flush=True)
            s.close()
        except Exception as e:  # reported below
            err.append(f"rank {r}: {e!r}")
            bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    W.close()
    if err:
        print(err)
        sys.exit(1)
    import numpy as np
    P = np.array(out)
    print("world", N, a.config, "max over ranks per phase", P.max(axis=0).round(4).tolist(),
          "mean", P.mean(axis=0).round(4).tolist())


if __name__ == "__main__":
    main()

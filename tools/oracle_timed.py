"""Full, timed, single-threaded oracle run (SURVEY §8(d) "Oracle timing"):
O0-O8 of oracle/rsi_oracle.c over EVERY head of one BASELINE-shape config in
one thread, wall time per phase (steady clock, generation excluded), printed
as one JSON line. Run on the GPU box's host to record the CPU baseline that
bench.py's sampled cpu_baseline estimates.

    python tools/oracle_timed.py orkut > gpurun_out/oracle_orkut.json
"""
import json
import os
import platform
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import gen  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    name = sys.argv[1]
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    t0 = time.perf_counter()
    g = gen.config_graph(name) if name != "karate" else gen.load_fixture("karate")[0]
    gen_s = time.perf_counter() - t0
    oracle.build()
    ph = {}
    t = time.perf_counter()
    tg = oracle.select_targets(g.comm, k if name != "karate" else 2)
    ph["O0_targets"] = time.perf_counter() - t
    t = time.perf_counter()
    oracle.border(g)
    ph["O1_border"] = time.perf_counter() - t
    t = time.perf_counter()
    f, _ = oracle.counts(g, tg)
    ph["O2_counts"] = time.perf_counter() - t
    t = time.perf_counter()
    w = oracle.weights(f)
    ph["O3_weights"] = time.perf_counter() - t
    t = time.perf_counter()
    wmax = oracle.omega_max(w)
    ph["O4_omega_max"] = time.perf_counter() - t
    t = time.perf_counter()
    oracle.pred(g)
    ph["O5a_pred_lists"] = time.perf_counter() - t
    t = time.perf_counter()
    R, nI, nII = oracle.rsi(g, tg, w, wmax)
    ph["O5_O7_rsi_all_heads"] = time.perf_counter() - t
    t = time.perf_counter()
    ids, _ = oracle.topk(R, 25)
    ph["O8_topk"] = time.perf_counter() - t
    total = sum(ph.values())
    print(json.dumps({"config": name, "n": g.n, "m": g.m, "k": int(tg.size), "threads": 1,
                      "cpu": cpu_model(), "nproc": os.cpu_count(), "gen_s": round(gen_s, 1),
                      "phase_s": {a: round(b, 3) for a, b in ph.items()}, "total_s": round(total, 2),
                      "GTEPS": g.m / total / 1e9, "top5": [int(x) for x in ids[:5]],
                      "sum_nI": int(nI.sum()), "sum_nII": int(nII.sum()),
                      "nonzero_R": int(np.count_nonzero(R))}), flush=True)


if __name__ == "__main__":
    main()

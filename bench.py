#!/usr/bin/env python
"""RSI hot-path benchmark (arXiv 2508.01485 on B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config orkut|lj|dblp|karate]
                    [--impl ours|reference] [--K 25]

One step = the whole hot path on one synthetic
graph resident in HBM: rs_set_communities (target selection + labels) ->
rs_score (border, histogram, weights, G' lists, Type-I/II triad sums,
finalize) -> rs_topk (K = 25). Metric: RSI-scored edges/s (GTEPS) = m /
step time. Each timed step is bracketed by CUDA events on the library's
stream; L2 is flushed (a 512 MiB write) between steps, outside the events.
For N > 1 (torchrun), heads are split into work-balanced ranges, ranks merge
top-K with NCCL, and the time is the max over ranks.

--impl reference times the CPU oracle (oracle/, single thread) on a bounded
sample of the same workload (the reference arm of this tier).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import gen  # noqa: E402

METRIC = "RSI-scored edges/sec (GTEPS)"
UNIT = "GTEPS"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--no-awcc", action="store_true", help="skip the NEXT-1/3/4 evaluation timings")
    p.add_argument("--config", default="orkut", choices=["orkut", "lj", "dblp", "karate", "friendster"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--K", type=int, default=25)
    p.add_argument("--k", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-mgpu", action="store_true", help="skip the emulated multi-GPU model leg")
    p.add_argument("--phases", action="store_true", help="print per-phase ms to stderr")
    p.add_argument("--mg-mode", default="sharded", choices=["sharded", "replicated"],
                   help="N > 1: Phase A sharded + exchanged, or replicated on every rank (RS_REPLICATE_A)")
    return p.parse_args()


def load_graph(name, alloc=None):
    if name == "karate":
        g, _ = gen.load_fixture("karate")
        return g
    return gen.config_graph(name, alloc=alloc)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    5 ms during the timed region (nvidia-smi is too slow for a 100 ms region)."""

    def __init__(self, index=0, period_s=0.005):
        self.index = index
        self.period = period_s
        self.rows = []
        self.maxclk = None
        self._stop = threading.Event()
        self._t = None
        self.err = None

    def _sample(self):
        N = self._N
        clk = N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)
        rs = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.rows.append((clk, [k for k, v in self._bits.items() if rs & v]))

    def _run(self):
        try:
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(self.period)
        except Exception as e:  # NVML failure mid-run: report it
            self.err = repr(e)

    def __enter__(self):
        # NVML is initialised and a first sample taken before the timed region
        # starts (the sampling thread alone could miss a short region)
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.maxclk = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
            self._bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                          "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                          "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap,
                          "hw_power_brake": N.nvmlClocksEventReasonHwPowerBrakeSlowdown}
            self._sample()
        except Exception as e:  # NVML unavailable: report it
            self.err = repr(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)
            try:
                self._sample()   # and one at the end of the region
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.maxclk, "reasons": [self.err or "no samples"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.maxclk, "reasons": reasons,
                "samples": len(self.rows), "source": "NVML, 5 ms period, timed region only"}


# ------------------------------------------------------------------ algorithmic bytes
def survey_bytes(n, D, Db, k, ntri, nprobe):
    """SURVEY §8(d)'s algorithmic-bytes table, term by term (4-byte ids, 1-byte
    labels, 8-byte values): the HEADLINE roofline bytes. librs's Phase A fuses
    §8(d)'s phases A (border + histogram + weights), B (P-list build) and C (B
    table), so its bytes are their sum; E || D is §8(d)'s D (Type-II) + E
    (Type-I: 4 B per probed entry + 16 B per matched triad); F is finalize."""
    A = 4 * D + 8 * n + 1 * D + 4 * n + 8 * k * n + 8 * n
    B = 4 * D + 8 * n + 1 * D + 4 * Db + 8 * n
    C = 4 * Db + 8 * Db + 8 * k * n
    Dt2 = 4 * Db + 8 * Db + 8 * Db + 8 * n
    E = 4 * nprobe + 16 * ntri
    F = 8 * n * 3
    return {"A": A + B + C, "ED": Dt2 + E, "F": F}


def fused_bytes(n, D, Db, k, ntri, nprobe):
    """The bytes librs's fused pipeline moves at least once (DESIGN.md §6
    kernel table): reported beside the survey figure, not as the headline."""
    A = 8 * (n + 1) + 4 * D + 1 * D + 1 * n + 4 * Db + 16 * k * n + 16 * n + 4 * Db + 6 * Db + 8 * Db + 16 * n
    E = 4 * nprobe + 20 * (Db // 2) + 32 * ntri + 8 * k * n
    D_ = 4 * Db + 16 * Db + 16 * n + 16 * n
    F = 16 * n + 24 * n + 16 * n + 8 * n + 4 * n + 8 * n
    return {"A": A, "ED": E + D_, "F": F}


def build_hash():
    """sha256 (16 hex) of librs's sources: ties an ncu capture to the build it measured."""
    import glob
    import hashlib
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(REPO, "paper_2508_01485_b200", "csrc", "*"))):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + fh.read())
    return h.hexdigest()[:16]


def ncu_record(config):
    """per-kernel ncu figures of the committed capture (profiles/ncu_kernels.json,
    written by tools/ncu_kernels.py from one `ncu --set full` run of bench.py)"""
    p = os.path.join(REPO, "profiles", "ncu_kernels.json")
    if not os.path.exists(p):
        return None
    rec = json.load(open(p))
    if rec.get("config") != config:
        return None
    rec["build_match"] = rec.get("build") == build_hash()
    return rec


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return reference_arm(a, rank, world)
    import torch
    import torch.distributed as dist
    import paper_2508_01485_b200 as rsb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    sh = stream.cuda_stream

    t0 = time.time()
    g = load_graph(a.config)
    gen_s = time.time() - t0
    n, D, m = g.n, g.nnz, g.m

    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(rsb.rs_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        sc = rsb.Scorer(local, sh, rank=rank, world=world, nccl_id=bytes(idt.cpu().numpy()))
    else:
        sc = rsb.Scorer(local, sh)

    # device-resident inputs
    rp_d = torch.from_numpy(g.rowptr).to(dev)
    col_d = torch.from_numpy(g.col).to(dev)
    comm_d = torch.from_numpy(g.comm).to(dev)
    ids_d = torch.empty(a.K, dtype=torch.int32, device=dev)
    sco_d = torch.empty(a.K, dtype=torch.float64, device=dev)
    sc.load_csr(rp_d, col_d, validate=False)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    mgf = rsb.RS_REPLICATE_A if (world > 1 and a.mg_mode == "replicated") else 0

    def step():
        sc.set_communities(comm_d, a.k)
        sc.score(gather=False, flags=mgf)
        sc.topk(a.K, ids_d, sco_d)

    # warm-up (also sizes every buffer)
    for _ in range(max(a.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    st = sc.score(stats=True, flags=mgf)
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    phase_ms = []
    launches0 = sc.launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xFF)            # L2 flush outside the timed events
            ev[i][0].record(stream)
            sc.set_communities(comm_d, a.k)
            s = sc.score(stats=a.phases, flags=mgf)
            sc.topk(a.K, ids_d, sco_d)
            ev[i][1].record(stream)
            if a.phases:
                phase_ms.append(s["ms_phase"][:4])
        torch.cuda.synchronize(dev)
    launches = sc.launches() - launches0
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / a.steps
    value = m / (ms_per_step * 1e-3) / 1e9

    # top-k latency (rs_topk alone, device-resident scores -> device ids), for the
    # bench's K and SURVEY §8(d)'s K = 5 and K = 1000
    def topk_ms(K, host=False):
        # rs_topk from device-resident scores to HOST ids (pinned
        # buffers; rs_topk returns once they are there: wall time); the device-
        # output variant is timed with CUDA events on the library stream
        if host:
            ib = torch.empty(K, dtype=torch.int32).pin_memory()
            sb = torch.empty(K, dtype=torch.float64).pin_memory()
        else:
            ib = torch.empty(K, dtype=torch.int32, device=dev)
            sb = torch.empty(K, dtype=torch.float64, device=dev)
        sc.topk(K, ib, sb)
        out = []
        for i in range(7):
            torch.cuda.synchronize(dev)
            if host:
                t0 = time.perf_counter()
                sc.topk(K, ib, sb)
                out.append(1e3 * (time.perf_counter() - t0))
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sc.topk(K, ib, sb)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                out.append(e0.elapsed_time(e1))
        return float(np.median(out))
    tk_ms = [topk_ms(a.K)]
    tk_more = {f"K={K}": round(topk_ms(K), 4) for K in (5, 1000)}
    tk_more.update({f"K={K} to host ids": round(topk_ms(K, host=True), 4) for K in (5, a.K, 1000)})
    sc.topk(a.K, ids_d, sco_d)

    # per-phase split of one step (stats on), for the roofline of the dominant phase
    ph = []
    for _ in range(3):
        with torch.cuda.stream(stream):
            flush.fill_(7)
        sc.set_communities(comm_d, a.k)
        s = sc.score(stats=True)
        ph.append([s["ms_phase"][0], s["ms_phase"][2], s["ms_phase"][3]])
    ph = np.median(np.array(ph), axis=0)
    names = ["A_hist_weights_lists", "ED_type1_type2", "F_finalize"]
    Db, nb, ntri, nprobe = st["n_pred_entries"], st["n_border"], st["n_triangles"], st["n_probes"]
    sb = survey_bytes(n, D, Db, a.k, ntri, nprobe)
    fb = fused_bytes(n, D, Db, a.k, ntri, nprobe)
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6550.0))
    # every phase against the HBM roof (phase time = CUDA events on the library
    # stream around the phase's launches, median of 3 steps); the dominant one is
    # the headline, with SURVEY §8(d)'s bytes (fused-pipeline bytes beside them)
    keys = {"A_hist_weights_lists": "A", "ED_type1_type2": "ED", "F_finalize": "F"}
    phases = {}
    for nm, ms in zip(names, ph):
        by, byf = sb[keys[nm]], fb[keys[nm]]
        gbs = by / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        gbf = byf / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        phases[nm] = {"ms": round(float(ms), 4), "survey_bytes": int(by), "GBps": round(gbs, 1),
                      "frac": round(gbs / hbm_peak, 4), "fused_bytes": int(byf), "fused_frac": round(gbf / hbm_peak, 4)}
    dom = max(phases, key=lambda x: phases[x]["ms"])
    ncu = ncu_record(a.config)
    traffic, kernels = None, None
    if ncu:
        per = ncu.get("phase_dram_bytes", {}).get(keys[dom])
        traffic = per
        kernels = ncu.get("kernels")
    roof = {"bound": "hbm", "kernel": dom, "achieved": phases[dom]["GBps"], "peak": hbm_peak, "unit": "GB/s",
            "frac": phases[dom]["frac"], "traffic": traffic,
            "traffic_over_alg": round(traffic / phases[dom]["survey_bytes"], 3) if traffic else None,
            "bytes_formula": "SURVEY §8(d) table (bench.py survey_bytes); fused-pipeline bytes as fused_*",
            "traffic_source": (f"profiles/ncu_kernels.json ({ncu.get('source')}, build {ncu.get('build')}, "
                               f"matches this build: {ncu['build_match']})") if ncu else None,
            "phases": phases, "ncu_kernels": kernels,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"}

    # NEXT-1: absolute AWCC of the top-K under cumulative random
    # edge / node removal, 5 %..75 % (16 steps), per trial; rs_awcc_removal is
    # host-synchronous, so its wall time is its latency
    awcc = None
    if not a.no_awcc:
        top = ids_d.cpu().numpy()
        awcc = {"S": int(top.size), "steps": 16}
        for mode in ("edge", "node"):
            sc.awcc_removal(top, mode, 5, 75, 1, 1)            # warm-up
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            _, mean = sc.awcc_removal(top, mode, 5, 75, 3, 2)
            torch.cuda.synchronize(dev)
            dt = (time.perf_counter() - t0) / 3
            items = m if mode == "edge" else n
            awcc[f"{mode}_ms_per_trial"] = round(dt * 1e3, 3)
            awcc[f"{mode}_Gitems_per_s"] = round(items / dt / 1e9, 2)
            awcc[f"{mode}_awcc_0_75"] = [round(float(mean[0]), 6), round(float(mean[-1]), 6)]

    # NEXT-4: SHII of the top-K under IC (p = 0.1, SPEC default) and LT, 2 runs each;
    # host-synchronous (a BFS level per launch), so wall time is its latency
    shii = None
    if not a.no_awcc:
        top = ids_d.cpu().numpy()
        shii = {"S": int(top.size), "runs": 2}
        for model in ("ic", "lt"):
            sc.shii(top[:1], model, 0.1, 1, 1)             # warm-up (buffers)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            _, _, mean = sc.shii(top, model, 0.1, 2, 3)
            dt = time.perf_counter() - t0
            shii[f"{model}_ms_per_diffusion"] = round(dt * 1e3 / (top.size * 2), 3)
            shii[f"{model}_mean_shii"] = round(float(mean), 6)

    # NEXT-3: the step with every literal variant on (RS_LITERAL_L | RS_GATE_L | RS_WMAX_EB)
    variants = None
    if not a.no_awcc:
        vf = rsb.RS_LITERAL_L | rsb.RS_GATE_L | rsb.RS_WMAX_EB
        vms = []
        for i in range(3 + a.warmup):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sc.set_communities(comm_d, a.k)
            sc.score(flags=vf)
            sc.topk(a.K, ids_d, sco_d)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if i >= a.warmup:
                vms.append(e0.elapsed_time(e1))
        variants = {"flags": "literal_L|gate_L|wmax_eb", "ms_per_step": round(float(np.median(vms)), 4)}
        sc.score()   # back to the adopted readings

    # NEXT-2: the all-communities mode (every community a target, sparse tables) on
    # an LFR-style LiveJournal-shape graph with 10 000 communities (Zipf 0.8 sizes)
    sparse = None
    if not a.no_awcc and world == 1:
        sparse = sparse_leg(a, rsb, dev, stream, sh, flush)

    mgpu = None
    if world == 1 and not a.no_mgpu:
        mgpu = multigpu_model(a, g, rsb, st, ms_per_step, tk_ms[0])

    e2e = None
    if not a.no_e2e:
        e2e = measure_e2e(a, g, rsb, dev, stream, sh, rank, world, st)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(g, a.k, budget_s=15.0, config=a.config)

    if rank == 0:
        clk_s = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{a.config}-shape DC-SBM (SURVEY §8(d))", "n": n, "m": m, "nnz": D,
                       "k_targets": a.k, "K": a.K, "seed": gen.CONFIGS.get(a.config, {}).get("seed"),
                       "n_border": nb, "pred_entries": Db, "triangles": ntri, "probes": nprobe, "omega_max": st["omega_max"],
                       "l2": "flushed between timed steps (512 MiB write)", "gen_s": round(gen_s, 1),
                       "parallelism": f"head-range x{world} (Phase A {a.mg_mode})" if world > 1 else "single GPU"},
            "roofline": roof,
            "topk_latency_ms": round(float(np.median(tk_ms)), 4),
            "topk_latency_ms_more": tk_more,
            # the method's lower bound is one fused pass (col_idx +
            # a 1-byte label per adjacency entry, offsets / own label / score per
            # vertex); the step time against that traffic at the HBM roof
            "lower_bound": {"bytes": int(5 * D + 20 * n), "ms_at_peak": round((5 * D + 20 * n) / (hbm_peak * 1e6), 4),
                            "frac_of_step": round((5 * D + 20 * n) / (hbm_peak * 1e6) / ms_per_step, 4)},
            "next_awcc_removal": awcc,
            "next_literal_variants": variants,
            "next_shii": shii,
            "next_all_communities": sparse,
            "multigpu_model": mgpu,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": int(launches),
            "clocks": clk_s, "step_ms_minmax": [round(min(step_ms), 4), round(max(step_ms), 4)],
        }
        print(json.dumps(line), flush=True)
    sc.close()
    if world > 1:
        dist.destroy_process_group()


# NVLink figures measured on this pool's B200s (B200_PROFILING.md): 8-rank
# all-reduce bus bandwidth at 1 GiB and a peer copy, per direction per GPU
NVLINK_ALLREDUCE_BUSBW = 725e9
NVLINK_PEER_BW = 770e9


def multigpu_model(a, g, rsb, st1, ms1, tk1, worlds=(2, 4, 8), reps=3):
    """Both multi-GPU modes: Phase A sharded + exchanged, and Phase A
    replicated on every rank (RS_REPLICATE_A, the north_star's replicated CSR and
    labels: only the Type-I limbs are exchanged); per N the faster is the
    modelled step."""
    sh = multigpu_model_mode(a, g, rsb, st1, ms1, tk1, worlds, reps, 0)
    rep = multigpu_model_mode(a, g, rsb, st1, ms1, tk1, worlds, reps, rsb.RS_REPLICATE_A)
    out = {"how": sh.pop("how"), "N1_ms_per_step": sh.pop("N1_ms_per_step")}
    rep.pop("how"), rep.pop("N1_ms_per_step")
    for N in worlds:
        key = f"N={N}"
        a_, b_ = sh.get(key, {}), rep.get(key, {})
        best = min((x for x in (("sharded", a_), ("replicated", b_)) if "step_ms_model" in x[1]),
                   key=lambda x: x[1]["step_ms_model"], default=None)
        out[key] = {"mode": best[0], "step_ms_model": best[1]["step_ms_model"],
                    "GTEPS_model": best[1]["GTEPS_model"], "speedup_vs_N1": best[1]["speedup_vs_N1"]} if best else {}
    out["sharded"] = sh
    out["replicated"] = rep
    return out


def multigpu_model_mode(a, g, rsb, st1, ms1, tk1, worlds, reps, flags):
    """The multi-GPU path on this one GPU: N emulated
    ranks (rs_create_emulated) in SERIAL mode -- inside rs_score the ranks take
    turns between collectives, so each rank's kernels run alone on the GPU and
    its rs_stats phase times are those of a GPU of its own. Per phase the max
    over ranks is taken (ranks wait for each other at every exchange); the
    exchanges are modelled from their exact byte counts at the measured NVLink
    figures (NCCL all-reduce moves 2(N-1)/N of the buffer per rank, an
    all-gather or reduce-scatter (N-1)/N of the total). Not a multi-GPU
    measurement: the box has one GPU."""
    import threading
    import torch
    n, D, k = g.n, g.nnz, a.k
    out = {"how": "per-rank phase times measured (serial emulated ranks, one GPU; the exchange phases' own "
                  "kernels included, their waits excluded), max over ranks; exchange bytes exact, at 725 GB/s "
                  "all-reduce bus bandwidth / 770 GB/s peer copy (measured, B200_PROFILING.md)",
           "N1_ms_per_step": round(ms1, 4)}
    for N in worlds:
        W = rsb.EmuWorld(N)
        W.serial(True)
        per, err, xb = [None] * N, [], [None] * N

        def main(r):
            try:
                stream = torch.cuda.Stream(device=0)
                s = rsb.Scorer(0, stream.cuda_stream, rank=r, world=N, emu=W)
                s.load_csr(g.rowptr, g.col)
                s.set_communities(g.comm, k)
                s.score(flags=flags)
                ph = []
                for _ in range(reps):
                    st_last = s.score(stats=True, flags=flags)
                    # the rank's own kernel time per phase: the collectives' waits
                    # (peers' turns, the emulated copies) taken out
                    ph.append(np.array(st_last["ms_phase"]) - np.array(st_last["ms_xwait"]))
                per[r] = np.median(np.array(ph), axis=0)
                xb[r] = (st_last["xchg_allreduce_bytes"], st_last["xchg_allgather_bytes"],
                         st_last["xchg_reduce_scatter_bytes"])
                s.close()
            except Exception as e:  # reported below
                err.append(repr(e))

        th = [threading.Thread(target=main, args=(r,)) for r in range(N)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        W.close()
        torch.cuda.empty_cache()
        if err:
            out[f"N={N}"] = {"error": err[0]}
            continue
        P = np.array(per)
        A, ED, F = float(P[:, 0].max()), float(P[:, 2].max()), float(P[:, 3].max())
        # the local kernels of the exchange phases (packing, unpacking, the hub fold)
        XL, LL = float(P[:, 1].max()), float(P[:, 4].max())
        # the exchanges: exact byte counts reported by librs (rs_stats), at the
        # measured NVLink figures; all-reduce buffers move 2(N-1)/N of their size
        # per rank, an all-gather (N-1)/N of the gathered total
        ar, ag, rsc = xb[0]
        x1 = (ar * 2 * (N - 1) / N / NVLINK_ALLREDUCE_BUSBW + ag * (N - 1) / N / NVLINK_PEER_BW
              + rsc * (N - 1) / N / NVLINK_PEER_BW)
        x2 = 0.0
        tk = tk1                                       # top-K: local select + a K x 12 B all-gather
        step = A + XL + ED + LL + F + 1e3 * (x1 + x2) + tk
        out[f"N={N}"] = {"A_ms_max": round(A, 4), "ED_ms_max": round(ED, 4), "F_ms_max": round(F, 4),
                         "xchg_local_ms_max": round(XL, 4), "limb_local_ms_max": round(LL, 4),
                         "A_ms_ranks": [round(float(x), 4) for x in P[:, 0]],
                         "ED_ms_ranks": [round(float(x), 4) for x in P[:, 2]],
                         "allreduce_MB": round(ar / 1e6, 1), "allgather_MB": round(ag / 1e6, 1),
                         "reduce_scatter_MB": round(rsc / 1e6, 1),
                         "exchange_ms": round(1e3 * x1, 4),
                         "step_ms_model": round(step, 4), "GTEPS_model": round(g.m / (step * 1e-3) / 1e9, 3),
                         "speedup_vs_N1": round(ms1 / step, 3)}
    return out


SPARSE_CFG = dict(base="lj", n_comm=10_000, zipf_s=0.8)


def sparse_leg(a, rsb, dev, stream, sh, flush):
    """One step = rs_set_communities(RS_ALL_COMMUNITIES) + rs_score + rs_topk on a
    device-resident LFR-style graph, L2 flushed between steps."""
    import torch
    t0 = time.time()
    g2 = gen.config_graph(SPARSE_CFG["base"], n_comm=SPARSE_CFG["n_comm"], zipf_s=SPARSE_CFG["zipf_s"])
    gen_s = time.time() - t0
    sc2 = rsb.Scorer(dev.index, sh)
    rp = torch.from_numpy(g2.rowptr).to(dev)
    cl = torch.from_numpy(g2.col).to(dev)
    cm = torch.from_numpy(g2.comm).to(dev)
    ids = torch.empty(a.K, dtype=torch.int32, device=dev)
    sco = torch.empty(a.K, dtype=torch.float64, device=dev)
    sc2.load_csr(rp, cl)
    ms, ph = [], []
    for i in range(a.warmup + 5):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sc2.set_communities(cm, rsb.RS_ALL_COMMUNITIES)
        sc2.score()
        sc2.topk(a.K, ids, sco)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= a.warmup:
            ms.append(e0.elapsed_time(e1))
    for i in range(3):
        with torch.cuda.stream(stream):
            flush.fill_(i)
        s = sc2.score(stats=True)
        ph.append([s["ms_phase"][0], s["ms_phase"][2], s["ms_phase"][3]])
    ph = np.median(np.array(ph), axis=0)
    step = float(np.median(ms))
    out = {"workload": f"{SPARSE_CFG['base']}-shape DC-SBM, {SPARSE_CFG['n_comm']} communities "
                       f"(Zipf {SPARSE_CFG['zipf_s']} sizes), targets = all", "n": g2.n, "m": g2.m, "k": sc2.k,
           "ms_per_step": round(step, 4), "GTEPS": round(g2.m / (step * 1e-3) / 1e9, 4),
           "phase_ms": {"tables_lists": round(float(ph[0]), 4), "ED_type1_type2": round(float(ph[1]), 4),
                        "F_finalize": round(float(ph[2]), 4)},
           "pred_entries": s["n_pred_entries"], "triangles": s["n_triangles"], "omega_max": s["omega_max"],
           "gen_s": round(gen_s, 1)}
    sc2.close()
    del rp, cl, cm
    return out


def measure_e2e(a, g, rsb, dev, stream, sh, rank, world, st):
    """Same metric through the public API from pinned HOST buffers: every step
    copies the CSR + labels host->device (rs_load_csr, rs_set_communities),
    scores, and reads the top-K ids back to the host."""
    import torch
    rp_h = torch.from_numpy(g.rowptr).pin_memory()
    col_h = torch.from_numpy(g.col).pin_memory()
    comm_h = torch.from_numpy(g.comm).pin_memory()
    ids_h = torch.empty(a.K, dtype=torch.int32).pin_memory()
    sco_h = torch.empty(a.K, dtype=torch.float64).pin_memory()
    if world > 1:
        import torch.distributed as dist
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(rsb.rs_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        sc = rsb.Scorer(int(dev.index), sh, rank=rank, world=world, nccl_id=bytes(idt.cpu().numpy()))
    else:
        sc = rsb.Scorer(int(dev.index), sh)

    def step():
        sc.load_csr(rp_h, col_h)
        sc.set_communities(comm_h, a.k)
        sc.score()
        sc.topk(a.K, ids_h, sco_h)

    for _ in range(2):
        step()
    steps = max(3, min(a.steps, 5))
    ts = []
    for _ in range(steps):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(ts) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    sc.close()
    h2d = g.rowptr.nbytes + g.col.nbytes + g.comm.nbytes
    d2h = a.K * (4 + 8)
    return {"value": round(g.m / (ms * 1e-3) / 1e9, 4), "unit": UNIT, "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


# ------------------------------------------------------------------ oracle arms
def oracle_globals(g, k):
    """O0-O4 over the whole graph (targets, border, counts, weights, omega_max)
    and the G' lists; returns (targets, w, wmax, seconds)."""
    import oracle
    t0 = time.perf_counter()
    t = oracle.select_targets(g.comm, k)
    oracle.border(g)
    f, _ = oracle.counts(g, t)
    w = oracle.weights(f)
    wmax = oracle.omega_max(w)
    oracle.pred(g)
    return t, w, wmax, time.perf_counter() - t0


def oracle_heads(g, t, w, wmax, heads):
    """O5-O7 on the given heads, single thread; returns (seconds, edges scored =
    sum of d(u)/2 over the heads: an undirected edge is scored through both ends)"""
    import oracle
    t0 = time.perf_counter()
    oracle.rsi(g, t, w, wmax, heads)
    dt = time.perf_counter() - t0
    return dt, float(np.diff(g.rowptr)[heads].sum()) / 2.0


def full_oracle_record(config):
    """the committed full single-thread oracle run of this config (tools/oracle_timed.py)"""
    p = os.path.join(REPO, "profiles", f"oracle_{config}.json")
    if not os.path.exists(p):
        return None
    r = json.load(open(p))
    return {"total_s": r.get("total_s"), "GTEPS": r.get("GTEPS"), "cpu": r.get("cpu"),
            "source": f"profiles/oracle_{config}.json (tools/oracle_timed.py, full, 1 thread)"}


def cpu_baseline(g, k, budget_s=15.0, config=""):
    """The oracle as it stands, one thread: O0-O4 over the whole graph, then
    O5-O7 on random head batches for about budget_s; the rate is edges scored /
    s over the batches (mean and standard error over the batches) and the
    single-thread whole-graph time it implies; the full run is cited if one
    was recorded for this config."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(0)
    t, w, wmax, glob_s = oracle_globals(g, k)
    probe_s, _ = oracle_heads(g, t, w, wmax, rng.choice(g.n, size=min(200, g.n), replace=False).astype(np.int64))
    per_head = max(probe_s / min(200, g.n), 1e-7)
    nb = 10
    batch = int(max(50, min(g.n // nb, budget_s / nb / per_head)))
    rates, heads_done, secs = [], 0, 0.0
    for _ in range(nb):
        h = rng.choice(g.n, size=batch, replace=False).astype(np.int64)
        dt, e = oracle_heads(g, t, w, wmax, h)
        rates.append(e / dt / 1e9)
        heads_done += h.size
        secs += dt
    rates = np.array(rates)
    mean, se = float(rates.mean()), float(rates.std(ddof=1) / np.sqrt(len(rates)))
    full_s = glob_s + g.m / (mean * 1e9)
    return {"value": round(g.m / full_s / 1e9, 7), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"O0-O4 on the whole graph ({glob_s:.1f}s) + O5-O7 on {nb} batches of {batch} random heads "
                      f"({secs:.1f}s): {mean:.3e} +- {se:.1e} (SE) GTEPS over the batches, i.e. ~{full_s:.0f}s "
                      f"single-thread for the whole graph",
            "batch_GTEPS_mean": mean, "batch_GTEPS_se": se, "extrapolated_full_s": round(full_s, 1),
            "full_run": full_oracle_record(config), "host_cores": os.cpu_count()}


def reference_arm(a, rank, world):
    """--impl reference: the oracle as it stands (oracle/, one thread) on the
    repo arm's workload. O0-O4 run once, untimed, before the steps; each
    (warm-up or timed) step is O5-O7 on a fresh random sample of heads sized so
    the run stays within minutes. ms_per_step is the measured time of exactly
    that work, value = edges scored by the sampled heads / time; the
    whole-graph extrapolation is a separate field."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    g = load_graph(a.config)
    rng = np.random.default_rng(0)
    t, w, wmax, glob_s = oracle_globals(g, a.k)
    probe_s, _ = oracle_heads(g, t, w, wmax, rng.choice(g.n, size=min(100, g.n), replace=False).astype(np.int64))
    per_head = max(probe_s / min(100, g.n), 1e-7)
    budget = 6.0 if a.config in ("orkut", "lj", "friendster") else 1.0
    nh = int(max(50, min(g.n, budget / per_head)))
    secs, edges = [], []
    for i in range(a.warmup + a.steps):
        h = rng.choice(g.n, size=nh, replace=False).astype(np.int64)
        dt, e = oracle_heads(g, t, w, wmax, h)
        if i >= a.warmup:
            secs.append(dt)
            edges.append(e)
    ms = 1e3 * float(np.mean(secs))
    value = float(np.sum(edges)) / float(np.sum(secs)) / 1e9
    full_s = glob_s + g.m / (value * 1e9)
    cpu = {"value": round(value, 7), "unit": UNIT, "kind": "oracle", "cores": 1,
           "sample": f"per step: O5-O7 on {nh} random heads (one thread); O0-O4 over the whole graph ran once "
                     f"before the steps ({glob_s:.1f}s, untimed)"}
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 7), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.config}-shape DC-SBM (SURVEY §8(d))", "n": g.n, "m": g.m, "k_targets": a.k,
                       "heads_per_step": nh},
            "cpu_baseline": cpu,
            "extrapolated_full_graph": {"seconds": round(full_s, 1), "GTEPS": round(g.m / full_s / 1e9, 7),
                                        "how": "O0-O4 time + m / measured edge rate (not timed as one run)",
                                        "full_run": full_oracle_record(a.config)},
            "e2e": {"value": round(value, 7), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

"""The unchanged oracle (rsi_oracle.c, O5-O7) split over head ranges on the
host cores ("a parity run with the same oracle code split over
head ranges on all host cores"): every head is still scored by one
single-threaded call of ``oracle_rsi``; this module only hands disjoint head
ranges to forked worker processes and concatenates their outputs in head order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): importable from tests/,
tools/ scripts that write golden files, and bench.py's oracle legs.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import rsi

_ARGS = None   # (g, targets, w, wmax) inherited by the forked workers


def _work(rng):
    g, t, w, wmax = _ARGS
    lo, hi = rng
    heads = np.arange(lo, hi, dtype=np.int64)
    t0 = time.perf_counter()
    R, nI, nII = rsi(g, t, w, wmax, heads)
    return lo, R, nI, nII, time.perf_counter() - t0


def rsi_all_heads(g, targets, w, wmax, procs=None, chunks_per_proc=48):
    """R, n_I, n_II for every vertex (head order = vertex id), computed by
    ``procs`` forked processes over contiguous head ranges. Returns
    (R, nI, nII, info) with info = {procs, wall_s, cpu_s}: cpu_s is the sum of
    the per-range single-thread times (the single-thread cost of O5-O7)."""
    global _ARGS
    n = g.n
    procs = procs or os.cpu_count() or 1
    nch = max(1, min(n, procs * chunks_per_proc))
    cuts = np.linspace(0, n, nch + 1).astype(np.int64)
    ranges = [(int(cuts[i]), int(cuts[i + 1])) for i in range(nch) if cuts[i + 1] > cuts[i]]
    R = np.zeros(n, dtype=np.float64)
    nI = np.zeros(n, dtype=np.int64)
    nII = np.zeros(n, dtype=np.int64)
    _ARGS = (g, targets, w, wmax)
    t0 = time.perf_counter()
    cpu = 0.0
    try:
        if procs == 1:
            outs = map(_work, ranges)
            for lo, r, a, b, s in outs:
                R[lo:lo + r.size], nI[lo:lo + r.size], nII[lo:lo + r.size] = r, a, b
                cpu += s
        else:
            with mp.get_context("fork").Pool(procs) as pool:
                for lo, r, a, b, s in pool.imap_unordered(_work, ranges):
                    R[lo:lo + r.size], nI[lo:lo + r.size], nII[lo:lo + r.size] = r, a, b
                    cpu += s
    finally:
        _ARGS = None
    return R, nI, nII, {"procs": procs, "wall_s": time.perf_counter() - t0, "cpu_s": cpu}

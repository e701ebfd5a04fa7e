"""ctypes wrapper of the plain-C RSI oracle (rsi_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2508_01485_b200) never imports this module, and this module never
imports the product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_P = ctypes.c_void_p


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "rsi_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        # -O2, no OpenMP, no -ffast-math: IEEE fp64, single thread
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        lib.oracle_select_targets.restype = i64
        lib.oracle_select_targets.argtypes = [i64, _P, i32, _P]
        lib.oracle_border.restype = i64
        lib.oracle_border.argtypes = [i64, _P, _P, _P, _P]
        lib.oracle_counts.argtypes = [i64, _P, _P, _P, i32, _P, _P, _P]
        lib.oracle_weights.argtypes = [i64, i32, _P, _P]
        lib.oracle_weights_closed_form.argtypes = [i64, i32, _P, _P]
        lib.oracle_omega_max.restype = ctypes.c_double
        lib.oracle_omega_max.argtypes = [i64, i32, _P]
        lib.oracle_pred.restype = i64
        lib.oracle_pred.argtypes = [i64, _P, _P, _P, _P, _P]
        lib.oracle_rsi.argtypes = [i64, _P, _P, _P, i32, _P, _P, ctypes.c_double, i64, _P, _P, _P, _P]
        lib.oracle_topk.restype = i64
        lib.oracle_topk.argtypes = [i64, _P, i64, _P, _P]
        lib.oracle_weights_variant.argtypes = [i64, i32, _P, i32, _P]
        lib.oracle_omega_max_eb.restype = ctypes.c_double
        lib.oracle_omega_max_eb.argtypes = [i64, _P, _P, _P, i32, _P, _P, i32, _P]
        lib.oracle_shii.restype = ctypes.c_double
        lib.oracle_shii.argtypes = [i64, _P, _P, _P, _P, i64, i32, ctypes.c_double, i32, ctypes.c_uint64, _P, _P]
        lib.oracle_mix64.restype = ctypes.c_uint64
        lib.oracle_mix64.argtypes = [ctypes.c_uint64]
        lib.oracle_awcc_removal.restype = i64
        lib.oracle_awcc_removal.argtypes = [i64, _P, _P, _P, _P, i64, i32, i32, i32, i32, ctypes.c_uint64, _P, _P]
        lib.oracle_tables_all.restype = i64
        lib.oracle_tables_all.argtypes = [i64, _P, _P, _P, i32, _P, _P, _P, _P, _P, _P, _P]
        lib.oracle_rsi_all.argtypes = [i64, _P, _P, _P, i32, _P, _P, _P, _P, _P, ctypes.c_double, i64, _P, _P, _P,
                                       _P]
        _lib = lib
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return a.ctypes.data


def select_targets(comm, k):
    comm = _c(comm, np.int32)
    out = np.zeros(max(k, 1), dtype=np.int32)
    nc = _load().oracle_select_targets(comm.size, _ptr(comm), k, _ptr(out))
    if nc < 0:
        raise ValueError(f"k={k} out of range")
    return out[:k]


def border(g):
    out = np.zeros(g.n, dtype=np.uint8)
    _load().oracle_border(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)),
                          _ptr(_c(g.comm, np.int32)), _ptr(out))
    return out


def counts(g, targets):
    targets = _c(targets, np.int32)
    k = targets.size
    f = np.zeros((g.n, k), dtype=np.int32)
    T = np.zeros(g.n, dtype=np.int32)
    _load().oracle_counts(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)),
                          _ptr(_c(g.comm, np.int32)), k, _ptr(targets), _ptr(f), _ptr(T))
    return f, T


def weights(f, closed_form=False):
    f = _c(f, np.int32)
    n, k = f.shape
    w = np.zeros((n, k), dtype=np.float64)
    fn = _load().oracle_weights_closed_form if closed_form else _load().oracle_weights
    fn(n, k, _ptr(f), _ptr(w))
    return w


def omega_max(w):
    w = _c(w, np.float64)
    return float(_load().oracle_omega_max(w.shape[0], w.shape[1], _ptr(w)))


def pred(g):
    off = np.zeros(g.n + 1, dtype=np.int64)
    rp, cl, cm = _c(g.rowptr, np.int64), _c(g.col, np.int32), _c(g.comm, np.int32)
    cnt = _load().oracle_pred(g.n, _ptr(rp), _ptr(cl), _ptr(cm), _ptr(off), None)
    lists = np.zeros(max(cnt, 1), dtype=np.int32)
    _load().oracle_pred(g.n, _ptr(rp), _ptr(cl), _ptr(cm), _ptr(off), _ptr(lists))
    return off, lists[:cnt]


def rsi(g, targets, w, wmax, heads=None):
    targets = _c(targets, np.int32)
    heads = np.arange(g.n, dtype=np.int64) if heads is None else _c(heads, np.int64)
    R = np.zeros(heads.size, dtype=np.float64)
    nI = np.zeros(heads.size, dtype=np.int64)
    nII = np.zeros(heads.size, dtype=np.int64)
    w = _c(w, np.float64)
    _load().oracle_rsi(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)),
                       _ptr(_c(g.comm, np.int32)), targets.size, _ptr(targets), _ptr(w), float(wmax),
                       heads.size, _ptr(heads), _ptr(R), _ptr(nI), _ptr(nII))
    return R, nI, nII


def topk(R, K):
    R = _c(R, np.float64)
    ids = np.zeros(max(K, 1), dtype=np.int32)
    sc = np.zeros(max(K, 1), dtype=np.float64)
    cnt = _load().oracle_topk(R.size, _ptr(R), K, _ptr(ids), _ptr(sc))
    return ids[:cnt], sc[:cnt]


LITERAL_L, GATE_L, WMAX_EB = 1, 2, 4   # NEXT-3 variant flags (oracle numbering)


def weights_variant(f, flags):
    """Eq. 3/5 weights under the literal |L| (flags & 1) and/or Algorithm 1's gate (flags & 2)"""
    f = _c(f, np.int32)
    n, k = f.shape
    w = np.zeros((n, k), dtype=np.float64)
    _load().oracle_weights_variant(n, k, _ptr(f), int(flags) & 3, _ptr(w))
    return w


def omega_max_eb(g, targets, f, w, flags):
    """omega_max over Algorithm 1's E_b"""
    targets = _c(targets, np.int32)
    return _load().oracle_omega_max_eb(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)),
                                       _ptr(_c(g.comm, np.int32)), targets.size, _ptr(targets),
                                       _ptr(_c(f, np.int32)), int(flags) & 3, _ptr(_c(w, np.float64)))


def run_variant(g, k, flags, K=25, targets=None):
    """O0-O8 with the NEXT-3 variants: weights per flags & 3, omega_max over E_b if
    flags & 4 (else over all cells)"""
    if targets is None:
        targets = select_targets(g.comm, k)
    targets = _c(targets, np.int32)
    b = border(g)
    f, T = counts(g, targets)
    w = weights_variant(f, flags)
    wmax = omega_max_eb(g, targets, f, w, flags) if flags & WMAX_EB else omega_max(w)
    off, pl = pred(g)
    R, nI, nII = rsi(g, targets, w, wmax)
    ids, sc = topk(R, K)
    return OracleResult(targets, b, f, T, w, wmax, off, pl, R, nI, nII, ids, sc)


def awcc_removal(g, S, mode="edge", step_pct=5, max_pct=75, trials=1, seed=0):
    """NEXT-1: per-trial |zeta_j(v)| int32[trials, J+1, |S|] and the
    mean absolute AWCC per step float64[J+1] (step 0 = no removal = AWCC)."""
    S = _c(S, np.int32)
    J1 = max_pct // step_pct + 1
    zeta = np.zeros((trials, J1, S.size), dtype=np.int32)
    mean = np.zeros(J1, dtype=np.float64)
    r = _load().oracle_awcc_removal(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)),
                                    _ptr(_c(g.comm, np.int32)), _ptr(S), S.size, 0 if mode == "edge" else 1,
                                    step_pct, max_pct, trials, int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(zeta), _ptr(mean))
    if r < 0:
        raise ValueError("oracle_awcc_removal: bad arguments")
    return zeta, mean


def shii(g, S, model="ic", p=0.1, runs=10, seed=0):
    """NEXT-4: (influenced int64[|S|, runs, 2] = {all, outside C(seed)},
    per-seed SHII float64[|S|], mean over S)"""
    S = _c(S, np.int32)
    out = np.zeros((S.size, runs, 2), dtype=np.int64)
    per = np.zeros(S.size, dtype=np.float64)
    m = _load().oracle_shii(g.n, _ptr(_c(g.rowptr, np.int64)), _ptr(_c(g.col, np.int32)), _ptr(_c(g.comm, np.int32)),
                            _ptr(S), S.size, 0 if model == "ic" else 1, float(p), int(runs),
                            int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(out), _ptr(per))
    return out, per, m


def mix64(z):
    return int(_load().oracle_mix64(int(z) & 0xFFFFFFFFFFFFFFFF))


@dataclass
class OracleResult:
    targets: np.ndarray
    border: np.ndarray
    f: np.ndarray
    T: np.ndarray
    omega: np.ndarray
    omega_max: float
    pred_off: np.ndarray
    pred: np.ndarray
    R: np.ndarray
    nI: np.ndarray
    nII: np.ndarray
    top_ids: np.ndarray
    top_scores: np.ndarray


def run(g, k=None, targets=None, K=25, heads=None) -> OracleResult:
    """O0-O8 end to end.  ``heads`` limits O5-O7 to a sample;
    top-K is then over the sampled heads' scores only (positions)."""
    if targets is None:
        targets = select_targets(g.comm, k)
    targets = _c(targets, np.int32)
    b = border(g)
    f, T = counts(g, targets)
    w = weights(f)
    wmax = omega_max(w)
    off, pl = pred(g)
    R, nI, nII = rsi(g, targets, w, wmax, heads)
    ids, sc = topk(R, K)
    return OracleResult(targets, b, f, T, w, wmax, off, pl, R, nI, nII, ids, sc)


# ---- NEXT-2: every community a target, rows kept as their nonzero columns ----
@dataclass
class TablesAll:
    targets: np.ndarray     # int32[k]: all communities, size desc / id asc (column order)
    off: np.ndarray         # int64[n+1]
    cols: np.ndarray        # int32[E]: nonzero columns of each row, ascending
    cnt: np.ndarray         # int32[E]: f_u(column)
    omega: np.ndarray       # f64[E]: omega_u(column)
    omega_abs: np.ndarray   # f64[n]: omega_u(c) of every absent column c
    omega_max: float


def tables_all(g):
    """O2-O4 with targets = all communities (oracle_tables_all)."""
    k = len(np.unique(g.comm))
    t = select_targets(g.comm, k)
    rp, cl, cm = _c(g.rowptr, np.int64), _c(g.col, np.int32), _c(g.comm, np.int32)
    E = max(g.nnz, 1)
    off = np.zeros(g.n + 1, dtype=np.int64)
    cols = np.zeros(E, dtype=np.int32)
    cnt = np.zeros(E, dtype=np.int32)
    om = np.zeros(E, dtype=np.float64)
    oa = np.zeros(g.n, dtype=np.float64)
    wm = ctypes.c_double(0.0)
    tot = _load().oracle_tables_all(g.n, _ptr(rp), _ptr(cl), _ptr(cm), k, _ptr(t), _ptr(off), _ptr(cols), _ptr(cnt),
                                    _ptr(om), _ptr(oa), ctypes.byref(wm))
    return TablesAll(t, off, cols[:tot].copy(), cnt[:tot].copy(), om[:tot].copy(), oa, float(wm.value))


def rsi_all(g, tab, heads):
    """O5-O7 with targets = all on the given heads (oracle_rsi_all)."""
    heads = _c(heads, np.int64)
    nh = heads.size
    R = np.zeros(nh, dtype=np.float64)
    nI = np.zeros(nh, dtype=np.int64)
    nII = np.zeros(nh, dtype=np.int64)
    rp, cl, cm = _c(g.rowptr, np.int64), _c(g.col, np.int32), _c(g.comm, np.int32)
    _load().oracle_rsi_all(g.n, _ptr(rp), _ptr(cl), _ptr(cm), tab.targets.size, _ptr(tab.targets), _ptr(tab.off),
                           _ptr(tab.cols), _ptr(tab.omega), _ptr(tab.omega_abs), tab.omega_max, nh, _ptr(heads),
                           _ptr(R), _ptr(nI), _ptr(nII))
    return R, nI, nII

"""Python binding of librs (include/rs.h): argument marshalling only.

Every step of the RSI path (arXiv 2508.01485, Algorithm 1 + Eq. 4) runs in the
CUDA kernels of librs.so (sm_100a). There is no CPU fallback: if librs.so is
missing or no CUDA device is present, the calls raise.

Low-level names mirror the C-ABI (``rs_create``, ``rs_load_csr``,
``rs_set_communities``, ``rs_score``, ``rs_topk``, getters); ``Scorer`` is a
thin object wrapper around one context. Arrays may be numpy arrays (host),
torch CPU tensors (host; pinned or not) or torch CUDA tensors (device).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librs.so")

RS_OK, RS_EINVAL, RS_ESTATE, RS_ENOMEM, RS_ECUDA, RS_ENCCL = 0, -1, -2, -3, -4, -5
RS_VALIDATE = 1
RS_GATHER_SCORES = 1
RS_REMOVE_EDGES, RS_REMOVE_NODES = 0, 1
RS_LITERAL_L, RS_GATE_L, RS_WMAX_EB = 1 << 16, 1 << 17, 1 << 18   # NEXT-3 variants (rs_score flags)
RS_REPLICATE_A = 1 << 20   # multi-GPU: Phase A on every rank over all vertices, no Phase A exchange
RS_ALL_COMMUNITIES = -1   # rs_set_communities k: every community a target (NEXT-2 sparse mode)


def RS_LOAD_CHUNK_LOG2(e: int) -> int:
    """rs_load_csr test hook: pipelined host col_idx copy in chunks of 2^e entries."""
    return (int(e) & 0x1F) << 8


def RS_E_SHARES(s: int) -> int:
    """rs_score test hook: Phase E as s sequential shares of the multi-GPU split."""
    return (int(s) & 0xFF) << 8
_STATUS = {0: "RS_OK", -1: "RS_EINVAL", -2: "RS_ESTATE", -3: "RS_ENOMEM", -4: "RS_ECUDA", -5: "RS_ENCCL"}


class RsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class rs_stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("n_border", ctypes.c_int64),
                ("n_pred_entries", ctypes.c_int64), ("n_triangles", ctypes.c_int64),
                ("n_probes", ctypes.c_int64), ("omega_max", ctypes.c_double), ("ms_phase", ctypes.c_float * 8),
                ("xchg_allreduce_bytes", ctypes.c_int64), ("xchg_allgather_bytes", ctypes.c_int64),
                ("xchg_reduce_scatter_bytes", ctypes.c_int64), ("ms_xwait", ctypes.c_float * 8)]

    def as_dict(self):
        return {"n": self.n, "m": self.m, "n_border": self.n_border, "n_pred_entries": self.n_pred_entries,
                "n_triangles": self.n_triangles, "n_probes": self.n_probes, "omega_max": self.omega_max,
                "ms_phase": [float(x) for x in self.ms_phase],
                "xchg_allreduce_bytes": self.xchg_allreduce_bytes, "xchg_allgather_bytes": self.xchg_allgather_bytes,
                "xchg_reduce_scatter_bytes": self.xchg_reduce_scatter_bytes,
                "ms_xwait": [float(x) for x in self.ms_xwait]}


_P = ctypes.c_void_p
_lib = None

# (name, restype, argtypes) for every symbol include/rs.h declares
SIGNATURES = [
    ("rs_create", ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _P]),
    ("rs_create_dist", ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _P, ctypes.c_int, ctypes.c_int, _P]),
    ("rs_nccl_unique_id", ctypes.c_int, [_P]),
    ("rs_nccl_selftest", ctypes.c_int, [ctypes.c_int, _P, ctypes.c_size_t]),
    ("rs_destroy", None, [_P]),
    ("rs_last_error", ctypes.c_char_p, [_P]),
    ("rs_load_csr", ctypes.c_int, [_P, ctypes.c_int64, _P, _P, ctypes.c_uint32]),
    ("rs_set_communities", ctypes.c_int, [_P, _P, _P, ctypes.c_int32]),
    ("rs_score", ctypes.c_int, [_P, _P, ctypes.POINTER(rs_stats), ctypes.c_uint32]),
    ("rs_topk", ctypes.c_int, [_P, ctypes.c_int64, _P, _P, ctypes.POINTER(ctypes.c_int64)]),
    ("rs_get_comm_tables", ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.POINTER(ctypes.c_int64)]),
    ("rs_get_counts", ctypes.c_int, [_P, _P, _P]),
    ("rs_get_weights", ctypes.c_int, [_P, _P, _P]),
    ("rs_get_border", ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_int64)]),
    ("rs_get_pred", ctypes.c_int, [_P, _P, _P, ctypes.POINTER(ctypes.c_int64)]),
    ("rs_get_triad_counts", ctypes.c_int, [_P, _P, _P]),
    ("rs_get_targets", ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_int32)]),
    ("rs_kernel_launches", ctypes.c_int64, [_P]),
    ("rs_debug_poison", None, [ctypes.c_int32]),
    ("rs_awcc_removal", ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_uint64, _P, _P, ctypes.POINTER(ctypes.c_int64)]),
    ("rs_shii", ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                               ctypes.c_uint64, _P, _P, ctypes.POINTER(ctypes.c_double)]),
    ("rs_emu_world_create", ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32]),
    ("rs_emu_world_destroy", None, [_P]),
    ("rs_create_emulated", ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _P, ctypes.c_int, ctypes.c_int, _P]),
    ("rs_emu_world_serial", ctypes.c_int, [_P, ctypes.c_int32]),
    ("rs_local_candidates", ctypes.c_int, [ctypes.c_int64, _P, _P, ctypes.c_int64, _P, _P]),
    ("rs_split_ranges", ctypes.c_int, [ctypes.c_int64, _P, ctypes.c_int32, _P]),
    ("rs_merge_candidates", ctypes.c_int, [ctypes.c_int64, _P, _P, ctypes.c_int64, _P, _P,
                                           ctypes.POINTER(ctypes.c_int64)]),
]


def load_library(path: str | None = None):
    """Load librs.so (build it first with paper_2508_01485_b200.build). Raises if absent.
    ``RS_LIBRARY`` overrides the path (experiment builds)."""
    global _lib
    if _lib is None:
        path = path or os.environ.get("RS_LIBRARY") or LIB_PATH
        if not os.path.exists(path):
            raise ImportError(f"librs.so not built at {path}; run `python -m paper_2508_01485_b200.build`")
        lib = ctypes.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(a):
    """Address of a numpy array / torch tensor (host or device); None -> NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported array type {type(a)}")


def _check(ctx, status):
    if status != RS_OK:
        raise RsError(status, load_library().rs_last_error(ctx).decode())


def _as(a, dtype):
    if hasattr(a, "data_ptr"):
        import torch
        want = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[dtype]
        if a.dtype != want:
            raise TypeError(f"expected {want}, got {a.dtype}")
        return a.contiguous()
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------ C-ABI mirrors
def rs_create(device: int = 0, stream: int | None = None):
    lib = load_library()
    h = _P()
    st = lib.rs_create(ctypes.byref(h), device, stream)
    if st != RS_OK:
        raise RsError(st, lib.rs_last_error(None).decode())
    return h


def rs_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    st = load_library().rs_nccl_unique_id(buf)
    if st != RS_OK:
        raise RsError(st, load_library().rs_last_error(None).decode())
    return bytes(buf)


def rs_nccl_selftest(device: int, stream=None, nbytes: int = 1 << 20) -> None:
    """include/rs.h rs_nccl_selftest: every NCCL-transport collective on a
    one-rank communicator, checked bit for bit; raises RsError on failure."""
    lib = load_library()
    st = lib.rs_nccl_selftest(int(device), _P(stream) if stream else None, int(nbytes))
    if st != RS_OK:
        raise RsError(st, lib.rs_last_error(None).decode())


def rs_create_dist(device: int, stream, rank: int, world: int, nccl_id: bytes):
    lib = load_library()
    h = _P()
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
    st = lib.rs_create_dist(ctypes.byref(h), device, stream, rank, world, buf)
    if st != RS_OK:
        raise RsError(st, lib.rs_last_error(h if h.value else None).decode())
    return h


def rs_destroy(ctx):
    load_library().rs_destroy(ctx)


def rs_load_csr(ctx, row_offsets, col_idx, flags: int = 0):
    ro, ci = _as(row_offsets, np.int64), _as(col_idx, np.int32)
    _check(ctx, load_library().rs_load_csr(ctx, int(ro.shape[0]) - 1, _ptr(ro), _ptr(ci), flags))


def rs_set_communities(ctx, community_of, k: int, targets=None):
    c = _as(community_of, np.int32)
    t = None if targets is None else _as(targets, np.int32)
    _check(ctx, load_library().rs_set_communities(ctx, _ptr(c), _ptr(t), int(k)))


def rs_score(ctx, scores_out=None, want_stats: bool = False, flags: int = 0):
    st = rs_stats()
    _check(ctx, load_library().rs_score(ctx, _ptr(scores_out), ctypes.byref(st) if want_stats else None, flags))
    return st.as_dict() if want_stats else None


def rs_topk(ctx, K: int, ids_out=None, scores_out=None):
    """Returns (ids, scores) numpy arrays when no output buffers are given."""
    n_alloc = ids_out is None
    if n_alloc:
        ids_out = np.empty(K, dtype=np.int32)
        scores_out = np.empty(K, dtype=np.float64)
    cnt = ctypes.c_int64(0)
    _check(ctx, load_library().rs_topk(ctx, int(K), _ptr(ids_out), _ptr(scores_out), ctypes.byref(cnt)))
    if n_alloc:
        return ids_out[:cnt.value], scores_out[:cnt.value]
    return cnt.value


def rs_get_counts(ctx, n, k):
    f = np.empty((n, k), dtype=np.int32)
    t = np.empty(n, dtype=np.int32)
    _check(ctx, load_library().rs_get_counts(ctx, _ptr(f), _ptr(t)))
    return f, t


def rs_get_weights(ctx, n, k):
    w = np.empty((n, k), dtype=np.float64)
    m = ctypes.c_double(0)
    _check(ctx, load_library().rs_get_weights(ctx, _ptr(w), ctypes.byref(m)))
    return w, m.value


def rs_get_border(ctx, n):
    bv = np.empty(n, dtype=np.int32)
    nb = ctypes.c_int64(0)
    _check(ctx, load_library().rs_get_border(ctx, _ptr(bv), ctypes.byref(nb)))
    return bv[:nb.value]


def rs_get_pred(ctx, n, nnz):
    off = np.empty(n + 1, dtype=np.int64)
    pr = np.empty(max(nnz, 1), dtype=np.int32)
    ne = ctypes.c_int64(0)
    _check(ctx, load_library().rs_get_pred(ctx, _ptr(off), _ptr(pr), ctypes.byref(ne)))
    return off, pr[:ne.value]


def rs_get_triad_counts(ctx, n):
    t1 = np.empty(n, dtype=np.int64)
    t2 = np.empty(n, dtype=np.int64)
    _check(ctx, load_library().rs_get_triad_counts(ctx, _ptr(t1), _ptr(t2)))
    return t1, t2


def rs_get_comm_tables(ctx, n):
    """All-communities mode: (off int64[n+1], cols int32[E], cnt int32[E], omega f64[E], omega_abs f64[n])."""
    lib = load_library()
    E = ctypes.c_int64(0)
    _check(ctx, lib.rs_get_comm_tables(ctx, None, None, None, None, None, ctypes.byref(E)))
    off = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(E.value, 1), dtype=np.int32)
    cnt = np.empty(max(E.value, 1), dtype=np.int32)
    om = np.empty(max(E.value, 1), dtype=np.float64)
    oa = np.empty(n, dtype=np.float64)
    _check(ctx, lib.rs_get_comm_tables(ctx, _ptr(off), _ptr(cols), _ptr(cnt), _ptr(om), _ptr(oa), ctypes.byref(E)))
    e = E.value
    return off, cols[:e], cnt[:e], om[:e], oa


def rs_get_targets(ctx):
    k = ctypes.c_int32(0)
    _check(ctx, load_library().rs_get_targets(ctx, None, ctypes.byref(k)))
    buf = np.empty(max(k.value, 1), dtype=np.int32)
    _check(ctx, load_library().rs_get_targets(ctx, _ptr(buf), ctypes.byref(k)))
    return buf[:k.value].copy()


def rs_debug_poison(byte: int) -> None:
    """test hook: fill every new librs device allocation with ``byte`` (-1 = off)"""
    load_library().rs_debug_poison(int(byte))


def rs_kernel_launches(ctx) -> int:
    return int(load_library().rs_kernel_launches(ctx))


def rs_awcc_removal(ctx, S, mode: str = "edge", step_pct: int = 5, max_pct: int = 75, trials: int = 1,
                    seed: int = 0):
    """NEXT-1: (zeta int32[trials, J+1, |S|], mean float64[J+1]) of the
    absolute AWCC of S under cumulative random edge or node removal."""
    Sa = _as(S, np.int32)
    nS = int(Sa.shape[0])
    J1 = max_pct // step_pct + 1 if step_pct > 0 else 1
    zeta = np.zeros((trials, J1, nS), dtype=np.int32)
    mean = np.zeros(J1, dtype=np.float64)
    steps = ctypes.c_int64(0)
    m = RS_REMOVE_EDGES if mode == "edge" else RS_REMOVE_NODES
    _check(ctx, load_library().rs_awcc_removal(ctx, _ptr(Sa), nS, m, int(step_pct), int(max_pct), int(trials),
                                               int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(zeta), _ptr(mean),
                                               ctypes.byref(steps)))
    return zeta[:, :steps.value], mean[:steps.value]


def rs_shii(ctx, S, model: str = "ic", p: float = 0.1, runs: int = 10, seed: int = 0):
    """NEXT-4: (influenced int64[|S|, runs, 2], per-seed SHII float64[|S|], mean)"""
    Sa = _as(S, np.int32)
    nS = int(Sa.shape[0])
    out = np.zeros((nS, max(runs, 1), 2), dtype=np.int64)
    per = np.zeros(max(nS, 1), dtype=np.float64)
    mean = ctypes.c_double(0.0)
    _check(ctx, load_library().rs_shii(ctx, _ptr(Sa), nS, 0 if model == "ic" else 1, float(p), int(runs),
                                       int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(out), _ptr(per), ctypes.byref(mean)))
    return out, per[:nS], mean.value


# ------------------------------------------------------------------ multi-GPU host protocol
def rs_split_ranges(work_incl, world: int) -> np.ndarray:
    """bounds int64[world+1] of the balanced contiguous split (include/rs.h)."""
    w = np.ascontiguousarray(work_incl, dtype=np.int64)
    b = np.empty(world + 1, dtype=np.int64)
    st = load_library().rs_split_ranges(int(w.shape[0]), _ptr(w) if w.size else None, int(world), _ptr(b))
    if st != RS_OK:
        raise RsError(st, "rs_split_ranges: invalid arguments")
    return b


def rs_local_candidates(scores, ids, K: int):
    """(keys uint64[K], ids int32[K]): a rank's Step-4 candidates, padded (0, INT32_MAX)."""
    sc = np.ascontiguousarray(scores, dtype=np.float64)
    i = np.ascontiguousarray(ids, dtype=np.int32)
    ko = np.empty(max(K, 1), dtype=np.uint64)
    io = np.empty(max(K, 1), dtype=np.int32)
    st = load_library().rs_local_candidates(int(sc.shape[0]), _ptr(sc) if sc.size else None,
                                            _ptr(i) if i.size else None, int(K), _ptr(ko), _ptr(io))
    if st != RS_OK:
        raise RsError(st, "rs_local_candidates: invalid arguments")
    return ko[:K].copy(), io[:K].copy()


class EmuWorld:
    """An emulated multi-GPU world (rs_emu_world): ``world`` ranks as host threads
    on one GPU, each with a Scorer(..., emu=this, rank=r, world=world)."""

    def __init__(self, world: int):
        h = _P()
        st = load_library().rs_emu_world_create(ctypes.byref(h), int(world))
        if st != RS_OK:
            raise RsError(st, "rs_emu_world_create: invalid world size")
        self.h, self.world = h, int(world)

    def serial(self, on: bool = True):
        """ranks take turns inside rs_score (each rank's phase times = a GPU of its own)"""
        load_library().rs_emu_world_serial(self.h, 1 if on else 0)

    def close(self):
        if self.h is not None:
            load_library().rs_emu_world_destroy(self.h)
            self.h = None


def rs_merge_candidates(keys, ids, K: int):
    """(ids, scores) of the merged top-K of gathered (key, id) candidates."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    i = np.ascontiguousarray(ids, dtype=np.int32)
    out_i = np.empty(max(K, 1), dtype=np.int32)
    out_s = np.empty(max(K, 1), dtype=np.float64)
    cnt = ctypes.c_int64(0)
    st = load_library().rs_merge_candidates(int(k.shape[0]), _ptr(k) if k.size else None,
                                            _ptr(i) if i.size else None, int(K), _ptr(out_i), _ptr(out_s),
                                            ctypes.byref(cnt))
    if st != RS_OK:
        raise RsError(st, "rs_merge_candidates: invalid arguments")
    return out_i[:cnt.value].copy(), out_s[:cnt.value].copy()


def score_keys(scores) -> np.ndarray:
    """The Step 4 order key of non-negative scores: IEEE bits, -0.0 folded to +0.0."""
    b = np.ascontiguousarray(scores, dtype=np.float64).view(np.uint64).copy()
    b[b == np.uint64(0x8000000000000000)] = 0
    return b


# ------------------------------------------------------------------ object wrapper
class Scorer:
    """One librs context. ``stream`` is a raw cudaStream_t (e.g.
    ``torch.cuda.current_stream().cuda_stream``) or None for the default stream."""

    def __init__(self, device: int = 0, stream: int | None = None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, emu: "EmuWorld | None" = None):
        if emu is not None:
            h = _P()
            st = load_library().rs_create_emulated(ctypes.byref(h), int(device), stream, int(rank), int(world), emu.h)
            if st != RS_OK:
                raise RsError(st, load_library().rs_last_error(None).decode())
            self.ctx = h
        elif world > 1:
            self.ctx = rs_create_dist(device, stream, rank, world, nccl_id)
        else:
            self.ctx = rs_create(device, stream)
        self.n = self.nnz = self.k = 0

    def close(self):
        if self.ctx is not None:
            rs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_csr(self, rowptr, col, validate: bool = False, flags: int = 0):
        rs_load_csr(self.ctx, rowptr, col, (RS_VALIDATE if validate else 0) | flags)
        self.n = int(rowptr.shape[0]) - 1
        self.nnz = int(col.shape[0])

    def set_communities(self, comm, k: int, targets=None):
        """k = RS_ALL_COMMUNITIES: every community a target (self.k becomes their number)."""
        rs_set_communities(self.ctx, comm, k, targets)
        self.k = int(k) if k != RS_ALL_COMMUNITIES else len(rs_get_targets(self.ctx))

    def score(self, scores_out=None, stats: bool = False, gather: bool = False, flags: int = 0):
        return rs_score(self.ctx, scores_out, stats, (RS_GATHER_SCORES if gather else 0) | flags)

    def scores(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.float64)
        rs_score(self.ctx, out)
        return out

    def topk(self, K: int, ids_out=None, scores_out=None):
        return rs_topk(self.ctx, K, ids_out, scores_out)

    def counts(self):
        return rs_get_counts(self.ctx, self.n, self.k)

    def weights(self):
        return rs_get_weights(self.ctx, self.n, self.k)

    def border(self):
        return rs_get_border(self.ctx, self.n)

    def pred(self):
        return rs_get_pred(self.ctx, self.n, self.nnz)

    def triad_counts(self):
        return rs_get_triad_counts(self.ctx, self.n)

    def comm_tables(self):
        return rs_get_comm_tables(self.ctx, self.n)

    def targets(self):
        return rs_get_targets(self.ctx)

    def shii(self, S, model="ic", p=0.1, runs=10, seed=0):
        return rs_shii(self.ctx, S, model, p, runs, seed)

    def awcc_removal(self, S, mode="edge", step_pct=5, max_pct=75, trials=1, seed=0):
        return rs_awcc_removal(self.ctx, S, mode, step_pct, max_pct, trials, seed)

    def launches(self) -> int:
        return rs_kernel_launches(self.ctx)

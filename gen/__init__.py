"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

INPUT GENERATION ONLY: nothing here computes any part of the RSI method
(no histogram, entropy, weight, triad or ranking arithmetic).  Both sides of
the parity check consume these inputs; neither side imports the other.

* ``rsgen(...)`` / ``config_graph(name)``: the C DC-SBM generator (rsgen.c),
  SURVEY.md §8(d) parameter table, bit-identical for any thread count.
* ``planted_partition(...)``: small numpy planted-partition graphs for the
  n in [20, 200], 3-6 community recipe of SPEC S:542.
* ``load_fixture(name)``: the text fixtures under tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librsgen.so")
_REPO = os.path.dirname(_HERE)
GOLDEN = os.path.join(_REPO, "tests", "golden")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "rsgen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m_target", ctypes.c_int64), ("gamma", ctypes.c_double),
                ("dmax", ctypes.c_double), ("n_comm", ctypes.c_int32), ("zipf_s", ctypes.c_double),
                ("mu", ctypes.c_double), ("tau", ctypes.c_double), ("oversample", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.rsgen_create.restype = ctypes.c_void_p
        lib.rsgen_create.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(ctypes.c_int)]
        lib.rsgen_n.restype = ctypes.c_int64
        lib.rsgen_n.argtypes = [ctypes.c_void_p]
        lib.rsgen_nnz.restype = ctypes.c_int64
        lib.rsgen_nnz.argtypes = [ctypes.c_void_p]
        lib.rsgen_fill.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.rsgen_destroy.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass
class Graph:
    """Canonical CSR (symmetric, rows strictly ascending, no self-loops) + labels."""
    rowptr: np.ndarray   # int64[n+1]
    col: np.ndarray      # int32[nnz]
    comm: np.ndarray     # int32[n], community id >= 0
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.rowptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    @property
    def m(self) -> int:
        return self.nnz // 2


def rsgen(n, m_target, gamma, dmax, n_comm, zipf_s=1.2, mu=0.2, tau=0.3, seed=1,
          oversample=1.0, name="rsgen", alloc=None) -> Graph:
    """Generate a DC-SBM graph.  ``alloc(shape, dtype)`` may return e.g. pinned
    torch tensors' numpy views; default numpy.empty."""
    lib = _load()
    p = _Params(int(n), int(m_target), float(gamma), float(dmax), int(n_comm), float(zipf_s),
                float(mu), float(tau), float(oversample), int(seed) & 0xFFFFFFFFFFFFFFFF)
    st = ctypes.c_int(0)
    h = lib.rsgen_create(ctypes.byref(p), ctypes.byref(st))
    if not h:
        raise RuntimeError(f"rsgen failed with status {st.value}")
    try:
        nn, nnz = lib.rsgen_n(h), lib.rsgen_nnz(h)
        alloc = alloc or (lambda shape, dt: np.empty(shape, dtype=dt))
        rowptr = alloc((nn + 1,), np.int64)
        col = alloc((nnz,), np.int32)
        comm = alloc((nn,), np.int32)
        lib.rsgen_fill(h, rowptr.ctypes.data, col.ctypes.data, comm.ctypes.data)
    finally:
        lib.rsgen_destroy(h)
    return Graph(rowptr, col, comm, name)


# SURVEY.md §8(d) configs (n, m from SNAP com-* counts; shapes are synthetic).
CONFIGS = {
    "dblp": dict(n=317_080, m_target=1_049_866, gamma=2.6, dmax=343, n_comm=64, seed=0x52534901),
    "lj": dict(n=3_997_962, m_target=34_681_189, gamma=2.4, dmax=14_815, n_comm=64, seed=0x52534902),
    "orkut": dict(n=3_072_441, m_target=117_185_083, gamma=2.2, dmax=33_313, n_comm=64, seed=0x52534903),
    "friendster": dict(n=65_608_366, m_target=1_806_067_135, gamma=2.3, dmax=5_214, n_comm=64,
                       seed=0x52534904),
}
# dedup compensation per config (measured once; realized m is always reported)
OVERSAMPLE = {"dblp": 1.079, "lj": 1.047, "orkut": 1.078, "friendster": 1.05}


def config_graph(name: str, scale: float = 1.0, alloc=None, **over) -> Graph:
    """A §8(d) config; ``scale`` < 1 shrinks n and m proportionally (parity-size
    versions of the same shape)."""
    c = dict(CONFIGS[name])
    c.update(over)
    if scale != 1.0:
        c["n"] = max(64, int(c["n"] * scale))
        c["m_target"] = max(64, int(c["m_target"] * scale))
    c.setdefault("oversample", OVERSAMPLE.get(name, 1.0))
    return rsgen(name=f"{name}@{scale:g}", alloc=alloc, **c)


def planted_partition(n: int, n_comm: int, p_in: float, p_out: float, seed: int) -> Graph:
    """Small G(n; p_in, p_out) planted partition (SPEC S:542 recipe), numpy RNG."""
    rng = np.random.default_rng(seed)
    comm = rng.integers(0, n_comm, size=n).astype(np.int32)
    same = comm[:, None] == comm[None, :]
    prob = np.where(same, p_in, p_out)
    upper = np.triu(rng.random((n, n)) < prob, k=1)
    adj = upper | upper.T
    return from_adjacency(adj, comm, name=f"pp(n={n},c={n_comm},seed={seed})")


def from_adjacency(adj: np.ndarray, comm, name="") -> Graph:
    adj = np.asarray(adj, dtype=bool)
    np.fill_diagonal(adj, False)
    deg = adj.sum(1)
    rowptr = np.zeros(adj.shape[0] + 1, dtype=np.int64)
    np.cumsum(deg, out=rowptr[1:])
    col = np.nonzero(adj)[1].astype(np.int32)  # row-major -> rows ascending
    return Graph(rowptr, col, np.asarray(comm, dtype=np.int32), name)


def from_edges(n: int, edges, comm, name="") -> Graph:
    adj = np.zeros((n, n), dtype=bool)
    for a, b in edges:
        if a != b:
            adj[a, b] = adj[b, a] = True
    return from_adjacency(adj, comm, name)


def load_fixture(name: str) -> tuple[Graph, dict]:
    """Parse tests/golden/<name>.txt: '# ...' comments, 'n N', 'edges a-b ...',
    'comm c0 c1 ...', 'targets t0 t1 ...' (optional), and 'expect key value...'
    lines returned in a dict (each expectation is cited in the file)."""
    path = os.path.join(GOLDEN, name + ".txt")
    n = None
    edges, comm, meta = [], None, {}
    with open(path) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            key, *rest = line.split()
            if key == "n":
                n = int(rest[0])
            elif key == "edges":
                for tok in rest:
                    a, b = tok.split("-")
                    edges.append((int(a), int(b)))
            elif key == "comm":
                comm = [int(x) for x in rest]
            else:
                meta[key] = rest
    g = from_edges(n, edges, comm, name)
    return g, meta

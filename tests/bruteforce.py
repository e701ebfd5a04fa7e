"""Independent brute-force definition of RSI for tiny graphs (pure numpy/Python).

Written directly from PAPER.md, separately from oracle/rsi_oracle.c, as the
"brute force on tiny inputs" pin for the oracle: literal O(n^3) triple
enumeration of the Eq.6 indicator over every ordered (u, w, v),
entropies in natural log divided by ln 2 (a different route than the
oracle's log2), and per-head sums with math.fsum (exactly rounded, so order
independent).  Shares no code with oracle/ or the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np


def adjacency(g):
    n = g.n
    A = np.zeros((n, n), dtype=bool)
    for u in range(n):
        A[u, g.col[g.rowptr[u]:g.rowptr[u + 1]]] = True
    return A


def select_targets(comm, k):
    ids, sizes = np.unique(np.asarray(comm), return_counts=True)
    order = sorted(range(len(ids)), key=lambda i: (-sizes[i], ids[i]))  # P:846, C-15
    return np.array([ids[i] for i in order[:k]], dtype=np.int32)


def brute(g, targets):
    A = adjacency(g)
    C = np.asarray(g.comm)
    n = g.n
    k = len(targets)
    colmap = {int(t): i for i, t in enumerate(targets)}
    col = np.array([colmap.get(int(c), -1) for c in C])
    deg = A.sum(1)

    border = np.array([bool(np.any(A[u] & (C != C[u]))) for u in range(n)])
    f = np.zeros((n, k), dtype=np.int64)
    for v in range(n):
        for x in np.nonzero(A[v])[0]:
            if col[x] >= 0:
                f[v, col[x]] += 1

    omega = np.zeros((n, k))
    for v in range(n):
        L_all = int(np.count_nonzero(f[v]))
        if L_all <= 1:
            continue
        for i in range(k):
            others = [f[v, j] for j in range(k) if j != i and f[v, j] > 0]      # L(u,v), Eq.2
            Y = sum(others)
            H = -sum((fj / Y) * math.log(fj / Y) for fj in others) / math.log(2.0)  # Eq.3
            omega[v, i] = H * (L_all - 1)                                         # Eq.5, Alg.2 L
    wmax = float(omega.max()) if omega.size else 0.0

    R = np.zeros(n)
    nI = np.zeros(n, dtype=np.int64)
    nII = np.zeros(n, dtype=np.int64)
    for u in range(n):
        if col[u] < 0 or deg[u] < 2:
            continue
        terms = []
        for w in range(n):
            if w == u or not A[u, w] or C[w] == C[u]:
                continue
            for v in range(n):
                if v == u or v == w or not A[w, v] or C[v] == C[w]:
                    continue
                type1 = A[u, v] and C[u] != C[v] and col[v] >= 0
                type2 = C[u] == C[v]
                if not (type1 or type2):
                    continue
                if type1:
                    nI[u] += 1
                else:
                    nII[u] += 1
                if wmax > 0:
                    cu, cv = col[u], col[v]
                    p = (omega[v, cu] / wmax) * (omega[w, cv] / wmax) * (omega[w, cu] / wmax)
                    terms.append(p ** (1.0 / 3.0))
        if wmax > 0:
            R[u] = math.fsum(terms) / (deg[u] * (deg[u] - 1))
    order = sorted(range(n), key=lambda i: (-R[i], i))
    return dict(border=border, f=f, omega=omega, omega_max=wmax, R=R, nI=nI, nII=nII, order=order)

"""Work statistics of the Type-I triangle phase (Phase E) on a generated
config: |P|, the rank orientation, heavy/light split, work items and probe
volume. Host-side analysis tool (numpy), not part of the product path.
usage: python tools/e_stats.py [config] [scale] [k]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import gen  # noqa: E402


def main(name="orkut", scale=1.0, k=5, chunk=64, heavy_deg=128):
    g = gen.config_graph(name, scale)
    n, rp, col, comm = g.n, g.rowptr, g.col, g.comm
    deg = np.diff(rp)
    row = np.repeat(np.arange(n, dtype=np.int32), deg)
    foreign = comm[col] != comm[row]
    pcnt = np.bincount(row[foreign], minlength=n)
    sizes = np.bincount(comm)
    order = np.lexsort((np.arange(sizes.size), -sizes))
    is_t = np.zeros(sizes.size, bool)
    is_t[order[:k]] = True
    tv = is_t[comm]
    # rank (|P|, id): z above x
    r_src, r_dst = row[foreign], col[foreign]
    del row, foreign
    up = (pcnt[r_dst] > pcnt[r_src]) | ((pcnt[r_dst] == pcnt[r_src]) & (r_dst > r_src))
    pplus = np.bincount(r_src[up], minlength=n)
    pminus = pcnt - pplus
    # probe volume: for each y, sum over x in P-(y) (x below y: edges (y, x) with not up) of |P+(x)|
    dn = ~up
    ys, xs = r_src[dn], r_dst[dn]
    keep = (pplus[xs] > 0) & (pplus[ys] > 0) & (tv[xs] | tv[ys])
    ys, xs = ys[keep], xs[keep]
    probes = pplus[xs].astype(np.int64)
    heavy_y = deg[ys] >= heavy_deg
    print(f"{name}@{scale}: n={n} nnz={col.size} |P| entries={pcnt.sum()} G' edges={pcnt.sum() // 2}")
    print(f"probe volume {probes.sum():.4e} ({probes.sum() / col.size:.3f} per adjacency entry); "
          f"heavy-y share {probes[heavy_y].sum() / probes.sum():.3f}")
    hy = np.where((deg >= heavy_deg) & (pplus > 0) & (pminus > 0))[0]
    items = np.ceil(pminus[hy] / chunk).astype(np.int64)
    print(f"heavy y: {hy.size}, items {items.sum()}, P+(y) > 256: {(pplus[hy] > 256).sum()} "
          f"(their probe share {probes[heavy_y & (pplus[ys] > 256)].sum() / probes.sum():.3f})")
    # per-item probes (approx: per y / items)
    per_y = np.bincount(ys[heavy_y], weights=probes[heavy_y], minlength=n)[hy]
    per_item = per_y / items
    q = np.percentile(per_item, [10, 50, 90, 99])
    print(f"probes per item p10/50/90/99 = {q.round(0)}; items with > 2048 probes (unmapped @kPiece=4,map 512): "
          f"{(per_item > 2048).mean():.3f}")
    print(f"|P+(x)| of probed x: mean {probes.mean():.1f}, p99 {np.percentile(probes, 99):.0f}, "
          f"max {probes.max()}")
    light = ~heavy_y
    print(f"light y: {np.unique(ys[light]).size}, light probe volume {probes[light].sum():.3e}, "
          f"light (x,y) pairs {light.sum():.3e}")
    print(f"|P+(y)| heavy: p50 {np.median(pplus[hy]):.0f} p90 {np.percentile(pplus[hy], 90):.0f} "
          f"max {pplus[hy].max()}; |P-(y)| p50 {np.median(pminus[hy]):.0f} max {pminus[hy].max()}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "orkut", float(a[1]) if len(a) > 1 else 1.0, int(a[2]) if len(a) > 2 else 5)


def py_buckets(name="orkut", scale=1.0, k=5):
    """probe share by |P+(y)| bucket, and by target status of (x, y, z)"""
    g = gen.config_graph(name, scale)
    n, rp, col, comm = g.n, g.rowptr, g.col, g.comm
    deg = np.diff(rp)
    row = np.repeat(np.arange(n, dtype=np.int32), deg)
    foreign = comm[col] != comm[row]
    pcnt = np.bincount(row[foreign], minlength=n)
    sizes = np.bincount(comm)
    order = np.lexsort((np.arange(sizes.size), -sizes))
    is_t = np.zeros(sizes.size, bool)
    is_t[order[:k]] = True
    tv = is_t[comm]
    r_src, r_dst = row[foreign], col[foreign]
    del row, foreign
    up = (pcnt[r_dst] > pcnt[r_src]) | ((pcnt[r_dst] == pcnt[r_src]) & (r_dst > r_src))
    pplus = np.bincount(r_src[up], minlength=n)
    pplus_t = np.bincount(r_src[up & tv[r_dst]], minlength=n)
    dn = ~up
    ys, xs = r_src[dn], r_dst[dn]
    keep = (pplus[xs] > 0) & (pplus[ys] > 0) & (tv[xs] | tv[ys])
    ys, xs = ys[keep], xs[keep]
    both = tv[xs] & tv[ys]
    probes = pplus[xs].astype(np.int64)
    probes_t = np.where(both, pplus[xs], pplus_t[xs]).astype(np.int64)
    print(f"probes {probes.sum():.4e}; with target-prefix pruning {probes_t.sum():.4e} "
          f"({probes_t.sum() / probes.sum():.3f}); both-target pairs {both.mean():.3f}")
    pyv = pplus[ys]
    for lo, hi in [(0, 32), (32, 64), (64, 128), (128, 256), (256, 1 << 30)]:
        m = (pyv >= lo) & (pyv < hi)
        print(f"|P+(y)| in [{lo},{hi}): probe share {probes[m].sum() / probes.sum():.3f}")


def orientation_compare(name="orkut", scale=1.0, k=5):
    """probe volume (with target-run pruning) for the rank (|P|, id) orientation
    vs the rank (degree, id) orientation"""
    g = gen.config_graph(name, scale)
    n, rp, col, comm = g.n, g.rowptr, g.col, g.comm
    deg = np.diff(rp)
    row = np.repeat(np.arange(n, dtype=np.int32), deg)
    foreign = comm[col] != comm[row]
    pcnt = np.bincount(row[foreign], minlength=n)
    sizes = np.bincount(comm)
    order = np.lexsort((np.arange(sizes.size), -sizes))
    is_t = np.zeros(sizes.size, bool)
    is_t[order[:k]] = True
    tv = is_t[comm]
    r_src, r_dst = row[foreign], col[foreign]
    del row, foreign
    for label, key in [("|P|", pcnt), ("degree", deg)]:
        up = (key[r_dst] > key[r_src]) | ((key[r_dst] == key[r_src]) & (r_dst > r_src))
        pplus = np.bincount(r_src[up], minlength=n)
        pplus_t = np.bincount(r_src[up & tv[r_dst]], minlength=n)
        dn = ~up
        ys, xs = r_src[dn], r_dst[dn]
        keep = (pplus[xs] > 0) & (pplus[ys] > 0) & (tv[xs] | tv[ys])
        ys, xs = ys[keep], xs[keep]
        both = tv[xs] & tv[ys]
        probes_t = np.where(both, pplus[xs], pplus_t[xs]).astype(np.int64)
        print(f"orientation by {label}: probes {probes_t.sum():.4e}, max |P+| {pplus.max()}, "
              f"pairs {ys.size:.3e}")


def direction_stats(name="orkut", scale=1.0, k=5):
    """probe volume if each (x, y) pair probed its shorter side (id orientation,
    target-run pruning): sum of |P+(x)| vs sum of min(|P+(x)|, c |P+(y)| log2 |P+(x)|)"""
    g = gen.config_graph(name, scale)
    n, rp, col, comm = g.n, g.rowptr, g.col, g.comm
    deg = np.diff(rp)
    # internal order: degree descending, stable
    order = np.argsort(-deg, kind="stable")
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    row = np.repeat(np.arange(n, dtype=np.int32), deg)
    foreign = comm[col] != comm[row]
    sizes = np.bincount(comm)
    corder = np.lexsort((np.arange(sizes.size), -sizes))
    is_t = np.zeros(sizes.size, bool)
    is_t[corder[:k]] = True
    tv = is_t[comm]
    r_src, r_dst = row[foreign], col[foreign]
    del row, foreign
    up = rank[r_dst] < rank[r_src]              # dst above src
    pplus = np.bincount(r_src[up], minlength=n)
    pplus_t = np.bincount(r_src[up & tv[r_dst]], minlength=n)
    dn = ~up
    ys, xs = r_src[dn], r_dst[dn]
    keep = (pplus[xs] > 0) & (pplus[ys] > 0) & (tv[xs] | tv[ys])
    ys, xs = ys[keep], xs[keep]
    both = tv[xs] & tv[ys]
    px = np.where(both, pplus[xs], pplus_t[xs]).astype(np.float64)
    py = np.where(both, pplus[ys], pplus_t[ys]).astype(np.float64)
    print(f"forward probes {px.sum():.4e}")
    for c in [1, 2, 4]:
        cost = np.minimum(px, c * py * np.log2(np.maximum(px, 2)))
        rev = px > c * py * np.log2(np.maximum(px, 2))
        print(f"c={c}: hybrid cost {cost.sum():.4e}, reversed pairs {rev.mean():.3f}, "
              f"reversed probes {py[rev].sum():.3e} (searches), saved forward {px[rev].sum():.3e}")

// Phase E — the Type-I part of Step 3 (Algorithm 1): closed triads
// over three communities (Eq. 6) found as triangles of G'.
//
// G' has an edge between u and w iff they are adjacent in G and C(u) != C(w)
// (P:493), so the three communities of a G' triangle are pairwise distinct:
// every Type-I triad is a (head, mid) ordering of a G' triangle. G' is
// oriented by internal id (degree-descending: z is above u iff z < u; P+(u)
// is the prefix of P(u)), and each triangle z < y < x is found exactly once
// from its middle vertex y, as z in P+(x) ∩ P+(y) for x in P-(y) (the paper's
// "common predecessor" search, with filter/binary-search probes
// instead of a merge). Only triangles with two target vertices can carry a
// term (reading C-27): a pair (x, y) of targets probes all of P+(x), a pair
// with one target only the target run of P+(x), a pair without none.
//
// Each triangle adds the grouped terms of its (up to) three heads
//   head x: a_y(c_x) a_z(c_x) (a_z(c_y) + a_y(c_z))
//   head y: a_x(c_y) a_z(c_y) (a_z(c_x) + a_x(c_z))
//   head z: a_x(c_z) a_y(c_z) (a_y(c_x) + a_x(c_y))
// with a_v(c) = 0 for a non-target column c, each expression symmetric in the
// two other vertices (the numbering changes no bit of the result). a_x(c_z)
// comes from the weight Phase A stored beside z in P+(x) (read at the probe's
// own index). Sums are exact fixed point (C-12); the highest-degree heads are
// striped over kHubStripes accumulators (same-address atomics serialise).
//
// Heavy middle vertices (degree >= 128): work items (y, 64 positions of
// P-(y)), a warp per item from a global queue, heaviest first. The warp puts a
// 4096-bit filter and a sorted copy of P+(y) in shared memory, lists the
// item's predecessors x, and cuts every probed prefix of P+(x) into aligned
// 16-byte pieces: a lane probes one piece per round (the next round's load in
// flight), filter candidates are packed with one warp scan and verified 32 at a
// time by binary search in the run of P+(y) they can belong to. Head terms:
// y's in registers, x's in shared 20-bit limbs, z's by RED. Light middle
// vertices: a warp per 32 consecutive y, pairs and then probes flattened over
// the lanes. COUNT mode (parity getter) counts the ordered (head, mid) target
// pairs instead.
#include "rs_phase.cuh"
#include <cstdlib>

namespace rs {

constexpr int kChunkE = 64;      // positions of P(y) per work item
#ifndef RS_EXP_PYCAP
#define RS_EXP_PYCAP 128
#endif
#ifndef RS_EXP_E_MINB
#define RS_EXP_E_MINB 4
#endif
constexpr int kPyCap = RS_EXP_PYCAP;   // P+(y) kept in shared memory (sorted copy + labels)
constexpr int kBmWords = 128;    // 4096-bit membership filter of P+(y)
constexpr int kPiece = 4;        // consecutive P+(x) entries one lane probes per round
constexpr int kQCapE = 160;      // candidate queue (31 + 32 * kPiece < 160)
#ifndef RS_EXP_PSWORDS
#define RS_EXP_PSWORDS 128
#endif
constexpr int kPsWords = RS_EXP_PSWORDS;    // piece-start bitmap: items of at most 4096 pieces (else binary search)
constexpr int kWarpsE = 8;
#ifndef RS_EXP_QBATCH
#define RS_EXP_QBATCH 4
#endif
constexpr int kQBatch = RS_EXP_QBATCH;   // heavy work items per queue pop
#ifndef RS_EXP_E_REUSE
#define RS_EXP_E_REUSE 1                     // reuse the filter / P+(y) copy when consecutive items share y
#endif
#ifndef RS_EXP_E_RING
#define RS_EXP_E_RING 0                      // probe rounds staged in shared memory by cp.async (0: registers; measured 2 / 3 / 4 / 6 stages: E||D +0.04 / +0.08 / +0.20 / +0.22 ms, fewer resident blocks)
#endif
#ifndef RS_EXP_E_XPRE
#define RS_EXP_E_XPRE 0                      // load the next item's x list during this item (measured: E||D +0.03 ms, spills; off)
#endif
#ifndef RS_EXP_E_YSKIP
#define RS_EXP_E_YSKIP 1                     // skip the filter of probe rounds without any z < y
#endif
#ifndef RS_EXP_E_DEPTH
#define RS_EXP_E_DEPTH 1                     // probe rounds in flight ahead of the one being filtered (1 or 2; 2: E||D +0.02 ms, spills)
#endif

// membership filter bit of z (top 12 bits of a multiplicative hash)
__device__ __forceinline__ uint32_t bm_bit(int32_t z) {
    return ((uint32_t)z * 0x85EBCA6Bu) >> 20;
}

// position of z in the sorted list p[0, len), or -1
__device__ __forceinline__ int find_sorted(const int32_t *p, int len, int32_t z) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (p[mid] < z) lo = mid + 1; else hi = mid;
    }
    return (lo < len && p[lo] == z) ? lo : -1;
}
__device__ __forceinline__ int find_sorted_g(const int32_t *p, int len, int32_t z) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(p + mid) < z) lo = mid + 1; else hi = mid;
    }
    return (lo < len && __ldg(p + lo) == z) ? lo : -1;
}

__device__ __forceinline__ double amat_at(const CdeArgs &a, int32_t v, int c) {
    return c < a.k ? __ldg(a.amat + (int64_t)v * a.k + c) : 0.0;
}

__device__ __forceinline__ bool owned(const CdeArgs &a, int64_t h) { return h >= a.head_lo && h < a.head_hi; }

// global exact accumulation of a head's (partial) Type-I sum (3 limbs for the
// wide heads, VRec::wide = h < n_wide)
__device__ __forceinline__ void acc_add(const CdeArgs &a, int32_t h, const U128 &q) {
    const bool wide = is_wide(a, h);
    unsigned long long *acc = a.acc1 + 3 * (int64_t)h;
    if (h < a.n_hub) {
        const int stripe = (int)(((blockIdx.x * blockDim.x + threadIdx.x) >> 5) & (kHubStripes - 1));
        acc = a.acc_hub + 3 * ((int64_t)stripe * a.n_hub + h);
    }
    if (wide) fx_red3(acc, q);
    else fx_red2(acc, q);
}

// position of z in the DESCENDING list p[0, len), or -1
__device__ __forceinline__ int find_desc_g(const int32_t *p, int len, int32_t z) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(p + mid) > z) lo = mid + 1; else hi = mid;
    }
    return (lo < len && __ldg(p + lo) == z) ? lo : -1;
}

// The probed range of P+(x) for the pair (y, x in P-(y)): a triangle z < y < x
// needs z in P+(y), so only the entries of P+(x) below y can close one (about
// half of P+(x) on average). Phase A stores P+(x) as its target run descending
// at [0, t) and the other run ascending at [t, |P+|), so those entries are one
// contiguous range: the tail of the target run and (if x and y are both
// targets, C-27) the head of the other run, found by two binary searches in
// lockstep. Returns the range's memory start, its length and the number of
// target entries at its front. All-communities mode: one ascending run.
// Measured on the Orkut shape (probes 394 M -> 202 M with the cut, 1xB200):
// Phase E+D 3.84 ms without the cut, 4.29 ms with it, 3.87 ms cutting only
// lists of >= 64 entries -- the two binary searches per pair in the item setup
// cost more than the probes they save (short lists: 1-2 aligned pieces either
// way). Off by default; -DRS_EXP_CUT_MIN=n cuts lists of >= n entries.
#ifndef RS_EXP_CUT_MIN
#define RS_EXP_CUT_MIN 0x7fffffff
#endif
template <bool SPARSE>
__device__ __forceinline__ void cut_range(const int32_t *__restrict__ pplus, int64_t bx, int pp, int t, int32_t y,
                                          bool both, bool any, int64_t &rs, int &len, int &tb) {
    if (!any) { rs = bx; len = 0; tb = 0; return; }
    if (pp < RS_EXP_CUT_MIN) {   // experiment: no cut below this list length
        // free bound: the ids are distinct and >= 0, so at most y entries of a run
        // lie below y -- the tail of the descending target run, the head of the
        // ascending other run (exact; 6 % fewer probes on the Orkut shape, mostly
        // for the hub middle vertices with small ids)
        const int yb = y;
        if constexpr (SPARSE) {
            rs = bx; len = min(pp, yb); tb = len;
        } else {
            const int mt = min(t, yb), mo = both ? min(pp - t, yb) : 0;
            rs = bx + (t - mt); tb = mt; len = mt + mo;
        }
        return;
    }
    if constexpr (SPARSE) {
        int lo = 0, hi = pp;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(pplus + bx + mid) < y) lo = mid + 1; else hi = mid;
        }
        rs = bx; len = lo; tb = lo;
    } else {
        int lo1 = 0, hi1 = t, lo2 = 0, hi2 = both ? pp - t : 0;   // #target entries >= y, #others < y
        while (lo1 < hi1 || lo2 < hi2) {
            const int m1 = (lo1 + hi1) >> 1, m2 = (lo2 + hi2) >> 1;
            const int32_t v1 = lo1 < hi1 ? __ldg(pplus + bx + m1) : 0;
            const int32_t v2 = lo2 < hi2 ? __ldg(pplus + bx + t + m2) : 0;
            if (lo1 < hi1) { if (v1 >= y) lo1 = m1 + 1; else hi1 = m1; }
            if (lo2 < hi2) { if (v2 < y) lo2 = m2 + 1; else hi2 = m2; }
        }
        rs = bx + lo1; tb = t - lo1; len = tb + lo2;
    }
}

// shared-memory per-item accumulator: four 20-bit limbs of q (< 2^80) added with
// native 32-bit shared atomics (64-bit shared atomics are CAS loops); exact
// while a slot receives at most CdeArgs::slot_cap terms per item (the top limb
// then cannot wrap; x slots with longer probed P+(x) go straight to the global
// limbs).
__device__ __forceinline__ void smem_red4(uint32_t *acc4, const U128 &q) {
    const uint32_t l0 = (uint32_t)(q.lo & 0xFFFFFull), l1 = (uint32_t)((q.lo >> 20) & 0xFFFFFull);
    const uint32_t l2 = (uint32_t)((q.lo >> 40) & 0xFFFFFull), l3 = (uint32_t)((q.lo >> 60) | (q.hi << 4));
    if (l0) atomicAdd(acc4 + 0, l0);
    if (l1) atomicAdd(acc4 + 1, l1);
    if (l2) atomicAdd(acc4 + 2, l2);
    if (l3) atomicAdd(acc4 + 3, l3);
}
__device__ __forceinline__ U128 from4(const uint32_t *acc4) {
    U128 s = U128{(unsigned long long)acc4[0], 0ull};
    s = u128_add(s, U128{(unsigned long long)acc4[1] << 20, 0ull});
    s = u128_add(s, U128{(unsigned long long)acc4[2] << 40, (unsigned long long)acc4[2] >> 24});
    s = u128_add(s, U128{(unsigned long long)acc4[3] << 60, (unsigned long long)acc4[3] >> 4});
    return s;
}

// a work item: positions [64 chunk, 64 chunk + 64) of P-(y), with y's record
struct __align__(16) EItem {
    int64_t by;            // start of y's slot (rowptr[y]): P(y) in pidx, P+(y) runs in pplus
                           // (multi-GPU: the packed offset of P+(y))
    int32_t y, chunk;
    int32_t pyl;           // |P+(y)| | lab(y) << 24
    int32_t pm;            // |P-(y)|
    int32_t pyt;           // |P+_T(y)|
    uint32_t mbase;        // multi-GPU: offset of P-(y) in the packed heavy lists
};
struct EItems {
    const EItem *items;    // work items of the heavy middle vertices, heaviest first
    const int32_t *total;  // number of items (device scalar, written by the item scan)
};

struct ESmem {             // one warp's shared memory
    uint32_t bm[kBmWords];
    int32_t py[kPyCap];     // P+(y): target run, then the other run, each ascending
    longlong2 xl[kChunkE];  // {x's slot start, (x << 32) | (lab(x) << 24) | |P+_T(x)|}
    int2 xn[kChunkE];       // {probed length of P+(x) (its target run, or all of it), -}
    uint32_t xa[4 * kChunkE];
    int32_t pe[kChunkE];    // end of each list's pieces
    int2 q[kQCapE];         // candidates {((offset of z in P+(x)) + 4) << 6 | x slot, z}
    uint32_t ps[kPsWords];  // bit p: piece p is the first piece of a list
#if RS_EXP_E_RING
    int4 ring[RS_EXP_E_RING][32];   // probe pieces in flight (cp.async), one per lane per round
    int rtag[RS_EXP_E_RING][32];    // their tags (-1: no piece)
#endif
};

__host__ __device__ constexpr size_t e_stride_bytes(int k) {
    return ((sizeof(ESmem) + 15) / 16) * 16 + ((8 * (size_t)k + 15) / 16) * 16;
}

// multi-GPU: the heavy items are dealt to the ranks in blocks of e_blk
// consecutive items, block b to rank b mod world. Measured (8 emulated ranks,
// Orkut shape, E || D max / mean over ranks): e_blk 1 1.07 / 0.85 ms, 4 1.38 /
// 1.22, 32 1.36 / 1.21, 256 1.38 / 1.21 -- keeping a y's items together on one
// rank (filter reuse) loses to spreading them, so 1 is the default
// (32-bit: item counts stay below 2^32; the common one-GPU / e_blk = 1 case is
// a multiply-add, the default e_perm = 2 constant shifts -- profiled: the 64-bit
// divisions of the general form were 2 % of the kernel's instructions)
__device__ __forceinline__ unsigned e_item(unsigned qi, int r, int world, int blk) {
    if (blk == 1) return qi * (unsigned)world + (unsigned)r;
    const unsigned B = (unsigned)blk;
    return ((qi / B) * (unsigned)world + (unsigned)r) * B + qi % B;
}
// within each group of kQBatch * P items, batch b takes items b, b + P,
// b + 2P, ... (a P x kQBatch transpose of the heaviest-first order)
__device__ __forceinline__ unsigned e_perm_map(unsigned g, int P, unsigned n_all) {
    if (P <= 1) return g;
    if (P == 2) {
        constexpr unsigned G2 = 2u * kQBatch;
        const unsigned base = g - g % G2, o = g % G2;
        if (base + G2 > n_all) return g;
        return base + (o / kQBatch) + 2u * (o % kQBatch);
    }
    const unsigned G = (unsigned)P * kQBatch, base = g - g % G, o = g % G;
    if (base + G > n_all) return g;
    return base + (o / kQBatch) + (unsigned)P * (o % kQBatch);
}
__device__ __forceinline__ unsigned long long e_rank_items(unsigned long long n_all, int r, int world, int blk) {
    const unsigned long long B = (unsigned long long)blk;
    const unsigned long long nb = (n_all + B - 1) / B, W = (unsigned long long)world, R = (unsigned long long)r;
    if (nb <= R) return 0ull;
    const unsigned long long mine = (nb - R + W - 1) / W;           // blocks r, r + W, ... < nb
    unsigned long long cnt = mine * B;
    if ((nb - 1) % W == R) cnt -= nb * B - n_all;                   // the last, partial block is this rank's
    return cnt;
}

// SPARSE (all-communities mode, k_sparse.cu): every vertex is a target, P+(u)
// is one ascending run in pidx, and the weights come from beside the list
// entries (wps: a_u(c_w), pwr: a_w(c_u)) instead of the dense rows.
template <bool COUNT, bool SPARSE>
__global__ void __launch_bounds__(kWarpsE * 32, RS_EXP_E_MINB) k_phase_e(CdeArgs a, EItems it, unsigned long long *queue_ctr) {
    extern __shared__ __align__(16) unsigned char e_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = a.k;
    unsigned char *base = e_smem + (size_t)wid * e_stride_bytes(SPARSE ? 0 : k);
    ESmem &S = *reinterpret_cast<ESmem *>(base);
    double *Ay = (double *)(base + ((sizeof(ESmem) + 15) / 16) * 16);
    unsigned long long ntri = 0, nprobe = 0;
    // multi-GPU: rank r takes the blocks of e_blk items b = r, r + world, ...
    // (heaviest first on every rank; e_item maps its queue index to the item)
    const unsigned long long n_all = (unsigned long long)*it.total;
    const unsigned long long n_items = e_rank_items(n_all, a.e_rank, a.e_world, a.e_blk);

    // the next item's index and its 32-byte record (word `lane` of it in lanes
    // 0-7) are fetched while the current item is processed
    const int32_t *items_w = reinterpret_cast<const int32_t *>(it.items);
    // items are popped kQBatch at a time: one same-address atomic per batch (the
    // queue counter is the one address every warp of the grid updates)
    unsigned long long qnext = 0;
    if (lane == 0) qnext = atomicAdd(queue_ctr, (unsigned long long)kQBatch);
    unsigned long long qbase = __shfl_sync(0xffffffffu, qnext, 0);
    unsigned long long qi = qbase;
    int32_t rec = (qi < n_items && lane < 8) ? __ldg(items_w + 8 * (size_t)(a.e_local ? (unsigned)qi : e_perm_map(e_item((unsigned)qi, a.e_rank, a.e_world, a.e_blk), a.e_perm, (unsigned)n_all)) + lane) : 0;
    // the items of one y are consecutive (a batch pop often brings two of them):
    // the filter, the sorted copy of P+(y) and y's weights built for the previous
    // item are reused when y repeats
    int32_t prev_y = -1;
    // the next item's x list, loaded during the current item's probes (its x
    // records prefetched into L2 after the first probe round): the setup of an
    // item is a chain of dependent gathers (P-(y) -> PRec(x) -> pieces)
    int32_t xpre[2] = {-1, -1};
    bool pre_ok = false;
    for (;;) {
        if (qi >= n_items) break;
        const bool last_of_batch = qi - qbase == (unsigned long long)(kQBatch - 1);
        if (last_of_batch && lane == 0) qnext = atomicAdd(queue_ctr, (unsigned long long)kQBatch);   // next batch
        // EItem words: by (0, 1), y (2), chunk (3), pyl (4), pm (5), pyt (6)
        const int64_t by = (int64_t)(uint32_t)__shfl_sync(0xffffffffu, rec, 0) |
                           ((int64_t)__shfl_sync(0xffffffffu, rec, 1) << 32);
        const int32_t y = __shfl_sync(0xffffffffu, rec, 2);
        const int chunk = __shfl_sync(0xffffffffu, rec, 3);
        const int pyl = __shfl_sync(0xffffffffu, rec, 4);
        const int ipm = __shfl_sync(0xffffffffu, rec, 5);
        const int pyt = __shfl_sync(0xffffffffu, rec, 6);
        const uint32_t mb = (uint32_t)__shfl_sync(0xffffffffu, rec, 7);
        const int py = pyl & 0xFFFFFF, ly = (int)((uint32_t)pyl >> 24);
        const int start = chunk * a.e_chunk, end = min(ipm, start + a.e_chunk);
        const bool ty = ly < k;
        const bool local = py <= kPyCap;            // sorted copy of P+(y) in smem
        // setup: the loads of P-(y) (x list), P+(y) (filter) and y's weights are
        // independent and issued together; then the x records, lab(z), a_x(c_y)
        int32_t xv[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int i = start + 32 * h + lane;
            // x in P-(y) (the suffix of P(y) in its slot; multi-GPU: packed): x > y
            xv[h] = pre_ok ? xpre[h] : (i < end ? __ldg(a.pidx + (a.mg ? (int64_t)mb : by + py) + i) : -1);
        }
        pre_ok = false;
        // i-th entry of P+(y) in ascending order within its run (the target run is
        // stored descending, the other run ascending after it)
        auto py_at = [&](int i) -> int64_t { return SPARSE ? by + i : (i < pyt ? by + pyt - 1 - i : by + i); };
        const bool fresh = !RS_EXP_E_REUSE || y != prev_y;   // warp-uniform
        const int32_t z0 = (fresh && lane < py) ? __ldg(a.pplus + py_at(lane)) : -1;
        const double ay0 = (fresh && !SPARSE && lane < k) ? __ldg(a.amat + (int64_t)y * k + lane) : 0.0;
        // x's record and label; its weight a_x(c_y) (and, all-communities mode,
        // a_y(c_x)) is gathered only by the lanes that verify a triangle (most
        // (y, x) pairs close none), from x's position kept in S.xn[slot].y
        PRec pcx[2];
        int lxv[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            pcx[h] = xv[h] >= 0 ? a.pc2[xv[h]] : PRec{(int)0xFF000000, 0, 0};
            lxv[h] = pr_lab(pcx[h]);                      // the label rides in the record
        }
        if (fresh) {
            __syncwarp();                                   // the previous item's readers are done
            for (int w = lane; w < kBmWords; w += 32) S.bm[w] = 0u;
            if constexpr (!SPARSE) {
                if (lane < k) Ay[lane] = ay0;
                for (int c = lane + 32; c < k; c += 32) Ay[c] = __ldg(a.amat + (int64_t)y * k + c);
            }
            __syncwarp();
            for (int i = lane; i < py; i += 32) {
                const int32_t z = i == lane ? z0 : __ldg(a.pplus + py_at(i));
                const uint32_t b = bm_bit(z);
                atomicOr(&S.bm[b >> 5], 1u << (b & 31));
                if (local) {
                    S.py[i] = z;
                }
            }
            prev_y = y;
        }
        // the next item's record, in flight during this item
        if (last_of_batch) {
            qbase = __shfl_sync(0xffffffffu, qnext, 0);
            qi = qbase;
        } else {
            qi++;
        }
        rec = (qi < n_items && lane < 8) ? __ldg(items_w + 8 * (size_t)(a.e_local ? (unsigned)qi : e_perm_map(e_item((unsigned)qi, a.e_rank, a.e_world, a.e_blk), a.e_perm, (unsigned)n_all)) + lane) : 0;
        // the item's predecessors x. A triangle carries a term only if two of its
        // vertices are targets: with both x and y targets every z < y of P+(x) is
        // probed, with one of them only those of the target run, with neither
        // nothing (cut_range). Each probed range is cut into pieces numbered
        // across the item.
        int nx = 0, npieces = 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int lx = lxv[h];
            const bool tx = lx < k;
            int64_t bx;
            int lenx, t;
            cut_range<SPARSE>(a.pplus, pr_start(pcx[h]), pr_plus(pcx[h]), pr_plus_t(pcx[h]), y, tx && ty,
                              xv[h] >= 0 && (tx || ty), bx, lenx, t);
            const bool use = lenx > 0;
            nprobe += (unsigned)lenx;
            // aligned 16-byte pieces covering [bx, bx + lenx)
            const int pieces = use ? (int)(((bx + lenx - 1) >> 2) - (bx >> 2) + 1) : 0;
            int incl = pieces;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const unsigned has = __ballot_sync(0xffffffffu, use);
            if (use) {
                const int slot = nx + __popc(has & ((1u << lane) - 1u));
                S.xl[slot] = make_longlong2(bx, ((long long)xv[h] << 32) | ((long long)(lx & 0xFF) << 24) | t);
                S.xn[slot] = make_int2(lenx, start + 32 * h + lane);   // x's position in P-(y)
                S.xa[4 * slot] = 0u;
                S.xa[4 * slot + 1] = 0u;
                S.xa[4 * slot + 2] = 0u;
                S.xa[4 * slot + 3] = 0u;
                S.pe[slot] = npieces + incl;
            }
            nx += __popc(has);
            npieces += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (npieces == 0) continue;
#ifdef RS_EXP_SETUP_ONLY
        if (npieces >= 0) continue;
#endif
        // piece -> list: bit p of S.ps marks the first piece of a list, so the list
        // of piece p0 + lane is (lists started before p0) + popc(word & lanes <= lane) - 1
        const bool mapped = npieces <= 32 * kPsWords;
        if (mapped) {
            for (int w = lane; w < ((npieces + 31) >> 5); w += 32) S.ps[w] = 0u;
            __syncwarp();
            for (int s = lane; s < nx; s += 32) {
                const int st = s ? S.pe[s - 1] : 0;
                atomicOr(&S.ps[st >> 5], 1u << (st & 31));
            }
            __syncwarp();
        }
#if RS_EXP_E_XPRE
        if (qi < n_items) {                                 // warp-uniform: the next item exists
            const int64_t byn = (int64_t)(uint32_t)__shfl_sync(0xffffffffu, rec, 0) |
                                ((int64_t)__shfl_sync(0xffffffffu, rec, 1) << 32);
            const int32_t yn = __shfl_sync(0xffffffffu, rec, 2);
            const int chn = __shfl_sync(0xffffffffu, rec, 3);
            const int pyn = __shfl_sync(0xffffffffu, rec, 4) & 0xFFFFFF;
            const int pmn = __shfl_sync(0xffffffffu, rec, 5);
            const uint32_t mbn = (uint32_t)__shfl_sync(0xffffffffu, rec, 7);
            const int sn = chn * a.e_chunk, en = min(pmn, sn + a.e_chunk);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int i = sn + 32 * h + lane;
                xpre[h] = i < en ? __ldg(a.pidx + (a.mg ? (int64_t)mbn : byn + pyn) + i) : -1;
            }
            pre_ok = true;
            if (yn != y) {                                  // a new y: its P+(y) runs and weight row
                if (32 * lane < pyn) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.pplus + byn + 32 * lane));
                if (!SPARSE && lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.amat + (int64_t)yn * k));
            }
        }
#endif
        int lists_before = 0;
        auto fetch = [&](int p0, int32_t (&z)[kPiece], int &tag) {
            const int p = p0 + lane;
            int slot;
            if (mapped) {
                const uint32_t wd = S.ps[p0 >> 5];
                slot = lists_before + __popc(wd & (0xFFFFFFFFu >> (31 - lane))) - 1;
                lists_before += __popc(wd);
            } else {
                int lo = 0, hi = nx;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (S.pe[mid] <= p) lo = mid + 1; else hi = mid;
                }
                slot = lo;
            }
            int off = 0;   // offset in P+(x) of the piece's first entry (-3..-1 for a head piece)
            if (p < npieces) {
                const int64_t bx = S.xl[slot].x;
                const int lenx = S.xn[slot].x;
                const int q = p - (slot ? S.pe[slot - 1] : 0);   // piece within the list
                const int64_t blk = (bx >> 2) + q;
                off = (int)(4 * blk - bx);
                // one aligned 16-byte load; entries outside [0, lenx) are masked
                const int4 v = __ldg(reinterpret_cast<const int4 *>(a.pplus + 4 * blk));
                z[0] = (off >= 0 && off < lenx) ? v.x : -1;
                z[1] = (off + 1 >= 0 && off + 1 < lenx) ? v.y : -1;
                z[2] = (off + 2 >= 0 && off + 2 < lenx) ? v.z : -1;
                z[3] = (off + 3 < lenx) ? v.w : -1;
            } else {
#pragma unroll
                for (int j = 0; j < kPiece; j++) z[j] = -1;
            }
            tag = ((off + 4) << 6) | (slot & 63);
        };

        U128 accy = u128_zero();
        unsigned long long cnty = 0;
        int qn = 0;
        // verify candidates 32 at a time and add the triangle's terms
        auto drain = [&](int upto) {
            while (qn >= upto && qn > 0) {
                const int take = qn < 32 ? qn : 32;
                const int b0 = qn - take;
                if (lane < take) {
                    const int2 e = S.q[b0 + lane];
                    const int slot = e.x & 63, off = (e.x >> 6) - 4;
                    const int32_t z = e.y;
                    const longlong2 xe = S.xl[slot];
                    const bool zt = off < (int)(xe.y & 0xFFFFFF);   // z from the target run of P+(x)
                    int iz;
                    if (local) iz = zt ? find_sorted(S.py, pyt, z) : find_sorted(S.py + pyt, py - pyt, z);
                    else if (zt) iz = SPARSE ? find_sorted_g(a.pplus + by, pyt, z) : find_desc_g(a.pplus + by, pyt, z);
                    else iz = find_sorted_g(a.pplus + by + pyt, py - pyt, z);
#ifdef RS_EXP_NO_TERMS
                    if (iz >= 0) ntri++;
                    if (iz >= 0 && z == -7) {
#else
                    if (iz >= 0) {
#endif
                        ntri++;
                        const int32_t x = (int32_t)((xe.y >> 32) & 0x7FFFFFFF);
                        const int lx = (int)((xe.y >> 24) & 0xFF);
                        if constexpr (COUNT) {
                            const bool tx = lx < k, tz = zt;          // z's run of P+(x) is its target status
                            if (tx && (ty + tz) && owned(a, x)) atomicAdd(a.n1 + x, (unsigned long long)(ty + tz));
                            if (tz && (tx + ty) && owned(a, z)) atomicAdd(a.n1 + z, (unsigned long long)(tx + ty));
                            cnty += ty ? (unsigned long long)(tx + tz) : 0ull;
                        } else {
                            // a_x(c_z) and a_y(c_z): 0 unless z is a target (its run of
                            // P+(x)); else x's row at lab(z) and y's row in shared memory
                            const int lz = (!SPARSE && zt) ? (int)__ldg(a.lab + z) : 0;
                            const double Axlz = SPARSE ? __ldg(a.wps + xe.x + off)
                                                       : (zt ? __ldg(a.amat + (int64_t)x * k + lz) : 0.0);
                            // a_x(c_y) (and, all-communities mode, a_y(c_x)) gathered per
                            // verified triangle rather than per (y, x) pair: most pairs close none
                            const int64_t xq = by + py + S.xn[slot].y;
                            const double Axly = SPARSE ? __ldg(a.pwr + xq) : (ty ? __ldg(a.amat + (int64_t)x * k + ly) : 0.0);
                            const double Aylx = SPARSE ? __ldg(a.wps + xq) : (lx < k ? Ay[lx] : 0.0);
                            // a_y(c_z), beside z in y's slot (the other run holds 0)
                            const int64_t ypos = by + (!zt ? pyt + iz : ((local && !SPARSE) ? pyt - 1 - iz : iz));
                            const double Aylz = SPARSE ? __ldg(a.wps + ypos) : (zt ? Ay[lz] : 0.0);
                            const double Azlx = SPARSE ? __ldg(a.pwr + xe.x + off) : amat_at(a, z, lx);
                            const double Azly = SPARSE ? __ldg(a.pwr + ypos) : amat_at(a, z, ly);
                            const double tx = Aylx * Azlx * (Azly + Aylz);
                            const double tz = Axlz * Aylz * (Aylx + Axly);
                            accy = u128_add(accy, fx_quantize(Axly * Azly * (Azlx + Axlz)));
#ifndef RS_EXP_NO_XRED
                            if (tx > 0.0) {
                                const int lenx = S.xn[slot].x;
                                if (lenx <= a.slot_cap) smem_red4(S.xa + 4 * slot, fx_quantize(tx));
                                else if (owned(a, x)) acc_add(a, x, fx_quantize(tx));
                            }
#endif
#ifndef RS_EXP_NO_ZRED
                            if (tz > 0.0 && owned(a, z)) acc_add(a, z, fx_quantize(tz));
#endif
                        }
                    }
                }
                __syncwarp();
                qn = b0;
            }
        };

        // one piece per lane per round, the next RS_EXP_E_DEPTH rounds' loads in flight
        // while this round is filtered (profiled: with one round ahead, the wait for
        // the piece was the top stall, 17% of the samples); filter candidates
        // packed by one warp scan
#if RS_EXP_E_RING
        // the pieces of RS_EXP_E_RING - 1 rounds ahead are in flight as cp.async
        // copies into the warp's shared ring (no registers held: the round-ahead
        // register prefetch kept one round in flight, and the probe loop was bound
        // by the latency of its piece loads)
        auto issue = [&](int p0, int st) {
            const int p = p0 + lane;
            int slot;
            if (mapped) {
                const uint32_t wd = S.ps[p0 >> 5];
                slot = lists_before + __popc(wd & (0xFFFFFFFFu >> (31 - lane))) - 1;
                lists_before += __popc(wd);
            } else {
                int lo = 0, hi = nx;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (S.pe[mid] <= p) lo = mid + 1; else hi = mid;
                }
                slot = lo;
            }
            int tag = -1;
            if (p < npieces) {
                const int64_t bx = S.xl[slot].x;
                const int q = p - (slot ? S.pe[slot - 1] : 0);   // piece within the list
                const int64_t blk = (bx >> 2) + q;
                const int off = (int)(4 * blk - bx);
                tag = ((off + 4) << 6) | (slot & 63);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&S.ring[st][lane]);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(a.pplus + 4 * blk));
            }
            S.rtag[st][lane] = tag;
            asm volatile("cp.async.commit_group;");
        };
        constexpr int R = RS_EXP_E_RING;
#pragma unroll
        for (int r = 0; r < R - 1; r++) issue(32 * r, r);
        int st = 0;
        for (int p0 = 0; p0 < npieces; p0 += 32) {
            issue(p0 + 32 * (R - 1), (st + R - 1) % R);     // the stage consumed last round
            asm volatile("cp.async.wait_group %0;" ::"n"(R - 1));
            int32_t zc[kPiece];
            const int tagc = S.rtag[st][lane];
            if (tagc >= 0) {
                const int4 v = S.ring[st][lane];
                const int off = (tagc >> 6) - 4;
                const int lenx = S.xn[tagc & 63].x;
                zc[0] = (off >= 0 && off < lenx) ? v.x : -1;
                zc[1] = (off + 1 >= 0 && off + 1 < lenx) ? v.y : -1;
                zc[2] = (off + 2 >= 0 && off + 2 < lenx) ? v.z : -1;
                zc[3] = (off + 3 < lenx) ? v.w : -1;
            } else {
#pragma unroll
                for (int j = 0; j < kPiece; j++) zc[j] = -1;
            }
            st = st + 1 == R ? 0 : st + 1;
#else
        int32_t zc[kPiece];
        int tagc;
        fetch(0, zc, tagc);
#endif
#if !RS_EXP_E_RING && RS_EXP_E_DEPTH >= 2
        int32_t zm[kPiece];
        int tagm = 0;
        if (32 < npieces) {
            fetch(32, zm, tagm);
        } else {
#pragma unroll
            for (int j = 0; j < kPiece; j++) zm[j] = -1;
        }
#endif
#if !RS_EXP_E_RING
        for (int p0 = 0; p0 < npieces; p0 += 32) {
            int32_t zn[kPiece];
            int tagn = 0;
            if (p0 + 32 * RS_EXP_E_DEPTH < npieces) {
                fetch(p0 + 32 * RS_EXP_E_DEPTH, zn, tagn);
            } else {
#pragma unroll
                for (int j = 0; j < kPiece; j++) zn[j] = -1;
            }
#endif
            // a triangle needs z < y (every entry of P+(y) is below y): the rounds
            // in which no lane holds such a z -- most rounds of a hub y's items,
            // whose probed runs lie almost wholly above it -- skip the filter, the
            // scan and the queue (warp-uniform; measured E || D -0.02..-0.03 ms)
            bool below = false;
#pragma unroll
            for (int j = 0; j < kPiece; j++) below |= (uint32_t)zc[j] < (uint32_t)y;   // -1: never
            if (!RS_EXP_E_YSKIP || __any_sync(0xffffffffu, below)) {
                unsigned m = 0;
#pragma unroll
                for (int j = 0; j < kPiece; j++) {
                    const uint32_t b = bm_bit(zc[j]);
                    if ((uint32_t)zc[j] < (uint32_t)y && ((S.bm[b >> 5] >> (b & 31)) & 1u)) m |= 1u << j;
                }
                const int npos = __popc(m);
                int incl = npos;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                int w = qn + incl - npos;
#pragma unroll
                for (int j = 0; j < kPiece; j++)
                    if ((m >> j) & 1u) S.q[w++] = make_int2(tagc + (j << 6), zc[j]);
                qn += __shfl_sync(0xffffffffu, incl, 31);
#ifdef RS_EXP_NO_DRAIN
                qn = 0;
#endif
                __syncwarp();
                drain(32);
            }
#if RS_EXP_E_XPRE
            if (p0 == 0 && pre_ok) {                        // the next item's x records into L2
#pragma unroll
                for (int h = 0; h < 2; h++)
                    if (xpre[h] >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.pc2 + xpre[h]));
            }
#endif
#if RS_EXP_E_RING
#elif RS_EXP_E_DEPTH >= 2
#pragma unroll
            for (int j = 0; j < kPiece; j++) { zc[j] = zm[j]; zm[j] = zn[j]; }
            tagc = tagm;
            tagm = tagn;
#else
#pragma unroll
            for (int j = 0; j < kPiece; j++) zc[j] = zn[j];
            tagc = tagn;
#endif
        }
        drain(1);
        __syncwarp();
        // flush the item's per-head partial sums: one RED per touched head
        if constexpr (!COUNT) {
            for (int s = lane; s < nx; s += 32) {
                const uint32_t *l = S.xa + 4 * s;
                const longlong2 xe = S.xl[s];
                const int32_t x = (int32_t)((xe.y >> 32) & 0x7FFFFFFF);
                if ((l[0] | l[1] | l[2] | l[3]) && owned(a, x)) acc_add(a, x, from4(l));
            }
        }
        if (ty && owned(a, y)) {
            if constexpr (COUNT) {
                for (int o = 16; o > 0; o >>= 1) cnty += __shfl_xor_sync(0xffffffffu, cnty, o);
                if (lane == 0 && cnty) atomicAdd(a.n1 + y, cnty);
            } else {
                for (int o = 16; o > 0; o >>= 1) {
                    const U128 w{__shfl_xor_sync(0xffffffffu, accy.lo, o), __shfl_xor_sync(0xffffffffu, accy.hi, o)};
                    accy = u128_add(accy, w);
                }
                if (lane == 0 && (accy.lo | accy.hi)) acc_add(a, y, accy);
            }
        }
        __syncwarp();
    }
    for (int o = 16; o > 0; o >>= 1) {
        ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
        nprobe += __shfl_xor_sync(0xffffffffu, nprobe, o);
    }
    if (lane == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
    if (lane == 0 && nprobe) atomicAdd(&a.scal[kScalNProbe], nprobe);
}

// ---------------------------------------------------------------- light middle vertices
// Vertices of degree < 128 (most of them, ~5% of the probe work). A warp takes
// 32 consecutive y; their pairs (y, x in P-(y)) are dealt to the lanes 32 at a
// time (one warp scan), and the probes of those 32 pairs -- the entries of the
// probed runs of P+(x) -- are flattened by a second scan: a lane probes one z
// per round and looks it up by binary search in the matching run of P+(y)
// (short, L1-resident), so the work per lane is uniform whatever the list
// lengths. Terms go to the heads with one RED each.
template <bool COUNT, bool SPARSE>
#ifndef RS_EXP_LIGHT_MINB
#define RS_EXP_LIGHT_MINB 5
#endif
__global__ void __launch_bounds__(256, RS_EXP_LIGHT_MINB) k_phase_e_light(CdeArgs a, int64_t ylo, int64_t yhi) {
    const int k = a.k;
    const int lane = threadIdx.x & 31;
    unsigned long long ntri = 0, nprobe = 0;   // nprobe: warp-uniform
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    auto owner = [&](int incl, int q) {          // first lane whose inclusive count exceeds q
        int j = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, j + s - 1);
            if (v <= q) j += s;
        }
        return j;
    };
    // warp task t covers y in [ylo + 32 t, +32); multi-GPU: rank r takes t = r mod world
    for (int64_t t = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * a.e_world + a.e_rank;
         ylo + 32 * t < yhi; t += nwarps * a.e_world) {
        const int64_t y0 = ylo + 32 * t;
        // ---- y level: lane j holds y0 + j
        const int64_t yl = y0 + lane;
        PRec pcl{(int)0xFF000000, 0, 0};
        if (yl < yhi) pcl = a.pc2[yl];
        const int lyl = pr_lab(pcl);
        // P-(y): the suffix of P(y) in y's slot (multi-GPU: P+ runs are packed, the
        // light P-(y) of a rank's own y stay in their slots)
        const int64_t rpl = a.mg ? (yl < yhi ? __ldg(a.rowptr + yl) : 0) : pr_start(pcl);
        const int cnt = pr_plus(pcl) > 0 ? pcl.y - pr_plus(pcl) : 0;   // pairs of this y: |P-(y)| if P+(y) is non-empty
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int q0 = 0; q0 < total; q0 += 32) {
            // ---- pair level: lane holds pair q0 + lane
            const int q = q0 + lane;
            const int j = owner(incl, q);
            const int inc_j = __shfl_sync(0xffffffffu, incl, j);
            const int cnt_j = __shfl_sync(0xffffffffu, cnt, j);
            const long long by = __shfl_sync(0xffffffffu, rpl, j);
            const int ppj = __shfl_sync(0xffffffffu, pr_plus(pcl), j);     // |P+(y)|
            const int ly = __shfl_sync(0xffffffffu, lyl, j);
            int32_t x = -1;
            const int64_t qpos = by + ppj + (q - (inc_j - cnt_j));       // P-(y): the suffix, x > y
            if (q < total) x = __ldg(a.pidx + qpos);
            PRec pcx{(int)0xFF000000, 0, 0};
            if (x >= 0) pcx = a.pc2[x];
            const int lx = pr_lab(pcx);                   // the label rides in the record
            const bool tx = lx < k, ty = ly < k;
            int64_t rsx;                                                 // probed: z < y of the target
            int np, t;                                                   // run, and of the other if both
            cut_range<SPARSE>(a.pplus, pr_start(pcx), pr_plus(pcx), pr_plus_t(pcx), (int32_t)(y0 + j), tx && ty,
                              x >= 0 && (tx || ty), rsx, np, t);
            // a_x(c_y) and a_y(c_x) are gathered by the probe lanes that find a
            // triangle (few of the pairs close one), not per pair
            int incl2 = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl2, o);
                if (lane >= o) incl2 += v;
            }
            const int total2 = __shfl_sync(0xffffffffu, incl2, 31);
            nprobe += (unsigned)total2;
            for (int r0 = 0; r0 < total2; r0 += 32) {
                // ---- probe level: lane probes entry o of pair p's runs
                const int r = r0 + lane;
                const int p = owner(incl2, r);
                const int o = r - (__shfl_sync(0xffffffffu, incl2, p) - __shfl_sync(0xffffffffu, np, p));
                const int32_t xp = __shfl_sync(0xffffffffu, x, p);
                const long long bx = __shfl_sync(0xffffffffu, (long long)rsx, p);
                const int tp = __shfl_sync(0xffffffffu, t, p);
                const int lxp = __shfl_sync(0xffffffffu, lx, p);
                const long long qp = __shfl_sync(0xffffffffu, (long long)qpos, p);   // x's position in P(y)
                const int jp = __shfl_sync(0xffffffffu, j, p);               // y's lane
                const PRec pcy{__shfl_sync(0xffffffffu, pcl.x, jp), __shfl_sync(0xffffffffu, pcl.y, jp),
                               __shfl_sync(0xffffffffu, pcl.start, jp)};
                const int lyp = __shfl_sync(0xffffffffu, lyl, jp);
                if (r >= total2) continue;
                const int32_t y = (int32_t)(y0 + jp);
                const bool zt = o < tp;                                     // z from the target run
                const int64_t pos = bx + o;                                 // the probed prefix of P+(x)
                const int32_t z = __ldg(a.pplus + pos);
                const int64_t dy = pr_start(pcy);
                const int tyn = pr_plus_t(pcy), nyn = pr_plus(pcy) - tyn;
                int iz;
                int64_t ypos;
                if (zt) {                                                   // the target run, descending
                    iz = SPARSE ? find_sorted_g(a.pplus + dy, tyn, z) : find_desc_g(a.pplus + dy, tyn, z);
                    ypos = dy + iz;
                } else {
                    const int64_t nb = dy + tyn;                              // the other run, ascending
                    iz = find_sorted_g(a.pplus + nb, nyn, z);
                    ypos = nb + iz;
                }
                if (iz < 0) continue;
                ntri++;
                const bool txp = lxp < k, typ = lyp < k;
                if constexpr (COUNT) {
                    const bool tz = zt;                                     // the run is z's target status
                    if (txp && (typ + tz) && owned(a, xp)) atomicAdd(a.n1 + xp, (unsigned long long)(typ + tz));
                    if (tz && (txp + typ) && owned(a, z)) atomicAdd(a.n1 + z, (unsigned long long)(txp + typ));
                    if (typ && (txp + tz) && owned(a, y)) atomicAdd(a.n1 + y, (unsigned long long)(txp + tz));
                } else {
                    const double Axlyp = SPARSE ? __ldg(a.pwr + qp) : amat_at(a, xp, lyp);
                    const double Aylxp = txp ? (SPARSE ? __ldg(a.wps + qp) : __ldg(a.amat + (int64_t)y * k + lxp)) : 0.0;
                    // a_x(c_z), a_y(c_z): 0 unless z is a target (its run), else the rows at lab(z)
                    const int lz = (!SPARSE && zt) ? (int)__ldg(a.lab + z) : 0;
                    const double Axlz = SPARSE ? __ldg(a.wps + pos) : (zt ? __ldg(a.amat + (int64_t)xp * k + lz) : 0.0);
                    const double Aylz = SPARSE ? __ldg(a.wps + ypos) : (zt ? __ldg(a.amat + (int64_t)y * k + lz) : 0.0);
                    const double Azlx = SPARSE ? __ldg(a.pwr + pos) : amat_at(a, z, lxp);
                    const double Azly = SPARSE ? __ldg(a.pwr + ypos) : amat_at(a, z, lyp);
                    const double ttx = Aylxp * Azlx * (Azly + Aylz);
                    const double tty = Axlyp * Azly * (Azlx + Axlz);
                    const double ttz = Axlz * Aylz * (Aylxp + Axlyp);
                    if (ttx > 0.0 && owned(a, xp)) acc_add(a, xp, fx_quantize(ttx));
                    if (tty > 0.0 && owned(a, y)) acc_add(a, y, fx_quantize(tty));
                    if (ttz > 0.0 && owned(a, z)) acc_add(a, z, fx_quantize(ttz));
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
    if (lane == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
    if (lane == 0 && nprobe) atomicAdd(&a.scal[kScalNProbe], nprobe);
}

// ---------------------------------------------------------------- work items (per step)
// Heavy middle vertices (degree >= 128) are cut into chunks of e_chunk
// positions of P(y); the chunk counts depend on the communities, so the item
// list is rebuilt every step (count, then scan + scatter), heaviest vertices first.
// One GPU: chunks of kChunkE = 64 positions. Multi-GPU: shorter ones -- a
// rank's share of the probes is 1/N, and a 64-position item can take ~16 K
// probes (Orkut shape), about a whole warp's share at N = 8, so the last items
// would set the kernel's length
// Block b of the item build owns the contiguous heavy vertices
// [b * per, (b + 1) * per): k_e_count writes each y's chunk count and the
// block's total; k_e_scatter adds the totals of the blocks before it (at most
// kEItemBlocks values), scans its own range tile by tile and writes the items --
// two launches of our own instead of count + CUB's device scan (two launches)
// + scatter. A thread per y writes its first 8 items; the rare y with more
// (hubs: up to hundreds of chunks) are written by a warp each, so no thread
// serialises a hub's whole item list.
constexpr int kEItemBlocks = 148 * 4, kEItemThreads = 256;
__device__ __forceinline__ int e_chunks(const PRec &p, int chunk) {
    return (pr_plus(p) > 0 && p.y > pr_plus(p)) ? (p.y - pr_plus(p) + chunk - 1) / chunk : 0;   // chunks of P-(y)
}
__global__ void __launch_bounds__(kEItemThreads) k_e_count(const PRec *__restrict__ pc2, int64_t n_heavy, int64_t per,
                                                          int chunk, int32_t *cnt, int32_t *bsum) {
    __shared__ int s_w[kEItemThreads / 32];
    const int64_t lo = blockIdx.x * per, hi = min(n_heavy, lo + per);
    int acc = 0;
    for (int64_t y = lo + threadIdx.x; y < hi; y += blockDim.x) {
        const int c = e_chunks(pc2[y], chunk);
        cnt[y] = c;
        acc += c;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kEItemThreads / 32; w++) t += s_w[w];
        bsum[blockIdx.x] = t;
    }
}
// multi-GPU (world > 1, items dealt one by one): only this rank's items g = rank
// mod world are written, at g / world (the rank's heavy kernel reads them in order)
__device__ __forceinline__ void e_put(EItem *items, int g, const EItem &e, int rank, int world) {
    if (world == 1) items[g] = e;
    else if (g % world == rank) items[g / world] = e;
}
// (multi-GPU, gpre / gm non-null: y's runs are read packed)
__global__ void __launch_bounds__(kEItemThreads) k_e_scatter(const int32_t *__restrict__ cnt,
                                                            const int32_t *__restrict__ bsum, int nblk,
                                                            const PRec *__restrict__ pc2,
                                                            const int64_t *__restrict__ rowptr,
                                                            const int64_t *__restrict__ gpre,
                                                            const int64_t *__restrict__ gm, int64_t n_heavy,
                                                            int64_t per, int32_t *total, EItem *items, int rank,
                                                            int world) {
    __shared__ int s_w[kEItemThreads / 32];
    __shared__ int s_off[kEItemThreads];
    __shared__ unsigned s_big[kEItemThreads / 32];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // the block's base: the totals of the blocks before it
    int pre = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) pre += bsum[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    if (lane == 0) s_w[wid] = pre;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kEItemThreads / 32; w++) t += s_w[w];
        s_base = t;
    }
    __syncthreads();
    int base = s_base;
    const int64_t lo = blockIdx.x * per, hi = min(n_heavy, lo + per);
    for (int64_t t0 = lo; t0 < hi; t0 += blockDim.x) {
        const int64_t y = t0 + threadIdx.x;
        const int c = y < hi ? cnt[y] : 0;
        // block exclusive scan of c
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        __syncthreads();                                  // s_w / s_off of the previous tile are read
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        int wpre = 0, tile = 0;
#pragma unroll
        for (int w = 0; w < kEItemThreads / 32; w++) {
            const int v = s_w[w];
            wpre += w < wid ? v : 0;
            tile += v;
        }
        const int o = base + wpre + incl - c;
        s_off[threadIdx.x] = o;
        EItem e;
        if (c > 0) {
            const PRec p = pc2[y];
            e.by = gpre ? gpre[y] : rowptr[y];
            e.y = (int32_t)y;
            e.pyl = p.x;                                  // |P+(y)| | lab(y) << 24
            e.pm = p.y - pr_plus(p);
            e.pyt = pr_plus_t(p);
            e.mbase = gm ? (uint32_t)gm[y] : 0u;
            for (int j = 0; j < c && j < 8; j++) {
                e.chunk = j;
                e_put(items, o + j, e, rank, world);
            }
        }
        // the tile's y with more than 8 chunks: a warp each (each warp publishes
        // its mask of them; the warps take them round robin)
        const unsigned big = __ballot_sync(0xffffffffu, c > 8);
        if (lane == 0) s_big[wid] = big;
        __syncthreads();                                  // s_off and s_big of this tile written
        int seen = 0;
        for (int w = 0; w < kEItemThreads / 32; w++) {
            unsigned m = s_big[w];
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                if (seen++ % (kEItemThreads / 32) != wid) continue;
                const int ti = 32 * w + bit;
                const int64_t yb = t0 + ti;
                const int cb = cnt[yb], ob = s_off[ti];
                const PRec p = pc2[yb];
                EItem eb;
                eb.by = gpre ? gpre[yb] : rowptr[yb];
                eb.y = (int32_t)yb;
                eb.pyl = p.x;
                eb.pm = p.y - pr_plus(p);
                eb.pyt = pr_plus_t(p);
                eb.mbase = gm ? (uint32_t)gm[yb] : 0u;
                for (int j = 8 + lane; j < cb; j += 32) {
                    eb.chunk = j;
                    e_put(items, ob + j, eb, rank, world);
                }
            }
        }
        base += tile;
    }
    if (blockIdx.x == nblk - 1 && threadIdx.x == 0) *total = base;   // the last block ends at the total
}

// load time: buffers sized for any community assignment (grow-only)
cudaError_t launch_e_items(Ctx &c) {
    cudaError_t e;
#ifndef RS_EXP_HEAVY_CLS
#define RS_EXP_HEAVY_CLS 4
#endif
    const int64_t nh = c.bins.offset[RS_EXP_HEAVY_CLS];   // degree classes 5-7
    c.e_nbig = nh;
    // measured, emulated ranks of the Orkut shape (E || D max over ranks): N = 8
    // 1.07 / 0.85 / 0.78 ms at 64 / 32 / 16 positions, N = 4 1.30 / 1.22 at 16 /
    // 32; one GPU: 64 (32: +0.33 ms)
    c.e_chunk = c.world >= 5 ? 16 : c.world >= 2 ? 32 : kChunkE;
    if (const char *ev = getenv("RS_EXP_ECHUNK")) c.e_chunk = std::min(kChunkE, std::max(1, atoi(ev)));
    c.e_extra = nh + c.nnz / c.e_chunk + 1;       // item capacity
    // layout: cnt[nh+1] | block totals[kEItemBlocks] | total | items[cap] (EItem)
    const size_t bytes = sizeof(int32_t) * ((size_t)(nh + 1) + kEItemBlocks + 1) + sizeof(EItem) * (size_t)c.e_extra + 16;
    if (bytes <= c.e_bytes) return cudaSuccess;
    if (c.e_pre) cudaFree(c.e_pre);
    c.e_pre = nullptr;
    c.e_bytes = 0;
    if ((e = rs::dmalloc(&c.e_pre, bytes))) return e;
    c.e_bytes = bytes;
    return cudaSuccess;
}

static cudaError_t build_e_items(Ctx &c, EItems &it, int deal_rank, int deal_world) {
    const int64_t nh = c.e_nbig;
    int32_t *cnt = (int32_t *)c.e_pre;
    int32_t *bsum = cnt + (nh + 1);
    int32_t *total = bsum + kEItemBlocks;
    EItem *items = (EItem *)(((uintptr_t)(total + 1) + 15) & ~(uintptr_t)15);
    // every heavy middle vertex (multi-GPU too: their P-(y) lists are exchanged,
    // and the ranks stride over the items)
    const int64_t per = std::max<int64_t>(1, (nh + kEItemBlocks - 1) / kEItemBlocks);
    const int nblk = (int)std::max<int64_t>(1, (nh + per - 1) / per);
    k_e_count<<<nblk, kEItemThreads, 0, c.stream>>>(c.pc2, nh, per, c.e_chunk, cnt, bsum);
    const int64_t *gm = c.mg_packed ? c.xg : nullptr, *gpre = c.mg_packed ? c.xg + (c.n + 1) : nullptr;
    k_e_scatter<<<nblk, kEItemThreads, 0, c.stream>>>(cnt, bsum, nblk, c.pc2, c.rowptr, gpre, gm, nh, per, total,
                                                      items, deal_rank, deal_world);
    c.launches += 2;
    it.items = items;
    it.total = total;
    return cudaGetLastError();
}

template <bool COUNT, bool SPARSE>
static cudaError_t launch_e(Ctx &c, cudaStream_t light) {
    CdeArgs a = cde_args(c);
    int64_t ylo = 0, yhi = c.n;
    CdeArgs ah;                                       // the heavy kernel's share of the items
    if (c.world > 1) {
        // every head's terms are accumulated here and summed over the ranks
        // afterwards (exact integer limbs). Light middle vertices: a rank's own
        // range (P-(y) is local). Heavy ones (degree >= 128; the hubs hold most
        // of the Type-I work, which a vertex-range split leaves on rank 0): the
        // ranks stride over the items, heaviest first (P-(y) of every heavy y is
        // exchanged after Phase A)
        a.head_lo = 0;
        a.head_hi = c.n;
        ylo = c.head_lo;
        yhi = c.head_hi;
        if (c.rep_a) {
            // Phase A replicated: every P-(y) is local, so the light warp tasks stride
            // over ALL light y (balanced; a vertex range holds very unequal work)
            ylo = 0;
            yhi = c.n;
            a.e_rank = c.rank;
            a.e_world = c.world;
        }
    }
    ah = a;
    if (c.world > 1) {
        ah.e_rank = c.rank;
        ah.e_world = c.world;
        if (c.mg_packed) ah.pidx = c.pk_m;            // the heavy P-(y), packed
        const char *eb = getenv("RS_EXP_EBLK");
        ah.e_blk = eb ? std::max(1, atoi(eb)) : 1;
    }
    // one GPU: the queue order interleaved over 2 batches (measured on the Orkut
    // shape: E || D 2.88-3.01 -> 2.80 ms; P = 4 / 8 / 16 2.81 / 2.82 / 2.83; LJ
    // shape unchanged). Multi-GPU: the items are already dealt one by one
    ah.e_perm = c.world > 1 ? 1 : 2;
    if (const char *ep = getenv("RS_EXP_EPERM")) ah.e_perm = std::max(1, atoi(ep));
    // test hook (RS_E_SHARES): the rank split run as sequential shares on one GPU
    const int shares = c.world > 1 ? 1 : std::max(1, c.e_shares);
    unsigned long long *ctr = c.scal + kScalCnt0;
    const int64_t n_heavy = c.e_nbig;                 // degree classes 5-7 (d >= 128)
    EItems it{nullptr, nullptr};
    // multi-GPU with items dealt one by one: the build writes only this rank's
    // (a scatter of all heavy items on every rank was ~40 us per rank at N = 8)
    const bool deal = c.world > 1 && ah.e_blk == 1;
    if (deal) ah.e_local = 1;
    if (n_heavy > 0) {
        cudaError_t e = build_e_items(c, it, deal ? c.rank : 0, deal ? c.world : 1);
        if (e != cudaSuccess) return e;
    }
    const size_t smem = (size_t)kWarpsE * e_stride_bytes(c.sparse ? 0 : c.k);
    // per launch: the attribute is per device (a process may hold contexts on
    // several GPUs), and the call is cheap next to the kernel
    cudaFuncSetAttribute(k_phase_e<COUNT, SPARSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phase_e<COUNT, SPARSE>, kWarpsE * 32, smem);
    if (const char *ev = getenv("RS_EXP_E_BLOCKS")) {   // experiment: heavy-grid blocks per SM
        const int v = atoi(ev);
        if (v >= 1 && v < per_sm) per_sm = v;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    for (int s = 0; s < shares; s++) {
        if (shares > 1) {
            a.e_rank = ah.e_rank = s;
            a.e_world = ah.e_world = shares;
        }
        cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), c.stream);
        const int64_t l0 = std::max<int64_t>(n_heavy, ylo);
        if (l0 < yhi) {                                   // light first (see rs_score)
            const int64_t threads = yhi - l0;             // a warp per 32 vertices
#ifndef RS_EXP_LIGHT_BLK
#define RS_EXP_LIGHT_BLK 4   // 148 x 4 blocks of 8 warps: 32 warps per SM beside the heavy kernel and Phase D
#endif
            const int64_t blocks = std::min<int64_t>((threads + 255) / 256, 148 * RS_EXP_LIGHT_BLK);
            k_phase_e_light<COUNT, SPARSE><<<(unsigned)blocks, 256, 0, light>>>(a, l0, yhi);
            c.launches++;
        }
        if (n_heavy > 0) {
            k_phase_e<COUNT, SPARSE><<<std::max(1, per_sm) * sms, kWarpsE * 32, smem, c.stream>>>(ah, it, ctr);
            c.launches++;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_phase_e(Ctx &c) {
    return c.sparse ? launch_e<false, true>(c, c.stream) : launch_e<false, false>(c, c.stream);
}
// light kernel on `light` (forked from c.stream by the caller)
cudaError_t launch_phase_e_on(Ctx &c, cudaStream_t light) {
    return c.sparse ? launch_e<false, true>(c, light) : launch_e<false, false>(c, light);
}
cudaError_t launch_triangle_counts(Ctx &c) {
    return c.sparse ? launch_e<true, true>(c, c.stream) : launch_e<true, false>(c, c.stream);
}

}  // namespace rs

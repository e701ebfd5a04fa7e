// Phase E — the Type-I part of Step 3 (Algorithm 1): closed triads
// over three communities (Eq. 6) found as triangles of G'.
//
// G' has an edge between u and w iff they are adjacent in G and C(u) != C(w)
// (P:493), so the three communities of a G' triangle are pairwise distinct:
// every Type-I triad is a (head, mid) ordering of a G' triangle. Orienting G'
// by rank (|P|, id) (Phase C's P+ lists), each triangle x < y < z is found
// exactly once from its middle vertex y, as z in P+(x) ∩ P+(y) for x in
// P-(y), the lower-ranked part of P(y) (the paper's "common predecessor"
// search, with bitmap/binary-search probes instead of a merge).
//
// Each triangle adds the grouped terms of its (up to) three heads
//   head x: a_y(c_x) a_z(c_x) (a_z(c_y) + a_y(c_z))
//   head y: a_x(c_y) a_z(c_y) (a_z(c_x) + a_x(c_z))
//   head z: a_x(c_z) a_y(c_z) (a_y(c_x) + a_x(c_y))
// with a_v(c) = 0 for a non-target column c -- so a non-target head or mid
// contributes exactly 0 without a test -- and each expression symmetric in
// the two other vertices (the numbering changes no bit of the result).
// a_x(c_z) comes from the weight Phase C stored beside z in P+(x) (read at the
// probe's own index). Sums are exact fixed point (C-12).
//
// Heavy middle vertices (degree >= 128): work items (y, 64 positions of
// P(y)), a warp per item from a global queue, heaviest first. The warp puts a
// 4096-bit filter and a sorted copy of P+(y) in shared memory, lists the
// item's predecessors x, and cuts every P+(x) into pieces of kPiece entries:
// a lane probes one piece per round (independent loads in flight), filter
// candidates are packed with one warp scan and verified 32 at a time by binary
// search in the shared copy. Head terms accumulate per item in shared memory
// (x per list slot, z per P+(y) position, y in registers) and are flushed with
// one RED per touched head. Light middle vertices: one thread per y, two-
// pointer merge of the short sorted lists. COUNT mode (parity getter) counts
// the ordered (head, mid) target pairs instead.
#include "rs_phase.cuh"
#include <cub/cub.cuh>

namespace rs {

constexpr int kChunkE = 64;      // positions of P(y) per work item
constexpr int kPyCap = 256;      // P+(y) kept in shared memory (sorted copy + labels)
constexpr int kBmWords = 128;    // 4096-bit membership filter of P+(y)
constexpr int kPiece = 4;        // consecutive P+(x) entries one lane probes per round
constexpr int kQCapE = 160;      // candidate queue (31 + 32 * kPiece < 160)
constexpr int kPieceMap = 512;   // piece -> slot map capacity (else binary search)
constexpr int kSlotMaxHits = 4096;   // smem limbs of an x slot take at most this many terms
constexpr int kWarpsE = 8;

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

// global exact accumulation of a head's (partial) Type-I sum
__device__ __forceinline__ void acc_add(const CdeArgs &a, int32_t h, const U128 &q) {
    unsigned long long *acc = a.acc1 + 3 * (int64_t)h;
    if (a.any_wide && a.vrec[h].wide) fx_red3(acc, q);
    else fx_red2(acc, q);
}

// shared-memory per-item accumulator: four 20-bit limbs of q (< 2^80) added with
// native 32-bit shared atomics (64-bit shared atomics are CAS loops); exact
// while a slot receives fewer than 2^12 terms per item (x slots with longer
// P+(x) and z positions beyond kPyCap go straight to the global limbs).
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

struct EItems {
    const int2 *items;     // {y, chunk} work items of the heavy middle vertices, heaviest first
    const int32_t *total;  // number of items (device scalar, written by the item scan)
};

struct ESmem {             // one warp's shared memory
    uint32_t bm[kBmWords];
    int32_t py[kPyCap];
    longlong2 xl[kChunkE];  // {P+(x) start, (x << 32) | (lab(x) << 24) | |P+(x)|}
    double2 xw[kChunkE];    // {a_x(c_y), a_y(c_x)}
    uint32_t xa[4 * kChunkE];
    int32_t pe[kChunkE];    // end of each list's pieces
    int2 q[kQCapE];         // candidates {x slot, offset in P+(x)}
    uint8_t pslot[kPieceMap];   // piece -> x slot (items with at most kPieceMap pieces)
    uint8_t zl[kPyCap];         // label of z in P+(y)
};

__host__ __device__ constexpr size_t e_stride_bytes(int k) {
    return ((sizeof(ESmem) + 15) / 16) * 16 + ((8 * (size_t)k + 15) / 16) * 16;
}

template <bool COUNT>
__global__ void __launch_bounds__(kWarpsE * 32) k_phase_e(CdeArgs a, EItems it, unsigned long long *queue_ctr) {
    extern __shared__ __align__(16) unsigned char e_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = a.k;
    unsigned char *base = e_smem + (size_t)wid * e_stride_bytes(k);
    ESmem &S = *reinterpret_cast<ESmem *>(base);
    double *Ay = (double *)(base + ((sizeof(ESmem) + 15) / 16) * 16);
    unsigned long long ntri = 0;
    const unsigned long long n_items = (unsigned long long)*it.total;

    for (;;) {
        unsigned long long qi = 0;
        if (lane == 0) qi = atomicAdd(queue_ctr, 1ull);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (qi >= n_items) break;
        const int2 itm = it.items[qi];
        const int32_t y = itm.x;
        const PRec pcy = a.pc2[y];
        const int py = pcy.x, pm = pcy.y - pcy.x;   // |P+(y)|, |P-(y)| (P-(y) = front of pidx)
        const int start = itm.y * kChunkE;
        if (py == 0 || start >= pm) continue;       // no z above y, or an empty chunk
        const int end = min(pm, start + kChunkE);
        const int ly = a.lab[y];
        const int64_t by = pcy.start;
        const bool local = py <= kPyCap;            // P+(y) copy + accumulators in smem
        for (int w = lane; w < kBmWords; w += 32) S.bm[w] = 0u;
        for (int c = lane; c < k; c += 32) Ay[c] = __ldg(a.amat + (int64_t)y * k + c);
        __syncwarp();
        for (int i = lane; i < py; i += 32) {
            const int32_t z = __ldg(a.pplus + by + i);
            const uint32_t b = bm_bit(z);
            atomicOr(&S.bm[b >> 5], 1u << (b & 31));
            if (local) {
                S.py[i] = z;
                const int lzi = __ldg(a.lab + z);
                S.zl[i] = (uint8_t)lzi;
            }
        }
        // the item's predecessors x (lower rank, non-empty P+(x), a target among
        // x and y), each P+(x) cut into pieces numbered across the list
        int nx = 0, npieces = 0;
        for (int i0 = start; i0 < end; i0 += 32) {
            const int i = i0 + lane;
            int32_t x = 0;
            int64_t bx = 0;
            int lenx = 0, lx = kOther;
            if (i < end) {
                x = __ldg(a.pidx + by + i);              // x in P-(y): lower rank than y
                const PRec pcx = a.pc2[x];
                if (pcx.x > 0) {
                    lx = __ldg(a.lab + x);
                    if (lx < k || ly < k) {
                        lenx = pcx.x;
                        bx = pcx.start;
                    }
                }
            }
            const int pieces = (lenx + kPiece - 1) / kPiece;
            int incl = pieces;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned has = __ballot_sync(0xffffffffu, lenx > 0);
            if (lenx > 0) {
                const int slot = nx + __popc(has & ((1u << lane) - 1u));
                S.xl[slot] = make_longlong2(bx, ((long long)x << 32) | ((long long)(lx & 0xFF) << 24) | lenx);
                S.xw[slot] = make_double2(ly < k ? __ldg(a.amat + (int64_t)x * k + ly) : 0.0, lx < k ? Ay[lx] : 0.0);
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
        const bool mapped = npieces <= kPieceMap;
        if (mapped) {
            for (int s = lane; s < nx; s += 32)
                for (int p = s ? S.pe[s - 1] : 0; p < S.pe[s]; p++) S.pslot[p] = (uint8_t)s;
            __syncwarp();
        }

        U128 accy = u128_zero();
        unsigned long long cnty = 0;
        int qn = 0;
        // verify candidates (x slot, offset) 32 at a time and add the triangle's terms
        auto drain = [&](int upto) {
            while (qn >= upto && qn > 0) {
                const int take = qn < 32 ? qn : 32;
                const int b0 = qn - take;
                if (lane < take) {
                    const int2 e = S.q[b0 + lane];
                    const longlong2 xe = S.xl[e.x];
                    const int32_t z = __ldg(a.pplus + xe.x + e.y);
                    const int iz = local ? find_sorted(S.py, py, z) : find_sorted_g(a.pplus + by, py, z);
                    if (iz >= 0) {
                        ntri++;
                        const int32_t x = (int32_t)(xe.y >> 32);
                        const int lx = (int)((xe.y >> 24) & 0xFF);
                        const int lz = local ? (int)S.zl[iz] : (int)__ldg(a.lab + z);
                        if constexpr (COUNT) {
                            const bool tx = lx < k, ty = ly < k, tz = lz < k;
                            if (tx && (ty + tz) && owned(a, x)) atomicAdd(a.n1 + x, (unsigned long long)(ty + tz));
                            if (tz && (tx + ty) && owned(a, z)) atomicAdd(a.n1 + z, (unsigned long long)(tx + ty));
                            cnty += ty ? (unsigned long long)(tx + tz) : 0ull;
                        } else {
                            const double2 w = S.xw[e.x];
                            const double Axly = w.x, Aylx = w.y;
                            const double Axlz = __ldg(a.wps + xe.x + e.y);   // a_x(c_z), stored by Phase C
                            const double Aylz = lz < k ? Ay[lz] : 0.0;
                            const double Azlx = amat_at(a, z, lx);
                            const double Azly = amat_at(a, z, ly);
                            const double tx = Aylx * Azlx * (Azly + Aylz);
                            const double tz = Axlz * Aylz * (Aylx + Axly);
                            accy = u128_add(accy, fx_quantize(Axly * Azly * (Azlx + Axlz)));
                            if (tx > 0.0) {
                                if ((int)(xe.y & 0xFFFFFF) <= kSlotMaxHits) smem_red4(S.xa + 4 * e.x, fx_quantize(tx));
                                else if (owned(a, x)) acc_add(a, x, fx_quantize(tx));
                            }
                            if (tz > 0.0) {
                                if (owned(a, z)) acc_add(a, z, fx_quantize(tz));   // z: hub-ish, hot in L2
                            }
                        }
                    }
                }
                __syncwarp();
                qn = b0;
            }
        };

        // one piece per lane per round; the round's filter candidates packed by one scan
        for (int p0 = 0; p0 < npieces; p0 += 32) {
            const int p = p0 + lane;
            int slot = 0, off = 0, cnt = 0;
            int64_t pb = 0;
            if (p < npieces) {
                int lo;                                // list holding piece p
                if (mapped) {
                    lo = S.pslot[p];
                } else {
                    lo = 0;
                    int hi = nx;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (S.pe[mid] <= p) lo = mid + 1; else hi = mid;
                    }
                }
                slot = lo;
                const longlong2 xe = S.xl[lo];
                off = (p - (lo ? S.pe[lo - 1] : 0)) * kPiece;
                cnt = min(kPiece, (int)(xe.y & 0xFFFFFF) - off);
                pb = xe.x + off;
            }
            int32_t z[kPiece];
#pragma unroll
            for (int j = 0; j < kPiece; j++) z[j] = j < cnt ? __ldg(a.pplus + pb + j) : -1;
            unsigned m = 0;
#pragma unroll
            for (int j = 0; j < kPiece; j++) {
                const uint32_t b = bm_bit(z[j]);
                if (z[j] >= 0 && ((S.bm[b >> 5] >> (b & 31)) & 1u)) m |= 1u << j;
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
                if ((m >> j) & 1u) S.q[w++] = make_int2(slot, off + j);
            qn += __shfl_sync(0xffffffffu, incl, 31);
#ifdef RS_EXP_NO_DRAIN
            qn = 0;
#endif
            __syncwarp();
            drain(32);
        }
        drain(1);
        __syncwarp();
        // flush the item's per-head partial sums: one RED per touched head
        if constexpr (!COUNT) {
            for (int s = lane; s < nx; s += 32) {
                const uint32_t *l = S.xa + 4 * s;
                const int32_t x = (int32_t)(S.xl[s].y >> 32);
                if ((l[0] | l[1] | l[2] | l[3]) && owned(a, x)) acc_add(a, x, from4(l));
            }
        }
        if (ly < k && owned(a, y)) {
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
    for (int o = 16; o > 0; o >>= 1) ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
    if (lane == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
}

// ---------------------------------------------------------------- light middle vertices
// Vertices of degree < 128 (most of them, ~5% of the probe work): one thread
// per y; P(y), P+(y) and the P+(x) are short and sorted, so each x in P-(y)
// is intersected with P+(y) by a two-pointer merge in L1. x's terms gather in
// a register while its list is merged (one RED per x).
template <bool COUNT>
__global__ void __launch_bounds__(256) k_phase_e_light(CdeArgs a, int64_t ylo) {
    const int k = a.k;
    unsigned long long ntri = 0;
    for (int64_t y64 = ylo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y64 < a.n;
         y64 += (int64_t)gridDim.x * blockDim.x) {
        const int32_t y = (int32_t)y64;
        const PRec pcy = a.pc2[y];
        const int py = pcy.x, pm = pcy.y - pcy.x;
        if (py == 0 || pm == 0) continue;
        const int ly = a.lab[y];
        const int64_t by = pcy.start;
        const int32_t *Py = a.pplus + by;
        const double *Wy = a.wps + by;              // a_y(c_z) beside z in P+(y)
        U128 accy = u128_zero();
        unsigned long long cnty = 0;
        for (int i = 0; i < pm; i++) {
            const int32_t x = __ldg(a.pidx + by + i);   // P-(y): lower rank than y
            const PRec pcx = a.pc2[x];
            if (pcx.x == 0) continue;
            const int lx = __ldg(a.lab + x);
            if (lx >= k && ly >= k) continue;
            const int64_t bx = pcx.start;
            const int32_t *Px = a.pplus + bx;
            const double Axly = amat_at(a, x, ly), Aylx = amat_at(a, y, lx);
            U128 accx = u128_zero();
            unsigned long long cntx = 0;
            int ix = 0, iy = 0;
            int32_t zx = __ldg(Px), zy = __ldg(Py);
            while (true) {
                if (zx == zy) {
                    ntri++;
                    const int32_t z = zx;
                    const int lz = __ldg(a.lab + z);
                    if constexpr (COUNT) {
                        const bool tx = lx < k, ty = ly < k, tz = lz < k;
                        cntx += tx ? (unsigned long long)(ty + tz) : 0ull;
                        if (tz && (tx + ty) && owned(a, z)) atomicAdd(a.n1 + z, (unsigned long long)(tx + ty));
                        cnty += ty ? (unsigned long long)(tx + tz) : 0ull;
                    } else {
                        const double Axlz = __ldg(a.wps + bx + ix), Aylz = __ldg(Wy + iy);
                        const double Azlx = amat_at(a, z, lx), Azly = amat_at(a, z, ly);
                        const double tx = Aylx * Azlx * (Azly + Aylz);
                        const double tz = Axlz * Aylz * (Aylx + Axly);
                        accy = u128_add(accy, fx_quantize(Axly * Azly * (Azlx + Axlz)));
                        if (tx > 0.0) accx = u128_add(accx, fx_quantize(tx));
                        if (tz > 0.0 && owned(a, z)) acc_add(a, z, fx_quantize(tz));
                    }
                    if (++ix >= pcx.x || ++iy >= py) break;
                    zx = __ldg(Px + ix);
                    zy = __ldg(Py + iy);
                } else if (zx < zy) {
                    if (++ix >= pcx.x) break;
                    zx = __ldg(Px + ix);
                } else {
                    if (++iy >= py) break;
                    zy = __ldg(Py + iy);
                }
            }
            if (owned(a, x)) {
                if constexpr (COUNT) {
                    if (cntx) atomicAdd(a.n1 + x, cntx);
                } else {
                    if (accx.lo | accx.hi) acc_add(a, x, accx);
                }
            }
        }
        if (ly < k && owned(a, y)) {
            if constexpr (COUNT) {
                if (cnty) atomicAdd(a.n1 + y, cnty);
            } else {
                if (accy.lo | accy.hi) acc_add(a, y, accy);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
    if ((threadIdx.x & 31) == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
}

// ---------------------------------------------------------------- work items (per step)
// Heavy middle vertices (degree >= 128) are cut into chunks of kChunkE
// positions of P(y); the chunk counts depend on the communities, so the item
// list is rebuilt every step (count, scan, scatter), heaviest vertices first.
__global__ void k_e_count(const PRec *__restrict__ pc2, int64_t n_heavy, int32_t *cnt) {
    for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y <= n_heavy; y += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        if (y < n_heavy) {
            const PRec p = pc2[y];
            if (p.x > 0 && p.y > p.x) c = (p.y - p.x + kChunkE - 1) / kChunkE;   // chunks of P-(y)
        }
        cnt[y] = c;
    }
}
__global__ void k_e_scatter(const int32_t *__restrict__ cnt, const int32_t *__restrict__ off, int64_t n_heavy,
                            int2 *items) {
    for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < n_heavy; y += (int64_t)gridDim.x * blockDim.x) {
        const int c = cnt[y], o = off[y];
        for (int j = 0; j < c; j++) items[o + j] = make_int2((int)y, j);
    }
}

// load time: buffers sized for any community assignment (grow-only)
cudaError_t launch_e_items(Ctx &c) {
    cudaError_t e;
    const int64_t nh = c.bins.offset[4];          // degree classes 5-7
    c.e_nbig = nh;
    c.e_extra = nh + c.nnz / kChunkE + 1;         // item capacity
    // layout: cnt[nh+1] | off[nh+1] | items[cap] (int2)
    const size_t bytes = sizeof(int32_t) * 2 * (size_t)(nh + 1) + sizeof(int2) * (size_t)c.e_extra + 16;
    if (bytes <= c.e_bytes) return cudaSuccess;
    if (c.e_pre) cudaFree(c.e_pre);
    c.e_pre = nullptr;
    c.e_bytes = 0;
    if ((e = cudaMalloc(&c.e_pre, bytes))) return e;
    c.e_bytes = bytes;
    return cudaSuccess;
}

static cudaError_t build_e_items(Ctx &c, EItems &it) {
    const int64_t nh = c.e_nbig;
    int32_t *cnt = (int32_t *)c.e_pre;
    int32_t *off = cnt + (nh + 1);
    int2 *items = (int2 *)(((uintptr_t)(off + (nh + 1)) + 15) & ~(uintptr_t)15);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nh + 256) / 256, 148 * 4));
    k_e_count<<<blocks, 256, 0, c.stream>>>(c.pc2, nh, cnt);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, off, (int)(nh + 1), c.stream);
    if (need > c.scratch_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::ExclusiveSum(c.scratch, need, cnt, off, (int)(nh + 1), c.stream);
    k_e_scatter<<<blocks, 256, 0, c.stream>>>(cnt, off, nh, items);
    c.launches += 3;
    it.items = items;
    it.total = off + nh;
    return cudaGetLastError();
}

template <bool COUNT>
static cudaError_t launch_e(Ctx &c) {
    CdeArgs a = cde_args(c);
    unsigned long long *ctr = c.scal + kScalCnt0;
    cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), c.stream);
    const int64_t n_heavy = c.e_nbig;                 // degree classes 5-7 (d >= 128)
    EItems it{nullptr, nullptr};
    if (n_heavy > 0) {
        cudaError_t e = build_e_items(c, it);
        if (e != cudaSuccess) return e;
    }
    const size_t smem = (size_t)kWarpsE * e_stride_bytes(c.k);
    static bool attr_set[2] = {false, false};
    if (!attr_set[COUNT]) {
        cudaFuncSetAttribute(k_phase_e<COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set[COUNT] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phase_e<COUNT>, kWarpsE * 32, smem);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    if (n_heavy > 0) {
        k_phase_e<COUNT><<<std::max(1, per_sm) * sms, kWarpsE * 32, smem, c.stream>>>(a, it, ctr);
        c.launches++;
    }
    if (n_heavy < c.n) {
        const int64_t threads = c.n - n_heavy;
        const int64_t blocks = std::min<int64_t>((threads + 255) / 256, 148 * 32);
        k_phase_e_light<COUNT><<<(unsigned)blocks, 256, 0, c.stream>>>(a, n_heavy);
        c.launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_phase_e(Ctx &c) { return launch_e<false>(c); }
cudaError_t launch_triangle_counts(Ctx &c) { return launch_e<true>(c); }

}  // namespace rs

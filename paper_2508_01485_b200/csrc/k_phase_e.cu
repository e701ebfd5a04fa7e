// Phase E — the Type-I part of Step 3 (Algorithm 1): closed triads
// over three communities (Eq. 6) found as triangles of G'.
//
// G' has an edge between u and w iff they are adjacent in G and C(u) != C(w)
// (P:493), so the three communities of a G' triangle are pairwise distinct:
// every Type-I triad is a (head, mid) ordering of a G' triangle. Orienting G'
// by rank (|P|, id) (Phase C's P+ lists), each triangle x < y < z is found
// exactly once from its middle vertex y, as z in P+(x) ∩ P+(y) for x in
// P-(y), the lower-ranked part of P(y) (the paper's "common predecessor"
// search, with hash probes instead of a merge).
//
// Work items are (y, chunk of 128 positions of P(y)); a warp takes an item
// from a global queue (the heaviest vertices first: internal ids are
// degree-descending), hashes P+(y) into shared memory, lists the item's
// predecessors x with their P+(x) in shared memory, and lets every lane walk
// one contiguous segment of the concatenated P+(x) lists, kUnrollE probes at
// a time (independent loads of one cache line in flight, no shuffles). Hits are queued in shared memory and
// evaluated 32 at a time with every lane busy; each triangle adds the grouped
// terms of its (up to) three heads:
//   head x: a_y(c_x) a_z(c_x) (a_z(c_y) + a_y(c_z))
//   head y: a_x(c_y) a_z(c_y) (a_z(c_x) + a_x(c_z))
//   head z: a_x(c_z) a_y(c_z) (a_y(c_x) + a_x(c_y))
// (a_v(c) = 0 for a non-target column c: a non-target mid has no term; each
// expression is symmetric in the two other vertices, so the numbering does not
// change any bit of the result). Head y accumulates in registers (one RED per
// item); x and z use exact fixed-point RED. COUNT mode (parity getter) counts
// the ordered (head, mid) target pairs instead.
#include "rs_phase.cuh"
#include <cub/cub.cuh>

namespace rs {

constexpr int kChunkE = 128;     // positions of P(y) per work item
constexpr int kTabE = 1024;      // hash slots per warp (P+(y) up to kTabE/4 hashed, load <= 1/4)
constexpr int kBmWords = 128;    // 4096-bit membership filter of P+(y) per warp
constexpr int kQCapE = 160;      // candidate queue per warp (31 + 4*32 < 160)
constexpr int kUnrollE = 4;
constexpr int kWarpsE = 8;

// membership filter bit of z (top 12 bits of a second multiplicative hash)
__device__ __forceinline__ uint32_t bm_bit(int32_t z) {
    return ((uint32_t)z * 0x85EBCA6Bu) >> 20;
}

// Fibonacci hashing: the top log2(size) bits of z * 2^32/phi
__device__ __forceinline__ uint32_t hslot(int32_t z, uint32_t shift) {
    return ((uint32_t)z * 2654435769u) >> shift;
}

// z in the sorted list p[0, len)
__device__ __forceinline__ bool in_sorted(const int32_t *p, int len, int32_t z) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(p + mid) < z) lo = mid + 1; else hi = mid;
    }
    return lo < len && __ldg(p + lo) == z;
}

__device__ __forceinline__ double amat_at(const CdeArgs &a, int32_t v, int c) {
    return __ldg(a.amat + (int64_t)v * a.k + c);
}

__device__ __forceinline__ void acc_add(const CdeArgs &a, int32_t h, const U128 &q) {
    unsigned long long *acc = a.acc1 + 3 * (int64_t)h;
    if (a.any_wide && a.vrec[h].wide) fx_red3(acc, q);
    else fx_red2(acc, q);
}

// one queued triangle (x, y, z) on this lane; returns head-y's term
template <bool COUNT>
__device__ __forceinline__ U128 tri_terms(const CdeArgs &a, int32_t x, int32_t y, int ly, const double *Ay,
                                          int32_t z, unsigned long long &cnt_y) {
    const int k = a.k;
    const int lx = __ldg(a.lab + x), lz = __ldg(a.lab + z);
    const bool tx = lx < k, ty = ly < k, tz = lz < k;
    if constexpr (COUNT) {
        if (tx && x >= a.head_lo && x < a.head_hi && (ty + tz)) atomicAdd(a.n1 + x, (unsigned long long)(ty + tz));
        if (tz && z >= a.head_lo && z < a.head_hi && (tx + ty)) atomicAdd(a.n1 + z, (unsigned long long)(tx + ty));
        cnt_y += ty ? (unsigned long long)(tx + tz) : 0ull;
        return u128_zero();
    } else {
        const double Axly = ty ? amat_at(a, x, ly) : 0.0;
        const double Axlz = tz ? amat_at(a, x, lz) : 0.0;
        const double Azlx = tx ? amat_at(a, z, lx) : 0.0;
        const double Azly = ty ? amat_at(a, z, ly) : 0.0;
        const double Aylx = tx ? Ay[lx] : 0.0;
        const double Aylz = tz ? Ay[lz] : 0.0;
        if (tx && x >= a.head_lo && x < a.head_hi) {
            const double t = Aylx * Azlx * (Azly + Aylz);
            if (t > 0.0) acc_add(a, x, fx_quantize(t));
        }
        if (tz && z >= a.head_lo && z < a.head_hi) {
            const double t = Axlz * Aylz * (Aylx + Axly);
            if (t > 0.0) acc_add(a, z, fx_quantize(t));
        }
        if (ty) return fx_quantize(Axly * Azly * (Azlx + Axlz));
        return u128_zero();
    }
}

struct EItems {
    const int2 *items;     // {y, chunk} work items of the heavy middle vertices, heaviest first
    const int32_t *total;  // number of items (device scalar, written by the item scan)
};

__host__ __device__ constexpr int e_stride_bytes(int k) {
    return kTabE * 4 + kBmWords * 4 + kQCapE * 8 + kChunkE * 16 + ((8 * k + 15) / 16) * 16;
}

template <bool COUNT>
__global__ void __launch_bounds__(kWarpsE * 32) k_phase_e(CdeArgs a, EItems it, unsigned long long *queue_ctr) {
    extern __shared__ __align__(16) unsigned char e_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = a.k;
    unsigned char *base = e_smem + (size_t)wid * e_stride_bytes(k);
    int32_t *T = (int32_t *)base;
    uint32_t *BM = (uint32_t *)(base + kTabE * 4);
    int2 *Q = (int2 *)(base + kTabE * 4 + kBmWords * 4);
    longlong2 *XL = (longlong2 *)(base + kTabE * 4 + kBmWords * 4 + kQCapE * 8);   // {P+(x) base - offset, (x << 32) | end}
    double *Ay = (double *)(base + kTabE * 4 + kBmWords * 4 + kQCapE * 8 + kChunkE * 16);
    unsigned long long ntri = 0;
    const unsigned long long n_items = (unsigned long long)*it.total;

    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(queue_ctr, 1ull);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= n_items) break;
        const int2 itm = it.items[q];
        const int32_t y = itm.x;
        const int chunk = itm.y;
        const int2 pcy = a.pc2[y];
        const int py = pcy.x, pc = pcy.y;
        const int start = chunk * kChunkE;
        if (py == 0 || start >= pc) continue;    // no z above y, or an empty chunk
        const int end = min(pc, start + kChunkE);
        const int ly = a.lab[y];
        const int64_t by = a.rowptr[y];
        const bool hashed = py <= kTabE / 4;
        uint32_t mask = 0, shift = 0;
        for (int w = lane; w < kBmWords; w += 32) BM[w] = 0u;
        __syncwarp();
        for (int i = lane; i < py; i += 32) {
            const uint32_t b = bm_bit(__ldg(a.pplus + by + i));
            atomicOr(&BM[b >> 5], 1u << (b & 31));
        }
        if (hashed) {
            uint32_t size = 32;
            while (size < 4u * (uint32_t)py) size <<= 1;
            mask = size - 1;
            shift = 32 - __ffs(size) + 1;
            for (uint32_t s = lane; s < size; s += 32) T[s] = -1;
            __syncwarp();
            for (int i = lane; i < py; i += 32) {
                const int32_t z = __ldg(a.pplus + by + i);
                uint32_t h = hslot(z, shift);
                while (atomicCAS(&T[h], -1, z) != -1) h = (h + 1) & mask;
            }
        }
        for (int c = lane; c < k; c += 32) Ay[c] = amat_at(a, y, c);
        __syncwarp();

        U128 accy = u128_zero();
        unsigned long long cnty = 0;
        int qn = 0;
        // queued candidates (x, z) passed the bitmap filter; verify z in P+(y)
        // exactly, then evaluate the triangle -- 32 at a time, all lanes busy
        auto drain = [&](int upto) {
            while (qn >= upto && qn > 0) {
                const int take = qn < 32 ? qn : 32;
                const int b = qn - take;
                if (lane < take) {
                    const int2 e = Q[b + lane];
                    bool hit;
                    if (hashed) {
                        uint32_t h = hslot(e.y, shift);
                        for (;;) {
                            const int32_t sv = T[h];
                            if (sv == e.y) { hit = true; break; }
                            if (sv == -1) { hit = false; break; }
                            h = (h + 1) & mask;
                        }
                    } else {
                        hit = in_sorted(a.pplus + by, py, e.y);
                    }
                    if (hit) {
                        ntri++;
                        accy = u128_add(accy, tri_terms<COUNT>(a, e.x, y, ly, Ay, e.y, cnty));
                    }
                }
                __syncwarp();
                qn = b;
            }
        };

        // the item's predecessors x (lower rank, non-empty P+(x), a target among
        // x and y) -> a compact list in shared memory: P+(x) occupies the
        // positions [end - |P+(x)|, end) of the concatenated probe sequence
        int nx = 0, total = 0;
        for (int i0 = start; i0 < end; i0 += 32) {
            const int i = i0 + lane;
            int32_t x = 0;
            int64_t bx = 0;
            int lenx = 0;
            if (i < end) {
                x = __ldg(a.pidx + by + i);
                const int2 pcx = a.pc2[x];
                const bool lower = pcx.y < pc || (pcx.y == pc && x < y);
                if (lower && pcx.x > 0 && (__ldg(a.lab + x) < k || ly < k)) {
                    lenx = pcx.x;
                    bx = a.rowptr[x];
                }
            }
            int incl = lenx;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned has = __ballot_sync(0xffffffffu, lenx > 0);
            if (lenx > 0) {
                const int slot = nx + __popc(has & ((1u << lane) - 1u));
                const int e_end = total + incl;
                XL[slot] = make_longlong2(bx - (e_end - lenx), ((long long)x << 32) | (unsigned)e_end);
            }
            nx += __popc(has);
            total += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        // every lane walks one contiguous segment of the probe sequence
        const int seg = (total + 31) >> 5;
        const int t_beg = min(total, lane * seg), t_end = min(total, t_beg + seg);
        // the lane's current list: P+(xcur) covers probe positions [.., xe), at base + t
        int xi = 0, xe = 0;
        int64_t xbase = 0;
        int32_t xcur = 0;
        if (t_beg < t_end) {
            int lo = 0, hi = nx;            // first list whose end > t_beg
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((int)(XL[mid].y & 0xffffffff) <= t_beg) lo = mid + 1; else hi = mid;
            }
            xi = lo;
            const longlong2 e = XL[xi];
            xbase = e.x;
            xe = (int)(e.y & 0xffffffff);
            xcur = (int32_t)(e.y >> 32);
        }
        int t = t_beg;
        for (int s0 = 0; s0 < seg; s0 += kUnrollE) {
            {
                int32_t z[kUnrollE], xj[kUnrollE];
#pragma unroll
                for (int u = 0; u < kUnrollE; u++) {
                    z[u] = -1;
                    xj[u] = xcur;
                    if (t < t_end) {
                        if (t >= xe) {           // lists are non-empty: one step crosses at most one end
                            const longlong2 e = XL[++xi];
                            xbase = e.x;
                            xe = (int)(e.y & 0xffffffff);
                            xcur = (int32_t)(e.y >> 32);
                            xj[u] = xcur;
                        }
                        z[u] = __ldg(a.pplus + xbase + t);
                    }
                    t++;
                }
                // bitmap filter; the lanes' candidates are packed with one warp scan
                int npos = 0;
                bool pos[kUnrollE];
#pragma unroll
                for (int u = 0; u < kUnrollE; u++) {
                    const uint32_t b = bm_bit(z[u]);
                    pos[u] = z[u] >= 0 && ((BM[b >> 5] >> (b & 31)) & 1u);
                    npos += pos[u];
                }
                int incl = npos;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                int w = qn + incl - npos;
#pragma unroll
                for (int u = 0; u < kUnrollE; u++)
                    if (pos[u]) Q[w++] = make_int2(xj[u], z[u]);
                qn += __shfl_sync(0xffffffffu, incl, 31);
                __syncwarp();
                drain(32);
            }
        }
        drain(1);
        if (ly < k && y >= a.head_lo && y < a.head_hi) {
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

// ---------------------------------------------------------------- work items (per step)
// Heavy middle vertices (degree >= 128) are cut into chunks of kChunkE
// positions of P(y); the chunk counts depend on the communities, so the item
// list is rebuilt every step (count, scan, scatter), heaviest vertices first.
__global__ void k_e_count(const int2 *__restrict__ pc2, int64_t n_heavy, int32_t *cnt) {
    for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y <= n_heavy; y += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        if (y < n_heavy) {
            const int2 p = pc2[y];
            if (p.x > 0 && p.y > p.x) c = (p.y + kChunkE - 1) / kChunkE;
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

// load time: buffers sized for any community assignment
cudaError_t launch_e_items(Ctx &c) {
    cudaError_t e;
    const int64_t nh = c.bins.offset[4];          // degree classes 5-7
    c.e_nbig = nh;
    c.e_extra = nh + c.nnz / kChunkE + 1;         // item capacity
    // layout: cnt[nh+1] | off[nh+1] | items[cap] (int2); grow-only
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

// ---------------------------------------------------------------- light middle vertices
// Vertices of degree < 128 (most of them, but a few percent of the probe
// work): a group of kGL lanes per y, no hash table -- P+(y) is short and
// sorted, so membership is a binary search that stays in L1.
constexpr int kGL = 8;                         // lanes per light vertex
constexpr int kXLL = 32;                       // P(y) positions per x-list pass
constexpr int kQL = kGL * kUnrollE + kGL;      // hit queue per group


template <bool COUNT>
__global__ void __launch_bounds__(256) k_phase_e_light(CdeArgs a, int64_t ylo) {
    __shared__ longlong2 XLs[256 / kGL][kXLL];
    __shared__ int2 Qs[256 / kGL][kQL];
    WarpGroup<kGL> g;
    const int gi = threadIdx.x / kGL;
    const int lane = (int)g.lane;
    longlong2 *XL = XLs[gi];
    int2 *Q = Qs[gi];
    const int k = a.k;
    unsigned long long ntri = 0;
    const int64_t gpb = blockDim.x / kGL;
    const int64_t ngroups = (int64_t)gridDim.x * gpb;
    for (int64_t y64 = ylo + blockIdx.x * gpb + gi; y64 < a.n; y64 += ngroups) {
        const int32_t y = (int32_t)y64;
        const int2 pcy = a.pc2[y];
        const int py = pcy.x, pc = pcy.y;
        if (py == 0 || pc == py) continue;
        const int ly = a.lab[y];
        const int64_t by = a.rowptr[y];
        const int32_t *Py = a.pplus + by;
        const double *Ay = a.amat + (int64_t)y * k;
        U128 accy = u128_zero();
        unsigned long long cnty = 0;
        int qn = 0;
        auto drain = [&](int upto) {
            while (qn >= upto && qn > 0) {
                const int take = qn < kGL ? qn : kGL;
                const int b = qn - take;
                if (lane < take) {
                    const int2 e = Q[b + lane];
                    accy = u128_add(accy, tri_terms<COUNT>(a, e.x, y, ly, Ay, e.y, cnty));
                }
                g.sync();
                qn = b;
            }
        };
        for (int i0 = 0; i0 < pc; i0 += kXLL) {
            const int iend = min(pc, i0 + kXLL);
            int nx = 0, total = 0;
            for (int j0 = i0; j0 < iend; j0 += kGL) {
                const int i = j0 + lane;
                int32_t x = 0;
                int64_t bx = 0;
                int lenx = 0;
                if (i < iend) {
                    x = __ldg(a.pidx + by + i);
                    const int2 pcx = a.pc2[x];
                    const bool lower = pcx.y < pc || (pcx.y == pc && x < y);
                    if (lower && pcx.x > 0 && (__ldg(a.lab + x) < k || ly < k)) {
                        lenx = pcx.x;
                        bx = a.rowptr[x];
                    }
                }
                int incl = lenx;
#pragma unroll
                for (int o = 1; o < kGL; o <<= 1) {
                    const int t = __shfl_up_sync(g.gmask, incl, o, kGL);
                    if (lane >= o) incl += t;
                }
                int cnt;
                const int r = g.rank(lenx > 0, &cnt);
                if (lenx > 0) {
                    const int e_end = total + incl;
                    XL[nx + r] = make_longlong2(bx - (e_end - lenx), ((long long)x << 32) | (unsigned)e_end);
                }
                nx += cnt;
                total += g.bcast(incl, kGL - 1);
            }
            g.sync();
            if (total > 0) {
                const int seg = (total + kGL - 1) / kGL;
                const int t_beg = min(total, lane * seg), t_end = min(total, t_beg + seg);
                int lo = 0, hi = nx;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((int)(XL[mid].y & 0xffffffff) <= t_beg) lo = mid + 1; else hi = mid;
                }
                int xi = lo, xe = 0;
                int64_t xbase = 0;
                int32_t xcur = 0;
                if (t_beg < t_end) {
                    const longlong2 e = XL[xi];
                    xbase = e.x;
                    xe = (int)(e.y & 0xffffffff);
                    xcur = (int32_t)(e.y >> 32);
                }
                int t = t_beg;
                for (int s0 = 0; s0 < seg; s0 += kUnrollE) {
                    int32_t z[kUnrollE], xj[kUnrollE];
#pragma unroll
                    for (int u = 0; u < kUnrollE; u++) {
                        z[u] = -1;
                        xj[u] = xcur;
                        if (t < t_end) {
                            if (t >= xe) {
                                const longlong2 e = XL[++xi];
                                xbase = e.x;
                                xe = (int)(e.y & 0xffffffff);
                                xcur = (int32_t)(e.y >> 32);
                                xj[u] = xcur;
                            }
                            z[u] = __ldg(a.pplus + xbase + t);
                        }
                        t++;
                    }
#pragma unroll
                    for (int u = 0; u < kUnrollE; u++) {
                        const bool hit = z[u] >= 0 && in_sorted(Py, py, z[u]);
                        int cnt;
                        const int r = g.rank(hit, &cnt);
                        if (hit) Q[qn + r] = make_int2(xj[u], z[u]);
                        qn += cnt;
                        if (lane == 0) ntri += cnt;
                    }
                    g.sync();
                    drain(kGL);
                }
            }
            g.sync();
        }
        drain(1);
        if (ly < k && y >= a.head_lo && y < a.head_hi) {
            if constexpr (COUNT) {
                cnty = g.sum(cnty);
                if (lane == 0 && cnty) atomicAdd(a.n1 + y, cnty);
            } else {
                accy = g.sum(accy);
                if (lane == 0 && (accy.lo | accy.hi)) acc_add(a, y, accy);
            }
        }
        g.sync();
    }
    for (int o = 16; o > 0; o >>= 1) ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
    if ((threadIdx.x & 31) == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
}

template <bool COUNT>
static cudaError_t launch_e(Ctx &c) {
    CdeArgs a = cde_args(c);
    unsigned long long *ctr = c.scal + kScalCnt0;
    cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), c.stream);
    const int64_t n_heavy = c.bins.offset[4];          // degree classes 5-7 (d >= 128)
    // light middle vertices on a side stream, concurrently with the heavy ones
    cudaEventRecord(c.ev_fork, c.stream);
    cudaStreamWaitEvent(c.side[0], c.ev_fork, 0);
    if (n_heavy < c.n) {
        const int64_t groups = c.n - n_heavy;
        const int64_t blocks = std::min<int64_t>((groups + 31) / 32, 148 * 8);
        k_phase_e_light<COUNT><<<(unsigned)blocks, 256, 0, c.side[0]>>>(a, n_heavy);
        c.launches++;
    }
    cudaEventRecord(c.ev_join[0], c.side[0]);
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
    const int grid = std::max(1, per_sm) * sms;
    if (n_heavy > 0) {
        k_phase_e<COUNT><<<grid, kWarpsE * 32, smem, c.stream>>>(a, it, ctr);
        c.launches++;
    }
    cudaStreamWaitEvent(c.stream, c.ev_join[0], 0);
    return cudaGetLastError();
}

cudaError_t launch_phase_e(Ctx &c) { return launch_e<false>(c); }
cudaError_t launch_triangle_counts(Ctx &c) { return launch_e<true>(c); }

}  // namespace rs

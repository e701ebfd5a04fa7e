// Load-time and community-time kernels:
//  - CSR contract check (C-17), degree classes for binned scheduling,
//  - community-size histogram, target selection (C-15), 8-bit labels.
#include "rs_internal.cuh"
#include "rs_protocol.h"
#include "rs_device.cuh"
#include <cub/cub.cuh>

namespace rs {

// ---------------------------------------------------------------- validation
// err codes: 1 row_offsets decreasing / bad, 2 col out of range, 3 not strictly
// ascending (unsorted or duplicate), 4 self-loop, 5 not symmetric.
__global__ void k_validate(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ col, int64_t n,
                           unsigned long long *scal) {
    int64_t u = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    for (; u < n; u += (int64_t)gridDim.x * (blockDim.x / 32)) {
        int64_t b = rowptr[u], e = rowptr[u + 1];
        int code = 0;
        if (e < b) code = 1;
        for (int64_t i = b + lane; i < e && !code; i += 32) {
            int32_t v = col[i];
            if (v < 0 || v >= n) { code = 2; break; }
            if (i > b && col[i - 1] >= v) { code = 3; break; }
            if (v == u) { code = 4; break; }
            // symmetric: u in N(v) (binary search in the sorted row of v)
            int64_t lo = rowptr[v], hi = rowptr[v + 1];
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (col[mid] < u) lo = mid + 1; else hi = mid;
            }
            if (lo >= rowptr[v + 1] || col[lo] != u) { code = 5; break; }
        }
        unsigned any = __ballot_sync(0xffffffffu, code != 0);
        if (any) {
            int first = __ffs(any) - 1;
            int c = __shfl_sync(0xffffffffu, code, first);
            if (lane == 0) {
                // keep the smallest offending row
                unsigned long long old = atomicMin(&scal[kScalErrRow], (unsigned long long)u);
                if ((unsigned long long)u <= old) atomicExch(&scal[kScalErr], (unsigned long long)c);
            }
        }
    }
}

cudaError_t launch_validate(Ctx &c, const int64_t *rp, const int32_t *col) {
    k_validate<<<148 * 8, 256, 0, c.stream>>>(rp, col, c.n, c.scal);
    c.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- internal numbering
// Vertices are renumbered by degree, descending (ties: ascending original id),
// once at load time. Every later gather then finds the high-degree vertices --
// the ones that appear in most adjacency and P lists -- packed at the front of
// each per-vertex table (L2-friendly), and the degree classes of the binned
// scheduler become contiguous ranges. Results are mapped back to original ids
// on output. Exact fixed-point sums make scores independent of the numbering.
__global__ void k_deg_iota(const int64_t *__restrict__ rp, int64_t n, uint32_t *deg, int32_t *iota) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        deg[u] = (uint32_t)(rp[u + 1] - rp[u]);
        iota[u] = (int32_t)u;
    }
}
__global__ void k_inv_perm(const int32_t *__restrict__ perm, int64_t n, int32_t *inv, const uint32_t *__restrict__ deg_s,
                           int64_t *d64) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        inv[perm[r]] = (int32_t)r;
        d64[r] = deg_s[r];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) d64[n] = 0;
}
// number of vertices with degree >= bin_lo(cls), cls = 1..7 (degrees sorted descending)
// (out[kNumBins]: degree >= 512, a split point of the row sorts)
__global__ void k_class_bounds(const uint32_t *__restrict__ deg_s, int64_t n, unsigned long long *out) {
    const int cls = threadIdx.x + 1;
    if (cls > kNumBins) return;
    const int64_t lo_deg = cls == kNumBins ? 512 : bin_lo(cls);
    int64_t lo = 0, hi = n;   // first r with deg_s[r] < lo_deg
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)deg_s[mid] >= lo_deg) lo = mid + 1; else hi = mid;
    }
    out[cls] = (unsigned long long)lo;
}

// rows of length in [lo, cap] sorted by one CTA each (cub::BlockRadixSort in
// shared memory, keys < 2^bits; padding keys 2^bits - 1 sort last)
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_row_sort(const int64_t *__restrict__ rowptr, int64_t r0, int64_t r1,
                                                      const int32_t *__restrict__ in, int32_t *out, int bits,
                                                      const int32_t *__restrict__ map) {
    using BRS = cub::BlockRadixSort<uint32_t, THREADS, ITEMS>;
    __shared__ typename BRS::TempStorage ts;
    const uint32_t pad = bits >= 32 ? 0xFFFFFFFFu : (1u << bits) - 1u;
    for (int64_t r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const int64_t b = rowptr[r];
        const int d = (int)(rowptr[r + 1] - b);
        uint32_t keys[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int idx = threadIdx.x * ITEMS + i;
            keys[i] = idx < d ? (uint32_t)(map ? __ldg(map + in[b + idx]) : in[b + idx]) : pad;
        }
        BRS(ts).Sort(keys, 0, bits);
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int idx = threadIdx.x * ITEMS + i;
            if (idx < d) out[b + idx] = (int32_t)keys[i];
        }
        __syncthreads();
    }
}

// bitonic sort of 32 J keys held by a warp (element i = 32 j + lane; partners
// across lanes by shuffle, within a lane by register swap), ascending
template <int J>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[J], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * J; k <<= 1) {
#pragma unroll
        for (int s = k >> 1; s > 0; s >>= 1) {
            if (s >= 32) {
#pragma unroll
                for (int j = 0; j < J; j++) {
                    const int pj = j ^ (s >> 5);
                    if (pj > j) {
                        const bool up = ((32 * j + lane) & k) == 0;
                        const uint32_t a = v[j], c = v[pj];
                        if ((a > c) == up) { v[j] = c; v[pj] = a; }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < J; j++) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[j], s);
                    const bool up = ((32 * j + lane) & k) == 0;
                    const bool low = (lane & s) == 0;
                    v[j] = (low == up) ? min(v[j], o) : max(v[j], o);
                }
            }
        }
    }
}

// rows of at most 32 J entries: a warp per row, bitonic sort in registers,
// padding keys 0xFFFFFFFF sort last
template <int J>
__global__ void __launch_bounds__(256) k_row_sort_warp(const int64_t *__restrict__ rowptr, int64_t r0, int64_t r1,
                                                       const int32_t *__restrict__ in, int32_t *out,
                                                       const int32_t *__restrict__ map) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < r1; r += nw) {
        const int64_t b = rowptr[r];
        const int d = (int)(rowptr[r + 1] - b);
        uint32_t v[J];
#pragma unroll
        for (int j = 0; j < J; j++) {
            const int i = 32 * j + lane;
            v[j] = i < d ? (uint32_t)(map ? __ldg(map + in[b + i]) : in[b + i]) : 0xFFFFFFFFu;
        }
        warp_bitonic<J>(v, lane);
#pragma unroll
        for (int j = 0; j < J; j++)
            if (32 * j + lane < d) out[b + 32 * j + lane] = (int32_t)v[j];
    }
}

// Load time, rows of the ORIGINAL numbering [v0, v1) (a chunk whose col_idx has
// arrived): each row is relabelled to internal ids and written at its internal
// position; rows shorter than 512 are sorted right here in registers (a warp per
// row), longer ones go unsorted to tmp for the class sorts of relabel_finish.
// Chunks let the host->device copy of col_idx overlap this pass.
template <int J>
__device__ __forceinline__ void relabel_sort_row(const int32_t *__restrict__ col_o, const int32_t *__restrict__ inv,
                                                 int64_t b, int d, int lane, int32_t *out) {
    uint32_t v[J];
#pragma unroll
    for (int j = 0; j < J; j++) {
        const int i = 32 * j + lane;
        v[j] = i < d ? (uint32_t)__ldg(inv + __ldg(col_o + b + i)) : 0xFFFFFFFFu;
    }
    warp_bitonic<J>(v, lane);
#pragma unroll
    for (int j = 0; j < J; j++)
        if (32 * j + lane < d) out[32 * j + lane] = (int32_t)v[j];
}
// rows of 512..8191 entries: a CTA per internal row r in [r0, r1) whose original
// row perm[r] lies in the chunk [v0, v1): relabel + block radix sort
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_relabel_sort_cta(const int64_t *__restrict__ rp_o,
                                                              const int32_t *__restrict__ col_o,
                                                              const int32_t *__restrict__ perm,
                                                              const int32_t *__restrict__ inv,
                                                              const int64_t *__restrict__ rp, int64_t r0, int64_t r1,
                                                              int64_t v0, int64_t v1, int32_t *out, int bits) {
    using BRS = cub::BlockRadixSort<uint32_t, THREADS, ITEMS>;
    __shared__ typename BRS::TempStorage ts;
    const uint32_t pad = bits >= 32 ? 0xFFFFFFFFu : (1u << bits) - 1u;
    for (int64_t r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const int64_t v = perm[r];
        if (v < v0 || v >= v1) continue;   // CTA-uniform
        const int64_t b = rp_o[v];
        const int d = (int)(rp_o[v + 1] - b);
        const int64_t o = rp[r];
        uint32_t keys[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int idx = threadIdx.x * ITEMS + i;
            keys[i] = idx < d ? (uint32_t)__ldg(inv + __ldg(col_o + b + idx)) : pad;
        }
        BRS(ts).Sort(keys, 0, bits);
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int idx = threadIdx.x * ITEMS + i;
            if (idx < d) out[o + idx] = (int32_t)keys[i];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_relabel_fused(const int64_t *__restrict__ rp_o, const int32_t *__restrict__ col_o,
                                                       const int32_t *__restrict__ inv, const int64_t *__restrict__ rp,
                                                       int64_t v0, int64_t v1, int32_t *tmp, int32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = v0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); v < v1; v += nw) {
        const int64_t b = rp_o[v];
        const int64_t d = rp_o[v + 1] - b;
        const int64_t o = rp[inv[v]];
        if (d >= 8192) {
            for (int64_t i = lane; i < d; i += 32) tmp[o + i] = __ldg(inv + __ldg(col_o + b + i));
        } else if (d >= 512) {
            continue;   // k_relabel_sort_cta
        } else if (d > 128) {
            relabel_sort_row<16>(col_o, inv, b, (int)d, lane, out + o);
        } else if (d > 32) {
            relabel_sort_row<4>(col_o, inv, b, (int)d, lane, out + o);
        } else if (d > 0) {
            relabel_sort_row<1>(col_o, inv, b, (int)d, lane, out + o);
        }
    }
}

// Sort every row of a CSR-shaped array (row r at [rowptr[r], rowptr[r+1])) by
// key = map ? map[in[e]] : in[e] (keys < 2^bits). Rows are in degree-descending
// order, so each length class is a contiguous range (c.rsplit, load time): rows
// >= 8192 with CUB's segmented radix sort (mapped keys gathered first), [512,
// 8192) one CTA per row (block radix sort sized to the class), < 512 a warp per
// row (register bitonic). Used at load time (adjacency by internal id) and by
// the all-communities mode (neighbour community codes, k_sparse.cu).
__global__ void k_gather_keys(const int32_t *__restrict__ in, const int32_t *__restrict__ map, int64_t cnt,
                              int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(map + in[i]);
}

cudaError_t sort_rows(Ctx &c, const int32_t *in, const int32_t *map, int32_t *out, int bits, void *tmp, size_t need,
                      int64_t upto) {
    // rows [0, upto) only: the class boundaries are clipped to it
    const int64_t n = std::min<int64_t>(c.n, upto);
    const int64_t r8192 = std::min(c.rsplit[0], n), r2048 = std::min(c.rsplit[1], n), r512 = std::min(c.rsplit[2], n);
    const int64_t r128 = std::min(c.rsplit[3], n), r32 = std::min(c.rsplit[4], n);
    cudaError_t e = cudaSuccess;
    if (r8192 > 0) {
        int64_t e8 = 0;
        if ((e = cudaMemcpy(&e8, c.rowptr + r8192, sizeof(int64_t), cudaMemcpyDeviceToHost))) return e;
        if (e8 > 0x7fffffff) return cudaErrorInvalidValue;   // CUB item counts are int
        const int32_t *src = in;
        if (map) {
            // mapped keys of the long rows, staged at the front of tmp
            int32_t *g = (int32_t *)tmp;
            const size_t gb = ((size_t)4 * e8 + 255) & ~(size_t)255;
            if (gb > need) return cudaErrorMemoryAllocation;
            k_gather_keys<<<148 * 8, 256, 0, c.stream>>>(in, map, e8, g);
            c.launches++;
            src = g;
            tmp = (char *)tmp + gb;
            need -= gb;
        }
        size_t t1 = 0;
        cub::DeviceSegmentedRadixSort::SortKeys(nullptr, t1, src, out, e8, (int)r8192, c.rowptr, c.rowptr + 1, 0,
                                                bits, c.stream);
        if (t1 > need) return cudaErrorMemoryAllocation;
        t1 = need;
        cub::DeviceSegmentedRadixSort::SortKeys(tmp, t1, src, out, e8, (int)r8192, c.rowptr, c.rowptr + 1, 0,
                                                bits, c.stream);
        c.launches++;
    }
    auto wgrid = [&](int64_t lo, int64_t hi) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((hi - lo + 7) / 8, 148 * 16)); };
    auto rows = [&](int64_t lo, int64_t hi) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(hi - lo, 148 * 32)); };
    if (r2048 > r8192) { k_row_sort<256, 32><<<rows(r8192, r2048), 256, 0, c.stream>>>(c.rowptr, r8192, r2048, in, out, bits, map); c.launches++; }
    if (r512 > r2048) { k_row_sort<256, 8><<<rows(r2048, r512), 256, 0, c.stream>>>(c.rowptr, r2048, r512, in, out, bits, map); c.launches++; }
    if (r128 > r512) { k_row_sort_warp<16><<<wgrid(r512, r128), 256, 0, c.stream>>>(c.rowptr, r512, r128, in, out, map); c.launches++; }
    if (r32 > r128) { k_row_sort_warp<4><<<wgrid(r128, r32), 256, 0, c.stream>>>(c.rowptr, r128, r32, in, out, map); c.launches++; }
    if (n > r32) { k_row_sort_warp<1><<<wgrid(r32, n), 256, 0, c.stream>>>(c.rowptr, r32, n, in, out, map); c.launches++; }
    return cudaGetLastError();
}

// temporaries of launch_relabel, carved from the caller's arena
size_t relabel_arena_bytes(int64_t n, int64_t nnz) {
    size_t need_sort = 0, need_scan = 0, need_seg = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need_sort, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                              (int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, need_scan, (int64_t *)nullptr, (int64_t *)nullptr, (int)(n + 1));
    // CUB's segmented radix sort takes int item counts: it only ever sorts the
    // rows of >= 8192 entries (sort_rows), whose total must stay below 2^31
    const int seg_items = (int)std::min<int64_t>(nnz, 0x7fffffff);
    size_t need_rad = 0;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, need_rad, (int32_t *)nullptr, (int32_t *)nullptr, seg_items,
                                            (int)n, (int64_t *)nullptr, (int64_t *)nullptr, 0, 32);
    const size_t cub_b = std::max(std::max(need_sort, need_scan), std::max(need_seg, need_rad));
    return 3 * (4 * (size_t)n + 256) + (8 * (size_t)(n + 1) + 256) + (4 * (size_t)std::max<int64_t>(nnz, 1) + 256) +
           cub_b + 256;
}

// Internal numbering, in three calls so that a host col_idx can stream in
// while rows are relabelled (rs_load_csr): prepare (degrees, permutation,
// internal offsets, degree classes; needs row_offsets only), rows (a chunk of
// original rows: relabel + sort the short ones), finish (sort the long rows).
cudaError_t launch_relabel_prepare(Ctx &c, const int64_t *rp_o, void *arena, size_t arena_bytes) {
    const int64_t n = c.n, nnz = c.nnz;
    char *ap = (char *)arena;
    auto carve = [&](size_t b) { void *p = ap; ap += (b + 255) & ~(size_t)255; return p; };
    uint32_t *deg = (uint32_t *)carve(4 * (size_t)n);
    uint32_t *deg_s = (uint32_t *)carve(4 * (size_t)n);
    int32_t *iota = (int32_t *)carve(4 * (size_t)n);
    int64_t *d64 = (int64_t *)carve(8 * (size_t)(n + 1));
    c.rl_tmpcol = (int32_t *)carve(4 * (size_t)std::max<int64_t>(nnz, 1));
    c.rl_tmp = ap;
    if ((size_t)(ap - (char *)arena) > arena_bytes) return cudaErrorMemoryAllocation;
    c.rl_need = arena_bytes - (size_t)(ap - (char *)arena);
    void *tmp = c.rl_tmp;
    const size_t need = c.rl_need;
    cudaError_t e = cudaSuccess;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_deg_iota<<<blocks, 256, 0, c.stream>>>(rp_o, n, deg, iota);
    size_t t1 = need;
    cub::DeviceRadixSort::SortPairsDescending(tmp, t1, deg, deg_s, iota, c.perm, (int)n, 0, 32, c.stream);
    k_inv_perm<<<blocks, 256, 0, c.stream>>>(c.perm, n, c.inv, deg_s, d64);
    t1 = need;
    cub::DeviceScan::ExclusiveSum(tmp, t1, d64, c.rowptr, (int)(n + 1), c.stream);
    k_class_bounds<<<1, 32, 0, c.stream>>>(deg_s, n, c.scal + kScalTk);
    c.launches += 5;
    unsigned long long ge[kNumBins + 1] = {0};
    uint32_t dmax = 0;
    cudaMemcpyAsync(ge, c.scal + kScalTk, sizeof(ge), cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(&dmax, deg_s, sizeof(uint32_t), cudaMemcpyDeviceToHost, c.stream);
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    if ((e = cudaGetLastError())) return e;
    c.rsplit[0] = (int64_t)ge[7];
    c.rsplit[1] = (int64_t)ge[6];
    c.rsplit[2] = (int64_t)ge[kNumBins];
    c.rsplit[3] = (int64_t)ge[5];
    c.rsplit[4] = (int64_t)ge[3];
    // ge[cls] = #vertices with degree >= bin_lo(cls); class cls = [ge[cls+1], ge[cls])
    ge[0] = (unsigned long long)n;
    for (int cls = 0; cls < kNumBins; cls++) {
        const int64_t hi = (int64_t)ge[cls];
        const int64_t lo = cls + 1 < kNumBins ? (int64_t)ge[cls + 1] : 0;
        c.bins.offset[cls] = lo;
        c.bins.count[cls] = hi - lo;
    }
    c.d_max = dmax;
    return cudaSuccess;
}

cudaError_t launch_relabel_rows(Ctx &c, const int64_t *rp_o, const int32_t *col_o, int64_t v0, int64_t v1) {
    if (v1 <= v0) return cudaSuccess;
    const int64_t warps = v1 - v0;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 16));
    k_relabel_fused<<<blocks, 256, 0, c.stream>>>(rp_o, col_o, c.inv, c.rowptr, v0, v1, c.rl_tmpcol, c.col);
    c.launches++;
    // rows of 512..8191 entries (internal [r8192, r512)) whose original row is in the chunk
    int bits = 1;
    while (bits < 31 && (1ll << bits) < c.n) bits++;
    const int64_t r8192 = c.rsplit[0], r2048 = c.rsplit[1], r512 = c.rsplit[2];
    auto rows = [&](int64_t lo, int64_t hi) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(hi - lo, 148 * 8)); };
    if (r2048 > r8192) {
        k_relabel_sort_cta<256, 32><<<rows(r8192, r2048), 256, 0, c.stream>>>(rp_o, col_o, c.perm, c.inv, c.rowptr,
                                                                               r8192, r2048, v0, v1, c.col, bits);
        c.launches++;
    }
    if (r512 > r2048) {
        k_relabel_sort_cta<256, 8><<<rows(r2048, r512), 256, 0, c.stream>>>(rp_o, col_o, c.perm, c.inv, c.rowptr,
                                                                             r2048, r512, v0, v1, c.col, bits);
        c.launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_relabel_finish(Ctx &c) {
    if (!c.nnz || c.rsplit[0] == 0) return cudaSuccess;   // no row of >= 8192 entries
    int bits = 1;
    while (bits < 31 && (1ll << bits) < c.n) bits++;
    return sort_rows(c, c.rl_tmpcol, nullptr, c.col, bits, c.rl_tmp, c.rl_need, c.rsplit[0]);
}

cudaError_t launch_relabel(Ctx &c, const int64_t *rp_o, const int32_t *col_o, void *arena, size_t arena_bytes) {
    cudaError_t e = launch_relabel_prepare(c, rp_o, arena, arena_bytes);
    if (e == cudaSuccess) e = launch_relabel_rows(c, rp_o, col_o, 0, c.n);
    if (e == cudaSuccess) e = launch_relabel_finish(c);
    return e;
}

// ---------------------------------------------------------------- log2 table
__global__ void k_log2_table(double *t, int64_t len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = i > 0 ? log2((double)i) : 0.0;
}
cudaError_t launch_log2_table(Ctx &c, double *t, int64_t len) {
    k_log2_table<<<148, 256, 0, c.stream>>>(t, len);
    c.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- communities
__global__ void k_minmax_i32(const int32_t *__restrict__ a, int64_t n, unsigned long long *out) {
    // out[0] = max(-min) trick: track min as max of (INT_MAX - v) via two atomics
    long long mn = INT64_MAX, mx = INT64_MIN;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long v = a[i];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        long long x = __shfl_xor_sync(0xffffffffu, mn, o); mn = x < mn ? x : mn;
        long long y = __shfl_xor_sync(0xffffffffu, mx, o); mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin((long long *)&out[0], mn);
        atomicMax((long long *)&out[1], mx);
    }
}

cudaError_t launch_minmax_i32(Ctx &c, const int32_t *a, int64_t n, int64_t *mn, int64_t *mx) {
    long long init[2] = {INT64_MAX, INT64_MIN};
    cudaMemcpyAsync(c.scal + kScalTk, init, sizeof(init), cudaMemcpyHostToDevice, c.stream);
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (blocks < 1) blocks = 1;
    k_minmax_i32<<<blocks, 256, 0, c.stream>>>(a, n, c.scal + kScalTk);
    c.launches++;
    long long res[2];
    cudaMemcpyAsync(res, c.scal + kScalTk, sizeof(res), cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    *mn = res[0];
    *mx = res[1];
    return e;
}

constexpr int kHistSmem = 8192;

// community sizes; an id outside [0, nbins) is not counted but flagged in
// scal[kScalErr] (12: negative, 13: >= nbins, i.e. the histogram must grow)
__global__ void k_comm_hist(const int32_t *__restrict__ comm, int64_t n, int32_t *hist, int64_t nbins,
                            unsigned long long *scal) {
    __shared__ int s[kHistSmem];
    const bool priv = nbins <= kHistSmem;
    if (priv) for (int i = threadIdx.x; i < nbins; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t cid = comm[i];
        if (cid < 0 || cid >= nbins) {
            atomicMax(&scal[kScalErr], cid < 0 ? 12ull : 13ull);
            continue;
        }
        if (priv) atomicAdd(&s[cid], 1); else atomicAdd(&hist[cid], 1);
    }
    __syncthreads();
    if (priv) for (int i = threadIdx.x; i < nbins; i += blockDim.x) if (s[i]) atomicAdd(&hist[i], s[i]);
}

// One CTA: target selection (k largest communities, ties ascending id, or the
// user's list), distinct count, and the community -> 8-bit code map:
// targets get their column 0..k-1; other present communities get k, k+1, ...
// in ascending id while codes last (<= 254); the rest share kOther (0xFF).
constexpr int kSelThreads = 1024;
__global__ void __launch_bounds__(kSelThreads) k_select(const int32_t *__restrict__ hist, int64_t nbins, int32_t k,
                                                        const int32_t *user_targets, int32_t *targets,
                                                        uint8_t *code, unsigned long long *scal) {
    __shared__ long long s_key[kSelThreads / 32];
    __shared__ int s_cnt[kSelThreads / 32];
    __shared__ int32_t s_t[kMaxK];
    __shared__ int s_base;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // distinct communities
    int cnt = 0;
    for (int64_t i = tid; i < nbins; i += blockDim.x) cnt += hist[i] > 0;
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_cnt[wid] = cnt;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int i = 0; i < kSelThreads / 32; i++) t += s_cnt[i];
        scal[kScalCnt0] = (unsigned long long)t;
        if (k > t) scal[kScalErr] = 10;   // k exceeds the number of communities
    }
    __syncthreads();
    if (scal[kScalErr]) return;
    if (user_targets) {
        if (tid < k) {
            int32_t t = user_targets[tid];
            bool ok = t >= 0 && t < nbins && hist[t] > 0;
            for (int j = 0; j < tid; j++) ok = ok && user_targets[j] != t;
            if (!ok) atomicExch(&scal[kScalErr], 11ull);
            s_t[tid] = t;
        }
        __syncthreads();
    } else {
        // k rounds of argmax over key = size * 2^32 + (2^31 - 1 - id): largest size, then smallest id
        for (int r = 0; r < k; r++) {
            long long best = -1;
            for (int64_t i = tid; i < nbins; i += blockDim.x) {
                int32_t h = hist[i];
                if (h <= 0) continue;
                bool taken = false;
                for (int j = 0; j < r; j++) taken |= (s_t[j] == (int32_t)i);
                if (taken) continue;
                long long key = ((long long)h << 32) | (long long)(0x7fffffff - (int32_t)i);
                best = key > best ? key : best;
            }
            for (int o = 16; o > 0; o >>= 1) { long long x = __shfl_xor_sync(0xffffffffu, best, o); best = x > best ? x : best; }
            if (lane == 0) s_key[wid] = best;
            __syncthreads();
            if (tid == 0) {
                long long b = -1;
                for (int i = 0; i < kSelThreads / 32; i++) b = s_key[i] > b ? s_key[i] : b;
                s_t[r] = 0x7fffffff - (int32_t)(b & 0xffffffffll);
            }
            __syncthreads();
        }
    }
    if (scal[kScalErr]) return;
    if (tid < k) targets[tid] = s_t[tid];
    // codes: ascending-id rank of non-target present communities
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int64_t base = 0; base < nbins; base += blockDim.x) {
        int64_t i = base + tid;
        int col = -1;
        bool present = false;
        if (i < nbins) {
            present = hist[i] > 0;
            for (int j = 0; j < k; j++) col = (s_t[j] == (int32_t)i) ? j : col;
        }
        bool other = present && col < 0;
        unsigned b = __ballot_sync(0xffffffffu, other);
        if (lane == 0) s_cnt[wid] = __popc(b);
        __syncthreads();
        int before = 0, all = 0;
        for (int w = 0; w < kSelThreads / 32; w++) { before += w < wid ? s_cnt[w] : 0; all += s_cnt[w]; }
        int rank = s_base + before + __popc(b & ((1u << lane) - 1u));
        if (i < nbins) {
            uint8_t cd = kOther;
            if (col >= 0) cd = (uint8_t)col;
            else if (other && k + rank < (int)kOther) cd = (uint8_t)(k + rank);
            code[i] = cd;
        }
        __syncthreads();
        if (tid == 0) s_base += all;
        __syncthreads();
    }
}

// internal vertex r gets the community of original vertex perm[r] and its code
__global__ void k_labels(const int32_t *__restrict__ comm_in, const int32_t *__restrict__ perm,
                         const uint8_t *__restrict__ code, int64_t n, int32_t *comm, uint8_t *lab) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t cid = comm_in[perm[r]];
        comm[r] = cid;
        lab[r] = code[cid];
    }
}

// n_wide: the vertices with d^2 >= wide_bound(k) (VRec::wide), a prefix of the
// degree-descending numbering
__global__ void k_nwide(const int64_t *__restrict__ rowptr, int64_t n, double bound, unsigned long long *out) {
    int64_t lo = 0, hi = n;   // first u with d(u)^2 < bound
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double d = (double)(rowptr[mid + 1] - rowptr[mid]);
        if (d * d >= bound) lo = mid + 1; else hi = mid;
    }
    *out = (unsigned long long)lo;
}

void launch_comm_hist(Ctx &c, int64_t nbins) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((c.n + 255) / 256, 148 * 4));
    k_comm_hist<<<blocks, 256, 0, c.stream>>>(c.comm_in, c.n, c.chist, nbins, c.scal);
    c.launches++;
}
void launch_nwide(Ctx &c, double bound) {
    k_nwide<<<1, 1, 0, c.stream>>>(c.rowptr, c.n, bound, c.scal + kScalNWide);
    c.nwide_k = -1;                                  // the dense path's cached n_wide is gone
    c.launches++;
}

cudaError_t launch_set_communities(Ctx &c, int64_t max_comm, const int32_t *user_targets) {
    const int64_t nbins = max_comm + 1;
    cudaMemsetAsync(c.chist, 0, sizeof(int32_t) * nbins, c.stream);
    int blocks = (int)std::min<int64_t>((c.n + 255) / 256, 148 * 4);
    if (blocks < 1) blocks = 1;
    k_comm_hist<<<blocks, 256, 0, c.stream>>>(c.comm_in, c.n, c.chist, nbins, c.scal);
    c.launches++;
    k_select<<<1, kSelThreads, 0, c.stream>>>(c.chist, nbins, c.k, user_targets, c.targets, c.ccode, c.scal);
    c.launches++;
    k_labels<<<blocks, 256, 0, c.stream>>>(c.comm_in, c.perm, c.ccode, c.n, c.comm_id, c.lab);
    // n_wide depends only on the graph and k: recomputed when either changed
    if (c.nwide_k != c.k) {
        k_nwide<<<1, 1, 0, c.stream>>>(c.rowptr, c.n, wide_bound(c.k), c.scal + kScalNWide);
        c.nwide_k = c.k;
        c.launches++;
    }
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

namespace rs {
// ---------------------------------------------------------------- multi-GPU partition
// Contiguous vertex ranges balanced by the work estimate d(u) + kVertexWork
// (prefix sum, then the first vertex whose prefix reaches r/world of the total).
// a vertex's Phase A work ~ d(u) entries plus a fixed per-vertex part (weights,
// records, the lists pass): worth about this many entries (from the per-rank
// Phase A times of the emulated 8-rank world)
#ifndef RS_EXP_VERTEX_WORK
#define RS_EXP_VERTEX_WORK 16
#endif
constexpr int64_t kVertexWork = RS_EXP_VERTEX_WORK;
__global__ void k_work(const int64_t *__restrict__ rowptr, int64_t n, int64_t *w) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        w[u] = rowptr[u + 1] - rowptr[u] + kVertexWork;
}
// boundaries of the head ranges (rs_protocol.h split_point, = rs_split_ranges)
__global__ void k_split(const int64_t *__restrict__ incl, int64_t n, int world, int64_t *bounds) {
    const int r = threadIdx.x;
    if (r <= world) bounds[r] = split_point(incl, n, world, r);
}
cudaError_t launch_partition(Ctx &c) {
    const int64_t n = c.n;
    int64_t *w = (int64_t *)c.scratch;
    int64_t *incl = w + n;
    int64_t *bounds = incl + n;
    void *tmp = bounds + (c.world + 1);
    size_t tmp_bytes = c.scratch_bytes - sizeof(int64_t) * (size_t)(2 * n + c.world + 1);
    k_work<<<148 * 4, 256, 0, c.stream>>>(c.rowptr, n, w);
    size_t need = 0;
    cub::DeviceScan::InclusiveSum(nullptr, need, w, incl, (int)n, c.stream);
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::InclusiveSum(tmp, need, w, incl, (int)n, c.stream);
    k_split<<<1, 1024, 0, c.stream>>>(incl, n, c.world, bounds);
    c.launches += 3;
    c.bounds.assign(c.world + 1, 0);
    cudaMemcpyAsync(c.bounds.data(), bounds, sizeof(int64_t) * (c.world + 1), cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    c.head_lo = c.bounds[c.rank];
    c.head_hi = c.bounds[c.rank + 1];
    return e;
}
}  // namespace rs

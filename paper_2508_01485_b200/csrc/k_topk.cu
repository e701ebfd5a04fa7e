// Step 4 (Algorithm 1, optional): top-K vertices by R, ties by ascending
// vertex id (C-14). Radix select over the IEEE bit patterns of the
// non-negative scores (monotone as unsigned integers once -0.0 is folded into
// +0.0), 6 digit passes of 11 bits; ties at the threshold are resolved by an
// id-ordered block scan; the K survivors are sorted (key desc, id asc).
#include "rs_internal.cuh"
#include "rs_device.cuh"
#include "rs_protocol.h"
#include <cub/cub.cuh>

namespace rs {

constexpr int kTkBlocks = 148 * 4;
constexpr int kTkThreads = 256;
constexpr int kTkSortMax = 4096;   // in-smem bitonic sort capacity
constexpr int kTkGatherSlot = 2040; // tk_hist word: the compact path's candidate count

// state slots at scal + kScalTk: [0] prefix, [1] krem (keys still to take at
// the threshold), [2] count of keys strictly above the current prefix
__device__ __forceinline__ unsigned long long score_key(double s) {
    return score_key_bits((unsigned long long)__double_as_longlong(s));   // -0.0 -> +0.0 (rs_protocol.h)
}

struct TkFilter {             // multi-GPU: only original ids whose internal id is owned
    const int32_t *inv;       // nullptr = no filter
    int64_t lo, hi;
    __device__ __forceinline__ bool keep(int64_t v) const {
        if (!inv) return true;
        const int64_t u = inv[v];
        return u >= lo && u < hi;
    }
};

// digit pass: 11-bit digits from the top (6 passes: 11 x 5 + 9). Blocks count
// the digits of the keys still matching the prefix into a shared histogram and
// add it to the global one; the last block to finish (ticket) picks the digit
// with a block scan from the top, updates the state and clears the histogram.
constexpr int kTkBits = 11, kTkBins = 1 << kTkBits, kTkPasses = 6;
__device__ __forceinline__ void tk_digit(int pass, int &shift, int &width) {
    const int hi = 64 - kTkBits * pass;
    width = hi < kTkBits ? hi : kTkBits;
    shift = hi - width;
}

// the compact path (k_tk_gather): once the keys sharing the threshold's top
// 22 bits -- and every key above them -- fit the final sort, the remaining
// passes over all n scores are skipped (*skip = how many were gathered)
__device__ __forceinline__ bool tk_skipped(const unsigned long long *skip) {
    return skip && *skip <= (unsigned long long)kTkSortMax;
}

__global__ void __launch_bounds__(kTkThreads) k_tk_pass(const double *__restrict__ score, int64_t lo, int64_t hi,
                                                        int pass, unsigned long long *st, unsigned int *hist,
                                                        unsigned int *ticket, TkFilter flt,
                                                        const unsigned long long *skip) {
    if (tk_skipped(skip)) return;
    __shared__ unsigned int h[kTkBins];
    __shared__ unsigned long long s_sum[kTkThreads];
    __shared__ bool s_last;
    for (int i = threadIdx.x; i < kTkBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int shift, width;
    tk_digit(pass, shift, width);
    const unsigned long long prefix = st[0];
    const int top = shift + width;      // bits above the digit must match the prefix
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        if (!flt.keep(i)) continue;
        const unsigned long long key = score_key(score[i]);
        const bool match = top >= 64 || ((key ^ prefix) >> top) == 0ull;
        if (match) atomicAdd(&h[(key >> shift) & (kTkBins - 1)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTkBins; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    // last block: thread t owns the 8 digits [kTkBins - 8 (t + 1), kTkBins - 8 t), scanned from the top
    constexpr int per = kTkBins / kTkThreads;
    const int t = threadIdx.x;
    unsigned int c[per];
    unsigned long long mine = 0;
#pragma unroll
    for (int j = 0; j < per; j++) {
        c[j] = __ldcg(hist + kTkBins - 1 - (per * t + j));   // descending digit order
        mine += c[j];
    }
    s_sum[t] = mine;
    __syncthreads();
    for (int o = 1; o < kTkThreads; o <<= 1) {   // inclusive scan (Hillis-Steele)
        const unsigned long long v = t >= o ? s_sum[t - o] : 0ull;
        __syncthreads();
        s_sum[t] += v;
        __syncthreads();
    }
    const unsigned long long krem = st[1];
    const unsigned long long before = t ? s_sum[t - 1] : 0ull;   // keys in higher digits
    // the crossing is in my digits (or there is none: fewer keys than krem, the
    // lowest thread takes digit 0 with every key above, as a full scan would)
    if ((before < krem && s_sum[t] >= krem) || (t == kTkThreads - 1 && s_sum[t] < krem)) {
        unsigned long long above = before;
        int dgt = 0;
#pragma unroll
        for (int j = 0; j < per; j++) {
            const int d = kTkBins - 1 - (per * t + j);
            if (above + c[j] >= krem) { dgt = d; break; }
            above += c[j];
        }
        st[0] = prefix | ((unsigned long long)dgt << shift);
        st[1] = krem - above;
        st[2] += above;
    }
    for (int i = threadIdx.x; i < kTkBins; i += blockDim.x) hist[i] = 0;   // ready for the next pass
    if (threadIdx.x == 0) *ticket = 0;
}

// keys above the threshold -> cand[0, count_gt) (any order); ties counted per block
__global__ void __launch_bounds__(kTkThreads) k_tk_above(const double *__restrict__ score, int64_t lo, int64_t hi,
                                                         const unsigned long long *st, unsigned long long *cand_key,
                                                         int32_t *cand_id, unsigned long long *cursor,
                                                         unsigned int *tie_cnt, int64_t chunk, TkFilter flt,
                                                         const unsigned long long *skip) {
    if (tk_skipped(skip)) return;
    __shared__ unsigned int s_ties;
    if (threadIdx.x == 0) s_ties = 0;
    __syncthreads();
    const unsigned long long T = st[0];
    const int64_t b0 = lo + blockIdx.x * chunk;
    const int64_t b1 = min(hi, b0 + chunk);
    unsigned int ties = 0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        if (!flt.keep(i)) continue;
        const unsigned long long key = score_key(score[i]);
        if (key > T) {
            const unsigned long long p = atomicAdd(cursor, 1ull);
            cand_key[p] = key;
            cand_id[p] = (int32_t)i;
        } else if (key == T) {
            ties++;
        }
    }
    for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_ties, ties);
    __syncthreads();
    if (threadIdx.x == 0) tie_cnt[blockIdx.x] = s_ties;
}

// ties in id order: block b takes its ties while their global rank < krem
__global__ void __launch_bounds__(kTkThreads) k_tk_ties(const double *__restrict__ score, int64_t lo, int64_t hi,
                                                        const unsigned long long *st, unsigned long long *cand_key,
                                                        int32_t *cand_id, const unsigned int *tie_cnt, int64_t chunk,
                                                        TkFilter flt, const unsigned long long *skip) {
    if (tk_skipped(skip)) return;
    __shared__ unsigned long long s_pre;
    __shared__ int s_w[kTkThreads / 32];
    const unsigned long long T = st[0];
    const unsigned long long krem = st[1];
    const unsigned long long gt = st[2];
    unsigned long long pre = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) pre += tie_cnt[b];
    for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    if (threadIdx.x == 0) s_pre = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_pre, pre);
    __syncthreads();
    unsigned long long base = s_pre;
    if (base >= krem || tie_cnt[blockIdx.x] == 0) return;
    const int64_t b0 = lo + blockIdx.x * chunk;
    const int64_t b1 = min(hi, b0 + chunk);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t t0 = b0; t0 < b1 && base < krem; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        const bool tie = i < b1 && flt.keep(i) && score_key(score[i]) == T;
        const unsigned m = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) s_w[wid] = __popc(m);
        __syncthreads();
        unsigned long long before = 0, all = 0;
        for (int w = 0; w < kTkThreads / 32; w++) { before += (w < wid) ? s_w[w] : 0; all += s_w[w]; }
        const unsigned long long r = base + before + __popc(m & ((1u << lane) - 1u));
        if (tie && r < krem) {
            cand_key[gt + r] = T;
            cand_id[gt + r] = (int32_t)i;
        }
        __syncthreads();
        base += all;
    }
}

// after the first two digit passes (the top 22 key bits of the threshold are
// known): every key whose top 22 bits are >= the threshold's -- the keys above
// it and those sharing its digits -- appended to the candidates (any order);
// *cnt counts them all. When they fit kTkSortMax the sort picks the K first by
// (key desc, id asc) and the later passes return at once
__global__ void __launch_bounds__(kTkThreads) k_tk_gather(const double *__restrict__ score, int64_t lo, int64_t hi,
                                                          const unsigned long long *st, unsigned long long *cand_key,
                                                          int32_t *cand_id, unsigned long long *cnt) {
    const unsigned long long top = st[0] >> 42;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = score_key(score[i]);
        if ((key >> 42) >= top) {
            const unsigned long long p = atomicAdd(cnt, 1ull);
            if (p < (unsigned long long)kTkSortMax) {
                cand_key[p] = key;
                cand_id[p] = (int32_t)i;
            }
        }
    }
}

__device__ __forceinline__ bool tk_before(unsigned long long ka, int32_t ia, unsigned long long kb, int32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// single CTA bitonic sort of cnt <= kTkSortMax candidates, writes the first `out` entries
__global__ void __launch_bounds__(1024) k_tk_sort(const unsigned long long *cand_key, const int32_t *cand_id,
                                                  int64_t cnt, int64_t out, int32_t *ids_out, double *scores_out,
                                                  const unsigned long long *dev_cnt) {
    __shared__ unsigned long long sk[kTkSortMax];
    __shared__ int32_t si[kTkSortMax];
    if (tk_skipped(dev_cnt)) cnt = (int64_t)*dev_cnt;   // the compact path's candidates
    int size = 1;
    while (size < cnt) size <<= 1;
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
        if (i < cnt) { sk[i] = cand_key[i]; si[i] = cand_id[i]; }
        else { sk[i] = 0ull; si[i] = 0x7fffffff; }
    }
    __syncthreads();
    for (int len = 2; len <= size; len <<= 1) {
        for (int j = len >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < size; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool asc = (i & len) == 0;   // "ascending" = our order
                    const bool swap = asc ? tk_before(sk[p], si[p], sk[i], si[i]) : tk_before(sk[i], si[i], sk[p], si[p]);
                    if (swap) {
                        unsigned long long tk = sk[i]; sk[i] = sk[p]; sk[p] = tk;
                        int32_t ti = si[i]; si[i] = si[p]; si[p] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < out; i += blockDim.x) {
        ids_out[i] = si[i];
        if (scores_out) scores_out[i] = __longlong_as_double((long long)sk[i]);
    }
}

__global__ void k_tk_copy_out(const unsigned long long *key, const int32_t *id, int64_t out, int32_t *ids_out,
                              double *scores_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < out; i += (int64_t)gridDim.x * blockDim.x) {
        ids_out[i] = id[i];
        if (scores_out) scores_out[i] = __longlong_as_double((long long)key[i]);
    }
}

// sort `cnt` (key, id) candidates by (key desc, id asc) and emit the first `out`
cudaError_t tk_sort_emit(Ctx &c, unsigned long long *key, int32_t *id, int64_t cnt, int64_t out, int32_t *ids_out,
                         double *scores_out, bool compact) {
    if (cnt <= kTkSortMax) {
        const unsigned long long *dev_cnt = compact ? c.tk_hist + kTkGatherSlot : nullptr;
        k_tk_sort<<<1, 1024, 0, c.stream>>>(key, id, cnt, out, ids_out, scores_out, dev_cnt);
        c.launches++;
        return cudaGetLastError();
    }
    // large K: two stable radix sorts (ids ascending, then keys descending)
    unsigned long long *key2 = key + cnt;
    int32_t *id2 = (int32_t *)(key2 + cnt);
    size_t need1 = 0, need2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need1, id, id2, key, key2, (int)cnt, 0, 32, c.stream);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need2, key2, key, id2, id, (int)cnt, 0, 64, c.stream);
    size_t need = std::max(need1, need2);
    if (need > c.scratch_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceRadixSort::SortPairs(c.scratch, need, id, id2, key, key2, (int)cnt, 0, 32, c.stream);
    cub::DeviceRadixSort::SortPairsDescending(c.scratch, need, key2, key, id2, id, (int)cnt, 0, 64, c.stream);
    c.launches += 2;
    k_tk_copy_out<<<148, 256, 0, c.stream>>>(key, id, out, ids_out, scores_out);
    c.launches++;
    return cudaGetLastError();
}

// local top-K of score[lo, hi) into (cand_key, cand_id)[0, K') sorted, K' = min(K, hi-lo)
cudaError_t launch_topk_select(Ctx &c, int64_t K, int64_t lo, int64_t hi, unsigned long long *cand_key,
                               int32_t *cand_id, const int32_t *own_inv, int64_t own_lo, int64_t own_hi,
                               bool compact) {
    TkFilter flt{own_inv, own_lo, own_hi};
    unsigned long long *st = c.scal + kScalTk;
    // tk_hist (2048 u64): digit histogram u32[kTkBins] | ticket | cursor | per-block tie counts
    unsigned int *hist = (unsigned int *)c.tk_hist;
    unsigned int *ticket = (unsigned int *)(c.tk_hist + kTkBins / 2);
    unsigned long long *cursor = c.tk_hist + kTkBins / 2 + 1;
    unsigned int *tie_cnt = (unsigned int *)(c.tk_hist + kTkBins / 2 + 8);
    const int64_t range = hi - lo;
    unsigned long long init[3] = {0ull, (unsigned long long)K, 0ull};
    cudaMemcpyAsync(st, init, sizeof(init), cudaMemcpyHostToDevice, c.stream);
    cudaMemsetAsync(c.tk_hist, 0, sizeof(unsigned long long) * (kTkBins / 2 + 2), c.stream);
    unsigned long long *gcnt = c.tk_hist + kTkGatherSlot;
    const unsigned long long *skip = compact ? gcnt : nullptr;
    if (compact) cudaMemsetAsync(gcnt, 0, sizeof(unsigned long long), c.stream);
    int blocks = (int)std::min<int64_t>((range + kTkThreads - 1) / kTkThreads, kTkBlocks);
    if (blocks < 1) blocks = 1;
    for (int pass = 0; pass < kTkPasses; pass++) {
        k_tk_pass<<<blocks, kTkThreads, 0, c.stream>>>(c.score, lo, hi, pass, st, hist, ticket, flt,
                                                      pass >= 2 ? skip : nullptr);
        c.launches++;
        if (compact && pass == 1) {
            k_tk_gather<<<blocks, kTkThreads, 0, c.stream>>>(c.score, lo, hi, st, cand_key, cand_id, gcnt);
            c.launches++;
        }
    }
    const int64_t chunk = (range + kTkBlocks - 1) / kTkBlocks;
    const int cblocks = (int)std::max<int64_t>(1, (range + chunk - 1) / std::max<int64_t>(chunk, 1));
    k_tk_above<<<cblocks, kTkThreads, 0, c.stream>>>(c.score, lo, hi, st, cand_key, cand_id, cursor, tie_cnt,
                                                     std::max<int64_t>(chunk, 1), flt, skip);
    k_tk_ties<<<cblocks, kTkThreads, 0, c.stream>>>(c.score, lo, hi, st, cand_key, cand_id, tie_cnt,
                                                    std::max<int64_t>(chunk, 1), flt, skip);
    c.launches += 2;
    return cudaGetLastError();
}

}  // namespace rs

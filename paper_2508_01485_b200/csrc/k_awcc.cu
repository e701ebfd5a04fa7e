// NEXT-1 — robustness evaluation of §VII.B: absolute AWCC of a
// vertex set S under cumulative random removal of edges or vertices.
//
// AWCC(S) = (1/|S|) sum_{v in S} |zeta(v)| / d(v), zeta(v) the community ids of
// v's neighbours; the absolute variant recomputes zeta over the
// survivors and keeps the original d(v). Removal (DESIGN C-28/C-29):
// trial t keys every item (undirected edge id min<<32|max, or vertex id, in the
// caller's original ids) with mix64(s_t ^ id) (SplitMix64 finaliser, a
// bijection: keys are distinct); step j removes the r_j = floor(j step% M/100)
// items of smallest key, i.e. those below T_j = the key of rank r_j.
//
// Per trial: (1) T_j for every step by one multi-rank radix select — a
// histogram of the top 12 key bits over all M items, the few bins holding a
// rank r_j gathered and sorted (CUB), T_j read at its rank; (2) per v in S one
// CTA: each neighbour's survival level L = #{j : it survives step j} (T is
// non-decreasing in j), per community the max level in a hash table in
// global scratch, |zeta_j(v)| = #{communities with max level > j}. Integer
// results: the caller averages them in a fixed order (bit-reproducible).
#include "rs_internal.cuh"
#include <cub/cub.cuh>
#include <vector>

namespace rs {

constexpr int kAwBits = 12, kAwBins = 1 << kAwBits;

__device__ __forceinline__ uint64_t aw_mix64(uint64_t z) {   // SplitMix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// the key of item i of the trial: edges are the internal entries (u, x) with
// perm[u] < perm[x] (one per undirected edge), ids in original numbering
struct AwItems {
    const int64_t *rowptr;
    const int32_t *col;
    const int32_t *perm;
    int64_t n;
    int mode;                 // 0 edges, 1 vertices
    uint64_t st;              // trial key salt
};

// visit every item of the trial (grid-stride over CSR entries or vertices)
template <class F>
__device__ __forceinline__ void aw_for_items(const AwItems &it, F f) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it.mode == 1) {
        for (int64_t v = t0; v < it.n; v += stride) f(aw_mix64(it.st ^ (uint64_t)it.perm[v]));
        return;
    }
    // edges: a warp per row of the internal CSR
    const int lane = threadIdx.x & 31;
    for (int64_t u = t0 >> 5; u < it.n; u += stride >> 5) {
        const uint32_t uo = (uint32_t)it.perm[u];
        for (int64_t e = it.rowptr[u] + lane; e < it.rowptr[u + 1]; e += 32) {
            const uint32_t xo = (uint32_t)it.perm[it.col[e]];
            if (uo < xo) f(aw_mix64(it.st ^ (((uint64_t)uo << 32) | xo)));
        }
    }
}

__global__ void __launch_bounds__(256) k_aw_hist(AwItems it, unsigned int *hist) {
    __shared__ unsigned int h[kAwBins];
    for (int i = threadIdx.x; i < kAwBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    aw_for_items(it, [&](uint64_t key) { atomicAdd(&h[key >> (64 - kAwBits)], 1u); });
    __syncthreads();
    for (int i = threadIdx.x; i < kAwBins; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// keys of the selected bins (slot[bin] >= 0) appended at their slot's cursor
__global__ void __launch_bounds__(256) k_aw_gather(AwItems it, const int *slot, unsigned long long *cursor,
                                                   uint64_t *out) {
    aw_for_items(it, [&](uint64_t key) {
        const int s = slot[key >> (64 - kAwBits)];
        if (s >= 0) out[atomicAdd(&cursor[s], 1ull)] = key;
    });
}

// per v in S: survival level of each neighbour, max level per community
// (open-addressing table of `cap` entries at tab + 2 cap * s), then
// zeta[j][s] = #{communities with level > j}
__global__ void __launch_bounds__(256) k_aw_zeta(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                                                 const int32_t *__restrict__ perm, const int32_t *__restrict__ inv,
                                                 const int32_t *__restrict__ comm_orig, const int32_t *__restrict__ S,
                                                 int64_t nS, int mode, uint64_t st, const uint64_t *__restrict__ T,
                                                 const int *__restrict__ all, int J1, int32_t *tab, int64_t cap,
                                                 int32_t *zeta) {
    __shared__ uint64_t sT[128];
    __shared__ int sA[128];
    __shared__ int cnt[129];
    for (int j = threadIdx.x; j < J1; j += blockDim.x) { sT[j] = T[j]; sA[j] = all[j]; }
    for (int j = threadIdx.x; j <= J1; j += blockDim.x) cnt[j] = 0;
    __syncthreads();
    // level of a key: the first step removing it (steps are nested)
    auto level = [&](uint64_t key) {
        int j = 0;
        while (j < J1 && !sA[j] && key >= sT[j]) j++;
        return j;
    };
    for (int64_t s = blockIdx.x; s < nS; s += gridDim.x) {
        const int32_t vo = S[s];
        const int64_t u = inv[vo];
        int32_t *keys = tab + 2 * cap * s, *lev = keys + cap;
        const int vlev = mode == 1 ? level(aw_mix64(st ^ (uint64_t)(uint32_t)vo)) : J1;   // v itself survives < vlev
        for (int64_t e = rowptr[u] + threadIdx.x; e < rowptr[u + 1]; e += blockDim.x) {
            const uint32_t xo = (uint32_t)perm[col[e]];
            const uint64_t id = mode == 0 ? ((((uint64_t)min((uint32_t)vo, xo)) << 32) | max((uint32_t)vo, xo))
                                          : (uint64_t)xo;
            const int L = min(level(aw_mix64(st ^ id)), vlev);
            if (L == 0) continue;
            const int32_t c = comm_orig[xo];
            uint32_t h = ((uint32_t)c * 0x9E3779B1u) & (uint32_t)(cap - 1);
            for (;;) {                                 // insert c (keys start at INT32_MIN = empty)
                const int32_t old = atomicCAS(keys + h, INT32_MIN, c);
                if (old == INT32_MIN || old == c) break;
                h = (h + 1) & (uint32_t)(cap - 1);
            }
            atomicMax(lev + h, L);
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < cap; i += blockDim.x)
            if (keys[i] != INT32_MIN) atomicAdd(&cnt[lev[i]], 1);
        __syncthreads();
        if (threadIdx.x == 0) {   // zeta_j = #{level > j}: suffix sums
            int acc = 0;
            for (int j = J1; j >= 1; j--) {
                acc += cnt[j];
                zeta[(int64_t)(j - 1) * nS + s] = acc;
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j <= J1; j += blockDim.x) cnt[j] = 0;
        __syncthreads();
    }
}

__global__ void k_aw_init(int32_t *tab, int64_t cap, int64_t nS) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap * nS; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / cap, k = i % cap;
        tab[2 * cap * s + k] = INT32_MIN;    // empty key
        tab[2 * cap * s + cap + k] = 0;      // level
    }
}

// degrees of the vertices of S (original ids)
__global__ void k_aw_deg(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ inv,
                         const int32_t *__restrict__ S, int64_t nS, int64_t *deg) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nS; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = inv[S[s]];
        deg[s] = rowptr[u + 1] - rowptr[u];
    }
}
cudaError_t launch_awcc_degrees(Ctx &c, const int32_t *S_dev, int64_t nS, int64_t *deg_dev) {
    k_aw_deg<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nS + 255) / 256, 148)), 256, 0, c.stream>>>(
        c.rowptr, c.inv, S_dev, nS, deg_dev);
    c.launches++;
    return cudaGetLastError();
}

// scratch bytes of launch_awcc_trial for M items
size_t awcc_scratch_bytes(int64_t M, int J1, int64_t cap, int64_t nS) {
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)std::max<int64_t>(M, 1),
                                   0, 64);
    return 2 * kAwBins * 8 + 3 * (size_t)J1 * 8 + 8 * (size_t)cap * nS + 16 * (size_t)std::max<int64_t>(M, 1) + need +
           16 * 256;
}

// one trial: thresholds, then zeta[J1][nS] on the device
cudaError_t launch_awcc_trial(Ctx &c, const int32_t *S_dev, int64_t nS, int mode, int step_pct, int J1,
                              uint64_t st, int32_t *zeta_dev, void *scratch, size_t scratch_bytes, int64_t cap) {
    cudaError_t e;
    const int64_t n = c.n;
    const int64_t M = mode == 0 ? c.nnz / 2 : n;
    AwItems it{c.rowptr, c.col, c.perm, n, mode, st};
    // scratch: hist u32[bins] | slot i32[bins] | cursor u64[J1] | T u64[J1] | all i32[J1] | table | gathered keys | cub
    char *p = (char *)scratch;
    auto carve = [&](size_t b) { char *q = p; p += (b + 255) & ~(size_t)255; return (void *)q; };
    unsigned int *hist = (unsigned int *)carve(sizeof(unsigned int) * kAwBins);
    int *slot = (int *)carve(sizeof(int) * kAwBins);
    unsigned long long *cursor = (unsigned long long *)carve(sizeof(unsigned long long) * J1);
    uint64_t *T = (uint64_t *)carve(sizeof(uint64_t) * J1);
    int *all = (int *)carve(sizeof(int) * J1);
    int32_t *tab = (int32_t *)carve(sizeof(int32_t) * 2 * cap * nS);
    const int blocks = 148 * 8;
    if ((e = cudaMemsetAsync(hist, 0, sizeof(unsigned int) * kAwBins, c.stream))) return e;
    k_aw_hist<<<blocks, 256, 0, c.stream>>>(it, hist);
    c.launches++;
    // ranks -> bins (host: J1 <= 101 ranks over 4096 bins)
    std::vector<unsigned int> h(kAwBins);
    if ((e = cudaMemcpyAsync(h.data(), hist, sizeof(unsigned int) * kAwBins, cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    std::vector<int> hslot(kAwBins, -1), jbin(J1, -1), jall(J1, 0);
    std::vector<int64_t> jin(J1, 0), binoff;          // rank inside the bin; offsets of selected bins
    std::vector<int> selbins;
    {
        int64_t below = 0;
        int b = 0;
        for (int j = 0; j < J1; j++) {
            const int64_t r = ((int64_t)j * step_pct * M) / 100;
            if (r >= M) { jall[j] = 1; continue; }
            while (below + h[b] <= (uint64_t)r) { below += h[b]; b++; }
            jbin[j] = b;
            jin[j] = r - below;
            if (hslot[b] < 0) { hslot[b] = (int)selbins.size(); selbins.push_back(b); }
        }
    }
    int64_t tot = 0;
    std::vector<unsigned long long> hcur(J1, 0);
    for (size_t s = 0; s < selbins.size(); s++) {
        binoff.push_back(tot);
        hcur[s] = (unsigned long long)tot;
        tot += h[selbins[s]];
    }
    uint64_t *keys = (uint64_t *)carve(sizeof(uint64_t) * std::max<int64_t>(tot, 1));
    uint64_t *keys2 = (uint64_t *)carve(sizeof(uint64_t) * std::max<int64_t>(tot, 1));
    void *cub_tmp = p;
    if ((size_t)(p - (char *)scratch) > scratch_bytes) return cudaErrorMemoryAllocation;
    const size_t cub_bytes = scratch_bytes - (size_t)(p - (char *)scratch);
    std::vector<uint64_t> hT(J1, 0);
    if (!selbins.empty()) {
        if ((e = cudaMemcpyAsync(slot, hslot.data(), sizeof(int) * kAwBins, cudaMemcpyHostToDevice, c.stream))) return e;
        if ((e = cudaMemcpyAsync(cursor, hcur.data(), sizeof(unsigned long long) * selbins.size(),
                                 cudaMemcpyHostToDevice, c.stream))) return e;
        k_aw_gather<<<blocks, 256, 0, c.stream>>>(it, slot, cursor, keys);
        c.launches++;
        // the gathered bins are disjoint key ranges: one sort orders every bin
        size_t need = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, keys, keys2, (int)tot, 0, 64, c.stream);
        if (need > cub_bytes) return cudaErrorMemoryAllocation;
        cub::DeviceRadixSort::SortKeys(cub_tmp, need, keys, keys2, (int)tot, 0, 64, c.stream);
        c.launches++;
        std::vector<uint64_t> sorted(tot);
        if ((e = cudaMemcpyAsync(sorted.data(), keys2, sizeof(uint64_t) * tot, cudaMemcpyDeviceToHost, c.stream)))
            return e;
        if ((e = cudaStreamSynchronize(c.stream))) return e;
        for (int j = 0; j < J1; j++)
            if (!jall[j]) hT[j] = sorted[binoff[hslot[jbin[j]]] + jin[j]];
    }
    if ((e = cudaMemcpyAsync(T, hT.data(), sizeof(uint64_t) * J1, cudaMemcpyHostToDevice, c.stream))) return e;
    if ((e = cudaMemcpyAsync(all, jall.data(), sizeof(int) * J1, cudaMemcpyHostToDevice, c.stream))) return e;
    // hash tables: keys INT32_MIN (empty), levels 0
    k_aw_init<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((cap * nS + 255) / 256, 148 * 8)), 256, 0,
                c.stream>>>(tab, cap, nS);
    c.launches++;
    k_aw_zeta<<<(unsigned)std::min<int64_t>(nS, 148 * 4), 256, 0, c.stream>>>(
        c.rowptr, c.col, c.perm, c.inv, c.comm_in, S_dev, nS, mode, st, T, all, J1, tab, cap, zeta_dev);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

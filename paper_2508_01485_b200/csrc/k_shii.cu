// NEXT-4 — structural hole influence index of §VII.A:
// SHII(u_s) = (influenced outside C(u_s)) / (influenced), averaged over
// Monte-Carlo runs of a diffusion from the seed u_s (DESIGN reading C-31).
//
// Run r of model m draws from s_r = mix64(seed + (2r + m + 1) * 0xD1B54A32D192ED03)
// (SplitMix64 finaliser), on the caller's (original) ids:
//  IC: the coin of a -> b succeeds iff mix64(s_r ^ (a << 32 | b)) < floor(p 2^64)
//      (every edge when p >= 1); the influenced set is what the seed reaches over
//      the succeeding directed edges -- one level-synchronous BFS, each edge of
//      a newly active vertex tested once.
//  LT: b activates once (active neighbours) >= need_b = max(1, ceil(theta_b d_b)),
//      theta_b = mix64(s_r ^ b) / 2^64, the ceiling taken exactly on the 128-bit
//      product; level-synchronous: each new activation increments its inactive
//      neighbours' counters, the increment that reaches need_b activates b.
// Both processes are monotone, so the final set does not depend on the order of
// the atomics. Per (seed, run) the device returns {influenced, outside}.
#include "rs_internal.cuh"
#include <vector>

namespace rs {

__device__ __forceinline__ uint64_t sh_mix64(uint64_t z) {   // SplitMix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct ShArgs {
    const int64_t *rowptr;
    const int32_t *col;
    const int32_t *perm;        // internal -> original id
    const int32_t *comm_orig;   // communities in original order
    int64_t n;
    int model;                  // 0 IC, 1 LT
    int all_live;               // IC with p >= 1
    uint64_t thr;               // IC: floor(p 2^64)
    uint64_t st;                // run salt
    int32_t c0;                 // community of the seed
    unsigned int *act;          // n flags
    int32_t *cnt;               // n LT counters
    int32_t *list;              // activated vertices in activation order (internal ids)
    unsigned long long *ctr;    // [0] list tail, [1] outside count
};

// expand the frontier list[head, tail): a warp per frontier vertex
__global__ void __launch_bounds__(256) k_sh_level(ShArgs a, int64_t head, int64_t tail) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t f = head + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); f < tail; f += nw) {
        const int32_t u = a.list[f];
        const uint64_t uo = (uint64_t)(uint32_t)a.perm[u];
        for (int64_t e = a.rowptr[u] + lane; e < a.rowptr[u + 1]; e += 32) {
            const int32_t b = a.col[e];
            if (a.act[b]) continue;
            const uint32_t bo = (uint32_t)a.perm[b];
            bool fire;
            if (a.model == 0) {
                fire = a.all_live || sh_mix64(a.st ^ ((uo << 32) | bo)) < a.thr;
            } else {
                const uint64_t key = sh_mix64(a.st ^ (uint64_t)bo);
                const uint64_t d = (uint64_t)(a.rowptr[b + 1] - a.rowptr[b]);
                const uint64_t lo = key * d, hi = __umul64hi(key, d);
                const int64_t need = (int64_t)hi + (lo != 0 ? 1 : 0);   // ceil(key d / 2^64)
                const int32_t old = atomicAdd(&a.cnt[b], 1);
                fire = (int64_t)old + 1 == (need < 1 ? 1 : need);
            }
            if (fire && atomicExch(&a.act[b], 1u) == 0u) {
                a.list[atomicAdd(&a.ctr[0], 1ull)] = b;
                if (a.comm_orig[bo] != a.c0) atomicAdd(&a.ctr[1], 1ull);
            }
        }
    }
}

__global__ void k_sh_reset(unsigned int *act, const int32_t *list, int64_t len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        act[list[i]] = 0u;
}

__global__ void k_sh_seed(ShArgs a, int32_t u) {
    a.act[u] = 1u;
    a.list[0] = u;
    a.ctr[0] = 1ull;
    a.ctr[1] = 0ull;
}

// one diffusion from the seed (original id) `seed_o`; {influenced, outside} to out2
cudaError_t launch_shii_run(Ctx &c, int32_t seed_o, int model, double p, uint64_t st, unsigned int *act,
                            int32_t *cnt, int32_t *list, unsigned long long *ctr, int64_t out2[2]) {
    cudaError_t e;
    ShArgs a;
    a.rowptr = c.rowptr; a.col = c.col; a.perm = c.perm; a.comm_orig = c.comm_in; a.n = c.n;
    a.model = model;
    a.all_live = p >= 1.0;
    a.thr = p >= 1.0 ? 0ull : (uint64_t)ldexp(p, 64);
    a.st = st;
    a.act = act; a.cnt = cnt; a.list = list; a.ctr = ctr;
    int32_t u = 0, c0 = 0;
    if ((e = cudaMemcpyAsync(&u, c.inv + seed_o, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaMemcpyAsync(&c0, c.comm_in + seed_o, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    a.c0 = c0;
    if (model == 1 && (e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * c.n, c.stream))) return e;
    k_sh_seed<<<1, 1, 0, c.stream>>>(a, u);
    c.launches++;
    int64_t head = 0, tail = 1;
    unsigned long long h2[2] = {1ull, 0ull};
    while (head < tail) {
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((tail - head + 7) / 8, 148 * 16));
        k_sh_level<<<(unsigned)blocks, 256, 0, c.stream>>>(a, head, tail);
        c.launches++;
        if ((e = cudaMemcpyAsync(h2, ctr, sizeof(h2), cudaMemcpyDeviceToHost, c.stream))) return e;
        if ((e = cudaStreamSynchronize(c.stream))) return e;
        head = tail;
        tail = (int64_t)h2[0];
    }
    out2[0] = (int64_t)h2[0];
    out2[1] = (int64_t)h2[1];
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((tail + 255) / 256, 148 * 8));
    k_sh_reset<<<(unsigned)blocks, 256, 0, c.stream>>>(act, list, tail);   // act back to all-zero
    c.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- IC, batched
// Up to 64 (seed, run) diffusions of the IC model at once, bit j of a vertex's
// word = diffusion j: act[v] the diffusions in which v is active, fr[v] those in
// which v became active in the last level. A level takes every frontier vertex
// u (a warp each) and every edge u -> b: the diffusions j active at u, not yet
// at b, whose coin of u -> b succeeds (run r_j's salt, the same coin as one
// diffusion at a time) activate b. IC's influenced set is reachability over the
// succeeding edges, so it does not depend on the order of the atomics; the
// adjacency of a frontier vertex is read once per level for all 64 diffusions
// instead of once per diffusion.
struct ShBatchArgs {
    const int64_t *rowptr;
    const int32_t *col;
    const int32_t *perm;
    int all_live;
    uint64_t thr;
    uint64_t st[64];            // run salt of diffusion j
    unsigned long long *act;    // n
    unsigned long long *fr;     // n, this level's new bits (read and cleared)
    unsigned long long *fn;     // n, the next level's new bits
    const int32_t *cur;         // this level's frontier vertices
    int32_t *nxt;               // the next level's
    unsigned long long *ctr;    // next frontier length
};

__global__ void __launch_bounds__(256) k_shb_level(ShBatchArgs a, int64_t len) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t f = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); f < len; f += nw) {
        const int32_t u = a.cur[f];
        const unsigned long long F = a.fr[u];
        __syncwarp();
        if (lane == 0) a.fr[u] = 0ull;               // written only by this level's readers
        const uint64_t uo = (uint64_t)(uint32_t)a.perm[u];
        for (int64_t e = a.rowptr[u] + lane; e < a.rowptr[u + 1]; e += 32) {
            const int32_t b = a.col[e];
            unsigned long long cand = F & ~*(volatile unsigned long long *)(a.act + b);
            if (!cand) continue;
            unsigned long long live = cand;
            if (!a.all_live) {
                const uint64_t key = (uo << 32) | (uint64_t)(uint32_t)a.perm[b];
                live = 0ull;
                while (cand) {
                    const int j = __ffsll((long long)cand) - 1;
                    cand &= cand - 1ull;
                    if (sh_mix64(a.st[j] ^ key) < a.thr) live |= 1ull << j;
                }
            }
            if (!live) continue;
            const unsigned long long old = atomicOr(a.act + b, live);
            const unsigned long long newly = live & ~old;
            if (!newly) continue;
            const unsigned long long oldn = atomicOr(a.fn + b, newly);
            if (oldn == 0ull) a.nxt[atomicAdd(a.ctr, 1ull)] = b;
        }
    }
}

// the seeds: diffusion j starts at internal vertex seed[j]
__global__ void k_shb_seed(const int32_t *seed, int nb, unsigned long long *act, unsigned long long *fr, int32_t *cur,
                           unsigned long long *ctr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ctr[0] = 0ull;
    for (int j = 0; j < nb; j++) {
        const int32_t u = seed[j];
        act[u] |= 1ull << j;
        if (fr[u] == 0ull) cur[ctr[0]++] = u;
        fr[u] |= 1ull << j;
    }
}

// per diffusion j: influenced = active vertices, outside = those whose community
// differs from the seed's (c0[j]); lane l counts bits l and l + 32
__global__ void __launch_bounds__(256) k_shb_count(const unsigned long long *__restrict__ act,
                                                   const int32_t *__restrict__ perm,
                                                   const int32_t *__restrict__ comm_orig, int64_t n,
                                                   const int32_t *__restrict__ c0, int nb,
                                                   unsigned long long *out) {
    __shared__ unsigned int s_cnt[4 * 32];
    for (int i = threadIdx.x; i < 4 * 32; i += blockDim.x) s_cnt[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int32_t c0a = lane < nb ? c0[lane] : 0, c0b = lane + 32 < nb ? c0[lane + 32] : 0;
    unsigned int ia = 0, oa = 0, ib = 0, ob = 0;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += warps * 32) {
        const int64_t v0 = base + lane;
        const unsigned long long A0 = v0 < n ? act[v0] : 0ull;
        const int32_t cv0 = A0 ? comm_orig[perm[v0]] : 0;
        unsigned nzm = __ballot_sync(0xffffffffu, A0 != 0ull);
        while (nzm) {
            const int src = __ffs(nzm) - 1;
            nzm &= nzm - 1u;
            const unsigned long long A = __shfl_sync(0xffffffffu, A0, src);
            const int32_t cv = __shfl_sync(0xffffffffu, cv0, src);
            const unsigned a1 = (unsigned)(A >> lane) & 1u, a2 = (unsigned)(A >> (lane + 32)) & 1u;
            ia += a1;
            oa += a1 & (unsigned)(cv != c0a);
            ib += a2;
            ob += a2 & (unsigned)(cv != c0b);
        }
    }
    atomicAdd(&s_cnt[lane], ia);
    atomicAdd(&s_cnt[32 + lane], ib);
    atomicAdd(&s_cnt[64 + lane], oa);
    atomicAdd(&s_cnt[96 + lane], ob);
    __syncthreads();
    if (threadIdx.x < 64) {
        const int j = threadIdx.x;
        if (j < nb) {
            atomicAdd(out + 2 * j, (unsigned long long)s_cnt[j]);
            atomicAdd(out + 2 * j + 1, (unsigned long long)s_cnt[64 + j]);
        }
    }
}

// nb <= 64 IC diffusions: diffusion j from internal seed seed_d[j] (device) with
// run salt st[j]; c0_d[j] its community; {influenced, outside} per diffusion to
// out2 (host, 2 nb). buf: 3 n u64 + 2 n int32 + 64 B counters, device.
cudaError_t launch_shii_ic_batch(Ctx &c, int nb, const int32_t *seed_d, const int32_t *c0_d, const uint64_t *st,
                                 double p, unsigned long long *buf, int64_t *out2) {
    cudaError_t e;
    const int64_t n = c.n;
    unsigned long long *act = buf, *fa = buf + n, *fb = buf + 2 * n;
    int32_t *la = (int32_t *)(buf + 3 * n), *lb = la + n;
    unsigned long long *ctr = (unsigned long long *)(lb + n);   // [0] list length, [2, 2 + 2 nb) counts
    if ((e = cudaMemsetAsync(buf, 0, sizeof(unsigned long long) * 3 * n, c.stream))) return e;
    if ((e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * (2 + 128), c.stream))) return e;
    k_shb_seed<<<1, 32, 0, c.stream>>>(seed_d, nb, act, fa, la, ctr);
    c.launches++;
    ShBatchArgs a;
    a.rowptr = c.rowptr; a.col = c.col; a.perm = c.perm;
    a.all_live = p >= 1.0;
    a.thr = p >= 1.0 ? 0ull : (uint64_t)ldexp(p, 64);
    for (int j = 0; j < 64; j++) a.st[j] = j < nb ? st[j] : 0ull;
    a.act = act;
    a.ctr = ctr;
    unsigned long long len = 0;
    if ((e = cudaMemcpyAsync(&len, ctr, sizeof(len), cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    bool flip = false;
    while (len > 0) {
        a.fr = flip ? fb : fa;
        a.fn = flip ? fa : fb;
        a.cur = flip ? lb : la;
        a.nxt = flip ? la : lb;
        if ((e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), c.stream))) return e;
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(((int64_t)len + 7) / 8, 148 * 16));
        k_shb_level<<<(unsigned)blocks, 256, 0, c.stream>>>(a, (int64_t)len);
        c.launches++;
        if ((e = cudaMemcpyAsync(&len, ctr, sizeof(len), cudaMemcpyDeviceToHost, c.stream))) return e;
        if ((e = cudaStreamSynchronize(c.stream))) return e;
        flip = !flip;
    }
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    k_shb_count<<<(unsigned)blocks, 256, 0, c.stream>>>(act, c.perm, c.comm_in, n, c0_d, nb, ctr + 2);
    c.launches++;
    std::vector<unsigned long long> h(2 * (size_t)nb);
    if ((e = cudaMemcpyAsync(h.data(), ctr + 2, sizeof(unsigned long long) * 2 * nb, cudaMemcpyDeviceToHost,
                             c.stream)))
        return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    for (int j = 0; j < 2 * nb; j++) out2[j] = (int64_t)h[j];
    return cudaGetLastError();
}

}  // namespace rs

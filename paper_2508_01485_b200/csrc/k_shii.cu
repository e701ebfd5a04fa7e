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

}  // namespace rs

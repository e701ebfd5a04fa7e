// Multi-GPU exchange helpers (SURVEY §8(e) option 2): every rank
// runs Phase A on its own vertex range only, then the ranks exchange what the
// other phases read of the 2-hop neighbourhood. Of the P lists, only the
// oriented runs P+(x) travel (Phase E probes P+(x) of any predecessor x;
// P-(y) and P(u) are read only for owned y, u): packed back to back in vertex
// order at gpre[x] = sum of |P+| over the vertices before x, all-gathered by
// segment, and unpacked into each vertex's CSR slot on the other ranks.
#include "rs_internal.cuh"
#include "rs_device.cuh"
#include <cub/cub.cuh>

namespace rs {

__global__ void k_plus_count(const PRec *__restrict__ pc2, int64_t n, int64_t *cnt) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x)
        cnt[x] = x < n ? (int64_t)pr_plus(pc2[x]) : 0;
}

// gpre[0..n]: exclusive prefix of |P+(x)| (gpre in the context scratch, the
// counts and the scan's temporary storage after it)
cudaError_t launch_plus_prefix(Ctx &c, int64_t *gpre) {
    const int64_t n = c.n;
    int64_t *cnt = gpre + (n + 1);
    void *tmp = cnt + (n + 1);
    const size_t used = sizeof(int64_t) * 2 * (size_t)(n + 1);
    if (used > c.scratch_bytes) return cudaErrorMemoryAllocation;
    const size_t tmp_bytes = c.scratch_bytes - used;
    k_plus_count<<<148 * 4, 256, 0, c.stream>>>(c.pc2, n, cnt);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, gpre, (int)(n + 1), c.stream);
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::ExclusiveSum(tmp, need, cnt, gpre, (int)(n + 1), c.stream);
    c.launches += 2;
    return cudaGetLastError();
}

// a warp per vertex: pack the owned vertices' runs (UNPACK = false), or copy
// every other vertex's run from the gathered buffer into its slot (true)
template <bool UNPACK>
__global__ void k_plus_pack(const PRec *__restrict__ pc2, const int64_t *__restrict__ gpre, int64_t n, int64_t lo,
                            int64_t hi, int32_t *__restrict__ pplus, double *__restrict__ wps,
                            int32_t *__restrict__ pk_id, double *__restrict__ pk_w) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t first = UNPACK ? 0 : lo, last = UNPACK ? n : hi;
    for (int64_t x = first + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); x < last; x += nw) {
        if (UNPACK && x >= lo && x < hi) continue;
        const PRec r = pc2[x];
        const int pp = pr_plus(r);
        const int64_t slot = pr_start(r), g = gpre[x];
        for (int i = lane; i < pp; i += 32) {
            if (UNPACK) {
                pplus[slot + i] = pk_id[g + i];
                wps[slot + i] = pk_w[g + i];
            } else {
                pk_id[g + i] = pplus[slot + i];
                pk_w[g + i] = wps[slot + i];
            }
        }
    }
}

cudaError_t launch_plus_pack(Ctx &c, const int64_t *gpre, bool unpack) {
    if (unpack)
        k_plus_pack<true><<<148 * 8, 256, 0, c.stream>>>(c.pc2, gpre, c.n, c.head_lo, c.head_hi, c.pplus, c.wps,
                                                        c.pk_id, c.pk_w);
    else
        k_plus_pack<false><<<148 * 8, 256, 0, c.stream>>>(c.pc2, gpre, c.n, c.head_lo, c.head_hi, c.pplus, c.wps,
                                                         c.pk_id, c.pk_w);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

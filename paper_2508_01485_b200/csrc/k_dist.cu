// Multi-GPU exchange helpers (SURVEY §8(e) option 2): every rank
// runs Phase A on its own vertex range only, then the ranks exchange what the
// other phases read of the 2-hop neighbourhood, as compactly as the exact
// results allow; everything derivable is rebuilt locally from replicated data
// (the CSR, the labels) and the gathered cube-root rows:
// * per vertex {|P|, |P+|, |P+_T|} (12 B): VRec and PRec are rebuilt from them
//   (a_self = a_u(C(u)) from the gathered row; head / wide from d(u) and lab);
// * the oriented runs P+(x): only their ids travel (4 B per entry), packed back
//   to back in vertex order at gpre[x] = sum of |P+| over the vertices before x;
//   Phase E reads them there (PRec start rebased to gpre[x]) and the weights
//   a_x(c_z) from the gathered rows: nothing is copied back into slots;
// * the P-(y) lists of the heavy middle vertices (degree >= 128; 4 B per
//   entry), packed at gm[y]: Phase E deals their work items over the ranks;
// * the B table: only the pushed integer sums (8 B per cell, summed over the
//   ranks); Phase D reads them with a_w(c) from the gathered rows (no rebuild
//   pass over the n k cells on every rank).
// P(u) and the light P-(y) stay local: they are read only for a rank's own u, y.
#include "rs_internal.cuh"
#include "rs_device.cuh"
#include <cub/cub.cuh>

namespace rs {

// MINUS = false: |P+(x)| for every x; true: |P-(y)| for the heavy y < n_heavy, else 0
template <bool MINUS>
__global__ void k_run_count(const PRec *__restrict__ pc2, int64_t n, int64_t n_heavy, int64_t *cnt) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = 0;
        if (x < n && (!MINUS || x < n_heavy)) {
            const PRec r = pc2[x];
            v = MINUS ? (int64_t)(r.y - pr_plus(r)) : (int64_t)pr_plus(r);
        }
        cnt[x] = v;
    }
}

// gpre[0..n]: exclusive prefix of |P+(x)| (or, minus, of the heavy |P-(y)|);
// the counts and the scan's temporary storage in the context scratch
cudaError_t launch_run_prefix(Ctx &c, int64_t *gpre, bool minus) {
    const int64_t n = c.n;
    int64_t *cnt = (int64_t *)c.scratch;
    void *tmp = cnt + (n + 1);
    const size_t used = sizeof(int64_t) * (size_t)(n + 1);
    if (used > c.scratch_bytes) return cudaErrorMemoryAllocation;
    const size_t tmp_bytes = c.scratch_bytes - used;
    if (minus) k_run_count<true><<<148 * 4, 256, 0, c.stream>>>(c.pc2, n, c.e_nbig, cnt);
    else k_run_count<false><<<148 * 4, 256, 0, c.stream>>>(c.pc2, n, c.e_nbig, cnt);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, gpre, (int)(n + 1), c.stream);
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::ExclusiveSum(tmp, need, cnt, gpre, (int)(n + 1), c.stream);
    c.launches += 2;
    return cudaGetLastError();
}

// pack the owned vertices' P+ runs (two runs each, as Phase A wrote them in
// their slots) back to back at gpre[x]. A warp takes 32 consecutive vertices
// and deals their entries to the lanes 32 at a time (a warp scan of the run
// lengths; most runs are a few entries): the packed writes are coalesced.
// After the all-gather every rank holds all runs packed, and Phase E reads
// them there (PRec start rebased to gpre[x], k_rebase): no copy back into slots
__global__ void k_plus_pack(const PRec *__restrict__ pc2, const int64_t *__restrict__ gpre, int64_t lo, int64_t hi,
                            const int32_t *__restrict__ pplus, int32_t *__restrict__ pk_id) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x0 = lo + 32 * ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); x0 < hi; x0 += 32 * nw) {
        const int64_t x = x0 + lane;
        int cnt = 0;
        int64_t slot = 0;
        if (x < hi) {
            const PRec r = pc2[x];
            cnt = pr_plus(r);
            slot = pr_start(r);
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t g0 = total ? gpre[x0] : 0;       // the first vertex's packed offset
        for (int q0 = 0; q0 < total; q0 += 32) {
            const int q = q0 + lane;
            int j = 0;                                    // the first lane whose inclusive count exceeds q
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, j + s - 1);
                if (v <= q) j += s;
            }
            const int i = q - (__shfl_sync(0xffffffffu, incl, j) - __shfl_sync(0xffffffffu, cnt, j));
            const int64_t sj = __shfl_sync(0xffffffffu, (long long)slot, j);
            if (q < total) pk_id[g0 + q] = pplus[sj + i];
        }
    }
}

// a warp per owned heavy vertex: its P-(y) (the suffix of P(y) in its slot) at gm[y]
__global__ void k_minus_pack(const PRec *__restrict__ pc2, const int64_t *__restrict__ gm, int64_t lo, int64_t hi,
                             const int32_t *__restrict__ pidx, int32_t *__restrict__ pk) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t y = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); y < hi; y += nw) {
        const PRec r = pc2[y];
        const int pp = pr_plus(r), pm = r.y - pp;
        const int64_t at = pr_start(r) + pp, g = gm[y];
        for (int i = lane; i < pm; i += 32) pk[g + i] = pidx[at + i];
    }
}
cudaError_t launch_minus_pack(Ctx &c, const int64_t *gm) {
    const int64_t hi = std::min(c.head_hi, c.e_nbig);
    if (c.head_lo < hi) {
        k_minus_pack<<<148 * 8, 256, 0, c.stream>>>(c.pc2, gm, c.head_lo, hi, c.pidx, c.pk_m);
        c.launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_plus_pack(Ctx &c, const int64_t *gpre) {
    k_plus_pack<<<148 * 8, 256, 0, c.stream>>>(c.pc2, gpre, c.head_lo, c.head_hi, c.pplus, c.pk_id);
    c.launches++;
    return cudaGetLastError();
}

// every vertex's PRec start -> its packed offset gpre[x] (|P+_T| kept above the offset bits)
__global__ void k_rebase(PRec *__restrict__ pc2, const int64_t *__restrict__ gpre, int64_t n) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const long long s = pc2[x].start;
        pc2[x].start = (s & ~((1ll << kPrShift) - 1)) | gpre[x];
    }
}
cudaError_t launch_rebase(Ctx &c, const int64_t *gpre) {
    k_rebase<<<148 * 8, 256, 0, c.stream>>>(c.pc2, gpre, c.n);
    c.launches++;
    return cudaGetLastError();
}

// {|P(u)|, |P+(u)|, |P+_T(u)|} of the owned vertices
__global__ void k_vx_pack(const VRec *__restrict__ vrec, const PRec *__restrict__ pc2, int64_t lo, int64_t hi,
                          int32_t *__restrict__ vx) {
    for (int64_t u = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < hi; u += (int64_t)gridDim.x * blockDim.x) {
        const PRec r = pc2[u];
        vx[3 * u] = vrec[u].pcnt;
        vx[3 * u + 1] = pr_plus(r);
        vx[3 * u + 2] = pr_plus_t(r);
    }
}
cudaError_t launch_vx_pack(Ctx &c) {
    const int64_t m = std::max<int64_t>(c.head_hi - c.head_lo, 1);
    k_vx_pack<<<(unsigned)std::min<int64_t>((m + 255) / 256, 148 * 8), 256, 0, c.stream>>>(c.vrec, c.pc2, c.head_lo,
                                                                                         c.head_hi, c.vx);
    c.launches++;
    return cudaGetLastError();
}

// VRec and PRec of every other vertex, as Phase A writes them (write_vrec, the
// PRec of phase_a_vertex), from the exchanged counts and the gathered row
__global__ void k_vx_unpack(const int32_t *__restrict__ vx, const int64_t *__restrict__ rowptr,
                            const uint8_t *__restrict__ lab, const double *__restrict__ amat, int k, double wide_bound,
                            int64_t n, int64_t lo, int64_t hi, VRec *__restrict__ vrec, PRec *__restrict__ pc2) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        if (u >= lo && u < hi) continue;
        const uint32_t lu = lab[u];
        const int64_t beg = rowptr[u], d = rowptr[u + 1] - beg;
        VRec v;
        v.a_self = lu < (uint32_t)k ? amat[u * k + lu] : 0.0;
        v.pcnt = vx[3 * u];
        v.lab = (uint8_t)lu;
        v.head = (lu < (uint32_t)k && d >= 2) ? 1 : 0;
        v.wide = ((double)d * (double)d >= wide_bound) ? 1 : 0;
        v.pad = 0;
        vrec[u] = v;
        PRec r;
        r.x = pr_pack(vx[3 * u + 1], lu);
        r.y = vx[3 * u];
        r.start = beg | ((long long)vx[3 * u + 2] << kPrShift);
        pc2[u] = r;
    }
}
cudaError_t launch_vx_unpack(Ctx &c) {
    k_vx_unpack<<<148 * 8, 256, 0, c.stream>>>(c.vx, c.rowptr, c.lab, c.amat, c.k, wide_bound(c.k), c.n, c.head_lo,
                                              c.head_hi, c.vrec, c.pc2);
    c.launches++;
    return cudaGetLastError();
}

// the B table of the Type-II pull: {B_w[c] (summed pushes), Q_w(c) = a_w(c)^2};
// a thread per w reads its cube-root row (coalesced across threads) and writes
// its k records, one per column array (coalesced across threads per column)
__global__ void k_b_rebuild(const unsigned long long *__restrict__ bsum, const double *__restrict__ amat, int64_t n,
                            int k, BQL *__restrict__ bql) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
        for (int c = 0; c < k; c++) {
            const double a = __ldg(amat + w * k + c);
            BQL r;
            r.b = __ldg(bsum + (int64_t)c * n + w);
            r.Q = a * a;
            bql[(int64_t)c * n + w] = r;
        }
    }
}
cudaError_t launch_b_rebuild(Ctx &c) {
    k_b_rebuild<<<148 * 8, 256, 0, c.stream>>>(c.bsum, c.amat, c.n, c.k, c.bql);
    c.launches++;
    return cudaGetLastError();
}

// multi-GPU, before the limb reduce-scatter: the kHubStripes copies of the
// hub heads' limbs added into acc1 (limb by limb: both use the head's own
// 2- or 3-limb format, so the sum is the one the REDs would have made)
__global__ void k_fold_hubs(unsigned long long *__restrict__ acc1, const unsigned long long *__restrict__ hub,
                            int64_t n_hub) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n_hub; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long v = acc1[i];
#pragma unroll
        for (int s = 0; s < kHubStripes; s++) v += hub[(int64_t)s * 3 * n_hub + i];
        acc1[i] = v;
    }
}
cudaError_t launch_fold_hubs(Ctx &c) {
    if (c.n_hub == 0) return cudaSuccess;
    k_fold_hubs<<<148 * 2, 256, 0, c.stream>>>(c.acc1, c.acc_hub, c.n_hub);
    c.launches++;
    c.hubs_folded = true;
    return cudaGetLastError();
}

}  // namespace rs

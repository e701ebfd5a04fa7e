// Parity getters and statistics: exports of the bit-exact artefacts of the last
// rs_score in ORIGINAL vertex ids (the kernels work in the internal
// degree-descending numbering). Not on the timed path.
#include "rs_internal.cuh"
#include "rs_device.cuh"
#include <cub/cub.cuh>

namespace rs {

// out[v*k + c] = in[inv[v]*k + c]: rows back to original order
template <class T>
__global__ void k_permute_rows(const T *__restrict__ in, const int32_t *__restrict__ inv, int64_t n, int k, T *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * k; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / k, c = i % k;
        out[i] = in[(int64_t)inv[v] * k + c];
    }
}
cudaError_t launch_permute_i32(Ctx &c, const int32_t *in, int k, int32_t *out) {
    k_permute_rows<int32_t><<<148 * 8, 256, 0, c.stream>>>(in, c.inv, c.n, k, out);
    c.launches++;
    return cudaGetLastError();
}
cudaError_t launch_permute_f64(Ctx &c, const double *in, int k, double *out) {
    k_permute_rows<double><<<148 * 8, 256, 0, c.stream>>>(in, c.inv, c.n, k, out);
    c.launches++;
    return cudaGetLastError();
}
cudaError_t launch_permute_u64(Ctx &c, const unsigned long long *in, int64_t *out) {
    k_permute_rows<long long><<<148 * 8, 256, 0, c.stream>>>((const long long *)in, c.inv, c.n, 1, (long long *)out);
    c.launches++;
    return cudaGetLastError();
}

__global__ void k_row_total(const int32_t *__restrict__ f, int64_t n, int k, int32_t *tot) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        int t = 0;
        for (int c = 0; c < k; c++) t += f[u * k + c];
        tot[u] = t;
    }
}
// total over an already permuted (original-order) f
cudaError_t launch_counts_total(Ctx &c, const int32_t *f_orig, int32_t *total_dev) {
    k_row_total<<<148 * 4, 256, 0, c.stream>>>(f_orig, c.n, c.k, total_dev);
    c.launches++;
    return cudaGetLastError();
}

__global__ void k_border_flag(const VRec *__restrict__ vrec, const int32_t *__restrict__ inv, int64_t n, int32_t *flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        flag[v] = vrec[inv[v]].pcnt > 0;
}
__global__ void k_border_scatter(const int32_t *__restrict__ flag, const int32_t *__restrict__ pos, int64_t n,
                                 int32_t *bv) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        if (flag[u]) bv[pos[u]] = (int32_t)u;
}

cudaError_t launch_border_list(Ctx &c, int32_t *bv_dev, int64_t *nb_host) {
    const int64_t n = c.n;
    int32_t *flag = (int32_t *)c.scratch;
    int32_t *pos = flag + n;
    void *tmp = pos + n;
    size_t tmp_bytes = c.scratch_bytes - 2 * sizeof(int32_t) * (size_t)n;
    k_border_flag<<<148 * 4, 256, 0, c.stream>>>(c.vrec, c.inv, n, flag);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, flag, pos, (int)n, c.stream);
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::ExclusiveSum(tmp, need, flag, pos, (int)n, c.stream);
    if (bv_dev) k_border_scatter<<<148 * 4, 256, 0, c.stream>>>(flag, pos, n, bv_dev);
    c.launches += 3;
    int32_t lp = 0, lf = 0;
    cudaMemcpyAsync(&lp, pos + n - 1, 4, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(&lf, flag + n - 1, 4, cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    *nb_host = (int64_t)lp + lf;
    return e;
}

__global__ void k_pcnt64(const VRec *__restrict__ vrec, const int32_t *__restrict__ inv, int64_t n, int64_t *out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = vrec[inv[v]].pcnt;
}
// original row v <- internal P list of inv[v], mapped to original ids (unsorted)
// P(u): ascending at rowptr[u] in pidx (Phase A)
__device__ __forceinline__ int32_t p_entry(const int64_t *rowptr, const int32_t *pidx, int64_t u, int i) {
    return pidx[rowptr[u] + i];
}

__global__ void k_pred_copy(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ pidx,
                            const PRec *__restrict__ pc2, const int32_t *__restrict__ inv, const int32_t *__restrict__ perm,
                            const int64_t *__restrict__ off, int64_t n, int32_t *out) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) / 32) {
        const int32_t u = inv[v];
        const PRec pr = pc2[u];
        for (int i = lane; i < pr.y; i += 32) out[off[v] + i] = perm[p_entry(rowptr, pidx, u, i)];
    }
}

cudaError_t launch_pred_export(Ctx &c, int64_t *off_dev, int32_t *pred_dev, int64_t *nent_host) {
    const int64_t n = c.n;
    int64_t *cnt = (int64_t *)c.scratch;
    int64_t *off = cnt + (n + 1);
    void *tmp = off + (n + 1);
    size_t tmp_bytes = c.scratch_bytes - 2 * sizeof(int64_t) * (size_t)(n + 1);
    k_pcnt64<<<148 * 4, 256, 0, c.stream>>>(c.vrec, c.inv, n, cnt);
    cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), c.stream);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, off, (int)(n + 1), c.stream);
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    cub::DeviceScan::ExclusiveSum(tmp, need, cnt, off, (int)(n + 1), c.stream);
    c.launches += 2;
    int64_t tot = 0;
    cudaMemcpyAsync(&tot, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return e;
    *nent_host = tot;
    if (off_dev) cudaMemcpyAsync(off_dev, off, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, c.stream);
    if (pred_dev && tot) {
        int32_t *unsorted = nullptr;
        void *stmp = nullptr;
        if ((e = rs::dmalloc(&unsorted, sizeof(int32_t) * tot))) return e;
        k_pred_copy<<<148 * 8, 256, 0, c.stream>>>(c.rowptr, c.pidx, c.pc2, c.inv, c.perm, off, n, unsorted);
        size_t sneed = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, sneed, unsorted, pred_dev, tot, (int)n, off, off + 1, c.stream);
        if ((e = rs::dmalloc(&stmp, std::max<size_t>(sneed, 1)))) { cudaFree(unsorted); return e; }
        cub::DeviceSegmentedSort::SortKeys(stmp, sneed, unsorted, pred_dev, tot, (int)n, off, off + 1, c.stream);
        c.launches += 2;
        e = cudaStreamSynchronize(c.stream);
        cudaFree(unsorted);
        cudaFree(stmp);
    }
    return e;
}

// n_II(u) = sum_{w in P(u)} (f_w[c_u] - 1): every v != u of C(u) adjacent to w
// (all such v are foreign to w) closes a Type-II triad (u, w, v).
// Written at out[perm[u]] (original order).
__global__ void k_type2_counts(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ pidx,
                               const PRec *__restrict__ pc2, const VRec *__restrict__ vrec, const int32_t *__restrict__ f,
                               const int32_t *__restrict__ perm, int64_t n, int k, int64_t lo, int64_t hi,
                               int64_t *out) {
    const int lane = threadIdx.x & 31;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; u < n;
         u += ((int64_t)gridDim.x * blockDim.x) / 32) {
        const VRec r = vrec[u];
        const PRec pr = pc2[u];
        long long s = 0;
        if (r.head && u >= lo && u < hi)
            for (int i = lane; i < r.pcnt; i += 32)
                s += (long long)f[(int64_t)p_entry(rowptr, pidx, u, i) * k + r.lab] - 1;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[perm[u]] = s;
    }
}
cudaError_t launch_type2_counts(Ctx &c, int64_t *t2_dev) {
    k_type2_counts<<<148 * 8, 256, 0, c.stream>>>(c.rowptr, c.pidx, c.pc2, c.vrec, c.f, c.perm, c.n, c.k,
                                                  c.head_lo, c.head_hi, t2_dev);
    c.launches++;
    return cudaGetLastError();
}

cudaError_t launch_type1_export(Ctx &c, int64_t *t1_dev) { return launch_permute_u64(c, c.n1, t1_dev); }

__global__ void k_stats(const VRec *__restrict__ vrec, int64_t n, unsigned long long *scal) {
    unsigned long long nb = 0, np = 0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const int pc = vrec[u].pcnt;
        nb += pc > 0;
        np += pc;
    }
    for (int o = 16; o > 0; o >>= 1) {
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
        np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&scal[kScalNBorder], nb);
        atomicAdd(&scal[kScalNPred], np);
    }
}
cudaError_t launch_stats(Ctx &c, int64_t out[4]) {
    cudaMemsetAsync(c.scal + kScalNBorder, 0, 2 * sizeof(unsigned long long), c.stream);
    k_stats<<<148 * 2, 256, 0, c.stream>>>(c.vrec, c.n, c.scal);
    c.launches++;
    unsigned long long v[4];
    cudaMemcpyAsync(v, c.scal + kScalNBorder, sizeof(v), cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    for (int i = 0; i < 4; i++) out[i] = (int64_t)v[i];
    return e;
}

}  // namespace rs

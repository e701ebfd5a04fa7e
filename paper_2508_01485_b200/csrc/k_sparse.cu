// All-communities mode (NEXT-2): every community is a target
// (rs_set_communities with k = RS_ALL_COMMUNITIES), so k is the number of
// distinct communities -- thousands on LFR-style graphs -- and the dense n*k
// tables of the k <= 254 path (P:428 notes that limitation) are replaced by a
// sparse per-vertex community table: u's distinct neighbour communities,
// ascending, with their counts f_u(c), cube-root weights a_u(c) and B_u[c]
// limbs, stored in u's own CSR slot (L(u) <= d(u) entries, no scan needed).
//
//   Step 2a: the neighbours' community columns of every row are
//     sorted (the load-time length-class row sorters with a gather map,
//     k_setup.cu sort_rows) and run-length encoded: f_u(c) for the present
//     columns, T(u) = d(u) (every neighbour is in a target), L_all(u) = runs.
//   Step 2b (Eq. 3, Eq. 5, Algorithm 2): omega_u(c) from the same
//     closed form as Phase A (C-26) for the present columns; every absent column
//     has f = 0 and the same weight H(f_u) (L_all - 1), kept once per vertex.
//   Step 2c: omega_max over ALL n*k cells (C-7): the present
//     cells, plus the absent-column weight when L_all(u) < k.
//   Step 2d: P(u) in place, ascending (prefix P+(u) = the part below u,
//     the orientation of Phase E), and beside each w of P(u): a_u(c_w) (own
//     table), a_w(c_u) and the position of c_u in w's table (binary search in
//     w's table), the push of a_u(c_u) into B_w[c_u] (exact 2-limb RED, v in
//     P(w) iff w in P(v)) and n_II(u) += f_w(c_u) - 1 (Type-II triads).
// Steps 3-4 reuse Phase D / E / finalize / top-K with the per-edge weights
// instead of dense rows (rs_phase.cuh CdeArgs::pwr).
#include "rs_phase.cuh"
#include <cub/cub.cuh>

namespace rs {

// ------------------------------------------------------------ target ranking
// key = size * 2^32 + (2^31 - 1 - id): descending order = largest community
// first, ties by ascending id (C-15) -- the column order of the k <= 254
// path's top-k selection, extended to every community.
__global__ void k_rank_keys(const int32_t *__restrict__ hist, int64_t nbins, unsigned long long *key, int32_t *id,
                            unsigned long long *scal) {
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbins; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = hist[i];
        key[i] = h > 0 ? ((unsigned long long)h << 32) | (unsigned long long)(0x7fffffff - (int32_t)i) : 0ull;
        id[i] = (int32_t)i;
        cnt += h > 0;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&scal[kScalCnt0], cnt);
}
__global__ void k_code_all(const int32_t *__restrict__ id_sorted, int64_t nbins, const unsigned long long *scal,
                           int32_t *code) {
    const int64_t nc = (int64_t)scal[kScalCnt0];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nbins; r += (int64_t)gridDim.x * blockDim.x)
        code[id_sorted[r]] = r < nc ? (int32_t)r : -1;
}
// internal vertex r: community id, its column; every vertex is in a target
// (8-bit label 0 < k for the shared Phase E / getters code)
__global__ void k_labels_all(const int32_t *__restrict__ comm_in, const int32_t *__restrict__ perm,
                             const int32_t *__restrict__ code, int64_t n, int32_t *comm, int32_t *cid, uint8_t *lab) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = comm_in[perm[r]];
        comm[r] = c;
        cid[r] = code[c];
        lab[r] = 0;
    }
}

size_t sparse_rank_bytes(int64_t nbins) {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need, (unsigned long long *)nullptr,
                                              (unsigned long long *)nullptr, (int32_t *)nullptr, (int32_t *)nullptr,
                                              (int)nbins, 0, 64);
    return 2 * (8 * (size_t)nbins + 256) + 2 * (4 * (size_t)nbins + 256) + need + 256;
}

cudaError_t launch_set_communities_all(Ctx &c, int64_t max_comm, int64_t *nc_out) {
    const int64_t nbins = max_comm + 1;
    char *ap = (char *)c.csort;
    auto carve = [&](size_t b) { void *p = ap; ap += (b + 255) & ~(size_t)255; return p; };
    unsigned long long *key = (unsigned long long *)carve(8 * (size_t)nbins);
    unsigned long long *key_s = (unsigned long long *)carve(8 * (size_t)nbins);
    int32_t *id = (int32_t *)carve(4 * (size_t)nbins);
    int32_t *id_s = (int32_t *)carve(4 * (size_t)nbins);
    size_t need = c.csort_bytes - (size_t)(ap - (char *)c.csort);
    cudaMemsetAsync(c.chist, 0, sizeof(int32_t) * nbins, c.stream);
    cudaMemsetAsync(c.scal + kScalCnt0, 0, sizeof(unsigned long long), c.stream);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((std::max(c.n, nbins) + 255) / 256, 148 * 4));
    launch_comm_hist(c, nbins);   // community sizes (k_setup.cu)
    k_rank_keys<<<blocks, 256, 0, c.stream>>>(c.chist, nbins, key, id, c.scal);
    cub::DeviceRadixSort::SortPairsDescending(ap, need, key, key_s, id, id_s, (int)nbins, 0, 64, c.stream);
    k_code_all<<<blocks, 256, 0, c.stream>>>(id_s, nbins, c.scal, c.code32);
    k_labels_all<<<blocks, 256, 0, c.stream>>>(c.comm_in, c.perm, c.code32, c.n, c.comm_id, c.cid, c.lab);
    c.launches += 4;
    unsigned long long nc = 0;
    cudaMemcpyAsync(&nc, c.scal + kScalCnt0, sizeof(nc), cudaMemcpyDeviceToHost, c.stream);
    cudaError_t e = cudaStreamSynchronize(c.stream);
    if (e) return e;
    *nc_out = (int64_t)nc;
    c.h_targets_all.assign((size_t)nc, 0);
    if (nc) cudaMemcpyAsync(c.h_targets_all.data(), id_s, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, c.stream);
    // heads whose Type-I sum could pass 2^31 use 3 limbs: omega <= log2(L - 1) (L - 1)
    // with L <= min(k, d_max), so the k <= 254 bound with k_eff = min(k, d_max + 1)
    const int keff = (int)std::max<int64_t>(2, std::min<int64_t>((int64_t)nc, c.d_max + 1));
    launch_nwide(c, wide_bound(keff));
    // B grid (BQL): a <= (keff log2(keff - 1))^(1/3), B sums at most d_max of them
    const double bmax = std::cbrt(2147483648.0 / (2.0 * wide_bound(keff))) * (double)std::max<int64_t>(c.d_max, 1);
    int q = 40;
    while (q > 16 && bmax * std::ldexp(1.0, q) >= std::ldexp(1.0, 62)) q--;
    c.bq = q;
    return cudaStreamSynchronize(c.stream);
}

// ------------------------------------------------------------ Step 2 tables
struct SpArgs {
    const int64_t *__restrict__ rowptr;
    const int32_t *__restrict__ col;
    const int32_t *__restrict__ cid;
    const int32_t *__restrict__ slab;    // neighbour columns, each row ascending
    const double *__restrict__ l2t;
    int64_t l2n;
    int64_t vlo, nverts, n, nc;
    double wide_bound;
    SRec *__restrict__ srec;
    CtEnt *__restrict__ ctk;
    unsigned long long *__restrict__ ctb;
    int bq;
    double *__restrict__ aself;
    double *__restrict__ xsum;          // X(u) = sum_c f log2 f (getters recompute weights from it)
    int32_t *__restrict__ pidx;
    double *__restrict__ wps;           // a_u(c_w) beside w in P(u)
    double *__restrict__ pwr;           // a_w(c_u)
    int64_t *__restrict__ prv;          // position of c_u in w's table
    VRec *__restrict__ vrec;
    PRec *__restrict__ pc2;
    unsigned long long *__restrict__ n2s;
    unsigned long long *scal;
};

__device__ __forceinline__ double sp_lg2(const double *l2t, int64_t l2n, int64_t x) {
    return x < l2n ? __ldg(l2t + x) : log2((double)x);
}

// omega for a column with count fc of a row with T, L_all, X (Algorithm 2's
// closed form, the same expression as Phase A's weight_of with the adopted
// readings C-3, C-4, C-6: H = 0 exactly when one community remains)
__device__ __forceinline__ double sp_weight(const double *l2t, int64_t l2n, int fc, int64_t T, int L_all, double X) {
    const int others = L_all - (fc > 0);
    if (L_all < 2 || others < 2) return 0.0;
    const int64_t Y = T - fc;
    const double xc = fc > 1 ? (double)fc * sp_lg2(l2t, l2n, fc) : 0.0;
    const double H = sp_lg2(l2t, l2n, Y) - (X - xc) / (double)Y;
    const double w = H * (double)(L_all - 1);
    return w > 0.0 ? w : 0.0;
}

template <class GR>
__device__ __forceinline__ double sp_table_vertex(const SpArgs &a, int64_t u, GR &g) {
    const int64_t beg = a.rowptr[u], end = a.rowptr[u + 1];
    const int64_t d = end - beg;
    const int cu = a.cid[u];
    // runs of the sorted neighbour columns: start of run j -> ctk[beg + j]
    int L = 0;
    for (int64_t base = beg; base < end; base += GR::size) {
        const int64_t e = base + g.lane;
        int s = -1;
        bool st = false;
        if (e < end) {
            s = a.slab[e];
            st = (e == beg) || (a.slab[e - 1] != s);
        }
        int tot;
        const int r = g.rank(st, &tot);
        if (st) {
            a.ctk[beg + L + r].x = s;
            a.ctk[beg + L + r].y = (int)(e - beg);
        }
        L += tot;
    }
    g.sync();
    // counts = distance to the next run start; X = sum f log2 f
    double X = 0.0;
    for (int j0 = 0; j0 < L; j0 += GR::size) {
        const int j = j0 + (int)g.lane;
        int cnt = 0;
        if (j < L) {
            const int st = a.ctk[beg + j].y;
            const int nx = j + 1 < L ? a.ctk[beg + j + 1].y : (int)d;
            cnt = nx - st;
        }
        g.sync();
        if (j < L) {
            a.ctk[beg + j].y = cnt;
            if (cnt > 1) X += (double)cnt * sp_lg2(a.l2t, a.l2n, cnt);
        }
        g.sync();
    }
    X = g.sum(X);
    const double wabs = sp_weight(a.l2t, a.l2n, 0, d, L, X);   // every absent column
    double wmax = (L < a.nc) ? wabs : 0.0;
    double as = 0.0;
    int found = 0;
    for (int j = (int)g.lane; j < L; j += GR::size) {
        const int tx = a.ctk[beg + j].x, ty = a.ctk[beg + j].y;
        const double w = sp_weight(a.l2t, a.l2n, ty, d, L, X);
        const double ac = w > 0.0 ? cube_root(w) : 0.0;
        a.ctk[beg + j].a = ac;
        a.ctb[beg + j] = 0ull;
        wmax = w > wmax ? w : wmax;
        if (tx == cu) { as = ac; found = 1; }
    }
    as = g.sum(as);           // at most one lane holds a non-zero value: exact
    found = g.sum(found);
    if (!found) as = wabs > 0.0 ? cube_root(wabs) : 0.0;
    if (g.lane == 0) {
        SRec r;
        r.beg = beg;
        r.L = L;
        r.cid = cu;
        a.srec[u] = r;
        a.aself[u] = as;
        a.xsum[u] = X;
    }
    g.sync();
    return wmax;
}

__device__ __forceinline__ void block_max_scal(double v, unsigned long long *scal) {
    __shared__ double s[32];
    for (int o = 16; o > 0; o >>= 1) { const double x = __shfl_xor_sync(0xffffffffu, v, o); v = x > v ? x : v; }
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) m = s[i] > m ? s[i] : m;
        if (m > 0.0) atomic_max_nonneg(&scal[kScalOmegaMaxBits], m);
    }
}

template <int G>
__global__ void __launch_bounds__(256) k_sp_table_warp(SpArgs a) {
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    double wmax = 0.0;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb) {
        const double w = sp_table_vertex(a, a.vlo + i, g);
        wmax = w > wmax ? w : wmax;
    }
    block_max_scal(wmax, a.scal);
}
__global__ void __launch_bounds__(kCtaThreads) k_sp_table_cta(SpArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    CtaGroup g(s_i, s_u);
    double wmax = 0.0;
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) {
        const double w = sp_table_vertex(a, a.vlo + i, g);
        wmax = w > wmax ? w : wmax;
    }
    block_max_scal(wmax, a.scal);
}

// ------------------------------------------------------------ Step 2d lists
template <int U, class GR>
__device__ __forceinline__ void sp_lists_vertex(const SpArgs &a, int64_t u, GR &g) {
    const int64_t beg = a.rowptr[u], end = a.rowptr[u + 1];
    const int64_t d = end - beg;
    const SRec su = a.srec[u];
    const int cu = su.cid;
    const double au = a.aself[u];
    const unsigned long long qs = bq_quantize(au, a.bq);   // the B grid (BQL)
    const bool push = qs != 0ull;
    int pc = 0, pp = 0;
    unsigned long long n2 = 0;
    for (int64_t base = beg; base < end; base += GR::size * U) {
        int32_t x[U];
        SRec sx[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int64_t e = base + j * GR::size + g.lane;
            x[j] = e < end ? __ldcs(a.col + e) : -1;
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (x[j] >= 0) sx[j] = a.srec[x[j]];
            else sx[j] = SRec{0, 0, cu};
        }
        // binary searches of every foreign entry, advanced in lockstep so the
        // 2U dependent load chains overlap: c_u in x's table (x is adjacent to u,
        // so present) and c_x in u's own table
        bool fr[U];
        int lo_r[U], hi_r[U], lo_o[U], hi_o[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            fr[j] = x[j] >= 0 && sx[j].cid != cu;
            lo_r[j] = 0; hi_r[j] = fr[j] ? sx[j].L : 0;
            lo_o[j] = 0; hi_o[j] = fr[j] ? su.L : 0;
        }
        for (;;) {
            bool more = false;
#pragma unroll
            for (int j = 0; j < U; j++) more |= (lo_r[j] < hi_r[j]) | (lo_o[j] < hi_o[j]);
            if (!more) break;
            int vr[U], vo[U];
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int mr = (lo_r[j] + hi_r[j]) >> 1, mo = (lo_o[j] + hi_o[j]) >> 1;
                vr[j] = lo_r[j] < hi_r[j] ? __ldg(&a.ctk[sx[j].beg + mr].x) : 0;
                vo[j] = lo_o[j] < hi_o[j] ? __ldg(&a.ctk[beg + mo].x) : 0;
            }
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int mr = (lo_r[j] + hi_r[j]) >> 1, mo = (lo_o[j] + hi_o[j]) >> 1;
                if (lo_r[j] < hi_r[j]) { if (vr[j] < cu) lo_r[j] = mr + 1; else hi_r[j] = mr; }
                if (lo_o[j] < hi_o[j]) { if (vo[j] < sx[j].cid) lo_o[j] = mo + 1; else hi_o[j] = mo; }
            }
        }
        double ao[U], ar[U];
        int cr[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int64_t p = sx[j].beg + lo_r[j];
            ao[j] = fr[j] ? __ldg(&a.ctk[beg + lo_o[j]].a) : 0.0;   // a_u(c_x)
            ar[j] = fr[j] ? __ldg(&a.ctk[p].a) : 0.0;               // a_x(c_u)
            cr[j] = fr[j] ? __ldg(&a.ctk[p].y) : 1;               // f_x(c_u)
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (base + j * GR::size < end) {          // group-uniform
                int tot, totp;
                const int r = g.rank(fr[j], &tot);
                g.rank(fr[j] && x[j] < (int32_t)u, &totp);
                if (fr[j]) {
                    const int64_t pos = beg + pc + r;
                    const int64_t p = sx[j].beg + lo_r[j];
                    a.pidx[pos] = x[j];
                    a.wps[pos] = ao[j];
                    a.pwr[pos] = ar[j];
                    a.prv[pos] = p;
                    n2 += (unsigned long long)(cr[j] - 1);
                    if (push) atomicAdd(&a.ctb[p], qs);   // u in P(x): a_u(c_u) into B_x[c_u]
                }
                pc += tot;
                pp += totp;
            }
        }
    }
    n2 = g.sum(n2);
    if (g.lane == 0) {
        VRec r;
        r.a_self = au;
        r.pcnt = pc;
        r.lab = 0;
        r.head = d >= 2 ? 1 : 0;
        r.wide = ((double)d * (double)d >= a.wide_bound) ? 1 : 0;
        r.pad = 0;
        a.vrec[u] = r;
        PRec q;
        q.x = pr_pack(pp, 0u);            // all-communities mode: every label is 0 (k_sparse lab)
        q.y = pc;
        q.start = beg | ((long long)pp << kPrShift);   // P+(u) is one (target) run
        a.pc2[u] = q;
        a.n2s[u] = d >= 2 ? n2 : 0ull;
    }
}

template <int G, int U>
__global__ void __launch_bounds__(256, 4) k_sp_lists_warp(SpArgs a) {
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb)
        sp_lists_vertex<U>(a, a.vlo + i, g);
}
__global__ void __launch_bounds__(kCtaThreads) k_sp_lists_cta(SpArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    CtaGroup g(s_i, s_u);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) sp_lists_vertex<4>(a, a.vlo + i, g);
}

static SpArgs sp_args(Ctx &c, const double *l2t, int64_t l2n) {
    SpArgs a;
    a.rowptr = c.rowptr; a.col = c.col; a.cid = c.cid; a.slab = c.pplus;
    a.l2t = l2t; a.l2n = l2n;
    a.vlo = 0; a.nverts = 0; a.n = c.n; a.nc = c.k;
    const int keff = (int)std::max<int64_t>(2, std::min<int64_t>((int64_t)c.k, c.d_max + 1));
    a.wide_bound = wide_bound(keff);
    a.srec = c.srec; a.ctk = c.ctk; a.ctb = c.ctb; a.bq = c.bq; a.aself = c.aself; a.xsum = c.xsum;
    a.pidx = c.pidx; a.wps = c.wps; a.pwr = c.pwr; a.prv = c.prv; a.vrec = c.vrec; a.pc2 = c.pc2; a.n2s = c.n2s;
    a.scal = c.scal;
    return a;
}

template <class K>
static void sp_grid(Ctx &c, K kern, int64_t nverts, int gpb, cudaStream_t s, const SpArgs &a) {
    int64_t blocks = (nverts + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * 16);
    if (blocks < 1) return;
    kern<<<(unsigned)blocks, 256, 0, s>>>(a);
    c.launches++;
}

// neighbour columns sorted per row into c.pplus (unused by this mode's Phase E,
// which probes P+(x) in pidx directly); temporaries from the load arena. On the
// library stream: the caller forks the table bins after it.
cudaError_t launch_sparse_sort(Ctx &c) {
    int bits = 1;
    while (bits < 31 && (1ll << bits) < (int64_t)c.k) bits++;
    return sort_rows(c, c.col, c.cid, c.pplus, bits, c.arena, c.arena_bytes, c.n);
}

cudaError_t launch_sparse_tables(Ctx &c, const double *l2t, int64_t l2n) {
    SpArgs base = sp_args(c, l2t, l2n);
    // groups: [0,8):4 [8,32):8 [32,128):16 [128,2048):32 [2048,inf):CTA
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        SpArgs a = base;
        a.vlo = c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_sp_table_cta<<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (cls == 5) sp_grid(c, k_sp_table_warp<32>, a.nverts, 8, s, a);
        else if (cls >= 3) sp_grid(c, k_sp_table_warp<16>, a.nverts, 16, s, a);
        else if (cls >= 1) sp_grid(c, k_sp_table_warp<8>, a.nverts, 32, s, a);
        else sp_grid(c, k_sp_table_warp<4>, a.nverts, 64, s, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_sparse_lists(Ctx &c) {
    SpArgs base = sp_args(c, nullptr, 0);
    // [0,8):4x2 [8,16):4x4 [16,32):8x4 [32,64):16x4 [64,2048):32x4 [2048,inf):CTAx4
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        SpArgs a = base;
        a.vlo = c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_sp_lists_cta<<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (cls >= 4) sp_grid(c, k_sp_lists_warp<32, 4>, a.nverts, 8, s, a);
        else if (cls == 3) sp_grid(c, k_sp_lists_warp<16, 4>, a.nverts, 16, s, a);
        else if (cls == 2) sp_grid(c, k_sp_lists_warp<8, 4>, a.nverts, 32, s, a);
        else if (cls == 1) sp_grid(c, k_sp_lists_warp<4, 4>, a.nverts, 64, s, a);
        else sp_grid(c, k_sp_lists_warp<4, 2>, a.nverts, 64, s, a);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ getters (dense views)
// counts f[v][c] (original vertex order, column order = rs_get_targets) and
// T(v) = d(v); the output is zeroed by the caller
__global__ void k_sp_counts_dense(const SRec *__restrict__ srec, const CtEnt *__restrict__ ctk,
                                  const int64_t *__restrict__ rowptr, const int32_t *__restrict__ perm, int64_t n,
                                  int64_t k, int32_t *f, int32_t *total) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const SRec r = srec[u];
        const int64_t o = perm[u];
        if (f)
            for (int j = 0; j < r.L; j++) {
                const CtEnt t = ctk[r.beg + j];
                f[o * k + t.x] = t.y;
            }
        if (total) total[o] = (int32_t)(rowptr[u + 1] - rowptr[u]);
    }
}
cudaError_t launch_sparse_counts_dense(Ctx &c, int32_t *f_dev, int32_t *total_dev) {
    k_sp_counts_dense<<<148 * 4, 256, 0, c.stream>>>(c.srec, c.ctk, c.rowptr, c.perm, c.n, c.k, f_dev, total_dev);
    c.launches++;
    return cudaGetLastError();
}

// weights omega[v][c] for every cell (absent columns: the row's f = 0 weight),
// from the same X and expression Step 2b used
__global__ void k_sp_weights_dense(const SRec *__restrict__ srec, const CtEnt *__restrict__ ctk,
                                   const double *__restrict__ xsum, const int64_t *__restrict__ rowptr,
                                   const int32_t *__restrict__ perm, const double *__restrict__ l2t, int64_t l2n,
                                   int64_t n, int64_t k, double *w) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const SRec r = srec[u];
        const int64_t o = perm[u];
        const int64_t d = rowptr[u + 1] - rowptr[u];
        const double X = xsum[u];
        const double wabs = sp_weight(l2t, l2n, 0, d, r.L, X);
        for (int64_t c = 0; c < k; c++) w[o * k + c] = wabs;
        for (int j = 0; j < r.L; j++) {
            const CtEnt t = ctk[r.beg + j];
            w[o * k + t.x] = sp_weight(l2t, l2n, t.y, d, r.L, X);
        }
    }
}
cudaError_t launch_sparse_weights_dense(Ctx &c, const double *l2t, int64_t l2n, double *w_dev) {
    k_sp_weights_dense<<<148 * 4, 256, 0, c.stream>>>(c.srec, c.ctk, c.xsum, c.rowptr, c.perm, l2t, l2n, c.n, c.k,
                                                      w_dev);
    c.launches++;
    return cudaGetLastError();
}

// the sparse tables themselves in original vertex order (rs_get_comm_tables):
// row lengths, offsets by scan, then columns / counts / weights per row
__global__ void k_sp_len(const SRec *__restrict__ srec, const int32_t *__restrict__ perm, int64_t n, int64_t *len) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        len[perm[u]] = srec[u].L;
}
__global__ void k_sp_export(const SRec *__restrict__ srec, const CtEnt *__restrict__ ctk,
                            const double *__restrict__ xsum, const int64_t *__restrict__ rowptr,
                            const int32_t *__restrict__ perm, const int64_t *__restrict__ off,
                            const double *__restrict__ l2t, int64_t l2n, int64_t n, int32_t *cols, int32_t *cnt,
                            double *omega, double *omega_abs) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const SRec r = srec[u];
        const int64_t o = perm[u], dst = off[o];
        const int64_t d = rowptr[u + 1] - rowptr[u];
        const double X = xsum[u];
        for (int j = 0; j < r.L; j++) {
            const CtEnt t = ctk[r.beg + j];
            if (cols) cols[dst + j] = t.x;
            if (cnt) cnt[dst + j] = t.y;
            if (omega) omega[dst + j] = sp_weight(l2t, l2n, t.y, d, r.L, X);
        }
        if (omega_abs) omega_abs[o] = sp_weight(l2t, l2n, 0, d, r.L, X);
    }
}
cudaError_t launch_sparse_offsets(Ctx &c, int64_t *off_dev, int64_t *total) {
    int64_t *len = (int64_t *)c.scratch;
    void *tmp = (void *)(((uintptr_t)(len + c.n + 1) + 255) & ~(uintptr_t)255);
    const size_t used = (size_t)((char *)tmp - (char *)c.scratch);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, len, off_dev, (int)(c.n + 1), c.stream);
    if (used + need > c.scratch_bytes) return cudaErrorMemoryAllocation;
    cudaMemsetAsync(len + c.n, 0, sizeof(int64_t), c.stream);
    k_sp_len<<<148 * 4, 256, 0, c.stream>>>(c.srec, c.perm, c.n, len);
    cub::DeviceScan::ExclusiveSum(tmp, need, len, off_dev, (int)(c.n + 1), c.stream);
    c.launches += 2;
    cudaMemcpyAsync(total, off_dev + c.n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
    return cudaStreamSynchronize(c.stream);
}
cudaError_t launch_sparse_export(Ctx &c, const int64_t *off_dev, const double *l2t, int64_t l2n, int32_t *cols,
                                 int32_t *cnt, double *omega, double *omega_abs) {
    k_sp_export<<<148 * 4, 256, 0, c.stream>>>(c.srec, c.ctk, c.xsum, c.rowptr, c.perm, off_dev, l2t, l2n, c.n, cols,
                                              cnt, omega, omega_abs);
    c.launches++;
    return cudaGetLastError();
}

// n_II in original order (owned heads; 0 elsewhere)
__global__ void k_sp_type2(const unsigned long long *__restrict__ n2s, const int32_t *__restrict__ perm, int64_t n,
                           int64_t lo, int64_t hi, int64_t *out) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        out[perm[u]] = (u >= lo && u < hi) ? (int64_t)n2s[u] : 0;
}
cudaError_t launch_sparse_type2(Ctx &c, int64_t *t2_dev) {
    k_sp_type2<<<148 * 4, 256, 0, c.stream>>>(c.n2s, c.perm, c.n, c.head_lo, c.head_hi, t2_dev);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

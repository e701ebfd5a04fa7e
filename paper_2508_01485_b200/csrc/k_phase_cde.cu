// Phases C and D — Step 3 of Algorithm 1 for Type-II triads,
// the Type-I part being Phase E (k_phase_e.cu).
//
// Eq. 4's sum over valid triads (Eq. 6; Type-I and Type-II) is
// factorised so that no kernel enumerates Type-II triads one by one. With
// a_x(c) = omega_x(c)^(1/3) and P(u) the inter-community neighbours of u:
//   Type-II (C(v) = C(u); C-10):
//     sum_{w in P(u)} a_w(c_u)^2 * (B_w[c_u] - a_u(c_u)),
//     B_w[c] = sum_{v in P(w), col(v) = c} a_v(c)          (Phase C, Phase D)
// Phase C also orients G' by rank (|P|, id) for Phase E. Phase D adds the
// Type-I sum, divides by omega_max and d(u)(d(u)-1) once (the
// cube root of a product of normalised weights equals the product of cube
// roots divided by omega_max, C-8) and writes R in original vertex order.
// Sums are exact fixed point (C-12).
#include "rs_phase.cuh"

namespace rs {


// -1 padding of the two runs of P+(w) to multiples of 4 (aligned probes)
__device__ __forceinline__ void dense_pads(const CdeArgs &a, int64_t dw, int cap, int t, int no, int lane, int gs) {
    for (int i = lane; i < 8; i += gs) {
        const int64_t at = i < 4 ? (t + i < ceil4(t) ? dw + t + i : -1)
                                 : (no + (i - 4) < ceil4(no) ? dw + cap - 1 - (no + (i - 4)) : -1);
        if (at >= 0) {
            a.pd[at] = -1;
            a.wd[at] = 0.0;
        }
    }
}

// ============================================================================
// Phase C: B_w[c] for every column, Q_w[c] = a_w(c)^2, and the degree
// orientation of G' (P+(w): neighbours of larger (|P|, id)) for Phase E.
// ============================================================================
template <int U, class GR>
__device__ __forceinline__ void phase_c_vertex(const CdeArgs &a, int64_t w, GR &g) {
    const VRec rw = a.vrec[w];
    const int pc = rw.pcnt;
    const int64_t beg = a.rowptr[w];
    const int k = a.k;
    U128 B[8];
#pragma unroll
    for (int c = 0; c < 8; c++) B[c] = u128_zero();
    // w's own cube-root row: a_w(c_v) for every P+ entry v goes beside v (wd)
    const int64_t dw = a.dpos[w];
    const int cap = dcap(pc);
    double arow[8];
#pragma unroll
    for (int c = 0; c < 8; c++) arow[c] = c < k ? __ldg(a.amat + w * k + c) : 0.0;
    int ppc = 0, ppn = 0, pmc = 0;   // |P+_T|, |P+ \ P+_T|, |P-| so far
    for (int base = 0; base < pc; base += GR::size * U) {
        int32_t v[U];
        VRec rv[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            v[j] = i < pc ? a.pidx[beg + i] : -1;     // plain load: this kernel rewrites P lists
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (v[j] >= 0) rv[j] = a.vrec[v[j]];
            else { rv[j].lab = kOther; rv[j].pcnt = 0; rv[j].a_self = 0.0; }
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            const U128 q = fx_quantize(rv[j].a_self);
#pragma unroll
            for (int c = 0; c < 8; c++)
                if (rv[j].lab == c) B[c] = u128_add(B[c], q);
            if (base + j * GR::size < pc) {
                const bool plus = v[j] >= 0 && (rv[j].pcnt > pc || (rv[j].pcnt == pc && v[j] > (int32_t)w));
                const bool tgt = rv[j].lab < k;
                int tot, totn;
                const int r = g.rank(plus && tgt, &tot);
                const int rn = g.rank(plus && !tgt, &totn);
                if (plus) {
                    double wv = 0.0;
#pragma unroll
                    for (int c = 0; c < 8; c++) wv = (rv[j].lab == c) ? arow[c] : wv;
                    // target run ascending from the front, the rest descending from the back
                    const int64_t at = tgt ? dw + ppc + r : dw + cap - 1 - (ppn + rn);
                    a.pd[at] = v[j];
                    a.wd[at] = rv[j].wide ? -wv : wv;   // sign bit: v needs 3 limbs
                }
                // P-(w) compacted in place to the front of w's P list (every position
                // written has been read: the count of minus entries trails the reads)
                int totm;
                const int rm = g.rank(v[j] >= 0 && !plus, &totm);
                if (v[j] >= 0 && !plus) a.pidx[beg + pmc + rm] = v[j];
                ppc += tot;
                ppn += totn;
                pmc += totm;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 8; c++) B[c] = g.sum(B[c]);
    if (g.lane == 0) { PRec r; r.x = ppc + ppn; r.y = pc; r.start = dw | ((long long)ppc << kPrShift); a.pc2[w] = r; }
    if (pc == 0) return;   // w is in no P(u): its B/Q row is never read
    dense_pads(a, dw, cap, ppc, ppn, (int)g.lane, GR::size);
    for (int c = g.lane; c < k; c += GR::size) {
        U128 Bc = u128_zero();
#pragma unroll
        for (int j = 0; j < 8; j++) if (j == c) Bc = B[j];
        const double aw = a.amat[w * k + c];
        BQ r;
        r.B = fx_to_double(Bc);
        r.Q = aw * aw;
        a.bq[(int64_t)c * a.n + w] = r;
    }
}

// k > 8: B in shared memory as three 64-bit limbs per column (exact)
template <class GR>
__device__ __forceinline__ void phase_c_vertex_smem(const CdeArgs &a, int64_t w, GR &g, unsigned long long *sB) {
    const VRec rw = a.vrec[w];
    const int pc = rw.pcnt;
    const int64_t beg = a.rowptr[w];
    const int k = a.k;
    const int64_t dw = a.dpos[w];
    const int cap = dcap(pc);
    for (int c = g.lane; c < 3 * k; c += GR::size) sB[c] = 0ull;
    g.sync();
    int ppc = 0, ppn = 0, pmc = 0;
    for (int base = 0; base < pc; base += GR::size) {
        const int i = base + (int)g.lane;
        const bool valid = i < pc;
        int32_t v = 0;
        VRec rv;
        rv.lab = kOther; rv.pcnt = 0; rv.a_self = 0.0;
        if (valid) { v = a.pidx[beg + i]; rv = a.vrec[v]; }
        if (valid && rv.lab < k) fx_red3(sB + 3 * rv.lab, fx_quantize(rv.a_self));
        const bool plus = valid && (rv.pcnt > pc || (rv.pcnt == pc && v > (int32_t)w));
        const bool tgt = rv.lab < k;
        int tot, totn;
        const int r = g.rank(plus && tgt, &tot);
        const int rn = g.rank(plus && !tgt, &totn);
        if (plus) {
            const int64_t at = tgt ? dw + ppc + r : dw + cap - 1 - (ppn + rn);
            const double wv = tgt ? __ldg(a.amat + w * k + rv.lab) : 0.0;
            a.pd[at] = v;
            a.wd[at] = rv.wide ? -wv : wv;
        }
        int totm;
        const int rm = g.rank(valid && !plus, &totm);
        if (valid && !plus) a.pidx[beg + pmc + rm] = v;
        ppc += tot;
        ppn += totn;
        pmc += totm;
    }
    g.sync();
    if (g.lane == 0) { PRec r; r.x = ppc + ppn; r.y = pc; r.start = dw | ((long long)ppc << kPrShift); a.pc2[w] = r; }
    if (pc > 0) {
        dense_pads(a, dw, cap, ppc, ppn, (int)g.lane, GR::size);
        for (int c = g.lane; c < k; c += GR::size) {
            const double aw = a.amat[w * k + c];
            BQ r;
            r.B = fx_to_double(fx_from3(sB + 3 * c));
            r.Q = aw * aw;
            a.bq[(int64_t)c * a.n + w] = r;
        }
    }
    g.sync();
}

template <int G, int U, bool SMEM>
__global__ void __launch_bounds__(256, 4) k_phase_c_warp(CdeArgs a) {
    __shared__ unsigned long long sB[SMEM ? 8 * 3 * kMaxK : 1];
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb) {
        if constexpr (SMEM) phase_c_vertex_smem(a, a.vlo + i, g, sB + (threadIdx.x / 32) * 3 * kMaxK);
        else phase_c_vertex<U>(a, a.vlo + i, g);
    }
}

template <bool SMEM>
__global__ void __launch_bounds__(kCtaThreads, 4) k_phase_c_cta(CdeArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    __shared__ unsigned long long sB[SMEM ? 3 * kMaxK : 1];
    CtaGroup g(s_i, s_u);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) {
        if constexpr (SMEM) phase_c_vertex_smem(a, a.vlo + i, g, sB);
        else phase_c_vertex<4>(a, a.vlo + i, g);
    }
}

// ============================================================================
// Phase D: Type-II pull for every head (concurrent with Phase E: it needs only
// Phase C's B table), then the finalize pass adds the Type-I limbs and
// normalises.
// ============================================================================
template <int U, class GR>
__device__ __forceinline__ void phase_d_vertex(const CdeArgs &a, int64_t u, GR &g) {
    const VRec ru = a.vrec[u];
    if (!ru.head || u < a.head_lo || u >= a.head_hi) return;   // finalize writes R = 0
    const int cu = ru.lab;
    const double au = ru.a_self;
    const int pc = ru.pcnt;
    const PRec pr = a.pc2[u];
    const int pm = pc - pr.x;                  // P(u) = P-(u) (front of pidx) + P+(u) (pplus, two runs)
    const int pt = pm + pr_plus_t(pr);         // [pm, pt): target run; [pt, pc): the other run
    const int64_t dw = pr_start(pr), de = dw + dcap(pc) - 1 + pt;   // the other run: de - i, descending
    const int64_t beg = a.rowptr[u];
    U128 S = u128_zero();
    for (int base = 0; base < pc; base += GR::size * U) {
        int32_t w[U];
        BQ r[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            w[j] = i < pm ? __ldg(a.pidx + beg + i)
                          : (i < pt ? __ldg(a.pd + dw + i - pm) : (i < pc ? __ldg(a.pd + de - i) : -1));
        }
#pragma unroll
        for (int j = 0; j < U; j++)
            if (w[j] >= 0) r[j] = a.bq[(int64_t)cu * a.n + w[j]];
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (w[j] >= 0) {
                // B_w[c_u] includes a_u exactly, so the difference is >= 0 and exactly 0
                // when u is w's only neighbour in C(u) (Type-II needs v != u)
                const double t = r[j].Q * (r[j].B - au);
                S = u128_add(S, fx_quantize(t));
            }
        }
    }
    S = g.sum(S);
    if (g.lane == 0) a.t2[u] = make_ulonglong2(S.lo, S.hi);   // the exact Type-II sum
}

// R(u) = (Type-II + Type-I) / omega_max / (d(d-1)) for every owned vertex, in
// original order (0 for non-heads, C-22)
__global__ void __launch_bounds__(256) k_finalize(CdeArgs a) {
    const double wmax = __longlong_as_double((long long)a.scal[kScalOmegaMaxBits]);
    for (int64_t u = a.head_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < a.head_hi;
         u += (int64_t)gridDim.x * blockDim.x) {
        const VRec ru = a.vrec[u];
        double R = 0.0;
        if (ru.head) {
            const ulonglong2 t = a.t2[u];
            U128 S{t.x, t.y};
            const bool wide = a.any_wide && ru.wide;
            const unsigned long long *acc = a.acc1 + 3 * u;
            S = u128_add(S, wide ? fx_from3(acc) : fx_from2(acc));
            if (u < a.n_hub)
                for (int s = 0; s < kHubStripes; s++) {
                    const unsigned long long *h = a.acc_hub + 3 * ((int64_t)s * a.n_hub + u);
                    S = u128_add(S, wide ? fx_from3(h) : fx_from2(h));
                }
            const double d = (double)(a.rowptr[u + 1] - a.rowptr[u]);
            if (wmax > 0.0) R = fx_to_double(S) / wmax / (d * (d - 1.0));
        }
        a.score[a.perm[u]] = R;
    }
}

template <int G, int U>
__global__ void __launch_bounds__(256) k_phase_d_warp(CdeArgs a) {
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb)
        phase_d_vertex<U>(a, a.vlo + i, g);
}

__global__ void __launch_bounds__(kCtaThreads) k_phase_d_cta(CdeArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    CtaGroup g(s_i, s_u);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) phase_d_vertex<4>(a, a.vlo + i, g);
}

// ============================================================================
// launchers
// ============================================================================
template <class K>
static void launch_grid(Ctx &c, K kern, int64_t groups, int gpb, cudaStream_t s, const CdeArgs &a) {
    int64_t blocks = (groups + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * 16);
    if (blocks < 1) return;
    kern<<<(unsigned)blocks, 256, 0, s>>>(a);
    c.launches++;
}

// P-list phases: |P| is about a quarter of d, so a class uses a smaller group
// than in Phase A (lanes x loads per lane): [0,32):4x2 [32,64):4x4 [64,128):8x4
// [128,2048):32x4 [2048,inf):CTAx4
template <bool SMEM>
static void launch_c_bins(Ctx &c) {
    CdeArgs base = cde_args(c);
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        CdeArgs a = base;
        a.vlo = c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_phase_c_cta<SMEM><<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (SMEM || cls == 5) launch_grid(c, k_phase_c_warp<32, 4, SMEM>, a.nverts, 8, s, a);
        else if (cls == 4) launch_grid(c, k_phase_c_warp<8, 4, SMEM>, a.nverts, 32, s, a);
        else if (cls == 3) launch_grid(c, k_phase_c_warp<4, 4, SMEM>, a.nverts, 64, s, a);
        else launch_grid(c, k_phase_c_warp<4, 2, SMEM>, a.nverts, 64, s, a);
    }
}

cudaError_t launch_phase_c(Ctx &c) {
    if (c.k <= 8) launch_c_bins<false>(c);
    else launch_c_bins<true>(c);
    return cudaGetLastError();
}

cudaError_t launch_phase_d(Ctx &c) {
    CdeArgs base = cde_args(c);
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        CdeArgs a = base;
        a.vlo = c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_phase_d_cta<<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (cls == 5) launch_grid(c, k_phase_d_warp<32, 4>, a.nverts, 8, s, a);
        else if (cls == 4) launch_grid(c, k_phase_d_warp<8, 4>, a.nverts, 32, s, a);
        else if (cls == 3) launch_grid(c, k_phase_d_warp<4, 4>, a.nverts, 64, s, a);
        else launch_grid(c, k_phase_d_warp<4, 2>, a.nverts, 64, s, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_finalize(Ctx &c) {
    CdeArgs a = cde_args(c);
    const int64_t m = c.head_hi - c.head_lo;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 8));
    k_finalize<<<(unsigned)blocks, 256, 0, c.stream>>>(a);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

// Phase D -- Step 3 of Algorithm 1 for Type-II triads, the Type-I
// part being Phase E (k_phase_e.cu), and the finalize pass.
//
// Eq. 4's sum over valid triads (Eq. 6; Type-I and Type-II) is
// factorised so that no kernel enumerates Type-II triads one by one. With
// a_x(c) = omega_x(c)^(1/3) and P(u) the inter-community neighbours of u:
//   Type-II (C(v) = C(u); C-10):
//     sum_{w in P(u)} a_w(c_u)^2 * (B_w[c_u] - a_u(c_u)),
//     B_w[c] = sum_{v in P(w), col(v) = c} a_v(c)   (pushed by each v in Phase A)
// The finalize pass adds the Type-I sum, divides by omega_max and d(u)(d(u)-1)
// once (the cube root of a product of normalised weights equals
// the product of cube roots divided by omega_max, C-8) and writes R in original
// vertex order. Sums are exact fixed point (C-12).
#include "rs_phase.cuh"

namespace rs {


// ============================================================================
// Phase D: Type-II pull for every head (concurrent with Phase E: it needs only
// Phase A's B table), then the finalize pass adds the Type-I limbs and
// normalises.
// ============================================================================
// SPARSE (all-communities mode, k_sparse.cu): a_w(c_u) and the position of
// B_w[c_u] in w's community table are stored beside w in P(u)
template <int U, bool SPARSE, class GR>
__device__ __forceinline__ void phase_d_vertex(const CdeArgs &a, int64_t u, GR &g) {
    const VRec ru = a.vrec[u];
    if (!ru.head || u < a.head_lo || u >= a.head_hi) return;   // finalize writes R = 0
    const int cu = ru.lab;
    const double au = ru.a_self;
    const int pc = ru.pcnt;
    const int64_t beg = a.rowptr[u];
    const BQL *bcol = SPARSE ? nullptr : a.bql + (int64_t)cu * a.n;
    const unsigned long long qa = bq_quantize(au, a.bq);   // a_u(c_u) on the B grid
    U128 S = u128_zero();
    for (int base = 0; base < pc; base += GR::size * U) {
        int32_t w[U];
        double Q[U], diff[U];
        int64_t pv[U];
        unsigned long long bq[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            if constexpr (SPARSE) {
                w[j] = i < pc ? 0 : -1;
                pv[j] = i < pc ? __ldg(a.prv + beg + i) : 0;
                Q[j] = i < pc ? __ldg(a.pwr + beg + i) : 0.0;
            } else {
                w[j] = i < pc ? __ldg(a.pidx + beg + i) : -1;
            }
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            if constexpr (SPARSE) {
                if (w[j] >= 0) {
                    bq[j] = a.ctb[pv[j]];
                    Q[j] *= Q[j];
                }
            } else if (a.bsum) {
                // the pushed sums and w's cube-root row, read directly (no BQL rebuild)
                if (w[j] >= 0) {
                    bq[j] = __ldg(a.bsum + (int64_t)cu * a.n + w[j]);
                    const double aw = __ldg(a.amat + (int64_t)w[j] * a.k + cu);
                    Q[j] = aw * aw;
                }
            } else {
                if (w[j] >= 0) {
                    const BQL r = bcol[w[j]];
                    bq[j] = r.b;
                    Q[j] = r.Q;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (w[j] >= 0) {
                // dense: B_w[c_u] - a_u(c_u) in integers on the B grid (exact; 0 when
                // u is w's only neighbour in C(u), v != u), converted once
                diff[j] = bq_to_double(bq[j] - qa, a.bq);
                const double t = Q[j] * diff[j];
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
            const bool wide = ru.wide;
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

#ifndef RS_EXP_D_MINB
#define RS_EXP_D_MINB 6
#endif
template <int G, int U, bool SPARSE>
__global__ void __launch_bounds__(256, RS_EXP_D_MINB) k_phase_d_warp(CdeArgs a) {
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb)
        phase_d_vertex<U, SPARSE>(a, a.vlo + i, g);
}

template <bool SPARSE>
__global__ void __launch_bounds__(kCtaThreads) k_phase_d_cta(CdeArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    CtaGroup g(s_i, s_u);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) phase_d_vertex<4, SPARSE>(a, a.vlo + i, g);
}

// ============================================================================
// launchers
// ============================================================================
#ifndef RS_EXP_D_BLK
#define RS_EXP_D_BLK 16   // warp-class grids: 148 x RS_EXP_D_BLK blocks of 8 warps (grid-stride)
#endif
template <class K>
static void launch_grid(Ctx &c, K kern, int64_t groups, int gpb, cudaStream_t s, const CdeArgs &a) {
    int64_t blocks = (groups + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * RS_EXP_D_BLK);
    if (blocks < 1) return;
    kern<<<(unsigned)blocks, 256, 0, s>>>(a);
    c.launches++;
}

// Type-II pull bins (lanes x loads per lane; |P| is about a quarter of d):
// [0,32):4x2 [32,64):4x4 [64,128):8x4 [128,2048):32x4 [2048,inf):CTAx4
#ifndef RS_EXP_D_CTA_CLS
#define RS_EXP_D_CTA_CLS 6   // first degree class run by a CTA per head
#endif
template <bool SPARSE>
static cudaError_t launch_phase_d_t(Ctx &c) {
    CdeArgs base = cde_args(c);
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        CdeArgs a = base;
        a.vlo = std::max<int64_t>(c.bins.offset[cls], c.head_lo);   // owned heads of the class
        a.nverts = std::min<int64_t>(c.bins.offset[cls] + c.bins.count[cls], c.head_hi) - a.vlo;
        if (a.nverts <= 0) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= RS_EXP_D_CTA_CLS) {
            k_phase_d_cta<SPARSE><<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (cls >= 5) launch_grid(c, k_phase_d_warp<32, 4, SPARSE>, a.nverts, 8, s, a);
        else if (cls == 4) launch_grid(c, k_phase_d_warp<8, 4, SPARSE>, a.nverts, 32, s, a);
        else if (cls == 3) launch_grid(c, k_phase_d_warp<4, 4, SPARSE>, a.nverts, 64, s, a);
        else launch_grid(c, k_phase_d_warp<4, 2, SPARSE>, a.nverts, 64, s, a);
    }
    return cudaGetLastError();
}
cudaError_t launch_phase_d(Ctx &c) { return c.sparse ? launch_phase_d_t<true>(c) : launch_phase_d_t<false>(c); }

cudaError_t launch_finalize(Ctx &c) {
    CdeArgs a = cde_args(c);
    if (c.hubs_folded) a.n_hub = 0;   // multi-GPU: the stripes are already in acc1
    const int64_t m = c.head_hi - c.head_lo;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 8));
    k_finalize<<<(unsigned)blocks, 256, 0, c.stream>>>(a);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

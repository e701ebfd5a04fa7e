// Phases C, E, D — Step 3 of Algorithm 1: the robust-triad sum of
// Eq. 4 over valid triads (Eq. 6; Type-I and Type-II), factorised so
// that no kernel enumerates triads one by one except closed Type-I triangles.
//
// With a_x(c) = omega_x(c)^(1/3) and P(u) the inter-community neighbours of u:
//   Type-II (C(v) = C(u); C-10):
//     sum_{w in P(u)} a_w(c_u)^2 * (B_w[c_u] - a_u(c_u)),
//     B_w[c] = sum_{v in P(w), col(v) = c} a_v(c)          (Phase C, Phase D)
//   Type-I (closed triad over three communities):
//     every triangle {x, y, z} of G' (edges of G joining different
//     communities, so the three communities are pairwise distinct) gives the
//     term a_m(c_h) a_w(c_m) a_w(c_h) to head h for each ordered (head h,
//     mid m) of target vertices, w the third vertex              (Phase E)
// The unnormalised sum is divided by omega_max and d(u)(d(u)-1) once (P:286,
// P:291; the cube root of a product of normalised weights equals the product of
// cube roots divided by omega_max, C-8). Sums are exact fixed point (C-12).
#include "rs_internal.cuh"
#include "rs_device.cuh"

namespace rs {

struct CdeArgs {
    const int64_t *__restrict__ rowptr;
    const int32_t *__restrict__ verts;
    int64_t nverts;
    int64_t n;
    int32_t k;
    const double *__restrict__ omega;
    const VRec *__restrict__ vrec;
    const int32_t *__restrict__ pidx;
    int32_t *__restrict__ pplus;
    int32_t *__restrict__ ppcnt;
    BQ *__restrict__ bq;
    unsigned long long *__restrict__ acc1;
    unsigned long long *__restrict__ n1;
    double *__restrict__ score;
    unsigned long long *scal;
    int64_t head_lo, head_hi;   // owned head range (multi-GPU); [0, n) on one GPU
};

// ============================================================================
// Phase C: B_w[c] for every column, Q_w[c] = a_w(c)^2, and the degree
// orientation of G' (P+(w): neighbours of larger (|P|, id)) for Phase E.
// ============================================================================
template <class GR>
__device__ __forceinline__ void phase_c_vertex(const CdeArgs &a, int64_t w, GR &g) {
    const VRec rw = a.vrec[w];
    const int pc = rw.pcnt;
    const int64_t beg = a.rowptr[w];
    const int k = a.k;
    U128 B[8];
#pragma unroll
    for (int c = 0; c < 8; c++) B[c] = u128_zero();
    int ppc = 0;
    for (int base = 0; base < pc; base += GR::size) {
        const int i = base + (int)g.lane;
        const bool valid = i < pc;
        int32_t v = 0;
        VRec rv;
        rv.lab = kOther; rv.pcnt = 0; rv.a_self = 0.0;
        if (valid) { v = __ldg(a.pidx + beg + i); rv = a.vrec[v]; }
        const U128 q = fx_quantize(rv.a_self);
#pragma unroll
        for (int c = 0; c < 8; c++)
            if (rv.lab == c) B[c] = u128_add(B[c], q);
        const bool plus = valid && (rv.pcnt > pc || (rv.pcnt == pc && v > (int32_t)w));
        int tot;
        const int r = g.rank(plus, &tot);
        if (plus) a.pplus[beg + ppc + r] = v;
        ppc += tot;
    }
#pragma unroll
    for (int c = 0; c < 8; c++) B[c] = g.sum(B[c]);
    if (g.lane == 0) a.ppcnt[w] = ppc;
    if (pc == 0) return;   // w is in no P(u): its B/Q row is never read
    for (int c = g.lane; c < k; c += GR::size) {
        U128 Bc = u128_zero();
#pragma unroll
        for (int j = 0; j < 8; j++) if (j == c) Bc = B[j];
        const double aw = cbrt(a.omega[w * k + c]);
        BQ r;
        r.B = fx_to_double(Bc);
        r.Q = aw * aw;
        a.bq[w * k + c] = r;
    }
}

// k > 8: B in shared memory as three 64-bit limbs per column (exact)
template <class GR>
__device__ __forceinline__ void phase_c_vertex_smem(const CdeArgs &a, int64_t w, GR &g, unsigned long long *sB) {
    const VRec rw = a.vrec[w];
    const int pc = rw.pcnt;
    const int64_t beg = a.rowptr[w];
    const int k = a.k;
    for (int c = g.lane; c < 3 * k; c += GR::size) sB[c] = 0ull;
    g.sync();
    int ppc = 0;
    for (int base = 0; base < pc; base += GR::size) {
        const int i = base + (int)g.lane;
        const bool valid = i < pc;
        int32_t v = 0;
        VRec rv;
        rv.lab = kOther; rv.pcnt = 0; rv.a_self = 0.0;
        if (valid) { v = __ldg(a.pidx + beg + i); rv = a.vrec[v]; }
        if (valid && rv.lab < k) fx_red3(sB + 3 * rv.lab, fx_quantize(rv.a_self));
        const bool plus = valid && (rv.pcnt > pc || (rv.pcnt == pc && v > (int32_t)w));
        int tot;
        const int r = g.rank(plus, &tot);
        if (plus) a.pplus[beg + ppc + r] = v;
        ppc += tot;
    }
    g.sync();
    if (g.lane == 0) a.ppcnt[w] = ppc;
    if (pc > 0) {
        for (int c = g.lane; c < k; c += GR::size) {
            const double aw = cbrt(a.omega[w * k + c]);
            BQ r;
            r.B = fx_to_double(fx_from3(sB + 3 * c));
            r.Q = aw * aw;
            a.bq[w * k + c] = r;
        }
    }
    g.sync();
}

template <int G, bool SMEM>
__global__ void __launch_bounds__(256) k_phase_c_warp(CdeArgs a) {
    __shared__ unsigned long long sB[SMEM ? 8 * 3 * kMaxK : 1];
    WarpGroup<G> g;
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb) {
        if constexpr (SMEM) phase_c_vertex_smem(a, a.verts[i], g, sB + (threadIdx.x / 32) * 3 * kMaxK);
        else phase_c_vertex(a, a.verts[i], g);
    }
}

template <bool SMEM>
__global__ void __launch_bounds__(kCtaThreads) k_phase_c_cta(CdeArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    __shared__ unsigned long long sB[SMEM ? 3 * kMaxK : 1];
    CtaGroup g(s_i, s_u);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) {
        if constexpr (SMEM) phase_c_vertex_smem(a, a.verts[i], g, sB);
        else phase_c_vertex(a, a.verts[i], g);
    }
}

// ============================================================================
// Phase D: Type-II pull for every head + Type-I limbs + finalize.
// ============================================================================
template <class GR>
__device__ __forceinline__ void phase_d_vertex(const CdeArgs &a, int64_t u, GR &g, double wmax) {
    const VRec ru = a.vrec[u];
    if (!ru.head || u < a.head_lo || u >= a.head_hi) {
        if (g.lane == 0 && u >= a.head_lo && u < a.head_hi) a.score[u] = 0.0;
        return;
    }
    const int cu = ru.lab;
    const double au = ru.a_self;
    const int pc = ru.pcnt;
    const int64_t beg = a.rowptr[u];
    const int64_t d = a.rowptr[u + 1] - beg;
    const int k = a.k;
    U128 S = u128_zero();
    for (int base = 0; base < pc; base += GR::size) {
        const int i = base + (int)g.lane;
        if (i < pc) {
            const int32_t w = __ldg(a.pidx + beg + i);
            const BQ r = a.bq[(int64_t)w * k + cu];
            // B_w[c_u] includes a_u exactly, so the difference is >= 0 and exactly 0
            // when u is w's only neighbour in C(u) (Type-II needs v != u)
            const double t = r.Q * (r.B - au);
            S = u128_add(S, fx_quantize(t));
        }
    }
    S = g.sum(S);
    if (g.lane == 0) {
        S = u128_add(S, fx_from3(a.acc1 + 3 * u));
        double R = 0.0;
        if (wmax > 0.0) R = fx_to_double(S) / wmax / ((double)d * (double)(d - 1));
        a.score[u] = R;
    }
}

template <int G>
__global__ void __launch_bounds__(256) k_phase_d_warp(CdeArgs a) {
    WarpGroup<G> g;
    const double wmax = __longlong_as_double((long long)a.scal[kScalOmegaMaxBits]);
    const int64_t gpb = blockDim.x / G;
    for (int64_t i = blockIdx.x * gpb + threadIdx.x / G; i < a.nverts; i += (int64_t)gridDim.x * gpb)
        phase_d_vertex(a, a.verts[i], g, wmax);
}

__global__ void __launch_bounds__(kCtaThreads) k_phase_d_cta(CdeArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    CtaGroup g(s_i, s_u);
    const double wmax = __longlong_as_double((long long)a.scal[kScalOmegaMaxBits]);
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) phase_d_vertex(a, a.verts[i], g, wmax);
}

// ============================================================================
// Phase E: triangles of G' by degree orientation (each found once from its
// lowest-ranked vertex x: y in P+(x), z in P+(x) ∩ P+(y)), P+(x) in a
// shared-memory hash set, the (y, z) work of a warp flattened so all 32
// lanes stay busy; every triangle scatters its Type-I terms with exact
// fixed-point RED (order independent).
// ============================================================================
constexpr int kEWarps = 4;
constexpr int kETab = 2048;          // hash slots per warp (P+(x) up to kETab/2)

__device__ __forceinline__ double wa(const CdeArgs &a, int32_t q, int c) {
    return cbrt(__ldg(a.omega + (int64_t)q * a.k + c));
}

__device__ __noinline__ void emit_triangle(const CdeArgs &a, int32_t x, int32_t y, int32_t z) {
    const int32_t vtx[3] = {x, y, z};
    int lab[3];
#pragma unroll
    for (int i = 0; i < 3; i++) lab[i] = a.vrec[vtx[i]].lab;
#pragma unroll
    for (int h = 0; h < 3; h++) {
        if (lab[h] >= a.k) continue;
        const int32_t uh = vtx[h];
        if (uh < a.head_lo || uh >= a.head_hi) continue;
#pragma unroll
        for (int m = 0; m < 3; m++) {
            if (m == h || lab[m] >= a.k) continue;
            const int wi = 3 - h - m;
            const double t = wa(a, vtx[m], lab[h]) * wa(a, vtx[wi], lab[m]) * wa(a, vtx[wi], lab[h]);
            fx_red3(a.acc1 + 3 * (int64_t)uh, fx_quantize(t));
            atomicAdd(a.n1 + uh, 1ull);
        }
    }
}

__device__ __forceinline__ uint32_t hslot(int32_t z, uint32_t mask) {
    return ((uint32_t)z * 2654435769u >> 7) & mask;
}

__global__ void __launch_bounds__(kEWarps * 32) k_phase_e(CdeArgs a) {
    __shared__ int32_t tab[kEWarps][kETab];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *T = tab[wid];
    unsigned long long ntri = 0;
    for (;;) {
        int64_t qi = 0;
        if (lane == 0) qi = (int64_t)atomicAdd(&a.scal[kScalCnt0], 1ull);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (qi >= a.nverts) break;
        const int32_t x = a.verts[a.nverts - 1 - qi];   // heaviest degree classes first
        const int px = a.ppcnt[x];
        if (px < 2) continue;
        const int64_t bx = a.rowptr[x];
        const bool hashed = px <= kETab / 2;
        uint32_t mask = 0;
        if (hashed) {
            uint32_t size = 64;
            while (size < 2u * (uint32_t)px) size <<= 1;
            mask = size - 1;
            for (uint32_t s = lane; s < size; s += 32) T[s] = -1;
            __syncwarp();
            for (int i = lane; i < px; i += 32) {
                const int32_t z = a.pplus[bx + i];
                uint32_t h = hslot(z, mask);
                while (atomicCAS(&T[h], -1, z) != -1) h = (h + 1) & mask;
            }
            __syncwarp();
        }
        for (int i0 = 0; i0 < px; i0 += 32) {
            const int iy = i0 + lane;
            int32_t y = 0;
            int64_t by = 0;
            int ly = 0;
            if (iy < px) { y = a.pplus[bx + iy]; by = a.rowptr[y]; ly = a.ppcnt[y]; }
            int incl = ly;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - ly;
            for (int t0 = 0; t0 < total; t0 += 32) {
                const int t = t0 + lane;
                // owner lane j: first lane with incl_j > t
                int j = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = j + step - 1;
                    const int v = __shfl_sync(0xffffffffu, incl, cand);
                    if (v <= t) j += step;
                }
                const int32_t yj = __shfl_sync(0xffffffffu, y, j);
                const int64_t byj = __shfl_sync(0xffffffffu, by, j);
                const int exj = __shfl_sync(0xffffffffu, excl, j);
                bool hit = false;
                int32_t z = 0;
                if (t < total) {
                    z = a.pplus[byj + (t - exj)];
                    if (hashed) {
                        uint32_t h = hslot(z, mask);
                        for (;;) {
                            const int32_t s = T[h];
                            if (s == z) { hit = true; break; }
                            if (s == -1) break;
                            h = (h + 1) & mask;
                        }
                    } else {
                        int64_t lo = bx, hi = bx + px;
                        while (lo < hi) {
                            const int64_t mid = (lo + hi) >> 1;
                            if (a.pplus[mid] < z) lo = mid + 1; else hi = mid;
                        }
                        hit = lo < bx + px && a.pplus[lo] == z;
                    }
                }
                const unsigned hb = __ballot_sync(0xffffffffu, hit);
                ntri += __popc(hb);
                if (hit) emit_triangle(a, x, yj, z);
            }
        }
        __syncwarp();
    }
    if (lane == 0 && ntri) atomicAdd(&a.scal[kScalNTri], ntri);
}

// ============================================================================
// launchers
// ============================================================================
static CdeArgs cde_args(Ctx &c) {
    CdeArgs a;
    a.rowptr = c.rowptr; a.verts = nullptr; a.nverts = 0; a.n = c.n; a.k = c.k;
    a.omega = c.omega; a.vrec = c.vrec; a.pidx = c.pidx; a.pplus = c.pplus; a.ppcnt = c.ppcnt;
    a.bq = c.bq; a.acc1 = c.acc1; a.n1 = c.n1; a.score = c.score; a.scal = c.scal;
    a.head_lo = c.head_lo; a.head_hi = c.head_hi;
    return a;
}

template <class K>
static void launch_grid(Ctx &c, K kern, int64_t groups, int gpb, cudaStream_t s, const CdeArgs &a) {
    int64_t blocks = (groups + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * 16);
    if (blocks < 1) return;
    kern<<<(unsigned)blocks, 256, 0, s>>>(a);
    c.launches++;
}

// P-list phases: |P| is about a quarter of d, so a class uses a smaller group
// than in Phase A: [0,16):4 [16,64):8 [64,128):16 [128,2048):32 [2048,inf):CTA
template <bool SMEM>
static void launch_c_bins(Ctx &c) {
    CdeArgs base = cde_args(c);
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        CdeArgs a = base;
        a.verts = c.binv + c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_phase_c_cta<SMEM><<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (SMEM || cls == 5) launch_grid(c, k_phase_c_warp<32, SMEM>, a.nverts, 8, s, a);
        else if (cls == 4) launch_grid(c, k_phase_c_warp<16, SMEM>, a.nverts, 16, s, a);
        else if (cls >= 2) launch_grid(c, k_phase_c_warp<8, SMEM>, a.nverts, 32, s, a);
        else launch_grid(c, k_phase_c_warp<4, SMEM>, a.nverts, 64, s, a);
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
        a.verts = c.binv + c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (!a.nverts) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= 6) {
            k_phase_d_cta<<<(unsigned)std::min<int64_t>(a.nverts, 148 * 8), kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (cls == 5) launch_grid(c, k_phase_d_warp<32>, a.nverts, 8, s, a);
        else if (cls == 4) launch_grid(c, k_phase_d_warp<16>, a.nverts, 16, s, a);
        else if (cls >= 2) launch_grid(c, k_phase_d_warp<8>, a.nverts, 32, s, a);
        else launch_grid(c, k_phase_d_warp<4>, a.nverts, 64, s, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_phase_e(Ctx &c) {
    CdeArgs a = cde_args(c);
    a.verts = c.binv;
    a.nverts = c.n;
    cudaMemsetAsync(c.scal + kScalCnt0, 0, sizeof(unsigned long long), c.stream);
    k_phase_e<<<148 * 7, kEWarps * 32, 0, c.stream>>>(a);
    c.launches++;
    return cudaGetLastError();
}

}  // namespace rs

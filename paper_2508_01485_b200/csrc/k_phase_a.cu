// Phase A — one streaming pass over the CSR:
//   Step 1 border test (Algorithm 1 lines P:254-263),
//   Step 2a neighbour-community histogram f[u][i] over the k targets,
//   Step 2b weights omega_u(C_i) = H(L_i) * (L_all - 1) (Eq. 3, Eq. 5, Algorithm 2
//           P:457-482, closed form of Eq. H_optimal P:417 with exact zeros) and
//           their cube roots a_u(C_i) used by every triad term (Eq. 4),
//   Step 2c omega_max partial maxima,
//   Step 2d G' predecessor list P(u) = {x in N(u): C(x) != C(u)}, written
//           in place at offset rowptr[u] (no scan needed), ascending,
// and, once u's weights are known, the inputs of Step 3: the orientation of G'
// by internal id (P+(u) = the prefix of P(u) below u, split into its target run
// and the rest, with a_u(c_z) beside each z) and u's pushes of a_u(c_u) into
// B_w[c_u] for every w in P(u) (v in P(w) iff w in P(v)), exact 2-limb REDs.
// Labels are the 8-bit community codes of rs_set_communities; only vertices of
// two uncoded ("other") communities fall back to comparing full int32 ids.
// Degree-binned: a group of G lanes (or a whole CTA for hubs) owns a vertex;
// each lane keeps U independent loads in flight (the row walk is
// latency-bound otherwise).
#include "rs_internal.cuh"
#include "rs_device.cuh"

namespace rs {


struct PhaseAArgs {
    const int64_t *__restrict__ rowptr;
    const int32_t *__restrict__ col;
    const int32_t *__restrict__ comm;
    const uint8_t *__restrict__ lab;
    int64_t vlo;                        // first vertex of the degree-class range
    int64_t nverts;
    int32_t k;
    double wide_bound;                  // d^2 above which a head's Type-I sum needs 3 limbs
    int variant;                        // NEXT-3 (rs_score flags >> 16): 1 literal |L|, 2 |L| > 1 gate, 4 E_b max
    int parity;                         // 1: getter pass, writes only the parity tables f and omega
    int bq;                             // B table grid: 2^-bq
    int64_t n;
    int32_t *__restrict__ pplus;
    double *__restrict__ wps;
    PRec *__restrict__ pc2;
    BQL *__restrict__ bql;
    const double *__restrict__ l2t;     // log2 of small integers
    int64_t l2n;
    int32_t *__restrict__ f;
    double *__restrict__ omega;
    double *__restrict__ amat;
    VRec *__restrict__ vrec;
    int32_t *__restrict__ pidx;
    unsigned long long *scal;
};

__device__ __forceinline__ double lg2(const PhaseAArgs &a, int64_t x) {
    return x < a.l2n ? __ldg(a.l2t + x) : log2((double)x);
}

// |L| of column c: Algorithm 2's L_all - 1 (reading C-3), or with the
// NEXT-3 literal variant Eq. 2's communities other than c
__device__ __forceinline__ int L_of(const PhaseAArgs &a, int fc, int L_all) {
    return (a.variant & 1) ? L_all - (fc > 0) : L_all - 1;
}

// omega for column c of a row with T, L_all, X = sum f log2 f (Algorithm 2),
// given xc = f_c log2 f_c and lgY = log2(T - f_c)
__device__ __forceinline__ double weight_from(const PhaseAArgs &a, int fc, int T, int L_all, double X, double xc,
                                              double lgY) {
    const int others = L_all - (fc > 0);   // nonzero columns of L(u, .) besides c
    if (L_all < 2 || others < 2) return 0.0; // one remaining community: H = 0 exactly
    const int L = L_of(a, fc, L_all);
    if ((a.variant & 2) && L <= 1) return 0.0;   // NEXT-3: Algorithm 1's gate
    const int Y = T - fc;                    // > 0
    const double H = lgY - (X - xc) / (double)Y;
    const double w = H * (double)L;
    return w > 0.0 ? w : 0.0;                // canonical +0.0
}
__device__ __forceinline__ double weight_of(const PhaseAArgs &a, int fc, int T, int L_all, double X) {
    if (L_all < 2 || L_all - (fc > 0) < 2) return 0.0;
    const double xc = fc > 1 ? (double)fc * lg2(a, fc) : 0.0;
    return weight_from(a, fc, T, L_all, X, xc, lg2(a, T - fc));
}

// does cell (u, c) count towards omega_max? All cells (C-7), or with the NEXT-3
// variant only Algorithm 1's E_b edges: u border, |L| > 1, and c = C(u)
// or u has a neighbour in c
__device__ __forceinline__ bool in_max(const PhaseAArgs &a, int fc, int L_all, int c, int lu, int pc) {
    if (!(a.variant & 4)) return true;
    return pc > 0 && L_of(a, fc, L_all) > 1 && (c == lu || fc > 0);
}

__device__ __forceinline__ void write_vrec(const PhaseAArgs &a, int64_t u, double a_self, int pc, uint8_t lu,
                                           int64_t d) {
    VRec r;
    r.a_self = a_self;
    r.pcnt = pc;
    r.lab = lu;
    r.head = (lu < a.k && d >= 2) ? 1 : 0;
    r.wide = ((double)d * (double)d >= a.wide_bound) ? 1 : 0;   // = (u < n_wide), degree-descending ids
    r.pad = 0;
    a.vrec[u] = r;
}

// Step 3 inputs of u (after its weights and amat row are written and the group
// synchronised): B pushes, the P+ runs with a_u(c_z), the PRec record. P+(u)
// is written as its target run DESCENDING at [0, pt) followed by the other run
// ascending at [pt, pp): the entries below any y then form one contiguous range
// around pt (Phase E probes only z < y).
template <int U, class GR>
__device__ __forceinline__ void phase_a_lists(const PhaseAArgs &a, int64_t u, GR &g, int64_t beg, int pc, int pp,
                                              int pt, int lu) {
    const int k = a.k;
    const double *arow = a.amat + u * k;           // this group's writes, plain loads
    const unsigned long long qs = lu < k ? bq_quantize(arow[lu], a.bq) : 0ull;
    const bool push = qs != 0ull;
    BQL *bcol = a.bql + (int64_t)(push ? lu : 0) * a.n;
    int ct = 0, cn = 0;
    for (int base = 0; base < pc; base += GR::size * U) {
        int32_t v[U];
        int lv[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            v[j] = i < pc ? a.pidx[beg + i] : -1;  // plain load: written by this group
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            lv[j] = (v[j] >= 0 && i < pp) ? (int)__ldg(a.lab + v[j]) : (int)kOther;
        }
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
#ifndef RS_EXP_NO_BPUSH
            if (push && v[j] >= 0) atomicAdd(&bcol[v[j]].b, qs);   // u in P(v): a_u(c_u) into B_v[c_u]
#endif
            if (base + j * GR::size < pp) {                      // group-uniform
                const bool inp = v[j] >= 0 && i < pp;
                const bool tgt = inp && lv[j] < k;
                int tt, tn;
                const int rt = g.rank(tgt, &tt);
                const int rn = g.rank(inp && !tgt, &tn);
                if (inp) {
                    // target run descending down from pt - 1, the rest ascending from pt
                    const int64_t at = tgt ? beg + pt - 1 - (ct + rt) : beg + pt + cn + rn;
                    a.pplus[at] = v[j];
                    a.wps[at] = tgt ? arow[lv[j]] : 0.0;
                }
                ct += tt;
                cn += tn;
            }
        }
    }
    if (g.lane == 0) {
        PRec r;
        r.x = pp;
        r.y = pc;
        r.start = beg | ((long long)ct << kPrShift);
        a.pc2[u] = r;
    }
}

// k <= 8: per-lane register histogram.
template <int U, class GR>
__device__ __forceinline__ double phase_a_vertex(const PhaseAArgs &a, int64_t u, GR &g) {
    const int64_t beg = a.rowptr[u], end = a.rowptr[u + 1];
    const uint8_t lu = a.lab[u];
    const int32_t cfull = (lu == kOther) ? a.comm[u] : 0;
    const int k = a.k;
    // per-lane histogram as 16-bit counters packed in two words (columns 0-3,
    // 4-7): one shift and one add per neighbour. A lane sees at most
    // ceil(d / G) neighbours < 2^16 (launch_phase_a_impl falls back to the
    // shared-memory histogram when d_max >= 2^22).
    unsigned long long h0 = 0ull, h1 = 0ull;
    int pc = 0, pp = 0, pt = 0;   // |P(u)|, |P+(u)| (foreign neighbours below u), |P+_T(u)|
    for (int64_t base = beg; base < end; base += GR::size * U) {
        int32_t x[U];
        uint8_t lx[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int64_t e = base + j * GR::size + g.lane;
            x[j] = e < end ? __ldcs(a.col + e) : -1;
        }
#pragma unroll
        for (int j = 0; j < U; j++) lx[j] = x[j] >= 0 ? __ldg(a.lab + x[j]) : kOther;
#pragma unroll
        for (int j = 0; j < U; j++) {
            const bool valid = x[j] >= 0;
            bool foreign = valid && (lx[j] != lu);
            if (valid && lx[j] == kOther && lu == kOther) foreign = __ldg(a.comm + x[j]) != cfull;
            const unsigned l = lx[j];
            if (l < (unsigned)k) {
                const unsigned long long inc = 1ull << ((l & 3u) * 16u);
                if (l < 4u) h0 += inc; else h1 += inc;
            }
            if (base + j * GR::size < end) {          // group-uniform
                int tot, totp, tott;
                const int r = g.rank(foreign, &tot);
                g.rank(foreign && x[j] < (int32_t)u, &totp);
                g.rank(foreign && x[j] < (int32_t)u && l < (unsigned)k, &tott);
                if (foreign && !a.parity) a.pidx[beg + pc + r] = x[j];
                pc += tot;
                pp += totp;
                pt += tott;
            }
        }
    }
    int cnt[8];
    if (end - beg < 65536) {          // group totals still fit the 16-bit fields
        h0 = g.sum(h0);
        h1 = g.sum(h1);
#pragma unroll
        for (int c = 0; c < 4; c++) {
            cnt[c] = (int)((h0 >> (16 * c)) & 0xFFFFull);
            cnt[c + 4] = (int)((h1 >> (16 * c)) & 0xFFFFull);
        }
    } else {
#pragma unroll
        for (int c = 0; c < 4; c++) {
            cnt[c] = g.sum((int)((h0 >> (16 * c)) & 0xFFFFull));
            cnt[c + 4] = g.sum((int)((h1 >> (16 * c)) & 0xFFFFull));
        }
    }
    int T = 0, L_all = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        T += cnt[c];
        L_all += cnt[c] > 0;
    }
    // Algorithm 2's X = sum f log2 f and every column's log2(T - f) with ONE
    // round of log2-table loads: lane l takes the columns l, l + G, ... (a
    // vertex's weights are a dependent chain after its row walk; a second
    // round of loads there cost ~0.4 ms of Phase A), X by a group sum
    constexpr int NC = GR::size >= 8 ? 1 : 8 / GR::size;
    int fcs[NC];
    double xcs[NC], lys[NC];
    double xpart = 0.0;
#pragma unroll
    for (int i = 0; i < NC; i++) {
        const int c = (int)g.lane + i * GR::size;
        int fc = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) fc = (j == c) ? cnt[j] : fc;
        fcs[i] = fc;
        xcs[i] = fc > 1 ? (double)fc * lg2(a, fc) : 0.0;
        lys[i] = (c < k && T - fc > 0) ? lg2(a, T - fc) : 0.0;
        xpart += xcs[i];
    }
    const double X = g.sum(xpart);
    const int64_t d = end - beg;
    double wmax = 0.0, a_self = 0.0;
#pragma unroll
    for (int i = 0; i < NC; i++) {
        const int c = (int)g.lane + i * GR::size;
        if (c >= k) continue;
        const int fc = fcs[i];
        const double w = weight_from(a, fc, T, L_all, X, xcs[i], lys[i]);
        const double ac = w > 0.0 ? cube_root(w) : 0.0;
        if (a.parity) {            // the parity tables, written only for the getters
            a.omega[u * k + c] = w;
            a.f[u * k + c] = fc;
        } else {
            a.amat[u * k + c] = ac;
            a.bql[(int64_t)c * a.n + u].Q = ac * ac;
        }
        if (in_max(a, fc, L_all, c, lu, pc)) wmax = w > wmax ? w : wmax;
        if (c == (int)lu) a_self = ac;
    }
    if (a.parity) return wmax;
    const int owner = (lu < k) ? (int)(lu % GR::size) : 0;
    if ((int)g.lane == owner) write_vrec(a, u, a_self, pc, lu, d);
    g.sync();
    phase_a_lists<U>(a, u, g, beg, pc, pp, pt, lu);
    return wmax;
}

// k > 8: histogram in shared memory (one warp or one CTA per vertex)
template <int U, class GR>
__device__ __forceinline__ double phase_a_vertex_smem(const PhaseAArgs &a, int64_t u, GR &g, int *hist) {
    const int64_t beg = a.rowptr[u], end = a.rowptr[u + 1];
    const uint8_t lu = a.lab[u];
    const int32_t cfull = (lu == kOther) ? a.comm[u] : 0;
    const int k = a.k;
    for (int c = g.lane; c < k; c += GR::size) hist[c] = 0;
    g.sync();
    int pc = 0, pp = 0, pt = 0;
    for (int64_t base = beg; base < end; base += GR::size * U) {
        int32_t x[U];
        uint8_t lx[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int64_t e = base + j * GR::size + g.lane;
            x[j] = e < end ? __ldcs(a.col + e) : -1;
        }
#pragma unroll
        for (int j = 0; j < U; j++) lx[j] = x[j] >= 0 ? __ldg(a.lab + x[j]) : kOther;
#pragma unroll
        for (int j = 0; j < U; j++) {
            const bool valid = x[j] >= 0;
            bool foreign = valid && (lx[j] != lu);
            if (valid && lx[j] == kOther && lu == kOther) foreign = __ldg(a.comm + x[j]) != cfull;
            if (valid && lx[j] < k) atomicAdd(&hist[lx[j]], 1);
            if (base + j * GR::size < end) {
                int tot, totp, tott;
                const int r = g.rank(foreign, &tot);
                g.rank(foreign && x[j] < (int32_t)u, &totp);
                g.rank(foreign && x[j] < (int32_t)u && lx[j] < k, &tott);
                if (foreign && !a.parity) a.pidx[beg + pc + r] = x[j];
                pc += tot;
                pp += totp;
                pt += tott;
            }
        }
    }
    g.sync();
    // T, L_all and X = sum f log2 f over the k columns, lane-strided + group sums
    // (one round of log2-table loads instead of k in sequence per lane)
    int Tp = 0, Lp = 0;
    double Xp = 0.0;
    for (int c = g.lane; c < k; c += GR::size) {
        const int v = hist[c];
        Tp += v;
        Lp += v > 0;
        if (v > 1) Xp += (double)v * lg2(a, v);
    }
    const int T = g.sum(Tp), L_all = g.sum(Lp);
    const double X = g.sum(Xp);
    const int64_t d = end - beg;
    double wmax = 0.0;
    for (int c = g.lane; c < k; c += GR::size) {
        const int fc = hist[c];
        const double w = weight_of(a, fc, T, L_all, X);
        const double ac = w > 0.0 ? cube_root(w) : 0.0;
        if (a.parity) {
            a.omega[u * k + c] = w;
            a.f[u * k + c] = fc;
        } else {
            a.amat[u * k + c] = ac;
            a.bql[(int64_t)c * a.n + u].Q = ac * ac;
        }
        if (in_max(a, fc, L_all, c, lu, pc)) wmax = w > wmax ? w : wmax;
    }
    g.sync();
    if (a.parity) return wmax;
    if (g.lane == 0) {
        double as = 0.0;
        if (lu < k) { const double w = weight_of(a, hist[lu], T, L_all, X); as = w > 0.0 ? cube_root(w) : 0.0; }
        write_vrec(a, u, as, pc, lu, d);
    }
    g.sync();
    phase_a_lists<U>(a, u, g, beg, pc, pp, pt, lu);
    g.sync();
    return wmax;
}

__device__ __forceinline__ void block_max_to_scal(double v, unsigned long long *scal) {
    __shared__ double s[32];
    for (int o = 16; o > 0; o >>= 1) { double x = __shfl_xor_sync(0xffffffffu, v, o); v = x > v ? x : v; }
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) m = s[i] > m ? s[i] : m;
        if (m > 0.0) atomic_max_nonneg(&scal[kScalOmegaMaxBits], m);
    }
}

template <int G, int U, bool SMEM>
__global__ void __launch_bounds__(256) k_phase_a_warp(PhaseAArgs a) {
    __shared__ int hist[SMEM ? 8 * 256 : 1];
    WarpGroup<G> g;
    const int64_t groups_per_block = blockDim.x / G;
    const int64_t gid = blockIdx.x * groups_per_block + threadIdx.x / G;
    const int64_t ngroups = (int64_t)gridDim.x * groups_per_block;
    double wmax = 0.0;
    for (int64_t i = gid; i < a.nverts; i += ngroups) {
        const int64_t u = (a.vlo + i);
        double w;
        if constexpr (SMEM) w = phase_a_vertex_smem<U>(a, u, g, hist + (threadIdx.x / 32) * 256);
        else w = phase_a_vertex<U>(a, u, g);
        wmax = w > wmax ? w : wmax;
    }
    block_max_to_scal(wmax, a.scal);
}

template <bool SMEM>
__global__ void __launch_bounds__(kCtaThreads) k_phase_a_cta(PhaseAArgs a) {
    __shared__ int s_i[kCtaWarps + 1];
    __shared__ unsigned long long s_u[2 * kCtaWarps];
    __shared__ int hist[SMEM ? 256 : 1];
    CtaGroup g(s_i, s_u);
    double wmax = 0.0;
    for (int64_t i = blockIdx.x; i < a.nverts; i += gridDim.x) {
        const int64_t u = (a.vlo + i);
        double w;
        if constexpr (SMEM) w = phase_a_vertex_smem<4>(a, u, g, hist);
        else w = phase_a_vertex<4>(a, u, g);
        wmax = w > wmax ? w : wmax;
    }
    block_max_to_scal(wmax, a.scal);
}

#ifndef RS_EXP_A_BLK
#define RS_EXP_A_BLK 16   // warp-class grids: 148 x RS_EXP_A_BLK blocks of 8 warps (grid-stride)
#endif
template <int G, int U, bool SMEM>
static void launch_warp_bin(Ctx &c, PhaseAArgs a, cudaStream_t s) {
    const int64_t gpb = 256 / G;
    int64_t blocks = (a.nverts + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * RS_EXP_A_BLK);
    if (blocks < 1) return;
    k_phase_a_warp<G, U, SMEM><<<(unsigned)blocks, 256, 0, s>>>(a);
    c.launches++;
}

// experiment knobs (lanes per vertex of classes 2-4, loads in flight of class 1)
#ifndef RS_EXP_A_G4
#define RS_EXP_A_G4 32
#endif
#ifndef RS_EXP_A_G3
#define RS_EXP_A_G3 8
#endif
#ifndef RS_EXP_A_G2
#define RS_EXP_A_G2 8
#endif
#ifndef RS_EXP_A_U3
#define RS_EXP_A_U3 4
#endif
#ifndef RS_EXP_A_U2
#define RS_EXP_A_U2 4
#endif
#ifndef RS_EXP_A_CTA_CLS
#define RS_EXP_A_CTA_CLS 7   // first degree class run by a CTA per vertex (class 6 on 32-lane groups)
#endif
#ifndef RS_EXP_A_U1
#define RS_EXP_A_U1 4
#endif
template <bool SMEM>
static void launch_bins_a(Ctx &c, PhaseAArgs base) {
    // class -> (lanes per vertex, loads in flight per lane), G*U about the row length:
    // [0,8):4x2 [8,16):4x4 [16,32):8x4 [32,64):8x4 [64,8192):32x4 [8192,inf):CTAx4 (bins: kNumBins)
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        PhaseAArgs a = base;
        a.vlo = c.bins.offset[cls];
        a.nverts = c.bins.count[cls];
        if (a.nverts == 0) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= RS_EXP_A_CTA_CLS) {
            int64_t blocks = std::min<int64_t>(a.nverts, 148 * 8);
            k_phase_a_cta<SMEM><<<(unsigned)blocks, kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (SMEM || cls >= 5) {
            launch_warp_bin<32, 4, SMEM>(c, a, s);
        } else if (cls == 4) {
            launch_warp_bin<RS_EXP_A_G4, 4, SMEM>(c, a, s);
        } else if (cls == 3) {
            launch_warp_bin<RS_EXP_A_G3, RS_EXP_A_U3, SMEM>(c, a, s);
        } else if (cls == 2) {
            launch_warp_bin<RS_EXP_A_G2, RS_EXP_A_U2, SMEM>(c, a, s);
        } else if (cls == 1) {
            launch_warp_bin<4, RS_EXP_A_U1, SMEM>(c, a, s);
        } else {
            launch_warp_bin<4, 2, SMEM>(c, a, s);
        }
    }
}

cudaError_t launch_phase_a_impl(Ctx &c, const double *l2t, int64_t l2n, bool parity) {
    PhaseAArgs a;
    a.rowptr = c.rowptr; a.col = c.col; a.comm = c.comm_id; a.lab = c.lab;
    a.vlo = 0; a.nverts = 0; a.k = c.k; a.l2t = l2t; a.l2n = l2n;
    // unnormalised grouped Type-I terms are < 2 * omega_max_bound; a head needs the
    // 3-limb accumulator when d^2 >= |P|^2 times that bound could reach 2^31 (fx_red2)
    a.wide_bound = wide_bound(c.k);
    a.variant = c.variant;
    a.parity = parity ? 1 : 0;
    a.bq = c.bq;
    a.f = c.f; a.omega = c.omega; a.amat = c.amat; a.vrec = c.vrec; a.pidx = c.pidx; a.scal = c.scal;
    a.n = c.n; a.pplus = c.pplus; a.wps = c.wps; a.pc2 = c.pc2; a.bql = c.bql;
    if (c.k <= 8 && c.d_max < (1ll << 22)) launch_bins_a<false>(c, a);
    else launch_bins_a<true>(c, a);
    return cudaGetLastError();
}

}  // namespace rs

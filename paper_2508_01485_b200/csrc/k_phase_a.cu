// Phase A — one streaming pass over the CSR:
//   Step 1 border test (Algorithm 1 lines P:254-263),
//   Step 2d G' predecessor list P(u) = {x in N(u): C(x) != C(u)}, written
//           in place at offset rowptr[u] (no scan needed), ascending, with the
//           8-bit label of each entry beside it (plab),
//   Step 2a neighbour-community histogram f[u][i] over the k targets,
//           read off P(u): a target column c != C(u) counts the entries of P(u)
//           labelled c, and f_u(C(u)) = d(u) - |P(u)| (every other neighbour
//           shares u's community),
//   Step 2b weights omega_u(C_i) = H(L_i) * (L_all - 1) (Eq. 3, Eq. 5, Algorithm 2
//           P:457-482, closed form of Eq. H_optimal P:417 with exact zeros) and
//           their cube roots a_u(C_i) used by every triad term (Eq. 4),
//   Step 2c omega_max partial maxima,
// and, once u's weights are known, the inputs of Step 3: the orientation of G'
// by internal id (P+(u) = the prefix of P(u) below u, split into its target run
// and the rest) and u's pushes of a_u(c_u) into
// B_w[c_u] for every w in P(u) (v in P(w) iff w in P(v)), exact integer REDs.
//
// The row walk is the only per-neighbour work: one coalesced column load, one
// 1-byte label gather, one compare and one ballot per neighbour (profiled
// round 1: the histogram, the P+ counts and their three ballots per neighbour
// made the walk instruction-bound at ~145 warp instructions per 32 neighbours).
// Everything else runs over P(u) (a quarter of the row at mu = 0.2).
// Labels are the 8-bit community codes of rs_set_communities; only vertices of
// two uncoded ("other") communities fall back to comparing full int32 ids.
// Degree-binned: a group of G lanes (or a whole CTA for hubs) owns a vertex;
// each lane keeps U independent loads in flight.
#include "rs_internal.cuh"
#include "rs_device.cuh"
#include <cstdio>
#include <cstdlib>
#include <type_traits>

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
    PRec *__restrict__ pc2;
    BQL *__restrict__ bql;
    const double *__restrict__ l2t;     // log2 of small integers
    int64_t l2n;
    int32_t *__restrict__ f;
    double *__restrict__ omega;
    double *__restrict__ amat;
    VRec *__restrict__ vrec;
    int32_t *__restrict__ pidx;
    uint8_t *__restrict__ plab;         // label of each P(u) entry, beside it
    unsigned long long *__restrict__ bsum;   // multi-GPU: the B pushes go here (k x n u64, summed over
                                        // the ranks, then rebuilt into BQL with Q); nullptr on one GPU
    unsigned long long *scal;
    int32_t hc;                         // vec walk: labels of vertices [0, hc) cached in shared memory
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

__device__ __forceinline__ void write_vrec(const PhaseAArgs &a, int64_t u, double a_self, int pc, uint32_t lu,
                                           int64_t d) {
    VRec r;
    r.a_self = a_self;
    r.pcnt = pc;
    r.lab = (uint8_t)lu;
    r.head = (lu < (uint32_t)a.k && d >= 2) ? 1 : 0;
    r.wide = ((double)d * (double)d >= a.wide_bound) ? 1 : 0;   // = (u < n_wide), degree-descending ids
    r.pad = 0;
    a.vrec[u] = r;
}

// Steps 1 + 2d for u: walk the row once and write P(u) (the foreign neighbours,
// ascending) and their labels in place at rowptr[u]. Returns |P(u)| and |P+(u)|
// (foreign neighbours below u) in every lane of the group. OTHER: u's
// community has no 8-bit code of its own, so neighbours coded kOther are
// compared by full community id.
template <int U, bool OTHER, class GR>
__device__ __forceinline__ void walk_row(const PhaseAArgs &a, int64_t u, int64_t beg, int d, uint32_t lu,
                                         int32_t cfull, GR &g, int &pc_out, int &pp_out) {
    const int32_t *__restrict__ row = a.col + beg;
    int32_t *__restrict__ pout = a.pidx + beg;
    uint8_t *__restrict__ lout = a.plab + beg;
    int pc = 0, ppl = 0;
    for (int base = 0; base < d; base += GR::size * U) {
        int32_t x[U];
        uint32_t l[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            x[j] = i < d ? __ldcs(row + i) : -1;
        }
#pragma unroll
        for (int j = 0; j < U; j++) l[j] = x[j] >= 0 ? (uint32_t)__ldg(a.lab + x[j]) : lu;
        bool f[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            f[j] = l[j] != lu;
            if (OTHER && x[j] >= 0 && l[j] == kOther) f[j] = __ldg(a.comm + x[j]) != cfull;
            ppl += (f[j] && x[j] < (int32_t)u) ? 1 : 0;
        }
        int r[U], tot[U];
        g.template rank_u<U>(f, r, tot);
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (f[j]) {
                pout[pc + r[j]] = x[j];
                lout[pc + r[j]] = (uint8_t)l[j];
            }
            pc += tot[j];
        }
    }
    pc_out = pc;
    pp_out = g.sum(ppl);
}

// Step 3 inputs of u (after its weights are known; au(c) = a_u(c)): B pushes
// and the P+ runs, reading P(u) and its labels back from this
// group's writes (k > 8 path). P+(u) is written as its
// target run DESCENDING at [0, pt) followed by the other run ascending at
// [pt, pp): an entry i of the prefix P+ has i predecessors in it, so its rank in
// the other run is i minus the targets before it (one ballot).
template <int U, class GR, class AU>
__device__ __forceinline__ void phase_a_lists(const PhaseAArgs &a, GR &g, int64_t beg, int pc, int pp, int pt,
                                              uint32_t lu, AU au) {
    const uint32_t k = (uint32_t)a.k;
    const unsigned long long qs = lu < k ? bq_quantize(au(lu), a.bq) : 0ull;
    const bool push = qs != 0ull;
    BQL *bcol = a.bql + (int64_t)(push ? lu : 0) * a.n;
    const int32_t *__restrict__ pin = a.pidx + beg;
    const uint8_t *__restrict__ lin = a.plab + beg;
    int ct = 0;
    for (int base = 0; base < pc; base += GR::size * U) {
        int32_t v[U];
        uint32_t lv[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            v[j] = i < pc ? pin[i] : -1;
            lv[j] = i < pc ? (uint32_t)lin[i] : kOther;
        }
#ifndef RS_EXP_NO_BPUSH
        if (push) {
#pragma unroll
            for (int j = 0; j < U; j++)
                if (v[j] >= 0) atomicAdd(&bcol[v[j]].b, qs);   // u in P(v): a_u(c_u) into B_v[c_u]
        }
#endif
        if (base < pp) {                                     // group-uniform: P+ is the prefix [0, pp)
            bool t[U];
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int i = base + j * GR::size + (int)g.lane;
                t[j] = i < pp && lv[j] < k;
            }
            int rt[U], tt[U];
            g.template rank_u<U>(t, rt, tt);
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int i = base + j * GR::size + (int)g.lane;
                if (i < pp) {
                    const int tb = ct + rt[j];                // target entries before i
                    const int64_t at = t[j] ? beg + pt - 1 - tb : beg + pt + (i - tb);
                    a.pplus[at] = v[j];
                }
                ct += tt[j];
            }
        }
    }
}

// The row walk of the k <= 8 path, scalar form (CTA groups, and the fallback):
// lane i of the group takes entries base + j G + i, U loads in flight, per-lane
// packed 16-bit histograms, one ballot per entry compacts P(u).
template <int U, class GR>
__device__ __forceinline__ void walk_scalar(const PhaseAArgs &a, int64_t u, int64_t beg, int d, uint32_t lu,
                                            int32_t cfull, bool wr, GR &g, int &pc_out, int &pp_out, int &pt_out,
                                            int (&cnt)[8]) {
    const uint32_t k = (uint32_t)a.k;
    const bool other = lu == kOther;                 // compare kOther neighbours by full id
    int32_t *__restrict__ pout = a.pidx + beg;
    uint8_t *__restrict__ lout = a.plab + beg;
    unsigned long long h0 = 0ull, h1 = 0ull;
    int pc = 0, ppl = 0, ptl = 0;
    const int dw = g.umax(d);
    for (int base = 0; base < dw; base += GR::size * U) {
        int32_t x[U];
        uint32_t l[U];
        bool f[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            x[j] = i < d ? __ldcs(a.col + beg + i) : -1;
        }
#pragma unroll
        for (int j = 0; j < U; j++) l[j] = x[j] >= 0 ? (uint32_t)__ldg(a.lab + x[j]) : lu;
#pragma unroll
        for (int j = 0; j < U; j++) {
            f[j] = l[j] != lu;
            if (other && x[j] >= 0 && l[j] == kOther) f[j] = __ldg(a.comm + x[j]) != cfull;
            if (x[j] >= 0 && l[j] < k) {
                const unsigned long long inc = 1ull << ((l[j] & 3u) * 16u);
                if (l[j] < 4u) h0 += inc; else h1 += inc;
            }
            const bool below = f[j] && x[j] < (int32_t)u;    // P+(u): foreign and above u
            ppl += below ? 1 : 0;
            ptl += (below && l[j] < k) ? 1 : 0;
        }
        int r[U], tot[U];
        g.template rank_u<U>(f, r, tot);
#pragma unroll
        for (int j = 0; j < U; j++) {
            if (f[j] && wr) {
                pout[pc + r[j]] = x[j];
                lout[pc + r[j]] = (uint8_t)l[j];
            }
            pc += tot[j];
        }
    }
    pp_out = g.sum(ppl);
    pt_out = g.sum(ptl);
    pc_out = pc;
    if (dw < 65536) {         // group totals still fit the 16-bit fields
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
}

// The row walk, vectorised (lockstep groups of G <= 32 lanes): the group reads
// its row as aligned 16-byte pieces of col (one LDG.128 per lane per piece,
// 16 G contiguous bytes per group; entries of the first and last piece outside
// the row are masked), so a lane holds 4 consecutive entries of each of its V
// pieces; the 4 V label gathers are independent. Branch-free per entry:
// histogram counts in packed fields (8-bit while a lane's share of the row
// cannot reach 256, PACK8; else 16-bit), P(u) compacted by ONE group scan of
// the per-lane foreign counts per piece (ascending order: piece, lane, slot).
// OTHER (warp-uniform): some group's vertex has no 8-bit code of its own.
extern __shared__ __align__(16) uint8_t s_lab[];   // vec walk: labels of vertices [0, PhaseAArgs::hc)

template <int V, bool PACK8, bool OTHER, int G>
__device__ __forceinline__ void walk_vec(const PhaseAArgs &a, int64_t u, int64_t beg, int d, uint32_t lu,
                                         int32_t cfull, bool wr, LockGroup<G> &g, int &pc_out, int &pp_out,
                                         int &pt_out, int (&cnt)[8]) {
    const uint32_t k = (uint32_t)a.k;
    const int head = (int)(beg & 3);                // entries of the first piece before the row
    const int hi = d > 0 ? d + head : 0;            // the row is window positions [head, hi)
    const int4 *__restrict__ wp = reinterpret_cast<const int4 *>(a.col + (beg - head));
    int32_t *__restrict__ pout = a.pidx + beg;
    uint8_t *__restrict__ lout = a.plab + beg;
    typedef typename std::conditional<PACK8, uint32_t, unsigned long long>::type H;
    H h0 = 0, h1 = 0;
    int pc = 0, ppl = 0, ptl = 0;
    const int dw = g.umax(hi);
    const int32_t u32 = (int32_t)u;
    for (int base = 0; base < dw; base += 4 * G * V) {
        int32_t x[V][4];
        uint32_t l[V][4];
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int w0 = base + 4 * (v * G + (int)g.lane);
            int4 q = make_int4(-1, -1, -1, -1);
            if (w0 < hi) q = __ldcs(wp + (w0 >> 2));
            x[v][0] = (w0 >= head && w0 < hi) ? q.x : -1;
            x[v][1] = (w0 + 1 >= head && w0 + 1 < hi) ? q.y : -1;
            x[v][2] = (w0 + 2 >= head && w0 + 2 < hi) ? q.z : -1;
            x[v][3] = (w0 + 3 < hi) ? q.w : -1;
        }
#pragma unroll
        for (int v = 0; v < V; v++)
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const int32_t xs = x[v][s];
                // the highest-degree vertices (the first ids) are most of the references:
                // their labels come from the block's shared copy (a random byte gather
                // from shared memory costs a few bank wavefronts, from L1 one per lane)
                l[v][s] = xs < 0 ? (uint32_t)kOther : xs < a.hc ? (uint32_t)s_lab[xs] : (uint32_t)__ldg(a.lab + xs);
            }
#pragma unroll
        for (int v = 0; v < V; v++) {
            unsigned fm = 0u;
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const int32_t xs = x[v][s];
                const uint32_t ls = l[v][s];
                bool f = xs >= 0 && ls != lu;
                if (OTHER && xs >= 0 && ls == kOther && lu == kOther) f = __ldg(a.comm + xs) != cfull;
                fm |= f ? (1u << s) : 0u;
                const bool tg = ls < k;                                  // invalid entries: kOther, never < k
                if constexpr (PACK8) {
                    const uint32_t inc = 1u << ((ls & 3u) * 8u);
                    h0 += (tg && ls < 4u) ? inc : 0u;
                    h1 += (tg && ls >= 4u) ? inc : 0u;
                } else {
                    const unsigned long long inc = 1ull << ((ls & 3u) * 16u);
                    h0 += (tg && ls < 4u) ? inc : 0ull;
                    h1 += (tg && ls >= 4u) ? inc : 0ull;
                }
                const bool below = f && xs < u32;                        // P+(u): foreign and above u
                ppl += below ? 1 : 0;
                ptl += (below && tg) ? 1 : 0;
            }
            // exclusive rank of this lane's first foreign entry in the piece round
            const int c = __popc(fm);
            int incl = c;
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o, G);
                if ((int)g.lane >= o) incl += t;
            }
            const int tot = __shfl_sync(0xffffffffu, incl, G - 1, G);
            int r = pc + incl - c;
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const bool f = (fm >> s) & 1u;
                if (f && wr) {
                    pout[r] = x[v][s];
                    lout[r] = (uint8_t)l[v][s];
                }
                r += f ? 1 : 0;
            }
            pc += tot;
        }
    }
    pp_out = g.sum(ppl);
    pt_out = g.sum(ptl);
    pc_out = pc;
    if constexpr (PACK8) {
        // 8-bit lane fields -> 16-bit fields (even / odd columns), then group sums
        // (a row has < 65536 entries on this path)
        const uint32_t a0 = g.sum(h0 & 0x00FF00FFu), a1 = g.sum((h0 >> 8) & 0x00FF00FFu);
        const uint32_t b0 = g.sum(h1 & 0x00FF00FFu), b1 = g.sum((h1 >> 8) & 0x00FF00FFu);
        cnt[0] = (int)(a0 & 0xFFFFu); cnt[2] = (int)(a0 >> 16);
        cnt[1] = (int)(a1 & 0xFFFFu); cnt[3] = (int)(a1 >> 16);
        cnt[4] = (int)(b0 & 0xFFFFu); cnt[6] = (int)(b0 >> 16);
        cnt[5] = (int)(b1 & 0xFFFFu); cnt[7] = (int)(b1 >> 16);
    } else if (dw < 65536) {
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
}

template <class GR> struct IsLock { static constexpr bool value = false; };
template <int G> struct IsLock<LockGroup<G>> { static constexpr bool value = true; };

// k <= 8: Steps 1, 2a-2d and the Step 3 inputs of u, in lockstep over the
// groups of a warp (LockGroup: warp-uniform loop bounds; u < 0 = no vertex).
// The row walk (walk_vec for lockstep groups, VEC pieces per lane per round;
// walk_scalar for CTAs) gives |P(u)|, |P+(u)|, |P+_T(u)| and the histogram. The
// lists pass reads P(u) and its labels back (L2) and takes a_u(c) from the lane
// that computed it (shuffle).
#ifndef RS_EXP_A_PF
#define RS_EXP_A_PF 0        // vec walk: prefetch the group's next row into L2 while this vertex runs (measured: no gain, off)
#endif
template <int U, class GR, int VEC = 0, bool PACK8 = false>
__device__ __forceinline__ double phase_a_vertex(const PhaseAArgs &a, int64_t u, GR &g, int64_t unext = -1) {
    const uint32_t k = (uint32_t)a.k;
    const bool valid = u >= 0;
    int64_t beg = 0;
    int d = 0;
    uint32_t lu = kOther;
    int32_t cfull = 0;
    int64_t nb = -1, ne = 0;
    if (RS_EXP_A_PF && VEC > 0 && unext >= 0) {     // issued with this vertex's own loads
        nb = __ldg(a.rowptr + unext);
        ne = __ldg(a.rowptr + unext + 1);
    }
    if (valid) {
        beg = a.rowptr[u];
        d = (int)(a.rowptr[u + 1] - beg);
        lu = a.lab[u];
        if (lu == kOther) cfull = a.comm[u];
    }
    if (RS_EXP_A_PF && VEC > 0 && nb >= 0) {
        // the next vertex's first two rounds of 16-byte pieces (a DRAM stream
        // otherwise first touched after this vertex's whole dependent chain)
        const int64_t p0 = (nb & ~3ll) + 4 * (int64_t)g.lane;
        if (p0 < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.col + p0));
        if (p0 + 4 * GR::size < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.col + p0 + 4 * GR::size));
    }
    const bool wr = valid && !a.parity;
    int pc, pp, pt;
    int cnt[8];
    if constexpr (VEC > 0 && IsLock<GR>::value) {
        // warp-uniform: the full-id comparison only where some group needs it
        if (__any_sync(0xffffffffu, lu == kOther))
            walk_vec<VEC, PACK8, true>(a, u, beg, d, lu, cfull, wr, g, pc, pp, pt, cnt);
        else
            walk_vec<VEC, PACK8, false>(a, u, beg, d, lu, cfull, wr, g, pc, pp, pt, cnt);
    } else {
        walk_scalar<U>(a, u, beg, d, lu, cfull, wr, g, pc, pp, pt, cnt);
    }
    int T = 0, L_all = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        T += cnt[c];
        L_all += cnt[c] > 0;
    }
    // Algorithm 2's X = sum f log2 f and every column's log2(T - f) with ONE
    // round of log2-table loads: lane l takes the columns l, l + G, ... (a
    // vertex's weights are a dependent chain after its row walk), X by a group sum
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
        lys[i] = (c < (int)k && T - fc > 0) ? lg2(a, T - fc) : 0.0;
        xpart += xcs[i];
    }
    const double X = g.sum(xpart);
    double wmax = 0.0;
    double acn[NC];
#pragma unroll
    for (int i = 0; i < NC; i++) {
        const int c = (int)g.lane + i * GR::size;
        acn[i] = 0.0;
        if (c >= (int)k) continue;
        const int fc = fcs[i];
        const double w = weight_from(a, fc, T, L_all, X, xcs[i], lys[i]);
        const double ac = w > 0.0 ? cube_root(w) : 0.0;
        acn[i] = ac;
        if (valid) {
            if (a.parity) {            // the parity tables, written only for the getters
                a.omega[u * k + c] = w;
                a.f[u * k + c] = fc;
            } else {
                a.amat[u * k + c] = ac;
                if (!a.bsum) a.bql[(int64_t)c * a.n + u].Q = ac * ac;
            }
            if (in_max(a, fc, L_all, c, (int)lu, pc)) wmax = w > wmax ? w : wmax;
        }
    }
    if (a.parity) return wmax;
    // a_u(c) of a column c < k: from the lane (c % G, slot c / G) that computed it
    const double *arow = a.amat + u * k;
    auto au = [&](uint32_t c) -> double {
        if constexpr (GR::size <= 32) {
            double v = 0.0;
#pragma unroll
            for (int i = 0; i < NC; i++) {
                const double t = g.from(acn[i], (int)(c % GR::size));
                v = ((int)(c / GR::size) == i) ? t : v;
            }
            return v;
        } else {
            return arow[c];                      // CTA: this block's writes (after the barrier)
        }
    };
    g.sync();
    const double aself = au(lu < k ? lu : 0u);
    if (valid && g.lane == 0) write_vrec(a, u, lu < k ? aself : 0.0, pc, lu, d);
    // Step 3 inputs: B pushes and the P+ runs, reading P(u) back
    const unsigned long long qs = (valid && lu < k) ? bq_quantize(aself, a.bq) : 0ull;
    // the pushes: into B_v's record, or (multi-GPU) the plain u64 sums
    const int64_t col0 = (int64_t)(qs ? lu : 0) * a.n;
    unsigned long long *bpush = a.bsum ? a.bsum + col0 : &a.bql[col0].b;
    const int bstride = a.bsum ? 1 : 2;                 // u64 words per entry
    const int32_t *__restrict__ pin = a.pidx + beg;
    const uint8_t *__restrict__ lin = a.plab + beg;
    int ct = 0;
    const int pcw = g.umax(wr ? pc : 0);
    for (int base = 0; base < pcw; base += GR::size * U) {
        int32_t v[U];
        uint32_t lv[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            v[j] = (wr && i < pc) ? pin[i] : -1;
            lv[j] = (wr && i < pc) ? (uint32_t)lin[i] : kOther;
        }
#ifndef RS_EXP_NO_BPUSH
#pragma unroll
        for (int j = 0; j < U; j++)
            if (qs && v[j] >= 0) atomicAdd(bpush + (int64_t)v[j] * bstride, qs);   // u in P(v): a_u(c_u) into B_v[c_u]
#endif
        bool t[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            t[j] = v[j] >= 0 && i < pp && lv[j] < k;
        }
        int rt[U], tt[U];
        g.template rank_u<U>(t, rt, tt);
#pragma unroll
        for (int j = 0; j < U; j++) {
            const int i = base + j * GR::size + (int)g.lane;
            const double aw = au(lv[j] < k ? lv[j] : 0u);
            if (v[j] >= 0 && i < pp) {
                const int tb = ct + rt[j];                // target entries of P+ before i
                const int64_t at = t[j] ? beg + pt - 1 - tb : beg + pt + (i - tb);
                a.pplus[at] = v[j];
            }
            ct += tt[j];
        }
    }
    if (wr && g.lane == 0) {
        PRec r;
        r.x = pr_pack(pp, lu);
        r.y = pc;
        r.start = beg | ((long long)pt << kPrShift);
        a.pc2[u] = r;
    }
    return wmax;
}

// k > 8: histogram in shared memory (one warp or one CTA per vertex)
template <int U, class GR>
__device__ __forceinline__ double phase_a_vertex_smem(const PhaseAArgs &a, int64_t u, GR &g, int *hist) {
    const int64_t beg = a.rowptr[u];
    const int d = (int)(a.rowptr[u + 1] - beg);
    const uint32_t lu = a.lab[u];
    const int k = a.k;
    for (int c = g.lane; c < k; c += GR::size) hist[c] = 0;
    int pc, pp;
    if (a.parity) {
        pc = a.vrec[u].pcnt;
        pp = pr_plus(a.pc2[u]);
    } else if (lu == kOther) {
        walk_row<U, true>(a, u, beg, d, lu, a.comm[u], g, pc, pp);
    } else {
        walk_row<U, false>(a, u, beg, d, lu, 0, g, pc, pp);
    }
    g.sync();
    // Step 2a from the P list: shared-memory counts of the target labels
    const uint8_t *__restrict__ lp = a.plab + beg;
    int ptl = 0;
    for (int i = g.lane; i < pc; i += GR::size) {
        const uint32_t l = lp[i];
        if (l < (uint32_t)k) {
            atomicAdd(&hist[l], 1);
            ptl += i < pp;
        }
    }
    const int pt = g.sum(ptl);
    g.sync();
    if (lu < (uint32_t)k && g.lane == 0) hist[lu] = d - pc;
    g.sync();
    // T, L_all and X = sum f log2 f over the k columns, lane-strided + group sums
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
        if (in_max(a, fc, L_all, c, (int)lu, pc)) wmax = w > wmax ? w : wmax;
    }
    g.sync();
    if (a.parity) return wmax;
    if (g.lane == 0) {
        double as = 0.0;
        if (lu < (uint32_t)k) { const double w = weight_of(a, hist[lu], T, L_all, X); as = w > 0.0 ? cube_root(w) : 0.0; }
        write_vrec(a, u, as, pc, lu, d);
    }
    g.sync();
    const double *arow = a.amat + u * k;            // this group's writes, plain loads
    phase_a_lists<U>(a, g, beg, pc, pp, pt, lu, [&](uint32_t c) { return arow[c]; });
    if (g.lane == 0) {
        PRec r;
        r.x = pr_pack(pp, lu);
        r.y = pc;
        r.start = beg | ((long long)pt << kPrShift);
        a.pc2[u] = r;
    }
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

template <int G, int U, bool SMEM, int VEC = 0, bool PACK8 = false>
#ifndef RS_EXP_A_MINB
#define RS_EXP_A_MINB 5      // warp kernels: resident blocks of 256 per SM (5: 51 registers, no spill; 6 spills)
#endif
__global__ void __launch_bounds__(256, RS_EXP_A_MINB) k_phase_a_warp(PhaseAArgs a) {
    __shared__ int hist[SMEM ? 8 * 256 : 1];
    double wmax = 0.0;
    if constexpr (SMEM) {
        WarpGroup<G> g;
        const int64_t groups_per_block = blockDim.x / G;
        const int64_t gid = blockIdx.x * groups_per_block + threadIdx.x / G;
        const int64_t ngroups = (int64_t)gridDim.x * groups_per_block;
        for (int64_t i = gid; i < a.nverts; i += ngroups) {
            const double w = phase_a_vertex_smem<U>(a, a.vlo + i, g, hist + (threadIdx.x / 32) * 256);
            wmax = w > wmax ? w : wmax;
        }
    } else {
        // lockstep: a warp takes 32 / G consecutive vertices per step, all its
        // lanes iterate together (a group past the end takes no vertex)
        LockGroup<G> g;
        if constexpr (VEC > 0) {
            // the label cache: a.hc bytes (a multiple of 16), 16-byte loads
            for (int i = threadIdx.x; i < (a.hc >> 4); i += blockDim.x)
                reinterpret_cast<int4 *>(s_lab)[i] = __ldg(reinterpret_cast<const int4 *>(a.lab) + i);
            __syncthreads();
        }
        constexpr int gpw = 32 / G;
        const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
        const int gi = (int)((threadIdx.x & 31u) / G);
        for (int64_t i0 = warp * gpw; i0 < a.nverts; i0 += nwarps * gpw) {
            const int64_t i = i0 + gi;
            const int64_t inx = i + nwarps * gpw;          // this group's next vertex
            const double w = phase_a_vertex<U, LockGroup<G>, VEC, PACK8>(a, i < a.nverts ? a.vlo + i : -1, g,
                                                                         inx < a.nverts ? a.vlo + inx : -1);
            wmax = w > wmax ? w : wmax;
        }
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
template <int G, int U, bool SMEM, int VEC = 0, bool PACK8 = false>
static void launch_warp_bin(Ctx &c, PhaseAArgs a, cudaStream_t s) {
    const int64_t gpb = 256 / G;
    int64_t blocks = (a.nverts + gpb - 1) / gpb;
    blocks = std::min<int64_t>(blocks, 148 * RS_EXP_A_BLK);
    if (blocks < 1) return;
    const size_t dyn = VEC > 0 ? (size_t)a.hc : 0;
    if (dyn > 48 * 1024)
        cudaFuncSetAttribute(k_phase_a_warp<G, U, SMEM, VEC, PACK8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k_phase_a_warp<G, U, SMEM, VEC, PACK8><<<(unsigned)blocks, 256, dyn, s>>>(a);
    c.launches++;
}

// the vectorised walk (walk_vec): V 16-byte pieces per lane per round; 8-bit
// histogram fields when a lane's share of the class's longest row stays < 256
template <int G>
static void launch_vec_bin(Ctx &c, PhaseAArgs a, cudaStream_t s, int V, int64_t dhi) {
    const bool p8 = (dhi + 3) / G + 4 * V < 256;
    if (V >= 2) {
        if (p8) launch_warp_bin<G, 4, false, 2, true>(c, a, s);
        else launch_warp_bin<G, 4, false, 2, false>(c, a, s);
    } else {
        if (p8) launch_warp_bin<G, 4, false, 1, true>(c, a, s);
        else launch_warp_bin<G, 4, false, 1, false>(c, a, s);
    }
}
static int a_vec() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("RS_A_VEC");   // 0: the scalar walk; 1 / 2: pieces per lane per round
        v = e ? std::max(0, std::min(2, atoi(e))) : 1;
    }
    return v;
}

#ifndef RS_EXP_A_CTA_CLS
#define RS_EXP_A_CTA_CLS 7   // first degree class run by a CTA per vertex (class 6 on 32-lane groups)
#endif
// lanes per vertex G and loads in flight per lane U of the warp classes 0..6
// (lockstep groups); the environment variables RS_A_LANES="g0,...,g6" and
// RS_A_LOADS="u0,...,u6" override them (experiments)
static void a_config(int cls, int *G, int *U) {
    static int lanes[7] = {4, 4, 4, 8, 16, 16, 32};
    static int loads[7] = {2, 4, 4, 4, 4, 4, 4};
    static bool init = false;
    if (!init) {
        init = true;
        int v[7];
        if (const char *e = getenv("RS_A_LANES")) {
            const int n = sscanf(e, "%d,%d,%d,%d,%d,%d,%d", v, v + 1, v + 2, v + 3, v + 4, v + 5, v + 6);
            for (int i = 0; i < n; i++)
                if (v[i] == 4 || v[i] == 8 || v[i] == 16 || v[i] == 32) lanes[i] = v[i];
        }
        if (const char *e = getenv("RS_A_LOADS")) {
            const int n = sscanf(e, "%d,%d,%d,%d,%d,%d,%d", v, v + 1, v + 2, v + 3, v + 4, v + 5, v + 6);
            for (int i = 0; i < n; i++)
                if (v[i] == 2 || v[i] == 4 || v[i] == 8) loads[i] = v[i];
        }
    }
    *G = lanes[cls];
    *U = loads[cls];
}

// class -> lanes per vertex G (a_lanes) x loads in flight per lane U (4; 2 for
// the class [0, 8)); [8192, inf) a CTA x 4. The warp kernels run their groups
// in lockstep: consecutive vertices of the degree-descending numbering have
// nearly equal degrees, so the warp-maximum trip count wastes little.
template <bool SMEM>
static void launch_bins_a(Ctx &c, PhaseAArgs base, int64_t lo, int64_t hi) {
    for (int cls = kNumBins - 1; cls >= 0; cls--) {
        PhaseAArgs a = base;
        a.vlo = std::max<int64_t>(c.bins.offset[cls], lo);   // the class, restricted to [lo, hi)
        a.nverts = std::min<int64_t>(c.bins.offset[cls] + c.bins.count[cls], hi) - a.vlo;
        if (a.nverts <= 0) continue;
        cudaStream_t s = c.side[cls];
        if (cls >= RS_EXP_A_CTA_CLS) {
            int64_t blocks = std::min<int64_t>(a.nverts, 148 * 8);
            k_phase_a_cta<SMEM><<<(unsigned)blocks, kCtaThreads, 0, s>>>(a);
            c.launches++;
        } else if (SMEM) {
            launch_warp_bin<32, 4, true>(c, a, s);
        } else {
            int G, U;
            a_config(cls, &G, &U);
            const int V = a_vec();
            const int64_t dhi = bin_lo(cls + 1) - 1;
            if (V > 0) {
                switch (G) {
                    case 4: launch_vec_bin<4>(c, a, s, V, dhi); break;
                    case 8: launch_vec_bin<8>(c, a, s, V, dhi); break;
                    case 16: launch_vec_bin<16>(c, a, s, V, dhi); break;
                    default: launch_vec_bin<32>(c, a, s, V, dhi); break;
                }
                continue;
            }
            const int key = G * 10 + U;
            switch (key) {
                case 42: launch_warp_bin<4, 2, false>(c, a, s); break;
                case 44: launch_warp_bin<4, 4, false>(c, a, s); break;
                case 82: launch_warp_bin<8, 2, false>(c, a, s); break;
                case 84: launch_warp_bin<8, 4, false>(c, a, s); break;
                case 162: launch_warp_bin<16, 2, false>(c, a, s); break;
                case 164: launch_warp_bin<16, 4, false>(c, a, s); break;
                case 168: launch_warp_bin<16, 8, false>(c, a, s); break;
                case 324: launch_warp_bin<32, 4, false>(c, a, s); break;
                case 328: launch_warp_bin<32, 8, false>(c, a, s); break;
                default: launch_warp_bin<32, 4, false>(c, a, s); break;
            }
        }
    }
}

// vertices [lo, hi) only (a rank's own range in the multi-GPU path)
cudaError_t launch_phase_a_impl(Ctx &c, const double *l2t, int64_t l2n, bool parity, int64_t lo, int64_t hi) {
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
    a.plab = c.plab;
    a.bsum = (c.bsum_mode && !parity) ? c.bsum : nullptr;
    a.n = c.n; a.pplus = c.pplus; a.pc2 = c.pc2; a.bql = c.bql;
    {
        // label cache of the vec walk: the first hc vertex ids (highest degrees),
        // RS_A_HC bytes per block (default 0: off)
        static int hc_env = -1;
        if (hc_env < 0) {
            const char *e = getenv("RS_A_HC");
            hc_env = e ? std::max(0, std::min(200 * 1024, atoi(e))) : 0;   // measured: 16 / 32 / 40 KB cost A +0.08 / +0.23 / +0.73 ms (the L1 it takes caches the hub labels already)
        }
        a.hc = (int32_t)(std::min<int64_t>(hc_env, c.n) & ~15ll);   // whole 16-byte pieces of lab
    }
    if (c.k <= 8) launch_bins_a<false>(c, a, lo, hi);
    else launch_bins_a<true>(c, a, lo, hi);
    return cudaGetLastError();
}

}  // namespace rs

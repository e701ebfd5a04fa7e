// Shared argument block of the P-list phases (D, E) and the finalize pass.
#pragma once
#include "rs_internal.cuh"

#include "rs_device.cuh"
#include <algorithm>
#include <cmath>

namespace rs {

struct CdeArgs {
    const int64_t *__restrict__ rowptr;
    int64_t vlo;                        // first vertex of the range
    int64_t nverts;
    int64_t n;
    int32_t k;
    const double *__restrict__ amat;    // n*k cube roots a_v(c), row-major
    const VRec *__restrict__ vrec;
    const int32_t *__restrict__ pidx;   // P(u) ascending at rowptr[u]: P+(u) prefix, P-(u) suffix
    const int32_t *__restrict__ pplus;  // P+(u) at rowptr[u]: target run + other run (see PRec)
    const double *__restrict__ wps;     // all-communities mode: a_u(c_w) beside each w of P(u)
    const PRec *__restrict__ pc2;       // {|P+(u)|, |P(u)|, rowptr[u] | |P+_T(u)| << 40}
    const BQL *__restrict__ bql;        // column-major: bql[c*n + w]
    const unsigned long long *__restrict__ bsum;   // non-null: B sums read here, Q from amat (no BQL rebuild)
    unsigned long long *__restrict__ acc1;  // 3 limbs per vertex (Type-I)
    unsigned long long *__restrict__ acc_hub;  // striped limbs of vertices < n_hub
    int64_t n_hub;
    unsigned long long *__restrict__ n1;    // Type-I triad counts (COUNT mode)
    ulonglong2 *__restrict__ t2;            // exact Type-II sum per head (Phase D)
    double *__restrict__ score;         // original vertex order
    const int32_t *__restrict__ perm;   // internal -> original id
    const uint8_t *__restrict__ lab;    // 8-bit community codes
    unsigned long long *scal;
    int64_t head_lo, head_hi;           // owned head range (multi-GPU); [0, n) on one GPU
    int32_t e_rank, e_world;            // Phase E: this rank's share of the middle vertices
    int32_t e_blk;                      // Phase E: heavy items dealt to the ranks in blocks of e_blk
    int32_t e_perm;                     // Phase E: the queue order interleaved over e_perm batches
    int32_t e_chunk;                    // Phase E: positions of P-(y) per heavy work item
    int32_t e_local;                    // Phase E: the item list holds only this rank's items (dealt at build)
    int32_t mg;                         // multi-GPU: P+ runs packed (pplus = the gathered runs, PRec start
                                        // = packed offset); heavy P-(y) at item.mbase of pidx (packed)
    int64_t n_wide;                     // heads [0, n_wide) use the 3-limb Type-I accumulator
    // all-communities mode (k_sparse.cu): weights per G' edge instead of dense rows
    const double *__restrict__ pwr;     // a_w(c_u) beside each w of P(u) (wps: a_u(c_w))
    const int64_t *__restrict__ prv;    // position of c_u in w's community table
    const unsigned long long *__restrict__ ctb;   // B_w[c] beside each column of w's table
    int bq;                             // B grid 2^-bq (BQL, ctb)
    int slot_cap;                       // Phase E: an x slot's shared 20-bit limbs take at most this many terms
};

// VRec::wide by internal id: d(h)^2 >= wide_bound, d non-increasing in h
__device__ __forceinline__ bool is_wide(const CdeArgs &a, int64_t h) { return h < a.n_wide; }

inline CdeArgs cde_args(Ctx &c) {
    CdeArgs a;
    a.rowptr = c.rowptr; a.vlo = 0; a.nverts = 0; a.n = c.n; a.k = c.k;
    a.amat = c.amat; a.vrec = c.vrec; a.pidx = c.pidx; a.pc2 = c.pc2;
    a.pplus = c.mg_packed ? c.pk_id : c.pplus; a.wps = c.wps; a.mg = c.mg_packed ? 1 : 0;
    a.bql = c.bql; a.bsum = (c.bsum_direct && !c.sparse) ? c.bsum : nullptr; a.acc1 = c.acc1; a.acc_hub = c.acc_hub; a.n_hub = c.n_hub; a.n1 = c.n1; a.t2 = c.t2; a.score = c.score; a.scal = c.scal;
    a.perm = c.perm; a.lab = c.lab;
    a.n_wide = c.n_wide;
    a.head_lo = c.head_lo; a.head_hi = c.head_hi;
    a.e_rank = 0; a.e_world = 1; a.e_blk = 1; a.e_perm = 1; a.e_chunk = c.e_chunk; a.e_local = 0;
    a.pwr = c.pwr; a.prv = c.prv; a.ctb = c.ctb; a.bq = c.bq;
    {
        // Phase E's per-item x slots (smem_red4): a grouped Type-I term is < 2 omega_max
        // <= 2 k log2(k - 1) (wide_bound's weight bound), so one term adds < 32 k log2(k - 1) + 1
        // to the top 32-bit limb (bits 60..91 of q = term * 2^64); the slot takes at most
        // 2^32 / that many terms (4096 for every k <= 254; ~1000 at k = 10 000 communities)
        const double wb = 2147483648.0 / (2.0 * wide_bound(c.k));
        const double per = 32.0 * wb + 1.0;
        a.slot_cap = (int)std::min(4096.0, std::floor(4294967295.0 / per));
    }
    if (c.sparse) a.pplus = c.pidx;   // P+(u) is one ascending run: the prefix of P(u)
    return a;
}

}  // namespace rs

// Shared argument block of the P-list phases (C, D, E).
#pragma once
#include "rs_internal.cuh"
#include "rs_device.cuh"

namespace rs {

struct CdeArgs {
    const int64_t *__restrict__ rowptr;
    int64_t vlo;                        // first vertex of the range
    int64_t nverts;
    int64_t n;
    int32_t k;
    const double *__restrict__ amat;    // n*k cube roots a_v(c), row-major
    const VRec *__restrict__ vrec;
    int32_t *__restrict__ pidx;         // P(u) at rowptr[u]; after Phase C: P-(u) at its front
    int32_t *__restrict__ pd;           // P+(u): two runs in u's region (see PRec)
    double *__restrict__ wd;            // a_u(c_z) beside each z of P+(u); sign bit: z is wide
    const int64_t *__restrict__ dpos;   // start of u's region
    PRec *__restrict__ pc2;             // {|P+(u)|, |P(u)|, start | |P+_T(u)| << 40}
    BQ *__restrict__ bq;                // column-major: bq[c*n + w]
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
    bool any_wide;                      // some head may need the 3-limb Type-I accumulator
    double wide_bound;                  // |P(h)|^2 >= wide_bound: head h is wide (VRec::wide)
};

// the 3-limb rule of VRec::wide from |P(h)| alone
__device__ __forceinline__ bool is_wide(const CdeArgs &a, int p) {
    return a.any_wide && (double)p * (double)p >= a.wide_bound;
}

inline CdeArgs cde_args(Ctx &c) {
    CdeArgs a;
    a.rowptr = c.rowptr; a.vlo = 0; a.nverts = 0; a.n = c.n; a.k = c.k;
    a.amat = c.amat; a.vrec = c.vrec; a.pidx = c.pidx; a.pc2 = c.pc2;
    a.pd = c.pd; a.wd = c.wd; a.dpos = c.dpos;
    a.bq = c.bq; a.acc1 = c.acc1; a.acc_hub = c.acc_hub; a.n_hub = c.n_hub; a.n1 = c.n1; a.t2 = c.t2; a.score = c.score; a.scal = c.scal;
    a.perm = c.perm; a.lab = c.lab;
    a.any_wide = (double)c.d_max * (double)c.d_max >= wide_bound(c.k);
    a.wide_bound = wide_bound(c.k);
    a.head_lo = c.head_lo; a.head_hi = c.head_hi;
    a.e_rank = 0; a.e_world = 1;
    return a;
}

}  // namespace rs

// Internal declarations of librs (B200 / sm_100a). Not part of the ABI.
// The oracle (oracle/) shares nothing with this tree: no header, helper,
// constant or table.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "../../include/rs.h"

#ifdef RS_WITH_NCCL
#include <nccl.h>
#endif

namespace rs {

// Test hook (rs_debug_poison): when >= 0, every device allocation librs makes
// is filled with this byte before use, so a kernel that reads memory nobody
// wrote gives results that change with the byte (tests/test_gpu_hygiene.py
// runs the pipeline under several bytes and requires identical bits; this
// stands in for compute-sanitizer initcheck, which is closed on this pool).
extern int g_poison;
template <class T>
inline cudaError_t dmalloc(T **p, size_t bytes) {
    cudaError_t e = cudaMalloc((void **)p, bytes);
    if (e == cudaSuccess && g_poison >= 0) e = cudaMemset((void *)*p, g_poison, bytes);
    return e;
}

#ifdef RS_WITH_NCCL
// NCCL is resolved at run time (dlopen) so that librs uses the libnccl already
// loaded in the process (e.g. the one torch.distributed brought) instead of
// linking a second, possibly different, copy.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char *(*GetErrorString)(ncclResult_t);
};
const NcclApi *nccl_api(std::string *err);
#endif

// The multi-GPU exchange layer (rs_xport.cu): NCCL, or an in-process emulated
// world of host threads on one GPU (rs_create_emulated). Collectives are
// blocking with respect to the host only for the emulated transport.
struct Xport {
    std::string msg;   // last transport error
    virtual ~Xport() {}
    // every rank holds buf; rank r's segment is [off[r], off[r] + len[r]) bytes: copy all segments everywhere
    virtual cudaError_t allgatherv(void *buf, const size_t *off, const size_t *len, cudaStream_t s) = 0;
    virtual cudaError_t allreduce_u64(unsigned long long *buf, size_t count, bool max, cudaStream_t s) = 0;
    virtual cudaError_t allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // u64 sums of rank r's segment [off[r], off[r] + len[r]) (in u64 words) over
    // all ranks, delivered to rank r only (the other segments are left as they are)
    virtual cudaError_t reduce_scatterv_u64(unsigned long long *buf, const size_t *off, const size_t *len,
                                            cudaStream_t s) = 0;
    // rs_score brackets (the emulated world's serial mode times each rank's
    // compute alone on the GPU: ranks take turns between collectives)
    virtual void score_begin() {}
    virtual void score_end(cudaStream_t) {}
    // the phase (rs_stats.ms_phase index) the next collectives belong to, and the
    // stream time this rank spent inside that phase's collectives (emulated
    // world: waiting for the peers, the device copies; 0 where not measured)
    int tag = 0;
    virtual float wait_ms(int) { return 0.f; }
};
struct EmuWorld;
Xport *make_emu_xport(EmuWorld *w, int rank);
#ifdef RS_WITH_NCCL
Xport *make_nccl_xport(ncclComm_t comm, int world);
#endif

constexpr int kMaxK = 254;        // target columns (uint8 label 0xFF = "other")
constexpr uint8_t kOther = 0xFF;  // community without its own 8-bit code
constexpr int kNumBins = 8;       // degree classes (load time)
// degree class c holds vertices with bin_lo(c) <= d < bin_lo(c+1); in the
// internal (degree-descending) numbering class c is the range
// [bins.offset[c], bins.offset[c] + bins.count[c]), class 7 first
__host__ __device__ constexpr int64_t bin_lo(int i) {
    return i <= 0 ? 0 : i == 1 ? 8 : i == 2 ? 16 : i == 3 ? 32 : i == 4 ? 64 : i == 5 ? 128 : i == 6 ? 2048
         : i == 7 ? 8192 : INT64_MAX;
}

// 16-byte per-vertex record gathered by the P-list phases (one sector / 2).
struct __align__(16) VRec {
    double a_self;     // omega_v(C(v))^(1/3) (unnormalised) if C(v) is a target, else 0
    int32_t pcnt;      // |P(v)|: inter-community neighbours (G' in-degree)
    uint8_t lab;       // 8-bit community code (< k: target column)
    uint8_t head;      // 1 if v can be an RSI head: target community and d(v) >= 2
    uint8_t wide;      // Type-I sum of this head needs the 3-limb accumulator (d(v)^2 >= wide_bound)
    uint8_t pad;
};

// Per-vertex G' record written by Phase A, gathered once per predecessor x by
// Phase E. G' is oriented by internal id: z is above u iff z < u, i.e. iff z
// has the higher degree (the numbering is degree-descending), so P+(u) is the
// prefix of the ascending list P(u) = pidx[rowptr[u], +|P|) and P-(u) its
// suffix. Phase A also copies P+(u) to pplus at the same offset as two runs:
// the entries in a target community in DESCENDING order at [0, t), the others
// ascending at [t, |P+|), so the entries below any y form one contiguous range
// around t. Phase E reads a_u(c_z) from u's row at lab(z) (0 for the other
// run); round 2 dropped the copy Phase A wrote beside each entry (Orkut shape:
// Phase A 1.78 -> 1.60 ms, E unchanged). (All-communities mode: pplus is pidx
// itself, one ascending run, t = |P+|; wps holds a_u(c_w) beside each w.)
// t = |P+_T(u)| is packed above bit 40 of `start` (offsets < 2^40).
// x also carries u's 8-bit label above bit 24, so Phase E gets a predecessor's
// label with the record it gathers anyway (one random 1-byte gather less per
// (y, x) pair); |P+(u)| < 2^24.
struct __align__(16) PRec {
    int x;             // |P+(u)| (orientation out-degree) | lab(u) << 24
    int y;             // |P(u)|
    long long start;   // rowptr[u] | (|P+_T(u)| << 40)
};
constexpr int kPrShift = 40;
__host__ __device__ __forceinline__ int pr_plus(const PRec &r) { return r.x & 0xFFFFFF; }
__host__ __device__ __forceinline__ int pr_lab(const PRec &r) { return (int)((unsigned)r.x >> 24); }
__host__ __device__ __forceinline__ int pr_pack(int pp, unsigned lab) { return (int)((unsigned)pp | (lab << 24)); }
// Type-I accumulation of the n_hub highest-degree heads is striped over
// kHubStripes copies (a RED picks its copy by warp): a hub closes up to
// millions of triangles, and same-address atomics serialise in the L2.
constexpr int kHubStripes = 16;
constexpr int64_t kHubMax = 1 << 16;
__host__ __device__ __forceinline__ int ceil4(int v) { return (v + 3) & ~3; }
__host__ __device__ __forceinline__ long long pr_start(const PRec &r) { return r.start & ((1ll << kPrShift) - 1); }
__host__ __device__ __forceinline__ int pr_plus_t(const PRec &r) { return (int)(r.start >> kPrShift); }

// Per (vertex, column) record read by the Type-II pull (Phase D), half a sector.
// B_w[c] = sum_{v in P(w), col(v)=c} a_v(c) is pushed by every such v during
// Phase A (v is in P(w) iff w is in P(v)) as one 64-bit integer RED of a_v(c)
// rounded once to the 2^-bq grid (bq_quantize): the sum is exact and order-free,
// and B_w[c] - a_u(c) is taken in integers, so it is exactly 0 when u is w's
// only such neighbour. bq = 40 unless a_max * d_max needs more integer bits
// (Ctx::bq); the rounding of each a (>= 0.01 when non-zero) is < 5e-11 relative.
struct __align__(16) BQL {
    unsigned long long b;        // sum of bq_quantize(a_v(c)) over the pushes
    double Q;                    // a_w(c)^2 = omega_w(c)^(2/3), written by w
};

// Per-vertex record of the all-communities mode, gathered once per neighbour.
struct __align__(16) SRec {
    long long beg;     // rowptr[v]: v's community table and lists start here
    int32_t L;         // number of distinct communities among N(v) (table length)
    int32_t cid;       // column of C(v)
};

// One entry of a vertex's sparse community table (all-communities mode): the
// column, its count and a_u(c) = omega_u(c)^(1/3) in one 16-byte record, so the
// binary search that finds a column also brings its weight.
struct __align__(16) CtEnt {
    int32_t x;         // column (community rank)
    int32_t y;         // f_u(column)
    double a;          // a_u(column)
};

struct Bins {
    int64_t count[kNumBins] = {0};
    int64_t offset[kNumBins + 1] = {0};
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side[kNumBins + 1] = {nullptr};   // forked streams: concurrent bins (+ light Phase E)
    cudaEvent_t ev_fork = nullptr, ev_join[kNumBins + 1] = {nullptr};
    cudaEvent_t ev_phase[8] = {nullptr};
    cudaEvent_t ev_zero = nullptr;   // accumulators zeroed for the next rs_score (side stream)
    bool acc_zero = false;           // acc1 / acc_hub are zero once ev_zero completes
    bool bql_zero = false;           // the dense B table's limbs are zero once ev_zero completes
    bool bsum_zero = false;          // the plain B sums (bsum mode) are zero once ev_zero completes
    bool parity_ok = false;          // f / omega written for the last rs_score (getters)
    std::string err;
    int64_t launches = 0;

    // multi-GPU
    int rank = 0, world = 1;
#ifdef RS_WITH_NCCL
    ncclComm_t comm = nullptr;
#endif
    Xport *xp = nullptr;                       // world > 1: the exchange transport (owned)
    int32_t *pk_id = nullptr;                  // world > 1: packed P+ runs of all ranks (ids), at gpre[x]
    int64_t pk_cap = 0;
    int32_t *pk_m = nullptr;                   // world > 1: packed P- lists of the heavy vertices, at gm[y]
    int64_t pkm_cap = 0;
    int64_t *xg = nullptr;                     // world > 1: gm[0..n] | gpre[0..n] (exclusive prefixes)
    int64_t xg_cap = 0;
    bool rep_a = false;                        // multi-GPU: Phase A replicated on every rank (RS_REPLICATE_A)
    bool mg_packed = false;                    // Phase E reads the packed runs (PRec start = gpre[x])
    int64_t xar_bytes = 0, xag_bytes = 0;      // world > 1: bytes all-reduced / all-gathered in the last rs_score
    int64_t xrs_bytes = 0;                     //   and reduce-scattered
    bool hubs_folded = false;                  // the hub stripes were folded into acc1 (multi-GPU)
    unsigned long long *bsum = nullptr;        // world > 1: B pushes (k x n), summed over the ranks
    int32_t *vx = nullptr;                     // world > 1: {|P|, |P+|, |P+_T|} per vertex, exchanged
    int64_t dist_cap = 0;                      // n * k the two above were sized for
    bool bsum_mode = false;                    // this rs_score pushes into bsum (multi-GPU; RS_EXP_BSUM)
    bool bsum_direct = false;                  // ... and Phase D reads bsum + amat directly (no BQL rebuild)
    unsigned long long *tk_gkey = nullptr;     // world > 1: gathered top-K candidates (world * K)
    int32_t *tk_gid = nullptr;
    int64_t tk_gcap = 0;
    int64_t head_lo = 0, head_hi = 0;          // owned vertex range [lo, hi)
    std::vector<int64_t> bounds;               // world+1 range boundaries

    // graph (load time)
    int64_t n = 0, nnz = 0;
    int64_t *rowptr = nullptr;   // n+1
    int32_t *col = nullptr;      // nnz
    int32_t *perm = nullptr;     // n: original id of internal vertex r (degree-descending order)
    int32_t *inv = nullptr;      // n: internal id of original vertex v
    Bins bins;
    int64_t rsplit[5] = {0};     // first row of degree < 8192, 2048, 512, 128, 32 (row-sort classes)
    int32_t *rl_tmpcol = nullptr;   // load-time temporaries (arena): unsorted long rows,
    void *rl_tmp = nullptr;         //   CUB scratch
    size_t rl_need = 0;
    std::vector<cudaEvent_t> ev_chunk;   // col_idx chunks copied (host input, rs_load_csr)
    int64_t d_max = 0;
    int64_t *e_pre = nullptr;    // Phase E work items: prefix of extra chunks of the e_nbig largest rows
    int64_t e_nbig = 0, e_extra = 0;
    int e_chunk = 64;            // Phase E: positions of P-(y) per heavy work item (<= kChunkE)
    size_t e_bytes = 0;
    bool loaded = false;

    // communities (set time)
    int32_t *comm_in = nullptr;  // n: communities as given (original order)
    int32_t *comm_id = nullptr;  // n: communities in internal order
    uint8_t *lab = nullptr;      // n
    int32_t *chist = nullptr;    // community sizes, cap entries
    uint8_t *ccode = nullptr;    // community id -> 8-bit code
    int64_t ccap = 0;
    int64_t cmax = 0;            // largest community id measured (sizes the histogram)
    int32_t *targets = nullptr;  // kMaxK
    int32_t k = 0;
    int32_t h_targets[kMaxK];
    bool has_comm = false;

    // all-communities mode (NEXT-2, rs_set_communities with k = RS_ALL_COMMUNITIES):
    // every community is a target (k = number of distinct communities, any size);
    // per-vertex sparse community tables replace the dense n*k tables
    bool sparse = false;
    std::vector<int32_t> h_targets_all;  // the k target ids in column order
    int32_t *cid = nullptr;      // n: column of C(u) (internal order)
    int32_t *code32 = nullptr;   // community id -> column (ccap entries)
    SRec *srec = nullptr;        // n: {rowptr, L(u), cid} gathered per neighbour
    CtEnt *ctk = nullptr;        // nnz: u's distinct neighbour columns ascending at rowptr[u]: {column, f_u(c), a_u(c)}
    unsigned long long *ctb = nullptr;   // nnz: B_u[c] on the 2^-bq grid (see BQL) beside each column
    double *pwr = nullptr;       // nnz: a_w(c_u) beside each w of P(u) (pidx order); wps holds a_u(c_w)
    int64_t *prv = nullptr;      // nnz: position of c_u in w's table, beside each w of P(u)
    double *aself = nullptr;     // n: a_u(c_u)
    double *xsum = nullptr;      // n: X(u) = sum_c f_u(c) log2 f_u(c) (Algorithm 2)
    unsigned long long *n2s = nullptr;  // n: Type-II triad counts (all-communities mode)
    void *csort = nullptr;       // community ranking temporaries (grow-only)
    size_t csort_bytes = 0;
    int64_t sp_cap = 0;          // nnz the sparse buffers were sized for

    // score (per rs_score)
    int32_t *f = nullptr;        // n*k counts
    double *omega = nullptr;     // n*k weights (unnormalised)
    VRec *vrec = nullptr;        // n
    int32_t *pidx = nullptr;     // nnz, P(u) ascending at rowptr[u] (P+(u) its prefix, see PRec)
    uint8_t *plab = nullptr;     // nnz, the 8-bit label of each P(u) entry, beside it (Phase A)
    int32_t *pplus = nullptr;    // nnz, P+(u) at rowptr[u] as a target run and the other run
    double *wps = nullptr;       // nnz, all-communities mode only: a_u(c_w) beside each w of P(u)
    PRec *pc2 = nullptr;         // n: {|P+(u)|, |P(u)|, rowptr[u] | |P+_T(u)| << 40}
    double *amat = nullptr;      // n*k cube roots a_u(C_i) = omega_u(C_i)^(1/3)
    BQL *bql = nullptr;          // k*n, column-major: bql[c*n + w]
    int64_t n_wide = 0;          // vertices [0, n_wide) (degree^2 >= wide_bound) use 3 Type-I limbs
    int32_t nwide_k = 0;         // the k scal[kScalNWide] was computed for (0: none; reset by rs_load_csr)
    int bq = 40;                 // fraction bits of the B table's integer sums (BQL)
    unsigned long long *acc1 = nullptr;  // 3*n fixed-point limbs of the Type-I sum (2 used unless wide)
    unsigned long long *acc_hub = nullptr;  // kHubStripes copies of the limbs of the first n_hub vertices
    int64_t n_hub = 0;                   //   (the highest degrees: contended heads), summed by Phase D
    unsigned long long *n1 = nullptr;    // n Type-I triad counts
    ulonglong2 *t2 = nullptr;            // n exact Type-II sums (Phase D, read by the finalize pass)
    double *score = nullptr;     // n, ORIGINAL vertex order
    unsigned long long *scal = nullptr;  // device scalars (see kScal*)
    int64_t k_alloc = 0;         // k the per-score buffers were sized for
    int64_t kn_alloc = 0;        // ... and n
    bool scored = false;
    int e_shares = 1;            // test hook: Phase E run as this many rank shares (rs_score flags)
    int variant = 0;             // NEXT-3 literal variants (rs_score flags >> 16)

    // top-k scratch
    unsigned long long *tk_hist = nullptr;   // 256 * 8
    unsigned long long *tk_cand = nullptr;   // candidates (key, id) pairs
    int64_t tk_cap = 0;

    // device scratch for reductions / validation
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    // grow-only arena for load-time staging and relabel temporaries; buffer capacities
    void *arena = nullptr;
    size_t arena_bytes = 0;
    int64_t cap_n = 0, cap_nnz = 0;
};

// device scalar slots in Ctx::scal
enum {
    kScalOmegaMaxBits = 0,   // omega_max as IEEE bits (non-negative => monotone)
    kScalErr = 1,            // first validation error code (0 = none)
    kScalErrRow = 2,         // row of the first error
    kScalCnt0 = 3,           // generic counters
    kScalNBorder = 4,
    kScalNPred = 5,
    kScalNTri = 6,
    kScalNProbe = 7,         // Phase E: entries of P+ lists probed
    kScalTk = 8,             // top-k state (8 slots; load time: degree class bounds, 9 slots)
    kScalNWide = 17,         // n_wide (rs_set_communities)
    kScalCount = 32
};

// |P(h)|^2 at or above which head h's unnormalised Type-I sum could reach 2^31
// (grouped terms are < 2 * omega_max <= 2 (k-1) log2(k-1)): such heads use the
// 3-limb accumulator (fx_red3) instead of fx_red2.
inline double wide_bound(int k) {
    // omega <= H |L| <= log2(k - 1) * k covers the literal |L| (<= k) of NEXT-3 too
    const double km1 = (double)(k - 1);
    const double wb = km1 > 1.0 ? (double)k * __builtin_log2(km1) : 2.0;
    return 2147483648.0 / (2.0 * wb);
}

// ---- kernels (launchers). Each returns cudaGetLastError() of the launch. ----
cudaError_t launch_validate(Ctx &c, const int64_t *rp, const int32_t *col);
size_t relabel_arena_bytes(int64_t n, int64_t nnz);
cudaError_t launch_relabel(Ctx &c, const int64_t *rp_o, const int32_t *col_o, void *arena, size_t arena_bytes);
cudaError_t launch_set_communities(Ctx &c, int64_t max_comm, const int32_t *user_targets);
cudaError_t launch_phase_a(Ctx &c);
cudaError_t launch_phase_e(Ctx &c);
cudaError_t launch_phase_d(Ctx &c);
cudaError_t launch_finalize(Ctx &c);
size_t awcc_scratch_bytes(int64_t M, int J1, int64_t cap, int64_t nS);
cudaError_t launch_shii_ic_batch(Ctx &c, int nb, const int32_t *seed_d, const int32_t *c0_d, const uint64_t *st,
                                 double p, unsigned long long *buf, int64_t *out2);
cudaError_t launch_shii_run(Ctx &c, int32_t seed_o, int model, double p, uint64_t st, unsigned int *act,
                            int32_t *cnt, int32_t *list, unsigned long long *ctr, int64_t out2[2]);
cudaError_t launch_awcc_degrees(Ctx &c, const int32_t *S_dev, int64_t nS, int64_t *deg_dev);
cudaError_t launch_awcc_trial(Ctx &c, const int32_t *S_dev, int64_t nS, int mode, int step_pct, int J1, uint64_t st,
                              int32_t *zeta_dev, void *scratch, size_t scratch_bytes, int64_t cap);
cudaError_t launch_phase_e_on(Ctx &c, cudaStream_t light);
cudaError_t launch_run_prefix(Ctx &c, int64_t *gpre, bool minus);
cudaError_t launch_plus_pack(Ctx &c, const int64_t *gpre);
cudaError_t launch_minus_pack(Ctx &c, const int64_t *gm);
cudaError_t launch_rebase(Ctx &c, const int64_t *gpre);
cudaError_t launch_vx_pack(Ctx &c);
cudaError_t launch_vx_unpack(Ctx &c);
cudaError_t launch_b_rebuild(Ctx &c);
cudaError_t launch_fold_hubs(Ctx &c);
cudaError_t launch_triangle_counts(Ctx &c);
cudaError_t launch_e_items(Ctx &c);
cudaError_t launch_topk(Ctx &c, int64_t K, int32_t *ids_dev, double *scores_dev, int64_t lo, int64_t hi);
cudaError_t launch_counts_total(Ctx &c, const int32_t *f_orig, int32_t *total_dev);
cudaError_t launch_permute_i32(Ctx &c, const int32_t *in, int k, int32_t *out);
cudaError_t launch_permute_f64(Ctx &c, const double *in, int k, double *out);
cudaError_t launch_border_list(Ctx &c, int32_t *bv_dev, int64_t *nb_host);
cudaError_t launch_pred_export(Ctx &c, int64_t *off_dev, int32_t *pred_dev, int64_t *nent_host);
cudaError_t launch_type2_counts(Ctx &c, int64_t *t2_dev);
cudaError_t launch_type1_export(Ctx &c, int64_t *t1_dev);
cudaError_t launch_stats(Ctx &c, int64_t out[4]);
cudaError_t sort_rows(Ctx &c, const int32_t *in, const int32_t *map, int32_t *out, int bits, void *tmp, size_t need,
                      int64_t upto);
cudaError_t launch_relabel_prepare(Ctx &c, const int64_t *rp_o, void *arena, size_t arena_bytes);
cudaError_t launch_relabel_rows(Ctx &c, const int64_t *rp_o, const int32_t *col_o, int64_t v0, int64_t v1);
cudaError_t launch_relabel_finish(Ctx &c);
void launch_comm_hist(Ctx &c, int64_t nbins);
void launch_nwide(Ctx &c, double bound);
// all-communities mode (k_sparse.cu)
size_t sparse_rank_bytes(int64_t nbins);
cudaError_t launch_set_communities_all(Ctx &c, int64_t max_comm, int64_t *nc_out);
cudaError_t launch_sparse_sort(Ctx &c);
cudaError_t launch_sparse_tables(Ctx &c, const double *l2t, int64_t l2n);
cudaError_t launch_sparse_lists(Ctx &c);
cudaError_t launch_sparse_counts_dense(Ctx &c, int32_t *f_dev, int32_t *total_dev);
cudaError_t launch_sparse_weights_dense(Ctx &c, const double *l2t, int64_t l2n, double *w_dev);
cudaError_t launch_sparse_type2(Ctx &c, int64_t *t2_dev);
cudaError_t launch_sparse_offsets(Ctx &c, int64_t *off_dev, int64_t *total);
cudaError_t launch_sparse_export(Ctx &c, const int64_t *off_dev, const double *l2t, int64_t l2n, int32_t *cols,
                                 int32_t *cnt, double *omega, double *omega_abs);
cudaError_t launch_minmax_i32(Ctx &c, const int32_t *a, int64_t n, int64_t *mn, int64_t *mx);

}  // namespace rs

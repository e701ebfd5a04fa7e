/*
 * rs.h — C-ABI of librs, the B200 (sm_100a) implementation of the hot path of
 * arXiv 2508.01485, "A Parallel Algorithm for Finding Robust Spanners in Large
 * Social Networks": per-vertex Robust Spanning Index (RSI, Eq. 4) scoring and
 * top-K robust-spanner selection over a community-labelled graph.
 *
 * Citations "P:n" are lines of the paper's LaTeX source; "C-n" are
 * the readings of ambiguous passages listed in DESIGN.md §3.
 *
 * Conventions for every entry point
 *  - Returns rs_status; RS_OK = 0. On any other status, rs_last_error(ctx)
 *    holds a one-line message naming the first offender. No call aborts the
 *    process or throws across the ABI.
 *  - Pointers are plain host or device addresses. Inputs are COPIED into
 *    context-owned device memory: the caller keeps ownership and may free or
 *    reuse its buffers when the call returns. Outputs go to caller-allocated
 *    buffers; an output pointer may be host memory (the call then
 *    synchronises the context stream before returning) or device memory
 *    (cudaPointerGetAttributes decides; the call is then stream-ordered and
 *    returns without synchronising).
 *  - All device work is issued on the context's stream (rs_create).
 *  - Call order: rs_load_csr -> rs_set_communities -> rs_score -> rs_topk /
 *    getters. Anything else returns RS_ESTATE. rs_load_csr invalidates
 *    communities and scores; rs_set_communities invalidates scores.
 *  - One context per host thread. Contexts are independent.
 */
#ifndef RS_H_
#define RS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RS_OK = 0,
    RS_EINVAL = -1,   /* an argument or input violates the contract below     */
    RS_ESTATE = -2,   /* call out of order (e.g. rs_score before communities)  */
    RS_ENOMEM = -3,   /* device allocation failed                              */
    RS_ECUDA = -4,    /* CUDA runtime / kernel error (message has cuda string) */
    RS_ENCCL = -5     /* NCCL error in a multi-GPU context                     */
} rs_status;

typedef struct rs_ctx rs_ctx;

/* Phase timings (device milliseconds, CUDA events on the context stream) and
 * size statistics of the last rs_score. */
typedef struct {
    int64_t n;                /* |V|                                            */
    int64_t m;                /* |E| undirected = nnz / 2                       */
    int64_t n_border;         /* |V_b| over all communities              */
    int64_t n_pred_entries;   /* sum over u of |P(u)| = |E_b|           */
    int64_t n_triangles;      /* triangles of G' (3 distinct communities) with at
                                 least two target vertices: the ones that carry
                                 Type-I terms (a term needs a target head and a
                                 target column among the other two)             */
    int64_t n_probes;         /* Phase E: P+ list entries probed (the Type-I
                                 intersection volume, bench roofline)           */
    double omega_max;         /* max weight over all cells (C-7)  */
    float ms_phase[8];        /* CUDA-event times on the context stream:
                                 [0] Phase A border/histogram/weights/G' lists,
                                     orientation, B-table pushes
                                 [1] multi-GPU: the exchange of Phase A's
                                     outputs; one GPU: the B-table rebuild
                                     when the pushes went to plain sums
                                 [2] Phase E Type-I triangles, concurrent with
                                     Phase D Type-II pull
                                 [3] finalize (sum, normalise)
                                 [4] multi-GPU: the sum of the Type-I limbs
                                     over the ranks [5..7] reserved */
    int64_t xchg_allreduce_bytes; /* multi-GPU: bytes of the buffers all-reduced
                                     in this rs_score (0 on one GPU)            */
    int64_t xchg_allgather_bytes; /* multi-GPU: total bytes all-gathered (every
                                     rank's segments together)                  */
    int64_t xchg_reduce_scatter_bytes; /* multi-GPU: total bytes reduce-scattered
                                     (every rank's segments together)           */
    float ms_xwait[8];        /* emulated world (rs_create_emulated): the part of
                                 ms_phase[i] this rank's stream spent inside
                                 collectives (waiting for the peers, the device
                                 copies); ms_phase[i] - ms_xwait[i] is its own
                                 kernel time. 0 elsewhere                       */
} rs_stats;

/* Flags for rs_load_csr. */
#define RS_VALIDATE   1u   /* check the CSR contract on the device (see rs_load_csr) */
/* Test hook: copy a host col_idx in chunks of 2^e entries (e = 4..30) with the
 * rows of each chunk relabelled as it arrives, whatever nnz (by default only
 * from 2^24 entries, in 2^24-entry chunks). Results must not change. */
#define RS_LOAD_CHUNK_LOG2(e) ((((uint32_t)(e)) & 0x1Fu) << 8)

/* rs_set_communities: every community is a target (sparse per-vertex tables). */
#define RS_ALL_COMMUNITIES (-1)

/* Flags for rs_score. */
#define RS_GATHER_SCORES 1u /* multi-GPU: make scores_out complete on every rank */
/* Test hook: run Phase E (Type-I) as s sequential shares of the multi-GPU
 * split by middle vertex (s = 2..255) on one GPU; results must not change. */
#define RS_E_SHARES(s)    (((uint32_t)(s) & 0xFFu) << 8)
#define RS_E_SHARES_OF(f) (((f) >> 8) & 0xFFu)
/* Multi-GPU: every rank runs Phase A (Steps 1-2d and the B table) over ALL
 * vertices from its replicated CSR and labels instead of its own range, so the
 * Phase A exchange disappears and the only collectives are the Type-I limb
 * reduce-scatter, the counters and the top-K merge. Results are
 * bitwise those of the sharded path and of one GPU. Ignored on one GPU. */
#define RS_REPLICATE_A (1u << 20)
/* NEXT-3 literal variants of the paper (DESIGN reading C-30; default = the
 * adopted readings C-3, C-4, C-7): */
#define RS_LITERAL_L (1u << 16) /* |L(u,v)| as Eq. 2 defines L: communities of
                                   N(v) other than C(u), instead of Algorithm 2's
                                   L_all - 1 for every column */
#define RS_GATE_L    (1u << 17) /* Algorithm 1's gate: omega = 0 unless |L| > 1 */
#define RS_WMAX_EB   (1u << 18) /* omega_max over Algorithm 1's E_b edges only:
                                   border v, |L| > 1, c = C(v) or v has a neighbour in c */

/* Create a context on CUDA device `device`. `cuda_stream` is a cudaStream_t
 * (NULL = the legacy default stream) on which all work is issued; the caller
 * keeps ownership of the stream and must keep it alive while ctx lives.
 * Errors: RS_EINVAL (out == NULL, bad device), RS_ECUDA. */
rs_status rs_create(rs_ctx **out, int device, void *cuda_stream);

/* Multi-GPU context: rank `rank` of `world` processes, one GPU each, that all
 * call the same sequence with the same inputs. `nccl_id` is the
 * 128-byte ncclUniqueId produced by rs_nccl_unique_id on rank 0 and broadcast
 * by the caller (e.g. with torch.distributed). Vertices are split into
 * work-balanced contiguous ranges (internal degree-descending numbering): a
 * rank runs Phase A (Steps 1-2) on its own vertices, exchanges what the other
 * phases read of the 2-hop neighbourhood (omega_max, the B table, the
 * cube-root rows, per-vertex records and the oriented P+ runs; DESIGN.md §7
 * gives the bytes), takes a share of the Type-I middle vertices (the per-head
 * limbs are then summed over the ranks) and finalizes its own heads; rs_topk
 * all-gathers K candidates per rank and merges them identically everywhere.
 * Supports explicit k <= 8 targets (RS_EINVAL otherwise, at
 * rs_set_communities); rs_get_pred is not available (a rank holds only its own
 * P lists; RS_ESTATE). Errors: RS_EINVAL, RS_ECUDA, RS_ENCCL. */
rs_status rs_create_dist(rs_ctx **out, int device, void *cuda_stream, int rank, int world,
                         const uint8_t nccl_id[128]);
/* Fill `id_out` (128 bytes, host) with a fresh ncclUniqueId. */
rs_status rs_nccl_unique_id(uint8_t id_out[128]);
/* Test hook: run every collective of the NCCL transport (the one rs_create_dist
 * uses: all-reduce sum and max, all-gather, the grouped-broadcast all-gather of
 * segments, the grouped-reduce reduce-scatter of segments) on a one-rank NCCL
 * communicator on `device`, on `cuda_stream` (NULL: a stream of its own), over
 * `bytes` (>= 64, multiple of 8) of device memory it allocates and frees, and
 * check every result bit for bit on the host. Only one GPU is available to this
 * build's tests; a world of one still resolves the library, creates a
 * communicator and runs each call through NCCL's kernels. RS_OK, RS_ENCCL (no
 * NCCL / a call failed), RS_ECUDA, RS_EINVAL (bad size); a wrong result is
 * RS_ECUDA with the mismatch in rs_last_error(NULL). */
rs_status rs_nccl_selftest(int device, void *cuda_stream, size_t bytes);

/* Emulated multi-GPU world (tests, one GPU): `world` ranks are host threads of
 * one process, each with its own context from rs_create_emulated on the same
 * device, each calling the same sequence as on a GPU of its own; the
 * collectives are host barriers plus device-to-device copies between the
 * contexts (no kernel waits on another). Everything else is the multi-GPU path
 * of rs_create_dist. rs_emu_world_create: 1 <= world <= 16, RS_EINVAL
 * otherwise; destroy the world after every context of it. */
typedef struct rs_emu_world rs_emu_world;
rs_status rs_emu_world_create(rs_emu_world **out, int32_t world);
void rs_emu_world_destroy(rs_emu_world *w);
rs_status rs_create_emulated(rs_ctx **out, int device, void *cuda_stream, int rank, int world, rs_emu_world *w);
/* Serial mode of an emulated world (on != 0): inside rs_score the ranks take
 * turns, rank 0 first, between consecutive collectives, so that each rank's
 * kernels run alone on the GPU and its rs_stats phase times are those of a GPU
 * of its own (the multi-GPU model of bench.py). RS_EINVAL if w is NULL. */
rs_status rs_emu_world_serial(rs_emu_world *w, int32_t on);

/* Free every device buffer owned by ctx. NULL is a no-op. */
void rs_destroy(rs_ctx *ctx);

/* Message for the last non-OK status on ctx (never NULL; "" if none).
 * ctx == NULL returns the message of the last failed rs_create. */
const char *rs_last_error(const rs_ctx *ctx);

/* Load the undirected input graph G = (V, E) in CSR form ("a row
 * pointer array ... and a 1D flattened neighbor list array").
 *   n            number of vertices, 1 <= n < 2^31.
 *   row_offsets  int64[n+1]; row_offsets[0] = 0, non-decreasing; row u's
 *                neighbours are col_idx[row_offsets[u] .. row_offsets[u+1]).
 *   col_idx      int32[row_offsets[n]], neighbour ids in [0, n).
 * Contract (P:81 simple undirected graph; C-17): every row strictly ascending
 * (sorted, no duplicates), no self-loops, and symmetric (v in N(u) iff u in
 * N(v)). With RS_VALIDATE the contract is checked on the device and a
 * violation returns RS_EINVAL naming the first offending row; without it the
 * input is trusted (results on a non-canonical input are unspecified).
 * The graph is copied; degree binning of the rows (a property of the graph
 * alone) is computed here. Errors: RS_EINVAL, RS_ENOMEM, RS_ECUDA. */
rs_status rs_load_csr(rs_ctx *ctx, int64_t n, const int64_t *row_offsets, const int32_t *col_idx,
                      uint32_t flags);

/* Set the non-overlapping community of every vertex ("community
 * IDs are considered user input") and the k target communities whose weights
 * omega_v(C_i) are computed.
 *   community_of  int32[n], each in [0, 2^28).
 *   targets       int32[k] distinct community ids present in community_of,
 *                 in column order, or NULL = the k largest communities,
 *                 ties by ascending community id (C-15).
 *   k             2 <= k <= min(254, number of distinct communities), or
 *                 RS_ALL_COMMUNITIES (targets must be NULL): every community
 *                 is a target, k = the number of distinct communities (>= 2,
 *                 any count; NEXT-2 all-communities mode). Columns are then
 *                 ordered like the top-k selection (size descending, ties by
 *                 ascending id) and rs_score keeps per-vertex sparse community
 *                 tables instead of dense n*k ones (P:428 names the dense
 *                 table's limit); scores are the same quantity as with
 *                 explicit targets = all communities. The NEXT-3 variant flags
 *                 of rs_score are not available in this mode (RS_EINVAL).
 * Target selection, the per-vertex column labels and the community-size
 * histogram run on the device. Errors: RS_EINVAL, RS_ESTATE, RS_ENOMEM, RS_ECUDA. */
rs_status rs_set_communities(rs_ctx *ctx, const int32_t *community_of, const int32_t *targets,
                             int32_t k);

/* Compute the RSI of every vertex (Algorithm 1 Steps 1-3; Eq. 4):
 *   R(u) = 1/(d(u)(d(u)-1)) * sum over valid triads (u,w,v) (Eq. 6, Type-I
 *          and Type-II) of (omega_v(u) omega_w(v) omega_w(u))^(1/3),
 * weights normalised by omega_max, d(u) the degree in G
 * (C-16). R(u) = +0.0 when C(u) is not a target, d(u) < 2, u is not a border
 * vertex, or omega_max = 0 (C-9, C-22). Each head's triad sum is accumulated
 * exactly in fixed point (C-12), so scores are bitwise independent of thread
 * schedule and GPU count.
 *   scores_out  double[n] (host or device) or NULL (scores stay on the device
 *               for rs_topk). In a multi-GPU context only the rank's head
 *               range is filled unless flags has RS_GATHER_SCORES.
 *   stats_out   rs_stats* (host) or NULL; requesting stats synchronises.
 * Errors: RS_ESTATE, RS_ECUDA, RS_ENCCL. */
rs_status rs_score(rs_ctx *ctx, double *scores_out, rs_stats *stats_out, uint32_t flags);

/* Top-K robust spanners (Algorithm 1 optional Step 4): the min(K, n)
 * vertices of largest R, ordered by descending R, ties by ascending vertex id
 * (C-14: zero scores are eligible). Radix select on the fp64 bit patterns.
 *   K          >= 1.
 *   ids_out    int32[min(K,n)] (host or device).
 *   scores_out double[min(K,n)] (host or device) or NULL.
 *   count_out  int64* (host) or NULL: receives min(K, n).
 * Multi-GPU: identical result on every rank (NCCL allgather of per-rank
 * candidates + the same deterministic merge). Errors: RS_EINVAL, RS_ESTATE,
 * RS_ECUDA, RS_ENCCL. */
rs_status rs_topk(rs_ctx *ctx, int64_t K, int32_t *ids_out, double *scores_out, int64_t *count_out);

/* ---- parity getters (bit-exact artefacts of the last rs_score) ---- */

/* Step 2a histogram: f_out int32[n*k] row-major, f[u*k+i] =
 * |{x in N(u): C(x) = targets[i]}|; total_out int32[n] = sum_i f[u*k+i]
 * (P:431 T). Either pointer may be NULL. Requires rs_score. In the
 * all-communities mode this is a dense view (n*k entries, k = number of
 * communities) of the sparse tables. */
rs_status rs_get_counts(rs_ctx *ctx, int32_t *f_out, int32_t *total_out);

/* Step 2b weights before normalisation (Eq. 3, Eq. 5, Algorithm 2 |L| rule):
 * omega_out double[n*k] row-major (column i = omega_u(C_i), Lemma 1) or NULL;
 * omega_max_out double* or NULL. Requires rs_score. All-communities mode: a
 * dense view (absent columns carry the row's f = 0 weight). */
rs_status rs_get_weights(rs_ctx *ctx, double *omega_out, double *omega_max_out);

/* Step 1 border vertices (over all communities): bv_out int32[|V_b|]
 * ascending (or NULL); nb_out int64* receives |V_b|. Requires rs_score. */
rs_status rs_get_border(rs_ctx *ctx, int32_t *bv_out, int64_t *nb_out);

/* Step 2d G' predecessor lists ((w -> u) in E_b iff (u,w) in E and
 * C(u) != C(w)): pred_off_out int64[n+1] and pred_out int32[|E_b|] (each list
 * ascending), either may be NULL; n_entries_out int64* receives |E_b|.
 * Requires rs_score. */
rs_status rs_get_pred(rs_ctx *ctx, int64_t *pred_off_out, int32_t *pred_out, int64_t *n_entries_out);

/* Step 3 valid-triad counts per head (the "removal" sets of P:236: triads in
 * which removing any one edge keeps C(w) reachable from u), counted for every
 * scored head (C(u) a target, d(u) >= 2) including zero-weight triads:
 * type1_out int64[n] Type-I, type2_out int64[n] Type-II; either may be NULL.
 * Requires rs_score. */
rs_status rs_get_triad_counts(rs_ctx *ctx, int64_t *type1_out, int64_t *type2_out);

/* All-communities mode only (RS_ALL_COMMUNITIES; RS_ESTATE otherwise): the
 * per-vertex sparse rows of the Step 2a/2b tables (Eq. 3, Eq. 5),
 * vertices in original order, each row's nonzero columns ascending (column i =
 * rs_get_targets()[i]). off_out int64[n+1] (row v = [off[v], off[v+1])),
 * cols_out / cnt_out int32[E], omega_out double[E] (omega_v(column)),
 * omega_abs_out double[n] (omega_v(c) of every column absent from the row);
 * any pointer may be NULL; n_entries_out receives E (query it first with the
 * arrays NULL to size them). Requires rs_score. */
rs_status rs_get_comm_tables(rs_ctx *ctx, int64_t *off_out, int32_t *cols_out, int32_t *cnt_out, double *omega_out,
                             double *omega_abs_out, int64_t *n_entries_out);

/* Target communities in column order (int32[k]) and k. Requires communities.
 * In the all-communities mode k can be large: query k with targets_out = NULL. */
rs_status rs_get_targets(rs_ctx *ctx, int32_t *targets_out, int32_t *k_out);

/* Number of librs kernels launched on ctx since creation (bench accounting). */
int64_t rs_kernel_launches(const rs_ctx *ctx);

/* Test hook, process-wide: byte in [0, 255] = every device allocation librs
 * makes from now on is filled with that byte before use; -1 = off (default).
 * A result that changes with the byte reveals a read of memory no kernel wrote
 * (tests/test_gpu_hygiene.py; the stand-in for compute-sanitizer initcheck). */
void rs_debug_poison(int32_t byte);

/* ---- NEXT-1: robustness evaluation (PAPER §VII.B). ----
 * Absolute AWCC of the vertex set S (original ids, e.g. the top-K of rs_topk)
 * under cumulative random removal: AWCC = (1/|S|) sum_{v in S} |zeta(v)|/d(v),
 * zeta(v) the community ids (as given to rs_set_communities) of v's surviving
 * neighbours, d(v) the ORIGINAL degree; a removed v contributes 0.
 * Trial t keys every item -- undirected edge {u, v} with id min << 32 | max, or
 * vertex v -- with mix64(s_t ^ id), mix64 the SplitMix64 finaliser and
 * s_t = mix64(seed + (2t + mode) * 0x9E3779B97F4A7C15); step j = 0..J
 * (J = max_pct / step_pct) removes the floor(j * step_pct * M / 100) items of
 * smallest key (M = |E| or |V|), so the removal sets are nested (DESIGN C-28,
 * C-29). zeta_out int32[trials][J+1][|S|] (host, or NULL) receives |zeta_j(v)|;
 * mean_out double[J+1] (host, or NULL) the mean over trials of each step's
 * AWCC (per trial: sum over S in order of |zeta|/d, / |S|; then the trial sum
 * in order, / trials); *steps_out = J + 1. S may be host or device memory.
 * Requires rs_load_csr and rs_set_communities. RS_EINVAL on an empty S, an
 * out-of-range id, a bad mode, step_pct < 1, max_pct outside [0, 100],
 * trials < 1 or more than 126 steps; RS_ENOMEM / RS_ECUDA on device errors. */
#define RS_REMOVE_EDGES 0
#define RS_REMOVE_NODES 1
rs_status rs_awcc_removal(rs_ctx *ctx, const int32_t *S, int64_t nS, int32_t mode, int32_t step_pct,
                          int32_t max_pct, int32_t trials, uint64_t seed, int32_t *zeta_out, double *mean_out,
                          int64_t *steps_out);

/* ---- NEXT-4: structural hole influence index (PAPER §VII.A). ----
 * SHII(u) = (influenced vertices outside C(u)) / (influenced vertices) of a
 * diffusion seeded at u, averaged over `runs` Monte-Carlo runs (the seed is
 * always influenced). Run r of model m draws from s_r = mix64(seed + (2r + m + 1)
 * * 0xD1B54A32D192ED03) on the caller's (original) ids (DESIGN reading C-31):
 * RS_DIFFUSE_IC, independent cascade with probability p: a newly active a
 * activates an inactive neighbour b iff mix64(s_r ^ (a << 32 | b)) < floor(p 2^64)
 * (always when p >= 1); RS_DIFFUSE_LT, linear threshold: theta_v = mix64(s_r ^ v)
 * / 2^64, an inactive v activates once (active neighbours) / d(v) >= theta_v with
 * at least one active neighbour (exact integer test). influenced_out
 * int64[|S|][runs][2] (host or NULL) receives {influenced, outside C(seed)};
 * shii_out double[|S|] (host or NULL) the per-seed means (summed in run order);
 * *mean_out the mean over S (in order). S may be host or device memory.
 * Requires rs_load_csr and rs_set_communities (C is community_of). RS_EINVAL on
 * an empty S, an out-of-range id, a bad model, p outside [0, 1] or runs < 1. */
#define RS_DIFFUSE_IC 0
#define RS_DIFFUSE_LT 1
rs_status rs_shii(rs_ctx *ctx, const int32_t *S, int64_t nS, int32_t model, double p, int32_t runs, uint64_t seed,
                  int64_t *influenced_out, double *shii_out, double *mean_out);

/* ---- Multi-GPU host protocol. Pure host functions on host
 * arrays, no context, no device work; rs_create_dist / rs_topk call them, and
 * they are exported so that the protocol can be exercised without GPUs. ---- */

/* Contiguous vertex ranges balanced by work: work_incl int64[n] is the
 * inclusive prefix sum of a non-negative per-vertex work estimate (librs uses
 * d(u) + 1 in its internal numbering). bounds_out int64[world+1]: rank r owns
 * [bounds[r], bounds[r+1]); bounds[0] = 0, bounds[world] = n, non-decreasing;
 * boundary r is the first vertex after the prefix reaches ceil(total r / world).
 * RS_EINVAL if n < 0, world < 1 or a pointer is NULL (work_incl may be NULL
 * when n == 0). */
rs_status rs_split_ranges(int64_t n, const int64_t *work_incl, int32_t world, int64_t *bounds_out);

/* A rank's candidate list of Step 4, on the host: the first min(K,
 * count) of the (score, id) pairs by (key descending, id ascending) -- key =
 * the IEEE bits of the non-negative score, -0.0 folded to +0.0 -- then
 * padding (0, INT32_MAX) up to K entries, into keys_out uint64[K] / ids_out
 * int32[K]. The same order and padding as the GPU's filtered local select of
 * rs_topk; used by the CPU tests of the protocol. RS_EINVAL on bad arguments. */
rs_status rs_local_candidates(int64_t count, const double *scores, const int32_t *ids, int64_t K,
                              uint64_t *keys_out, int32_t *ids_out);

/* Step 4 merge of the per-rank top-K candidate lists gathered from all
 * ranks: keys uint64[count] are the IEEE-754 bits of the non-negative scores
 * (-0.0 folded to +0.0: monotone as integers), ids int32[count] the original
 * vertex ids; padding entries are (0, INT32_MAX). Writes the first
 * min(K, count) by (key descending, id ascending) to ids_out int32[K] and, if
 * not NULL, their scores to scores_out double[K]; *count_out receives the
 * number written. Deterministic: every rank computes the same result. */
rs_status rs_merge_candidates(int64_t count, const uint64_t *keys, const int32_t *ids, int64_t K,
                              int32_t *ids_out, double *scores_out, int64_t *count_out);

#ifdef __cplusplus
}
#endif
#endif /* RS_H_ */

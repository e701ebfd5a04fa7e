// C-ABI of librs (include/rs.h): argument checking, device memory ownership,
// call-order state machine, stream fork/join for the degree bins, phase
// timing and the NCCL exchange steps of the multi-GPU path.
#include "rs_internal.cuh"
#include <vector>
#include "rs_protocol.h"
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <climits>
#include <string>
#include <dlfcn.h>

namespace rs {
cudaError_t launch_log2_table(Ctx &c, double *t, int64_t len);
cudaError_t launch_phase_a_impl(Ctx &c, const double *l2t, int64_t l2n, bool parity, int64_t lo, int64_t hi);
cudaError_t launch_topk_select(Ctx &c, int64_t K, int64_t lo, int64_t hi, unsigned long long *cand_key,
                               int32_t *cand_id, const int32_t *own_inv, int64_t own_lo, int64_t own_hi,
                               bool compact = false);
cudaError_t tk_sort_emit(Ctx &c, unsigned long long *key, int32_t *id, int64_t cnt, int64_t out, int32_t *ids_out,
                         double *scores_out, bool compact = false);
cudaError_t launch_partition(Ctx &c);
}  // namespace rs

using rs::Ctx;

int rs::g_poison = -1;

extern "C" void rs_debug_poison(int32_t byte) { rs::g_poison = (byte >= 0 && byte <= 255) ? (int)byte : -1; }

#ifdef RS_WITH_NCCL
const rs::NcclApi *rs::nccl_api(std::string *err) {
    static rs::NcclApi api;
    static int state = 0;   // 0 untried, 1 ok, -1 failed
    static std::string why;
    if (state == 0) {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char *path = getenv("RS_NCCL_LIBRARY");
            h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        state = -1;
        if (!h) {
            why = std::string("cannot load libnccl.so.2: ") + dlerror();
        } else {
            bool ok = true;
            auto sym = [&](const char *name) { void *p = dlsym(h, name); ok = ok && p; return p; };
            api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
            api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
            api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
            api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
            api.Reduce = (decltype(api.Reduce))sym("ncclReduce");
            api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
            if (ok) state = 1; else why = "libnccl.so.2 lacks a required symbol";
        }
    }
    if (state != 1) { if (err) *err = why; return nullptr; }
    return &api;
}
#endif

struct rs_ctx {
    Ctx c;
    double *l2t = nullptr;
    int64_t l2n = 0;
    int32_t *utargets = nullptr;     // device copy of user targets
    int32_t *stage_i32 = nullptr;    // device staging for host outputs
    double *stage_f64 = nullptr;
    int64_t stage_cap = 0;
    unsigned long long *cand_key = nullptr;
    int32_t *cand_id = nullptr;
    int64_t cand_cap = 0;
    size_t tk_scratch = 0;
};

static std::string g_create_err;
static constexpr int64_t kPipeMin = 1 << 24;     // pipelined host col_idx copy from this many entries
static constexpr int64_t kPipeChunk = 1 << 24;   // entries per copied chunk (64 MB)

static rs_status fail(rs_ctx *ctx, rs_status s, const std::string &m) {
    if (ctx) ctx->c.err = m; else g_create_err = m;
    return s;
}

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess) return fail(ctx, RS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#ifdef RS_WITH_NCCL
#define NK(expr)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess) return fail(ctx, RS_ENCCL, std::string(#expr) + ": " + rs::nccl_api(nullptr)->GetErrorString(r_)); \
    } while (0)
#define NCCL (*rs::nccl_api(nullptr))
#endif

// a collective of the exchange layer (rs_xport.cu)
#define XK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, RS_ENCCL, std::string(#expr) + ": " +                            \
                                           (c.xp->msg.empty() ? cudaGetErrorString(e_) : c.xp->msg)); \
    } while (0)

static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <class T>
static cudaError_t dalloc(T **p, size_t count) {
    if (*p) { cudaFree(*p); *p = nullptr; }
    if (count == 0) count = 1;
    return rs::dmalloc(p, sizeof(T) * count);
}
template <class T>
static void dfree(T *&p) {
    if (p) cudaFree(p);
    p = nullptr;
}

static void fork(Ctx &c) {
    cudaEventRecord(c.ev_fork, c.stream);
    for (int i = 0; i < rs::kNumBins + 1; i++) cudaStreamWaitEvent(c.side[i], c.ev_fork, 0);
}
static void join(Ctx &c) {
    for (int i = 0; i < rs::kNumBins + 1; i++) {
        cudaEventRecord(c.ev_join[i], c.side[i]);
        cudaStreamWaitEvent(c.stream, c.ev_join[i], 0);
    }
}

// ------------------------------------------------------------------ lifecycle
static rs_status create_common(rs_ctx **out, int device, void *cuda_stream) {
    rs_ctx *ctx = nullptr;
    if (!out) return fail(nullptr, RS_EINVAL, "rs_create: out is NULL");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return fail(nullptr, RS_EINVAL, "rs_create: no CUDA device " + std::to_string(device));
    }
    if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, RS_ECUDA, "rs_create: cudaSetDevice failed");
    ctx = new rs_ctx();
    Ctx &c = ctx->c;
    c.device = device;
    c.stream = (cudaStream_t)cuda_stream;
    for (int i = 0; i < rs::kNumBins + 1; i++) {
        CK(cudaStreamCreateWithFlags(&c.side[i], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c.ev_join[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_zero, cudaEventDisableTiming));
    for (int i = 0; i < 8; i++) CK(cudaEventCreate(&c.ev_phase[i]));
    CK(dalloc(&c.scal, rs::kScalCount));
    CK(cudaMemset(c.scal, 0, sizeof(unsigned long long) * rs::kScalCount));
    CK(dalloc(&c.tk_hist, 2048));
    CK(dalloc(&c.targets, rs::kMaxK));
    CK(dalloc(&ctx->utargets, rs::kMaxK));
    *out = ctx;
    return RS_OK;
}

extern "C" rs_status rs_create(rs_ctx **out, int device, void *cuda_stream) {
    return create_common(out, device, cuda_stream);
}

extern "C" rs_status rs_nccl_unique_id(uint8_t id_out[128]) {
#ifdef RS_WITH_NCCL
    if (!id_out) return fail(nullptr, RS_EINVAL, "rs_nccl_unique_id: NULL");
    std::string why;
    if (!rs::nccl_api(&why)) return fail(nullptr, RS_ENCCL, why);
    ncclUniqueId id;
    if (NCCL.GetUniqueId(&id) != ncclSuccess) return fail(nullptr, RS_ENCCL, "ncclGetUniqueId failed");
    memcpy(id_out, &id, 128);
    return RS_OK;
#else
    (void)id_out;
    return fail(nullptr, RS_ENCCL, "librs built without NCCL");
#endif
}

#ifdef RS_WITH_NCCL
// rs_nccl_selftest: each NcclXport collective on a one-rank communicator, results
// checked bit for bit (world 1: every collective leaves / copies its input)
static rs_status nccl_selftest_run(rs::Xport &xp, cudaStream_t s, size_t bytes) {
    rs_ctx *ctx = nullptr;
    const size_t nw = bytes / 8;
    std::vector<unsigned long long> h(nw), back(nw);
    for (size_t i = 0; i < nw; i++) h[i] = 0x9E3779B97F4A7C15ull * (i + 1) ^ (i << 7);
    unsigned long long *a = nullptr, *b = nullptr;
    CK(cudaMalloc((void **)&a, bytes));
    rs_status st = RS_OK;
    auto check = [&](const unsigned long long *d, const char *what) -> rs_status {
        cudaError_t e = cudaMemcpyAsync(back.data(), d, bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return fail(nullptr, RS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
        for (size_t i = 0; i < nw; i++)
            if (back[i] != h[i])
                return fail(nullptr, RS_ECUDA, std::string("rs_nccl_selftest: ") + what + " changed word " +
                                                   std::to_string(i));
        return RS_OK;
    };
    auto xk = [&](cudaError_t e, const char *what) -> rs_status {
        if (e == cudaSuccess) return RS_OK;
        return fail(nullptr, RS_ENCCL, std::string(what) + ": " + xp.msg);
    };
    const size_t off[1] = {0}, len_b[1] = {bytes}, len_w[1] = {nw};
    cudaError_t e = cudaMalloc((void **)&b, bytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a, h.data(), bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) st = fail(nullptr, RS_ECUDA, std::string("rs_nccl_selftest: ") + cudaGetErrorString(e));
    if (st == RS_OK) st = xk(xp.allreduce_u64(a, nw, false, s), "allreduce sum");
    if (st == RS_OK) st = check(a, "allreduce sum");
    if (st == RS_OK) st = xk(xp.allreduce_u64(a, nw, true, s), "allreduce max");
    if (st == RS_OK) st = check(a, "allreduce max");
    if (st == RS_OK) st = xk(xp.allgatherv(a, off, len_b, s), "allgatherv");
    if (st == RS_OK) st = check(a, "allgatherv");
    if (st == RS_OK) st = xk(xp.reduce_scatterv_u64(a, off, len_w, s), "reduce_scatterv");
    if (st == RS_OK) st = check(a, "reduce_scatterv");
    if (st == RS_OK) {
        e = cudaMemsetAsync(b, 0, bytes, s);
        if (e != cudaSuccess) st = fail(nullptr, RS_ECUDA, cudaGetErrorString(e));
    }
    if (st == RS_OK) st = xk(xp.allgather(a, b, bytes, s), "allgather");
    if (st == RS_OK) st = check(b, "allgather");
    cudaStreamSynchronize(s);
    cudaFree(a);
    if (b) cudaFree(b);
    return st;
}
#endif

extern "C" rs_status rs_nccl_selftest(int device, void *cuda_stream, size_t bytes) {
#ifdef RS_WITH_NCCL
    rs_ctx *ctx = nullptr;
    if (bytes < 64 || bytes % 8) return fail(nullptr, RS_EINVAL, "rs_nccl_selftest: bytes must be >= 64, a multiple of 8");
    std::string why;
    if (!rs::nccl_api(&why)) return fail(nullptr, RS_ENCCL, why);
    CK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)cuda_stream, own = nullptr;
    if (!s) {
        CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
        s = own;
    }
    ncclUniqueId id;
    ncclComm_t comm = nullptr;
    rs_status st = RS_OK;
    ncclResult_t r = NCCL.GetUniqueId(&id);
    if (r == ncclSuccess) r = NCCL.CommInitRank(&comm, 1, id, 0);
    if (r != ncclSuccess) {
        st = fail(nullptr, RS_ENCCL, std::string("rs_nccl_selftest: communicator: ") + NCCL.GetErrorString(r));
    } else {
        rs::Xport *xp = rs::make_nccl_xport(comm, 1);
        st = nccl_selftest_run(*xp, s, bytes);
        delete xp;
        NCCL.CommDestroy(comm);
    }
    if (own) cudaStreamDestroy(own);
    return st;
#else
    (void)device; (void)cuda_stream; (void)bytes;
    return fail(nullptr, RS_ENCCL, "librs built without NCCL");
#endif
}

extern "C" rs_status rs_create_dist(rs_ctx **out, int device, void *cuda_stream, int rank, int world,
                                    const uint8_t nccl_id[128]) {
    if (world < 1 || rank < 0 || rank >= world || !nccl_id)
        return fail(nullptr, RS_EINVAL, "rs_create_dist: bad rank/world/id");
    rs_status s = create_common(out, device, cuda_stream);
    if (s != RS_OK) return s;
    rs_ctx *ctx = *out;
    ctx->c.rank = rank;
    ctx->c.world = world;
#ifdef RS_WITH_NCCL
    if (world > 1) {
        std::string why;
        if (!rs::nccl_api(&why)) return fail(ctx, RS_ENCCL, why);
        ncclUniqueId id;
        memcpy(&id, nccl_id, 128);
        NK(NCCL.CommInitRank(&ctx->c.comm, world, id, rank));
        ctx->c.xp = rs::make_nccl_xport(ctx->c.comm, world);
    }
    return RS_OK;
#else
    if (world > 1) return fail(ctx, RS_ENCCL, "librs built without NCCL");
    return RS_OK;
#endif
}

namespace rs {
EmuWorld *emu_world_of(rs_emu_world *w);
int emu_world_size(EmuWorld *w);
}  // namespace rs

extern "C" rs_status rs_create_emulated(rs_ctx **out, int device, void *cuda_stream, int rank, int world,
                                        rs_emu_world *w) {
    if (!w || world < 1 || rank < 0 || rank >= world) return fail(nullptr, RS_EINVAL, "rs_create_emulated: bad rank/world");
    rs::EmuWorld *ew = rs::emu_world_of(w);
    if (!ew || rs::emu_world_size(ew) != world) return fail(nullptr, RS_EINVAL, "rs_create_emulated: world size mismatch");
    rs_status s = create_common(out, device, cuda_stream);
    if (s != RS_OK) return s;
    (*out)->c.rank = rank;
    (*out)->c.world = world;
    if (world > 1) (*out)->c.xp = rs::make_emu_xport(ew, rank);
    return RS_OK;
}

static void free_graph(rs_ctx *ctx) {
    Ctx &c = ctx->c;
    dfree(c.rowptr); dfree(c.col); dfree(c.perm); dfree(c.inv); dfree(c.scratch); dfree(ctx->l2t); dfree(c.e_pre); c.e_bytes = 0;
    dfree(c.comm_in); dfree(c.comm_id); dfree(c.lab); dfree(c.vrec); dfree(c.pidx); dfree(c.plab); dfree(c.pplus); dfree(c.wps); dfree(c.pc2); dfree(c.amat);
    dfree(c.acc1); dfree(c.acc_hub); dfree(c.t2); dfree(c.n1); dfree(c.score); dfree(c.f); dfree(c.omega); dfree(c.bql);
    dfree(c.cid); dfree(c.srec); dfree(c.ctk); dfree(c.ctb); dfree(c.pwr); dfree(c.prv); dfree(c.aself);
    dfree(c.xsum); dfree(c.n2s);
    dfree(c.pk_id); c.pk_cap = 0;
    dfree(c.pk_m); c.pkm_cap = 0;
    dfree(c.xg); c.xg_cap = 0;
    dfree(c.bsum); dfree(c.vx); c.dist_cap = 0;
    c.sp_cap = 0;
    c.k_alloc = 0; c.scratch_bytes = 0; c.loaded = c.has_comm = c.scored = false;
    c.cap_n = c.cap_nnz = 0;
    ctx->l2n = 0;
}

extern "C" void rs_destroy(rs_ctx *ctx) {
    if (!ctx) return;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (c.stream) cudaStreamSynchronize(c.stream);
    free_graph(ctx);
    dfree(c.chist); dfree(c.ccode); dfree(c.code32); dfree(c.csort); dfree(c.targets); dfree(c.scal); dfree(c.tk_hist); dfree(c.arena);
    dfree(ctx->utargets); dfree(ctx->stage_i32); dfree(ctx->stage_f64); dfree(ctx->cand_key); dfree(ctx->cand_id);
    dfree(c.tk_gkey); dfree(c.tk_gid);
    delete c.xp;
    c.xp = nullptr;
    for (int i = 0; i < rs::kNumBins + 1; i++) {
        if (c.side[i]) cudaStreamDestroy(c.side[i]);
        if (c.ev_join[i]) cudaEventDestroy(c.ev_join[i]);
    }
    if (c.ev_fork) cudaEventDestroy(c.ev_fork);
    if (c.ev_zero) cudaEventDestroy(c.ev_zero);
    for (cudaEvent_t ev : c.ev_chunk) cudaEventDestroy(ev);
    for (int i = 0; i < 8; i++) if (c.ev_phase[i]) cudaEventDestroy(c.ev_phase[i]);
#ifdef RS_WITH_NCCL
    if (c.comm) NCCL.CommDestroy(c.comm);
#endif
    delete ctx;
}

extern "C" const char *rs_last_error(const rs_ctx *ctx) {
    return ctx ? ctx->c.err.c_str() : g_create_err.c_str();
}

extern "C" int64_t rs_kernel_launches(const rs_ctx *ctx) { return ctx ? ctx->c.launches : 0; }

// ------------------------------------------------------------------ load
extern "C" rs_status rs_load_csr(rs_ctx *ctx, int64_t n, const int64_t *row_offsets, const int32_t *col_idx,
                                 uint32_t flags) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (n < 1 || n >= (1ll << 31)) return fail(ctx, RS_EINVAL, "rs_load_csr: n must be in [1, 2^31)");
    if (!row_offsets || !col_idx) return fail(ctx, RS_EINVAL, "rs_load_csr: NULL array");
    const bool dev_ro = is_device_ptr(row_offsets), dev_ci = is_device_ptr(col_idx);
    int64_t first = 0, nnz = 0;
    if (dev_ro) {
        CK(cudaMemcpy(&first, row_offsets, sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&nnz, row_offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    } else {
        first = row_offsets[0];
        nnz = row_offsets[n];
    }
    if (first != 0) return fail(ctx, RS_EINVAL, "rs_load_csr: row_offsets[0] != 0");
    if (nnz < 0) return fail(ctx, RS_EINVAL, "rs_load_csr: row_offsets[n] < 0");
    // buffers are reused when the new graph fits their capacity (no free/alloc per load)
    const bool fits = c.cap_n >= n && c.cap_nnz >= nnz;
    if (!fits) free_graph(ctx);
    c.loaded = c.has_comm = c.scored = false;
    c.acc_zero = c.bql_zero = c.bsum_zero = false;
    c.nwide_k = 0;
    c.n = n;
    c.nnz = nnz;
    // arena: host-input staging + relabel temporaries (grow-only)
    const size_t stage_b = (dev_ro ? 0 : 8 * (size_t)(n + 1) + 256) + (dev_ci ? 0 : 4 * (size_t)std::max<int64_t>(nnz, 1) + 256);
    const size_t arena_need = stage_b + rs::relabel_arena_bytes(n, nnz);
    if (arena_need > c.arena_bytes) {
        dfree(c.arena);
        c.arena_bytes = 0;
        CK(rs::dmalloc(&c.arena, arena_need));
        c.arena_bytes = arena_need;
    }
    char *ap = (char *)c.arena;
    // the caller's (original-id) CSR on the device: borrowed if already there
    const int64_t *rp_o = row_offsets;
    const int32_t *col_o = col_idx;
    if (!dev_ro) {
        int64_t *rp_tmp = (int64_t *)ap;
        ap += (8 * (size_t)(n + 1) + 255) & ~(size_t)255;
        CK(cudaMemcpyAsync(rp_tmp, row_offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, c.stream));
        rp_o = rp_tmp;
    }
    // host col_idx without validation: copied in chunks on a side stream while
    // the rows already there are relabelled (launch_relabel_rows below)
    const int chunk_log2 = (int)((flags >> 8) & 0x1Fu);   // RS_LOAD_CHUNK_LOG2 test hook
    const int64_t pipe_chunk = chunk_log2 >= 4 ? (1ll << chunk_log2) : kPipeChunk;
    const bool pipe = !dev_ci && !dev_ro && !(flags & RS_VALIDATE) && (nnz >= kPipeMin || chunk_log2 >= 4) && nnz > 0;
    int32_t *col_tmp = nullptr;
    if (!dev_ci) {
        col_tmp = (int32_t *)ap;
        ap += (4 * (size_t)std::max<int64_t>(nnz, 1) + 255) & ~(size_t)255;
        if (nnz && !pipe) CK(cudaMemcpyAsync(col_tmp, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c.stream));
        col_o = col_tmp;
    }
    if (flags & RS_VALIDATE) {
        unsigned long long init[3] = {0ull, ~0ull, 0ull};
        CK(cudaMemcpyAsync(c.scal + rs::kScalErr, init, 2 * sizeof(unsigned long long), cudaMemcpyHostToDevice, c.stream));
        CK(rs::launch_validate(c, rp_o, col_o));
        unsigned long long er[2];
        CK(cudaMemcpyAsync(er, c.scal + rs::kScalErr, sizeof(er), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        if (er[0]) {
            static const char *what[] = {"", "row_offsets decreasing", "col_idx out of range",
                                         "row not strictly ascending (unsorted or duplicate)", "self-loop",
                                         "graph not symmetric"};
            std::string m = std::string("rs_load_csr: ") + (er[0] < 6 ? what[er[0]] : "invalid") + " at row " +
                            std::to_string((long long)er[1]);
            return fail(ctx, RS_EINVAL, m);
        }
    }
    if (!fits) {
        CK(dalloc(&c.rowptr, n + 1));
        CK(dalloc(&c.col, nnz + 4));    // + 4: Phase A reads rows as aligned 16-byte pieces
        CK(dalloc(&c.perm, n));
        CK(dalloc(&c.inv, n));
        const size_t scratch = 24 * (size_t)(n + 1) + (64u << 20);
        CK(rs::dmalloc(&c.scratch, scratch));
        c.scratch_bytes = scratch;
        CK(dalloc(&c.comm_in, n));
        CK(dalloc(&c.comm_id, n));
        CK(dalloc(&c.lab, n));
        CK(dalloc(&c.vrec, n));
        CK(dalloc(&c.pidx, nnz));
        CK(dalloc(&c.plab, nnz));
        CK(dalloc(&c.pplus, nnz + 4));   // + 4: aligned 16-byte probes may read past the end
        CK(dalloc(&c.pc2, n));
        CK(dalloc(&c.acc1, 3 * n));
        c.n_hub = std::min<int64_t>(n, rs::kHubMax);
        CK(dalloc(&c.acc_hub, 3 * rs::kHubStripes * c.n_hub));
        CK(dalloc(&c.n1, n));
        CK(dalloc(&c.t2, n));
        CK(dalloc(&c.score, n));
        c.cap_n = n;
        c.cap_nnz = nnz;
    }
    // internal degree-descending numbering (k_setup.cu launch_relabel*)
    if (pipe) {
        // chunks of about kPipeChunk entries at original row boundaries
        std::vector<int64_t> cut{0};
        for (int64_t v = 0; v < n;) {
            const int64_t target = row_offsets[v] + pipe_chunk;
            int64_t w = std::upper_bound(row_offsets + v + 1, row_offsets + n + 1, target) - row_offsets - 1;
            if (w <= v) w = v + 1;
            if (w > n) w = n;
            cut.push_back(w);
            v = w;
        }
        const size_t nch = cut.size() - 1;
        while (c.ev_chunk.size() < nch) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            c.ev_chunk.push_back(ev);
        }
        cudaStream_t cs = c.side[rs::kNumBins];
        CK(cudaEventRecord(c.ev_fork, c.stream));   // the arena is free once earlier work is done
        CK(cudaStreamWaitEvent(cs, c.ev_fork, 0));
        for (size_t i = 0; i < nch; i++) {
            const int64_t e0 = row_offsets[cut[i]], e1 = row_offsets[cut[i + 1]];
            if (e1 > e0)
                CK(cudaMemcpyAsync(col_tmp + e0, col_idx + e0, sizeof(int32_t) * (e1 - e0), cudaMemcpyHostToDevice, cs));
            CK(cudaEventRecord(c.ev_chunk[i], cs));
        }
        CK(rs::launch_relabel_prepare(c, rp_o, ap, c.arena_bytes - (size_t)(ap - (char *)c.arena)));
        for (size_t i = 0; i < nch; i++) {
            CK(cudaStreamWaitEvent(c.stream, c.ev_chunk[i], 0));
            CK(rs::launch_relabel_rows(c, rp_o, col_o, cut[i], cut[i + 1]));
        }
        CK(rs::launch_relabel_finish(c));
    } else {
        CK(rs::launch_relabel(c, rp_o, col_o, ap, c.arena_bytes - (size_t)(ap - (char *)c.arena)));
    }
    CK(rs::launch_e_items(c));
    const int64_t l2n = std::min<int64_t>(c.d_max + 1, 1ll << 20);
    if (l2n > ctx->l2n) {
        CK(dalloc(&ctx->l2t, l2n));
        ctx->l2n = l2n;
        CK(rs::launch_log2_table(c, ctx->l2t, ctx->l2n));
    }
    c.head_lo = 0;
    c.head_hi = n;
    if (c.world > 1) CK(rs::launch_partition(c));
    CK(cudaStreamSynchronize(c.stream));
    c.loaded = true;
    return RS_OK;
}

// ------------------------------------------------------------------ communities
// all-communities mode (NEXT-2): every community is a target, sparse tables
static rs_status set_communities_all(rs_ctx *ctx, int64_t mx) {
    Ctx &c = ctx->c;
    const size_t need = rs::sparse_rank_bytes(mx + 1);
    if (need > c.csort_bytes) {
        dfree(c.csort);
        c.csort_bytes = 0;
        CK(rs::dmalloc(&c.csort, need));
        c.csort_bytes = need;
    }
    if (c.sp_cap < c.cap_nnz || !c.cid) {
        const int64_t n = c.cap_n, nnz = std::max<int64_t>(c.cap_nnz, 1);
        CK(dalloc(&c.cid, n)); CK(dalloc(&c.srec, n)); CK(dalloc(&c.aself, n)); CK(dalloc(&c.xsum, n));
        CK(dalloc(&c.n2s, n));
        CK(dalloc(&c.ctk, nnz)); CK(dalloc(&c.ctb, nnz));
        CK(dalloc(&c.pwr, nnz)); CK(dalloc(&c.prv, nnz)); CK(dalloc(&c.wps, nnz));
        c.sp_cap = c.cap_nnz;
    }
    int64_t nc = 0;
    CK(rs::launch_set_communities_all(c, mx, &nc));
    if (nc < 2) return fail(ctx, RS_EINVAL, "rs_set_communities: RS_ALL_COMMUNITIES needs at least 2 distinct communities");
    if (nc >= (1ll << 31)) return fail(ctx, RS_EINVAL, "rs_set_communities: too many communities");
    CK(cudaStreamSynchronize(c.stream));
    unsigned long long nw = 0;
    CK(cudaMemcpy(&nw, c.scal + rs::kScalNWide, sizeof(nw), cudaMemcpyDeviceToHost));
    c.n_wide = (int64_t)nw;
    c.k = (int32_t)nc;
    c.sparse = true;
    c.has_comm = true;
    return RS_OK;
}

extern "C" rs_status rs_set_communities(rs_ctx *ctx, const int32_t *community_of, const int32_t *targets, int32_t k) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.loaded) return fail(ctx, RS_ESTATE, "rs_set_communities: no graph loaded");
    if (!community_of) return fail(ctx, RS_EINVAL, "rs_set_communities: community_of is NULL");
    const bool all = k == RS_ALL_COMMUNITIES;
    if (!all && (k < 2 || k > rs::kMaxK))
        return fail(ctx, RS_EINVAL, "rs_set_communities: k must be in [2, 254] or RS_ALL_COMMUNITIES");
    if (all && targets) return fail(ctx, RS_EINVAL, "rs_set_communities: RS_ALL_COMMUNITIES takes targets = NULL");
    if (c.world > 1 && (all || k > 8))
        return fail(ctx, RS_EINVAL, "rs_set_communities: the multi-GPU path takes k <= 8 explicit-k targets");
    c.scored = false;
    c.has_comm = false;
    CK(cudaMemcpyAsync(c.comm_in, community_of, sizeof(int32_t) * c.n,
                       is_device_ptr(community_of) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    // the id range sizes the community histogram: measured (one host round trip)
    // on the first call and whenever an id reaches the current capacity; in the
    // steady state the histogram kernel itself flags out-of-range ids, so the
    // call synchronises with the host once (to report errors and the targets)
    auto grow = [&](bool &is_all_ok) -> rs_status {
        int64_t mn = 0, mx = 0;
        CK(rs::launch_minmax_i32(c, c.comm_in, c.n, &mn, &mx));
        if (mn < 0) return fail(ctx, RS_EINVAL, "rs_set_communities: negative community id");
        if (mx >= (1ll << 28)) return fail(ctx, RS_EINVAL, "rs_set_communities: community id >= 2^28");
        if (mx + 1 > c.ccap) {
            int64_t cap = std::max<int64_t>(mx + 1, 1024);
            CK(dalloc(&c.chist, cap));
            CK(dalloc(&c.ccode, cap));
            CK(dalloc(&c.code32, cap));
            c.ccap = cap;
        }
        c.cmax = mx;
        is_all_ok = true;
        return RS_OK;
    };
    bool ok = false;
    if (all || c.ccap == 0) {
        rs_status st = grow(ok);
        if (st != RS_OK) return st;
    }
    if (all) return set_communities_all(ctx, c.cmax);
    c.sparse = false;
    if (c.k_alloc != k || c.kn_alloc != c.n) {
        CK(dalloc(&c.f, (size_t)c.n * k));
        CK(dalloc(&c.omega, (size_t)c.n * k));
        CK(dalloc(&c.bql, (size_t)c.n * k));
        c.bql_zero = false;
        CK(dalloc(&c.amat, (size_t)c.n * k));
        c.k_alloc = k;
        c.kn_alloc = c.n;
    }
    c.k = k;
    const int32_t *ut = nullptr;
    if (targets) {
        CK(cudaMemcpyAsync(ctx->utargets, targets, sizeof(int32_t) * k,
                           is_device_ptr(targets) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
        ut = ctx->utargets;
    }
    unsigned long long er = 0, ndist = 0, nw = 0;
    for (int attempt = 0; attempt < 2; attempt++) {
        CK(cudaMemsetAsync(c.scal + rs::kScalErr, 0, sizeof(unsigned long long), c.stream));
        // histogram over the whole capacity (ids beyond the largest seen count 0)
        CK(rs::launch_set_communities(c, c.ccap - 1, ut));
        CK(cudaMemcpyAsync(&er, c.scal + rs::kScalErr, sizeof(er), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(&ndist, c.scal + rs::kScalCnt0, sizeof(ndist), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(c.h_targets, c.targets, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(&nw, c.scal + rs::kScalNWide, sizeof(nw), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        if (er != 12 && er != 13) break;
        // an id outside the histogram: measure the range (errors) and grow, once
        rs_status st = grow(ok);
        if (st != RS_OK) return st;
    }
    if (er == 12 || er == 13) return fail(ctx, RS_EINVAL, "rs_set_communities: community id out of range");
    c.n_wide = (int64_t)nw;
    {
        // B table grid: a <= (k log2(k - 1))^(1/3) (the wide_bound weight bound) and
        // B_w[c] sums at most d_max of them; keep 2 spare bits below 2^64
        const double wb = 2147483648.0 / (2.0 * rs::wide_bound(k));
        const double bmax = std::cbrt(wb) * (double)std::max<int64_t>(c.d_max, 1);
        int q = 40;
        while (q > 16 && bmax * std::ldexp(1.0, q) >= std::ldexp(1.0, 62)) q--;
        c.bq = q;
    }
    if (er == 10)
        return fail(ctx, RS_EINVAL, "rs_set_communities: k = " + std::to_string(k) + " exceeds the " +
                                        std::to_string((long long)ndist) + " distinct communities");
    if (er) return fail(ctx, RS_EINVAL, "rs_set_communities: targets must be distinct ids present in community_of");
    c.has_comm = true;
    return RS_OK;
}

// ------------------------------------------------------------------ multi-GPU exchange
// After each rank's Phase A shard (vertices [head_lo, head_hi)), every rank needs
// for ALL vertices what the other phases read of the 2-hop neighbourhood
// (k_dist.cu): omega_max (max), the B sums (k x n u64, integer sum of every
// rank's pushes), the cube-root rows (all-gather by segment), {|P|, |P+|,
// |P+_T|} per vertex and the ids of the oriented runs P+(x) (all-gathered;
// VRec, PRec and the weights beside P+ entries are rebuilt from them and the
// rows; Phase D reads the summed B pushes and the rows directly). Exact: every value is copied bit for bit, an integer sum, or
// recomputed by the same operation Phase A uses. Bytes: DESIGN.md §7.
static rs_status exchange_phase_a(rs_ctx *ctx) {
    Ctx &c = ctx->c;
    const int W = c.world;
    const int64_t n = c.n, k = c.k;
    std::vector<size_t> off(W), len(W);
    auto seg = [&](size_t per) {
        for (int r = 0; r < W; r++) {
            off[r] = (size_t)c.bounds[r] * per;
            len[r] = (size_t)(c.bounds[r + 1] - c.bounds[r]) * per;
        }
    };
    c.xar_bytes = 8 + 8 * n * k;
    c.xag_bytes = 0;
    c.xrs_bytes = 0;
    XK(c.xp->allreduce_u64(c.scal + rs::kScalOmegaMaxBits, 1, true, c.stream));
    XK(c.xp->allreduce_u64(c.bsum, (size_t)(n * k), false, c.stream));
    seg(sizeof(double) * k);
    XK(c.xp->allgatherv(c.amat, off.data(), len.data(), c.stream));
    CK(rs::launch_vx_pack(c));
    seg(3 * sizeof(int32_t));
    c.xag_bytes += (8 * k + 12) * n;
    XK(c.xp->allgatherv(c.vx, off.data(), len.data(), c.stream));
    CK(rs::launch_vx_unpack(c));
    if (!c.bsum_direct) CK(rs::launch_b_rebuild(c));
    // the heavy P-(y) lists (Phase E's items are dealt over the ranks): gm = prefix
    // of |P-(y)| over y < n_heavy in vertex order; the P+ runs: gpre = prefix of
    // |P+| in vertex order (every rank computes the same); one host read of the
    // segment bounds for both. Both travel packed and Phase E reads them packed
    if (c.xg_cap < n) {
        CK(dalloc(&c.xg, 2 * (size_t)(n + 1)));
        c.xg_cap = n;
    }
    int64_t *gm = c.xg;
    int64_t *gpre = c.xg + (n + 1);
    CK(rs::launch_run_prefix(c, gm, true));
    CK(rs::launch_run_prefix(c, gpre, false));
    std::vector<int64_t> hb(W + 1), gb(W + 1);
    for (int r = 0; r <= W; r++) {
        CK(cudaMemcpyAsync(&hb[r], gm + std::min<int64_t>(c.bounds[r], c.e_nbig), sizeof(int64_t),
                           cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(&gb[r], gpre + c.bounds[r], sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    }
    CK(cudaStreamSynchronize(c.stream));
    if (hb[W] > c.pkm_cap) {
        CK(dalloc(&c.pk_m, (size_t)hb[W]));
        c.pkm_cap = hb[W];
    }
    CK(rs::launch_minus_pack(c, gm));
    for (int r = 0; r < W; r++) {
        off[r] = (size_t)hb[r] * sizeof(int32_t);
        len[r] = (size_t)(hb[r + 1] - hb[r]) * sizeof(int32_t);
    }
    XK(c.xp->allgatherv(c.pk_m, off.data(), len.data(), c.stream));
    c.xag_bytes += 4 * hb[W];
    const int64_t total = gb[W];
    if (total + 4 > c.pk_cap) {                           // + 4: aligned 16-byte probes may read past the end
        CK(dalloc(&c.pk_id, (size_t)total + 4));
        c.pk_cap = total + 4;
    }
    CK(rs::launch_plus_pack(c, gpre));
    for (int r = 0; r < W; r++) {
        off[r] = (size_t)gb[r] * sizeof(int32_t);
        len[r] = (size_t)(gb[r + 1] - gb[r]) * sizeof(int32_t);
    }
    XK(c.xp->allgatherv(c.pk_id, off.data(), len.data(), c.stream));
    c.xag_bytes += 4 * total;
    // Phase E reads every P+ run packed: PRec start -> gpre[x] (after the pack,
    // which read the owned runs from their slots)
    CK(rs::launch_rebase(c, gpre));
    c.mg_packed = true;
    return RS_OK;
}

// ------------------------------------------------------------------ score
extern "C" rs_status rs_score(rs_ctx *ctx, double *scores_out, rs_stats *stats_out, uint32_t flags) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.has_comm) return fail(ctx, RS_ESTATE, "rs_score: call rs_load_csr and rs_set_communities first");
    const int64_t n = c.n;
    c.e_shares = (int)RS_E_SHARES_OF(flags);
    c.variant = (int)((flags >> 16) & 7u);
    if (c.sparse && c.variant)
        return fail(ctx, RS_EINVAL, "rs_score: the NEXT-3 variant flags need explicit targets (k <= 254)");
    if (c.xp) c.xp->score_begin();
    // multi-GPU, RS_REPLICATE_A: every rank runs Phase A over all vertices (the
    // replicated CSR and labels of the north_star's layout), so the only exchange
    // is the Type-I limb reduce-scatter; otherwise Phase A is sharded by range and
    // its outputs exchanged
    c.rep_a = c.world > 1 && (flags & RS_REPLICATE_A);
    const bool shard_a = c.world > 1 && !c.rep_a;
    c.hubs_folded = false;
    c.mg_packed = false;
    CK(cudaEventRecord(c.ev_phase[0], c.stream));
    // the accumulators (and the dense B table) were zeroed on a side stream at the
    // end of the previous rs_score, overlapping rs_topk; otherwise zero them here
    if (c.acc_zero || (!c.sparse && (c.bql_zero || c.bsum_zero))) CK(cudaStreamWaitEvent(c.stream, c.ev_zero, 0));
    if (!c.acc_zero) {
        CK(cudaMemsetAsync(c.acc1, 0, sizeof(unsigned long long) * 3 * n, c.stream));
        CK(cudaMemsetAsync(c.acc_hub, 0, sizeof(unsigned long long) * 3 * rs::kHubStripes * c.n_hub, c.stream));
    }
    c.acc_zero = false;
    c.parity_ok = false;
    CK(cudaMemsetAsync(c.scal + rs::kScalOmegaMaxBits, 0, sizeof(unsigned long long), c.stream));
    CK(cudaMemsetAsync(c.scal + rs::kScalNTri, 0, 2 * sizeof(unsigned long long), c.stream));   // NTri, NProbe
    if (c.sparse) {
        // all-communities mode: Steps 2a-2c into per-vertex community tables, then
        // Step 2d (P lists, per-edge weights, B pushes); each a degree-binned pass
        CK(rs::launch_sparse_sort(c));   // library stream, before the fork
        fork(c);
        CK(rs::launch_sparse_tables(c, ctx->l2t, ctx->l2n));
        join(c);
        fork(c);
        CK(rs::launch_sparse_lists(c));
        join(c);
    } else {
        {
            // the B pushes go to a plain k x n u64 table (half the bytes of the BQL
            // records, so the REDs hit L2 more often; Orkut shape: A 1.99 -> 1.84 ms)
            // and a streaming pass rebuilds BQL: worth it when the pushes per cell
            // (about D / (n k) x the foreign fraction) outweigh the rebuild's 32 B per
            // cell -- measured: Orkut shape (D / nk = 15) step -0.07..-0.11 ms, LJ
            // shape (3.5) +0.07 ms. Multi-GPU always (the sums are exchanged).
            // RS_EXP_BSUM=0/1 forces it off/on; =2 lets Phase D read the sums and
            // the rows directly instead of rebuilding (measured E||D +0.18 ms).
            const char *ex = getenv("RS_EXP_BSUM");
            const bool dense_enough = c.nnz >= 8 * n * (int64_t)c.k;
            c.bsum_mode = shard_a || (c.k <= 8 && (ex ? ex[0] != '0' : dense_enough));
            // multi-GPU: Phase D reads the summed pushes and the gathered rows directly
            // (the rebuild would be a pass over all n k cells on every rank)
            c.bsum_direct = c.bsum_mode && (shard_a || (ex && ex[0] == '2'));
        }
        if (c.bsum_mode) {
            if (c.dist_cap < n * c.k) {
                CK(dalloc(&c.bsum, (size_t)(n * c.k)));
                CK(dalloc(&c.vx, (size_t)(3 * n)));
                c.dist_cap = n * c.k;
                c.bsum_zero = false;
            }
            if (!c.bsum_zero) CK(cudaMemsetAsync(c.bsum, 0, sizeof(unsigned long long) * (size_t)n * c.k, c.stream));
        } else if (!c.bql_zero) {
            CK(cudaMemsetAsync(c.bql, 0, sizeof(rs::BQL) * (size_t)n * c.k, c.stream));   // B limbs
        }
        c.bql_zero = c.bsum_zero = false;
        // Phase A: border + histogram + weights + P lists + omega_max partials, the
        // orientation of G' and the B-table pushes
        fork(c);
        CK(rs::launch_phase_a_impl(c, ctx->l2t, ctx->l2n, false, shard_a ? c.head_lo : 0,
                                   shard_a ? c.head_hi : n));   // own range (sharded) or all
        join(c);
    }
    CK(cudaEventRecord(c.ev_phase[1], c.stream));
    c.xar_bytes = c.xag_bytes = c.xrs_bytes = 0;
    if (shard_a) {
        // multi-GPU: Phase A ran on this rank's vertices only; exchange what the
        // other phases read of the 2-hop neighbourhood (ms_phase[1])
        c.xp->tag = 1;
        rs_status st = exchange_phase_a(ctx);
        if (st != RS_OK) return st;
    } else if (c.bsum_mode && !c.sparse && !c.bsum_direct) {
        CK(rs::launch_b_rebuild(c));
    }
    CK(cudaEventRecord(c.ev_phase[2], c.stream));
    // Phase E (Type-I triangles) and Phase D (Type-II pull, which needs only
    // Phase A's B table) run concurrently: E heavy on the library stream, E light
    // and the D bins on the forked streams
    fork(c);
    CK(rs::launch_phase_d(c));                           // first: their blocks are queued ahead of
    CK(rs::launch_phase_e_on(c, c.side[rs::kNumBins]));  // the persistent heavy Phase E grid
    join(c);
    if (c.world > 1 && getenv("RS_DEBUG_E")) {      // per-rank Type-I work (balance diagnostics)
        unsigned long long v[2];
        CK(cudaMemcpyAsync(v, c.scal + rs::kScalNTri, sizeof(v), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        fprintf(stderr, "[rank %d] own [%lld, %lld) n_heavy %lld: triangles %llu probes %llu\n", c.rank,
                (long long)c.head_lo, (long long)c.head_hi, (long long)c.e_nbig, v[0], v[1]);
    }
    CK(cudaEventRecord(c.ev_phase[3], c.stream));
    if (c.world > 1) {
        // Phase E is split by middle vertex: sum every head's Type-I limbs (and the
        // triangle/probe counters) over the ranks; integer sums, exact in any order
        // the hub stripes are folded into the limbs first (exact integer adds), then
        // each rank receives only its own heads' sums (a reduce-scatter: half the
        // bytes an all-reduce moves)
        CK(rs::launch_fold_hubs(c));
        std::vector<size_t> off(c.world), len(c.world);
        for (int r = 0; r < c.world; r++) {
            off[r] = (size_t)(3 * c.bounds[r]);
            len[r] = (size_t)(3 * (c.bounds[r + 1] - c.bounds[r]));
        }
        c.xrs_bytes = 8 * 3 * n;
        c.xar_bytes += 16;
        c.xp->tag = 4;
        XK(c.xp->reduce_scatterv_u64(c.acc1, off.data(), len.data(), c.stream));
        XK(c.xp->allreduce_u64(c.scal + rs::kScalNTri, 2, false, c.stream));
    }
    CK(cudaEventRecord(c.ev_phase[4], c.stream));
    // multi-GPU: a rank writes only its heads' scores (scattered in original order)
    if (c.world > 1) CK(cudaMemsetAsync(c.score, 0, sizeof(double) * n, c.stream));
    // finalize: Type-II + Type-I sums, / omega_max / d(d-1), original order
    CK(rs::launch_finalize(c));
    CK(cudaEventRecord(c.ev_phase[5], c.stream));
    if (c.world > 1 && (flags & RS_GATHER_SCORES)) {
        // owned heads are a contiguous internal range, scattered in original order;
        // every other entry is +0.0 (all-zero bits) on a rank, so an integer sum of
        // the bit patterns gathers the scores exactly
        c.xar_bytes += 8 * n;
        c.xp->tag = 6;
        XK(c.xp->allreduce_u64((unsigned long long *)c.score, (size_t)n, false, c.stream));
    }
    // zero the accumulators (and the dense B table) for the next rs_score on a side
    // stream: it overlaps whatever the caller does next (rs_topk, getters)
    {
        cudaStream_t zs = c.side[rs::kNumBins];
        CK(cudaEventRecord(c.ev_fork, c.stream));
        CK(cudaStreamWaitEvent(zs, c.ev_fork, 0));
        CK(cudaMemsetAsync(c.acc1, 0, sizeof(unsigned long long) * 3 * n, zs));
        CK(cudaMemsetAsync(c.acc_hub, 0, sizeof(unsigned long long) * 3 * rs::kHubStripes * c.n_hub, zs));
        // the table the next pushes go to: the plain sums (bsum mode: BQL is
        // rewritten whole by the rebuild) or the BQL limbs
        if (!c.sparse && c.bsum_mode) {
            CK(cudaMemsetAsync(c.bsum, 0, sizeof(unsigned long long) * (size_t)n * c.k, zs));
            c.bsum_zero = true;
        } else if (!c.sparse) {
            CK(cudaMemsetAsync(c.bql, 0, sizeof(rs::BQL) * (size_t)n * c.k, zs));
            c.bql_zero = true;
        }
        CK(cudaEventRecord(c.ev_zero, zs));
        c.acc_zero = true;
    }
    c.scored = true;
    if (c.xp) c.xp->score_end(c.stream);
    if (scores_out) {
        const bool dev = is_device_ptr(scores_out);
        CK(cudaMemcpyAsync(scores_out, c.score, sizeof(double) * n,
                           dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
        if (!dev) CK(cudaStreamSynchronize(c.stream));
    }
    if (stats_out) {
        int64_t st[4];
        CK(rs::launch_stats(c, st));
        rs_stats s;
        memset(&s, 0, sizeof(s));
        s.n = n;
        s.m = c.nnz / 2;
        s.n_border = st[0];
        s.n_pred_entries = st[1];
        s.n_triangles = st[2];
        s.n_probes = st[3];
        unsigned long long wb = 0;
        CK(cudaMemcpy(&wb, c.scal + rs::kScalOmegaMaxBits, sizeof(wb), cudaMemcpyDeviceToHost));
        memcpy(&s.omega_max, &wb, sizeof(double));
        // ms_phase: [0] A (incl. zeroing) [1] the Phase A exchange (multi-GPU; else 0)
        // [2] E (Type-I) || D (Type-II) [3] finalize [4] the limb sum over the ranks
        CK(cudaEventElapsedTime(&s.ms_phase[0], c.ev_phase[0], c.ev_phase[1]));
        CK(cudaEventElapsedTime(&s.ms_phase[1], c.ev_phase[1], c.ev_phase[2]));
        CK(cudaEventElapsedTime(&s.ms_phase[2], c.ev_phase[2], c.ev_phase[3]));
        CK(cudaEventElapsedTime(&s.ms_phase[3], c.ev_phase[4], c.ev_phase[5]));
        CK(cudaEventElapsedTime(&s.ms_phase[4], c.ev_phase[3], c.ev_phase[4]));
        s.xchg_allreduce_bytes = c.world > 1 ? c.xar_bytes : 0;
        s.xchg_allgather_bytes = c.world > 1 ? c.xag_bytes : 0;
        s.xchg_reduce_scatter_bytes = c.world > 1 ? c.xrs_bytes : 0;
        if (c.xp)
            for (int i = 0; i < 8; i++) s.ms_xwait[i] = c.xp->wait_ms(i);
        *stats_out = s;
    }
    (void)flags;
    return RS_OK;
}

// ------------------------------------------------------------------ top-k
static rs_status ensure_cand(rs_ctx *ctx, int64_t cap) {
    if (cap <= ctx->cand_cap) return RS_OK;
    CK(dalloc(&ctx->cand_key, 2 * (size_t)cap + (size_t)cap / 2 + 2));   // key, key2, id2 (large-K sort)
    CK(dalloc(&ctx->cand_id, cap));
    ctx->cand_cap = cap;
    return RS_OK;
}
static rs_status ensure_stage(rs_ctx *ctx, int64_t cap) {
    if (cap <= ctx->stage_cap) return RS_OK;
    CK(dalloc(&ctx->stage_i32, cap));
    CK(dalloc(&ctx->stage_f64, cap));
    ctx->stage_cap = cap;
    return RS_OK;
}

extern "C" rs_status rs_topk(rs_ctx *ctx, int64_t K, int32_t *ids_out, double *scores_out, int64_t *count_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_topk: call rs_score first");
    if (K < 1) return fail(ctx, RS_EINVAL, "rs_topk: K must be >= 1");
    if (!ids_out) return fail(ctx, RS_EINVAL, "rs_topk: ids_out is NULL");
    const int64_t Kc = std::min<int64_t>(K, c.n);
    rs_status s = ensure_cand(ctx, Kc * c.world);
    if (s != RS_OK) return s;
    const bool dev_ids = is_device_ptr(ids_out);
    const bool dev_sc = scores_out ? is_device_ptr(scores_out) : true;
    int32_t *ids_d = ids_out;
    double *sc_d = scores_out;
    if (!dev_ids || !dev_sc) {
        s = ensure_stage(ctx, Kc);
        if (s != RS_OK) return s;
        if (!dev_ids) ids_d = ctx->stage_i32;
        if (scores_out && !dev_sc) sc_d = ctx->stage_f64;
    }
    if (c.world == 1) {
        // K <= 4096: the compact path (after two digit passes the keys sharing the
        // threshold's top 22 bits, and those above, usually fit the final sort:
        // the other four passes and the above / ties scans are skipped)
        const bool compact = Kc <= 4096 && !getenv("RS_EXP_TK_FULL");
        if (compact) {
            s = ensure_cand(ctx, 4096);
            if (s != RS_OK) return s;
        }
        CK(rs::launch_topk_select(c, Kc, 0, c.n, ctx->cand_key, ctx->cand_id, nullptr, 0, 0, compact));
        CK(rs::tk_sort_emit(c, ctx->cand_key, ctx->cand_id, Kc, Kc, ids_d, sc_d, compact));
    } else {
        // local top-K of the owned head range, padded with sentinels, all-gathered,
        // then the same deterministic merge on every rank
        const int64_t range = c.head_hi - c.head_lo;
        const int64_t Kl = std::min<int64_t>(Kc, range);
        unsigned long long *lk = ctx->cand_key;           // local sorted keys (Kc)
        int32_t *li = ctx->cand_id;
        s = ensure_stage(ctx, Kc);
        if (s != RS_OK) return s;
        const int64_t cnt = Kc * c.world;                 // gathered candidates
        if (cnt > c.tk_gcap) {
            CK(dalloc(&c.tk_gkey, (size_t)cnt));
            CK(dalloc(&c.tk_gid, (size_t)cnt));
            c.tk_gcap = cnt;
        }
        // pad: keys 0, ids INT32_MAX sort last
        CK(cudaMemsetAsync(lk, 0, sizeof(unsigned long long) * Kc, c.stream));
        CK(cudaMemsetAsync(li, 0x7f, sizeof(int32_t) * Kc, c.stream));
        if (Kl > 0) {
            // scores are in original order; keep the ids whose internal id is owned
            CK(rs::launch_topk_select(c, Kl, 0, c.n, lk, li, c.inv, c.head_lo, c.head_hi));
        }
        XK(c.xp->allgather(lk, c.tk_gkey, sizeof(unsigned long long) * Kc, c.stream));
        XK(c.xp->allgather(li, c.tk_gid, sizeof(int32_t) * Kc, c.stream));
        // world * K candidates: merged on the host by the exported protocol function
        std::vector<uint64_t> hk(cnt);
        std::vector<int32_t> hi(cnt), hid(Kc);
        std::vector<double> hs(Kc);
        CK(cudaMemcpyAsync(hk.data(), c.tk_gkey, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(hi.data(), c.tk_gid, sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        int64_t got = 0;
        rs_merge_candidates(cnt, hk.data(), hi.data(), Kc, hid.data(), hs.data(), &got);
        CK(cudaMemcpyAsync(ids_d, hid.data(), sizeof(int32_t) * Kc, cudaMemcpyHostToDevice, c.stream));
        if (sc_d) CK(cudaMemcpyAsync(sc_d, hs.data(), sizeof(double) * Kc, cudaMemcpyHostToDevice, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    }
    // the accumulators zeroed for the next rs_score on a side stream (forked at the
    // end of rs_score) overlap this call; the library stream waits for them here,
    // so a step timed on it includes that work
    if (c.acc_zero) CK(cudaStreamWaitEvent(c.stream, c.ev_zero, 0));
    if (!dev_ids) CK(cudaMemcpyAsync(ids_out, ids_d, sizeof(int32_t) * Kc, cudaMemcpyDeviceToHost, c.stream));
    if (scores_out && !dev_sc)
        CK(cudaMemcpyAsync(scores_out, sc_d, sizeof(double) * Kc, cudaMemcpyDeviceToHost, c.stream));
    if (!dev_ids || !dev_sc) CK(cudaStreamSynchronize(c.stream));
    if (count_out) *count_out = Kc;
    return RS_OK;
}

// ------------------------------------------------------------------ NEXT-1: robustness evaluation
static uint64_t host_mix64(uint64_t z) {   // SplitMix64 finaliser (same generator as k_awcc.cu)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

extern "C" rs_status rs_awcc_removal(rs_ctx *ctx, const int32_t *S, int64_t nS, int32_t mode, int32_t step_pct,
                                     int32_t max_pct, int32_t trials, uint64_t seed, int32_t *zeta_out,
                                     double *mean_out, int64_t *steps_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.has_comm) return fail(ctx, RS_ESTATE, "rs_awcc_removal: call rs_load_csr and rs_set_communities first");
    if (!S || nS < 1) return fail(ctx, RS_EINVAL, "rs_awcc_removal: S must be a non-empty vertex set");
    if (mode != RS_REMOVE_EDGES && mode != RS_REMOVE_NODES) return fail(ctx, RS_EINVAL, "rs_awcc_removal: bad mode");
    if (step_pct < 1 || max_pct < 0 || max_pct > 100 || trials < 1)
        return fail(ctx, RS_EINVAL, "rs_awcc_removal: need 1 <= step_pct, 0 <= max_pct <= 100, trials >= 1");
    const int J1 = max_pct / step_pct + 1;
    if (J1 > 127) return fail(ctx, RS_EINVAL, "rs_awcc_removal: at most 126 steps");
    std::vector<int32_t> hS(nS);
    CK(cudaMemcpy(hS.data(), S, sizeof(int32_t) * nS, is_device_ptr(S) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    for (int64_t i = 0; i < nS; i++)
        if (hS[i] < 0 || hS[i] >= c.n) return fail(ctx, RS_EINVAL, "rs_awcc_removal: vertex id out of range");
    const int64_t M = mode == RS_REMOVE_EDGES ? c.nnz / 2 : c.n;
    int64_t cap = 2;
    while (cap < 2 * std::max<int64_t>(c.d_max, 1)) cap <<= 1;          // per-vertex community table
    const size_t sbytes = rs::awcc_scratch_bytes(M, J1, cap, nS);
    char *buf = nullptr;
    CK(rs::dmalloc(&buf, sbytes + sizeof(int32_t) * (size_t)nS * (J1 + 1) + sizeof(int64_t) * nS + 1024));
    int32_t *S_dev = (int32_t *)buf;
    int32_t *zeta_dev = S_dev + nS;
    int64_t *deg_dev = (int64_t *)(((uintptr_t)(zeta_dev + (size_t)nS * J1) + 15) & ~(uintptr_t)15);
    void *scratch = (void *)(((uintptr_t)(deg_dev + nS) + 255) & ~(uintptr_t)255);
    rs_status st_ret = RS_OK;
    std::vector<int32_t> hz((size_t)nS * J1);
    std::vector<int64_t> hdeg(nS);
    std::vector<double> mean(J1, 0.0);
    cudaError_t e = cudaMemcpyAsync(S_dev, hS.data(), sizeof(int32_t) * nS, cudaMemcpyHostToDevice, c.stream);
    if (e == cudaSuccess) e = rs::launch_awcc_degrees(c, S_dev, nS, deg_dev);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hdeg.data(), deg_dev, sizeof(int64_t) * nS, cudaMemcpyDeviceToHost, c.stream);
    for (int32_t t = 0; t < trials && e == cudaSuccess; t++) {
        const uint64_t salt = host_mix64(seed + (uint64_t)(2 * (int64_t)t + mode) * 0x9E3779B97F4A7C15ull);
        e = rs::launch_awcc_trial(c, S_dev, nS, mode, step_pct, J1, salt, zeta_dev, scratch, sbytes, cap);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hz.data(), zeta_dev, sizeof(int32_t) * nS * J1, cudaMemcpyDeviceToHost, c.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
        if (e != cudaSuccess) break;
        // the trial's AWCC per step: |zeta|/d in S order, / |S| (the oracle's order)
        for (int j = 0; j < J1; j++) {
            double acc = 0.0;
            for (int64_t s = 0; s < nS; s++) {
                const int32_t z = hz[(size_t)j * nS + s];
                if (zeta_out) zeta_out[((int64_t)t * J1 + j) * nS + s] = z;
                if (hdeg[s] > 0) acc += (double)z / (double)hdeg[s];
            }
            mean[j] += acc / (double)nS;
        }
    }
    cudaFree(buf);
    if (e != cudaSuccess) return fail(ctx, RS_ECUDA, std::string("rs_awcc_removal: ") + cudaGetErrorString(e));
    for (int j = 0; j < J1; j++) mean[j] /= (double)trials;
    if (mean_out) memcpy(mean_out, mean.data(), sizeof(double) * J1);
    if (steps_out) *steps_out = J1;
    return st_ret;
}

// ------------------------------------------------------------------ NEXT-4: SHII
extern "C" rs_status rs_shii(rs_ctx *ctx, const int32_t *S, int64_t nS, int32_t model, double p, int32_t runs,
                             uint64_t seed, int64_t *influenced_out, double *shii_out, double *mean_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.has_comm) return fail(ctx, RS_ESTATE, "rs_shii: call rs_load_csr and rs_set_communities first");
    if (!S || nS < 1) return fail(ctx, RS_EINVAL, "rs_shii: S must be a non-empty vertex set");
    if (model != RS_DIFFUSE_IC && model != RS_DIFFUSE_LT) return fail(ctx, RS_EINVAL, "rs_shii: bad model");
    if (runs < 1 || !(p >= 0.0) || p > 1.0) return fail(ctx, RS_EINVAL, "rs_shii: need runs >= 1 and 0 <= p <= 1");
    std::vector<int32_t> hS(nS);
    CK(cudaMemcpy(hS.data(), S, sizeof(int32_t) * nS, is_device_ptr(S) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    for (int64_t i = 0; i < nS; i++)
        if (hS[i] < 0 || hS[i] >= c.n) return fail(ctx, RS_EINVAL, "rs_shii: vertex id out of range");
    if (model == RS_DIFFUSE_IC) {
        // IC: up to 64 (seed, run) diffusions at once (k_shii.cu, launch_shii_ic_batch),
        // diffusion j = (s, r) in seed-major order; the means summed in run order as below
        const int64_t total = nS * (int64_t)runs;
        std::vector<int64_t> res(2 * total);
        std::vector<int32_t> hu(64), hc(64);
        std::vector<uint64_t> st(64);
        unsigned long long *bb = nullptr;
        const size_t nbb = 3 * (size_t)c.n + (2 * sizeof(int32_t) * (size_t)c.n + 7) / 8 + 2 + 128 + 64;
        CK(rs::dmalloc(&bb, sizeof(unsigned long long) * nbb));
        int32_t *dsc = (int32_t *)(bb + nbb - 64);          // seeds | communities (64 each)
        cudaError_t e = cudaSuccess;
        std::vector<int32_t> hinv(1), hcomm(1);
        for (int64_t j0 = 0; j0 < total && e == cudaSuccess; j0 += 64) {
            const int nb = (int)std::min<int64_t>(64, total - j0);
            for (int j = 0; j < nb && e == cudaSuccess; j++) {
                const int64_t s = (j0 + j) / runs, r = (j0 + j) % runs;
                st[j] = host_mix64(seed + (uint64_t)(2 * r + model + 1) * 0xD1B54A32D192ED03ull);
                if (r == 0 || j == 0) {
                    e = cudaMemcpyAsync(hinv.data(), c.inv + hS[s], sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream);
                    if (e == cudaSuccess)
                        e = cudaMemcpyAsync(hcomm.data(), c.comm_in + hS[s], sizeof(int32_t), cudaMemcpyDeviceToHost,
                                            c.stream);
                    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
                }
                hu[j] = hinv[0];
                hc[j] = hcomm[0];
            }
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(dsc, hu.data(), sizeof(int32_t) * 64, cudaMemcpyHostToDevice, c.stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(dsc + 64, hc.data(), sizeof(int32_t) * 64, cudaMemcpyHostToDevice, c.stream);
            if (e == cudaSuccess)
                e = rs::launch_shii_ic_batch(c, nb, dsc, dsc + 64, st.data(), p, bb, res.data() + 2 * j0);
        }
        cudaFree(bb);
        if (e != cudaSuccess) return fail(ctx, RS_ECUDA, std::string("rs_shii: ") + cudaGetErrorString(e));
        double setmean = 0.0;
        for (int64_t s = 0; s < nS; s++) {
            double acc = 0.0;
            for (int32_t r = 0; r < runs; r++) {
                const int64_t j = s * runs + r;
                if (influenced_out) {
                    influenced_out[j * 2] = res[2 * j];
                    influenced_out[j * 2 + 1] = res[2 * j + 1];
                }
                acc += (double)res[2 * j + 1] / (double)res[2 * j];
            }
            const double sh = acc / (double)runs;
            if (shii_out) shii_out[s] = sh;
            setmean += sh;
        }
        if (mean_out) *mean_out = setmean / (double)nS;
        return RS_OK;
    }
    char *buf = nullptr;
    const size_t nb = sizeof(unsigned int) * c.n + 2 * sizeof(int32_t) * c.n + 64;
    CK(rs::dmalloc(&buf, nb));
    unsigned long long *ctr = (unsigned long long *)buf;
    unsigned int *act = (unsigned int *)(buf + 64);
    int32_t *cnt = (int32_t *)(act + c.n);
    int32_t *list = cnt + c.n;
    cudaError_t e = cudaMemsetAsync(act, 0, sizeof(unsigned int) * c.n, c.stream);
    double setmean = 0.0;
    for (int64_t s = 0; s < nS && e == cudaSuccess; s++) {
        double acc = 0.0;
        for (int32_t r = 0; r < runs && e == cudaSuccess; r++) {
            // run salt (shared by every seed of run r, as in the oracle)
            const uint64_t st = host_mix64(seed + (uint64_t)(2 * (int64_t)r + model + 1) * 0xD1B54A32D192ED03ull);
            int64_t o2[2] = {0, 0};
            e = rs::launch_shii_run(c, hS[s], model, p, st, act, cnt, list, ctr, o2);
            if (influenced_out) {
                influenced_out[(s * runs + r) * 2] = o2[0];
                influenced_out[(s * runs + r) * 2 + 1] = o2[1];
            }
            acc += (double)o2[1] / (double)o2[0];
        }
        const double sh = acc / (double)runs;
        if (shii_out) shii_out[s] = sh;
        setmean += sh;
    }
    cudaFree(buf);
    if (e != cudaSuccess) return fail(ctx, RS_ECUDA, std::string("rs_shii: ") + cudaGetErrorString(e));
    if (mean_out) *mean_out = setmean / (double)nS;
    return RS_OK;
}

// ------------------------------------------------------------------ multi-GPU host protocol
extern "C" rs_status rs_split_ranges(int64_t n, const int64_t *work_incl, int32_t world, int64_t *bounds_out) {
    if (n < 0 || world < 1 || !bounds_out || (n > 0 && !work_incl)) return RS_EINVAL;
    for (int r = 0; r <= world; r++) bounds_out[r] = rs::split_point(work_incl, n, world, r);
    return RS_OK;
}

extern "C" rs_status rs_local_candidates(int64_t count, const double *scores, const int32_t *ids, int64_t K,
                                         uint64_t *keys_out, int32_t *ids_out) {
    if (count < 0 || K < 0 || (count > 0 && (!scores || !ids)) || (K > 0 && (!keys_out || !ids_out))) return RS_EINVAL;
    std::vector<uint64_t> key(count);
    for (int64_t i = 0; i < count; i++) {
        uint64_t b;
        memcpy(&b, &scores[i], sizeof(b));
        key[i] = rs::score_key_bits(b);
    }
    std::vector<int64_t> ord(count);
    for (int64_t i = 0; i < count; i++) ord[i] = i;
    const int64_t take = std::min(K, count);
    std::partial_sort(ord.begin(), ord.begin() + take, ord.end(), [&](int64_t a, int64_t b) {
        return rs::cand_before(key[a], ids[a], key[b], ids[b]);
    });
    for (int64_t i = 0; i < K; i++) {
        keys_out[i] = i < take ? key[ord[i]] : 0ull;
        ids_out[i] = i < take ? ids[ord[i]] : INT32_MAX;
    }
    return RS_OK;
}

extern "C" rs_status rs_merge_candidates(int64_t count, const uint64_t *keys, const int32_t *ids, int64_t K,
                                         int32_t *ids_out, double *scores_out, int64_t *count_out) {
    if (count < 0 || K < 0 || (count > 0 && (!keys || !ids)) || (K > 0 && !ids_out)) return RS_EINVAL;
    std::vector<int64_t> ord(count);
    for (int64_t i = 0; i < count; i++) ord[i] = i;
    const int64_t out = std::min(K, count);
    std::partial_sort(ord.begin(), ord.begin() + out, ord.end(), [&](int64_t a, int64_t b) {
        return rs::cand_before(keys[a], ids[a], keys[b], ids[b]);
    });
    for (int64_t i = 0; i < out; i++) {
        ids_out[i] = ids[ord[i]];
        if (scores_out) {
            double d;
            memcpy(&d, &keys[ord[i]], sizeof(d));
            scores_out[i] = d;
        }
    }
    if (count_out) *count_out = out;
    return RS_OK;
}

// ------------------------------------------------------------------ getters
template <class T>
static rs_status out_copy(rs_ctx *ctx, T *dst, const T *src_dev, size_t count) {
    Ctx &c = ctx->c;
    CK(cudaMemcpyAsync(dst, src_dev, sizeof(T) * count,
                       is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return RS_OK;
}

// the dense parity tables f and omega are not written by rs_score: the first
// getter after it re-runs the Phase A histogram in its parity mode (same
// kernels, same arithmetic, only those two tables written)
static cudaError_t ensure_parity_tables(rs_ctx *ctx) {
    Ctx &c = ctx->c;
    if (c.parity_ok) return cudaSuccess;
    fork(c);
    // every vertex (in the multi-GPU path too: the parity walk reads only the
    // replicated CSR and labels)
    cudaError_t e = rs::launch_phase_a_impl(c, ctx->l2t, ctx->l2n, true, 0, c.n);
    join(c);
    if (e == cudaSuccess) c.parity_ok = true;
    return e;
}

extern "C" rs_status rs_get_counts(rs_ctx *ctx, int32_t *f_out, int32_t *total_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_counts: call rs_score first");
    int32_t *forig = nullptr;
    CK(rs::dmalloc(&forig, sizeof(int32_t) * (size_t)c.n * c.k));
    rs_status s = RS_OK;
    if (c.sparse) {
        // dense view of the sparse community tables
        int32_t *tot = (int32_t *)c.scratch;
        cudaError_t e = cudaMemsetAsync(forig, 0, sizeof(int32_t) * (size_t)c.n * c.k, c.stream);
        if (e == cudaSuccess) e = rs::launch_sparse_counts_dense(c, forig, tot);
        if (e == cudaSuccess && f_out) s = out_copy(ctx, f_out, forig, (size_t)c.n * c.k);
        if (e == cudaSuccess && s == RS_OK && total_out) s = out_copy(ctx, total_out, tot, (size_t)c.n);
        cudaFree(forig);
        CK(e);
        return s;
    }
    cudaError_t e = ensure_parity_tables(ctx);
    if (e == cudaSuccess) e = rs::launch_permute_i32(c, c.f, c.k, forig);
    if (e == cudaSuccess && f_out) s = out_copy(ctx, f_out, forig, (size_t)c.n * c.k);
    if (e == cudaSuccess && s == RS_OK && total_out) {
        int32_t *tmp = (int32_t *)c.scratch;
        e = rs::launch_counts_total(c, forig, tmp);
        if (e == cudaSuccess) s = out_copy(ctx, total_out, tmp, (size_t)c.n);
    }
    cudaFree(forig);
    CK(e);
    return s;
}

extern "C" rs_status rs_get_weights(rs_ctx *ctx, double *omega_out, double *omega_max_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_weights: call rs_score first");
    if (omega_out) {
        double *worig = nullptr;
        CK(rs::dmalloc(&worig, sizeof(double) * (size_t)c.n * c.k));
        cudaError_t e = c.sparse ? rs::launch_sparse_weights_dense(c, ctx->l2t, ctx->l2n, worig)
                                 : ensure_parity_tables(ctx);
        if (e == cudaSuccess && !c.sparse) e = rs::launch_permute_f64(c, c.omega, c.k, worig);
        rs_status s = e == cudaSuccess ? out_copy(ctx, omega_out, worig, (size_t)c.n * c.k) : RS_OK;
        cudaFree(worig);
        CK(e);
        if (s) return s;
    }
    if (omega_max_out) {
        unsigned long long wb = 0;
        CK(cudaMemcpyAsync(&wb, c.scal + rs::kScalOmegaMaxBits, 8, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        memcpy(omega_max_out, &wb, 8);
    }
    return RS_OK;
}

extern "C" rs_status rs_get_border(rs_ctx *ctx, int32_t *bv_out, int64_t *nb_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_border: call rs_score first");
    int64_t nb = 0;
    int32_t *tmp = nullptr;
    CK(rs::dmalloc(&tmp, sizeof(int32_t) * (size_t)c.n));
    cudaError_t e = rs::launch_border_list(c, tmp, &nb);
    if (e != cudaSuccess) { cudaFree(tmp); CK(e); }
    rs_status s = RS_OK;
    if (bv_out && nb) s = out_copy(ctx, bv_out, tmp, (size_t)nb);
    cudaFree(tmp);
    if (nb_out) *nb_out = nb;
    return s;
}

extern "C" rs_status rs_get_pred(rs_ctx *ctx, int64_t *pred_off_out, int32_t *pred_out, int64_t *n_entries_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_pred: call rs_score first");
    if (c.world > 1) return fail(ctx, RS_ESTATE, "rs_get_pred: a rank holds only its own P lists (multi-GPU)");
    int64_t *off = nullptr;
    int32_t *pr = nullptr;
    int64_t ne = 0;
    CK(rs::dmalloc(&off, sizeof(int64_t) * (size_t)(c.n + 1)));
    CK(rs::dmalloc(&pr, sizeof(int32_t) * (size_t)std::max<int64_t>(c.nnz, 1)));
    cudaError_t e = rs::launch_pred_export(c, off, pr, &ne);
    if (e != cudaSuccess) { cudaFree(off); cudaFree(pr); CK(e); }
    rs_status s = RS_OK;
    if (pred_off_out) s = out_copy(ctx, pred_off_out, off, (size_t)(c.n + 1));
    if (s == RS_OK && pred_out && ne) s = out_copy(ctx, pred_out, pr, (size_t)ne);
    cudaFree(off);
    cudaFree(pr);
    if (n_entries_out) *n_entries_out = ne;
    return s;
}

extern "C" rs_status rs_get_triad_counts(rs_ctx *ctx, int64_t *type1_out, int64_t *type2_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_triad_counts: call rs_score first");
    int64_t *tmp = (int64_t *)c.scratch;
    if (type1_out) {
        // Type-I triads are counted by re-running the triangle pass in COUNT mode
        // (kept off the timed rs_score path)
        CK(cudaMemsetAsync(c.n1, 0, sizeof(unsigned long long) * (size_t)c.n, c.stream));
        CK(rs::launch_triangle_counts(c));
        if (c.world > 1) XK(c.xp->allreduce_u64(c.n1, (size_t)c.n, false, c.stream));
        CK(rs::launch_type1_export(c, tmp));
        rs_status s = out_copy(ctx, type1_out, tmp, (size_t)c.n);
        if (s) return s;
    }
    if (type2_out) {
        // dense mode: n_II(u) = sum_{w in P(u)} (f_w[c_u] - 1) reads the count table f,
        // which rs_score does not write (parity tables, filled on demand)
        if (!c.sparse) CK(ensure_parity_tables(ctx));
        CK(c.sparse ? rs::launch_sparse_type2(c, tmp) : rs::launch_type2_counts(c, tmp));
        rs_status s = out_copy(ctx, type2_out, tmp, (size_t)c.n);
        if (s) return s;
    }
    return RS_OK;
}

extern "C" rs_status rs_get_comm_tables(rs_ctx *ctx, int64_t *off_out, int32_t *cols_out, int32_t *cnt_out,
                                        double *omega_out, double *omega_abs_out, int64_t *n_entries_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    if (!c.scored) return fail(ctx, RS_ESTATE, "rs_get_comm_tables: call rs_score first");
    if (!c.sparse) return fail(ctx, RS_ESTATE, "rs_get_comm_tables: needs the RS_ALL_COMMUNITIES mode");
    int64_t *off = nullptr;
    CK(rs::dmalloc(&off, sizeof(int64_t) * (size_t)(c.n + 1)));
    int64_t tot = 0;
    cudaError_t e = rs::launch_sparse_offsets(c, off, &tot);
    int32_t *cols = nullptr, *cnt = nullptr;
    double *om = nullptr, *oa = nullptr;
    const size_t E = (size_t)std::max<int64_t>(tot, 1);
    if (e == cudaSuccess && cols_out) e = rs::dmalloc(&cols, sizeof(int32_t) * E);
    if (e == cudaSuccess && cnt_out) e = rs::dmalloc(&cnt, sizeof(int32_t) * E);
    if (e == cudaSuccess && omega_out) e = rs::dmalloc(&om, sizeof(double) * E);
    if (e == cudaSuccess && omega_abs_out) e = rs::dmalloc(&oa, sizeof(double) * (size_t)c.n);
    if (e == cudaSuccess) e = rs::launch_sparse_export(c, off, ctx->l2t, ctx->l2n, cols, cnt, om, oa);
    rs_status s = RS_OK;
    if (e == cudaSuccess && off_out) s = out_copy(ctx, off_out, off, (size_t)(c.n + 1));
    if (e == cudaSuccess && s == RS_OK && cols_out && tot) s = out_copy(ctx, cols_out, cols, (size_t)tot);
    if (e == cudaSuccess && s == RS_OK && cnt_out && tot) s = out_copy(ctx, cnt_out, cnt, (size_t)tot);
    if (e == cudaSuccess && s == RS_OK && omega_out && tot) s = out_copy(ctx, omega_out, om, (size_t)tot);
    if (e == cudaSuccess && s == RS_OK && omega_abs_out) s = out_copy(ctx, omega_abs_out, oa, (size_t)c.n);
    cudaFree(off); cudaFree(cols); cudaFree(cnt); cudaFree(om); cudaFree(oa);
    CK(e);
    if (n_entries_out) *n_entries_out = tot;
    return s;
}

extern "C" rs_status rs_get_targets(rs_ctx *ctx, int32_t *targets_out, int32_t *k_out) {
    if (!ctx) return RS_EINVAL;
    Ctx &c = ctx->c;
    if (!c.has_comm) return fail(ctx, RS_ESTATE, "rs_get_targets: call rs_set_communities first");
    if (targets_out) memcpy(targets_out, c.sparse ? c.h_targets_all.data() : c.h_targets, sizeof(int32_t) * c.k);
    if (k_out) *k_out = c.k;
    return RS_OK;
}

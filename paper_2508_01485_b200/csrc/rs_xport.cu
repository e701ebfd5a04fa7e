// The exchange layer of the multi-GPU path: the
// handful of collectives rs_score / rs_topk issue between the ranks, behind
// one interface with two transports.
//
// * NcclXport: NCCL over NVLink (ncclAllReduce / ncclAllGather; a variable-size
//   all-gather is a group of ncclBroadcast, one per root's segment).
// * EmuXport: the ranks are host threads of ONE process on ONE GPU, each with
//   its own context (rs_create_emulated); a collective is a host barrier, then
//   device-to-device copies (or a summing kernel) reading the peers' buffers,
//   then a barrier. No kernel ever waits on another: every rank synchronises
//   its stream before the barrier. This runs rank r's whole pipeline -- its
//   Phase A shard, the exchanges, its Phase D / finalize range and its
//   filtered top-K select -- exactly as on a GPU of its own, so the tests can
//   check that the merged world gives the single-GPU bits
//   (tests/test_gpu_multirank.py); only the transport differs.
#include "rs_internal.cuh"
#include <condition_variable>
#include <mutex>
#include <vector>

namespace rs {

#ifdef RS_WITH_NCCL
struct NcclXport : Xport {
    ncclComm_t comm;
    int world;
    explicit NcclXport(ncclComm_t cm, int w) : comm(cm), world(w) {}
    cudaError_t err(ncclResult_t r, const char *what) {
        if (r == ncclSuccess) return cudaSuccess;
        msg = std::string(what) + ": " + nccl_api(nullptr)->GetErrorString(r);
        return cudaErrorUnknown;
    }
    cudaError_t allgatherv(void *buf, const size_t *off, const size_t *len, cudaStream_t s) override {
        const NcclApi &N = *nccl_api(nullptr);
        ncclResult_t r = N.GroupStart();
        for (int p = 0; p < world && r == ncclSuccess; p++)
            if (len[p]) r = N.Broadcast((char *)buf + off[p], (char *)buf + off[p], len[p], ncclUint8, p, comm, s);
        const ncclResult_t r2 = N.GroupEnd();
        return err(r != ncclSuccess ? r : r2, "ncclBroadcast (all-gather of segments)");
    }
    cudaError_t allreduce_u64(unsigned long long *buf, size_t count, bool max, cudaStream_t s) override {
        return err(nccl_api(nullptr)->AllReduce(buf, buf, count, ncclUint64, max ? ncclMax : ncclSum, comm, s),
                   "ncclAllReduce");
    }
    cudaError_t allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
        return err(nccl_api(nullptr)->AllGather(send, recv, bytes, ncclUint8, comm, s), "ncclAllGather");
    }
    cudaError_t reduce_scatterv_u64(unsigned long long *buf, const size_t *off, const size_t *len,
                                    cudaStream_t s) override {
        // unequal segments: one ncclReduce per root, grouped
        const NcclApi &N = *nccl_api(nullptr);
        ncclResult_t r = N.GroupStart();
        for (int p = 0; p < world && r == ncclSuccess; p++)
            if (len[p]) r = N.Reduce(buf + off[p], buf + off[p], len[p], ncclUint64, ncclSum, p, comm, s);
        const ncclResult_t r2 = N.GroupEnd();
        return err(r != ncclSuccess ? r : r2, "ncclReduce (reduce-scatter of segments)");
    }
};
Xport *make_nccl_xport(ncclComm_t comm, int world) { return new NcclXport(comm, world); }
#endif

// ---------------------------------------------------------------- emulated world
struct EmuWorld {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    std::vector<const void *> ptr;   // each rank's buffer of the current collective
    // serial mode (rs_emu_world_serial): inside rs_score the ranks take turns,
    // rank 0 first, between consecutive collectives, so each rank's kernels run
    // alone on the GPU and its phase times are those of a GPU of its own
    bool serial = false;
    int token = 0;                   // the rank whose turn it is
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            generation++;
            token = 0;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
    void turn_begin(int rank) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return token == rank; });
    }
    void turn_end(int rank) {
        std::unique_lock<std::mutex> lk(mu);
        if (token == rank) token = (rank + 1) % world;   // after the last rank: rank 0's next turn
        cv.notify_all();
    }
};

constexpr int kEmuMaxWorld = 16;
struct PtrPack {
    const unsigned long long *p[kEmuMaxWorld];
};

__global__ void k_reduce_u64(PtrPack src, int world, size_t count, bool max, unsigned long long *out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long v = src.p[0][i];
        for (int r = 1; r < world; r++) {
            const unsigned long long x = src.p[r][i];
            v = max ? (x > v ? x : v) : v + x;
        }
        out[i] = v;
    }
}

struct EmuXport : Xport {
    EmuWorld *W;
    int rank;
    unsigned long long *tmp = nullptr;
    size_t tmp_count = 0;
    EmuXport(EmuWorld *w, int r) : W(w), rank(r) {}
    ~EmuXport() override {
        if (tmp) cudaFree(tmp);
        for (Wait &x : waits) {
            cudaEventDestroy(x.e0);
            cudaEventDestroy(x.e1);
        }
    }
    // each collective of an rs_score: events on the rank's stream when it enters
    // (its buffer final) and when it resumes (the copies done, its turn again)
    struct Wait {
        cudaEvent_t e0, e1;
        int tag;
    };
    std::vector<Wait> waits;
    size_t nwait = 0;
    cudaStream_t wait_stream = nullptr;
    bool in_score = false;
    void score_begin() override {
        nwait = 0;
        in_score = W->serial;
        if (in_score) W->turn_begin(rank);
    }
    float wait_ms(int t) override {
        float sum = 0.f;
        for (size_t i = 0; i < nwait; i++) {
            if (waits[i].tag != t) continue;
            float ms = 0.f;
            if (cudaEventSynchronize(waits[i].e1) == cudaSuccess &&
                cudaEventElapsedTime(&ms, waits[i].e0, waits[i].e1) == cudaSuccess)
                sum += ms;
        }
        return sum;
    }
    void score_end(cudaStream_t s) override {
        if (!in_score) return;
        cudaStreamSynchronize(s);
        W->turn_end(rank);
        in_score = false;
    }
    cudaError_t publish(const void *p, cudaStream_t s) {
        const cudaError_t e = cudaStreamSynchronize(s);   // this rank's buffer is final
        if (nwait == 64) nwait = 63;                      // collectives outside rs_score: keep the last
        if (nwait == waits.size()) {
            Wait x{nullptr, nullptr, 0};
            cudaEventCreate(&x.e0);
            cudaEventCreate(&x.e1);
            waits.push_back(x);
        }
        waits[nwait].tag = tag;
        cudaEventRecord(waits[nwait].e0, s);
        wait_stream = s;
        if (in_score) W->turn_end(rank);
        W->ptr[rank] = p;
        W->barrier();
        return e;
    }
    // the end of a collective: in serial mode wait for this rank's turn again
    void resume() {
        if (in_score) W->turn_begin(rank);
        cudaEventRecord(waits[nwait].e1, wait_stream);
        nwait++;
    }
    cudaError_t allgatherv(void *buf, const size_t *off, const size_t *len, cudaStream_t s) override {
        cudaError_t e = publish(buf, s);
        for (int p = 0; p < W->world && e == cudaSuccess; p++)
            if (p != rank && len[p])
                e = cudaMemcpyAsync((char *)buf + off[p], (const char *)W->ptr[p] + off[p], len[p],
                                    cudaMemcpyDeviceToDevice, s);
        const cudaError_t e2 = cudaStreamSynchronize(s);
        W->barrier();                                      // every peer done reading
        resume();
        return e != cudaSuccess ? e : e2;
    }
    cudaError_t allreduce_u64(unsigned long long *buf, size_t count, bool max, cudaStream_t s) override {
        cudaError_t e = cudaSuccess;
        if (count > tmp_count) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            tmp_count = 0;
            e = cudaMalloc(&tmp, sizeof(unsigned long long) * count);
            if (e == cudaSuccess) tmp_count = count;
        }
        const cudaError_t ep = publish(buf, s);
        if (e == cudaSuccess) e = ep;
        if (e == cudaSuccess && count) {
            PtrPack pk;
            for (int r = 0; r < W->world; r++) pk.p[r] = (const unsigned long long *)W->ptr[r];
            const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 148 * 8);
            k_reduce_u64<<<blocks, 256, 0, s>>>(pk, W->world, count, max, tmp);
            e = cudaGetLastError();
        }
        const cudaError_t e2 = cudaStreamSynchronize(s);
        W->barrier();                                      // every peer done reading
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess && count)
            e = cudaMemcpyAsync(buf, tmp, sizeof(unsigned long long) * count, cudaMemcpyDeviceToDevice, s);
        resume();
        return e;
    }
    cudaError_t reduce_scatterv_u64(unsigned long long *buf, const size_t *off, const size_t *len,
                                    cudaStream_t s) override {
        const size_t count = len[rank];
        cudaError_t e = cudaSuccess;
        if (count > tmp_count) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            tmp_count = 0;
            e = cudaMalloc(&tmp, sizeof(unsigned long long) * count);
            if (e == cudaSuccess) tmp_count = count;
        }
        const cudaError_t ep = publish(buf, s);
        if (e == cudaSuccess) e = ep;
        if (e == cudaSuccess && count) {
            PtrPack pk;
            for (int r = 0; r < W->world; r++) pk.p[r] = (const unsigned long long *)W->ptr[r] + off[rank];
            const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 148 * 8);
            k_reduce_u64<<<blocks, 256, 0, s>>>(pk, W->world, count, false, tmp);
            e = cudaGetLastError();
        }
        const cudaError_t e2 = cudaStreamSynchronize(s);
        W->barrier();                                      // every peer done reading
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess && count)
            e = cudaMemcpyAsync(buf + off[rank], tmp, sizeof(unsigned long long) * count, cudaMemcpyDeviceToDevice, s);
        resume();
        return e;
    }
    cudaError_t allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
        cudaError_t e = publish(send, s);
        for (int p = 0; p < W->world && e == cudaSuccess; p++)
            e = cudaMemcpyAsync((char *)recv + (size_t)p * bytes, W->ptr[p], bytes, cudaMemcpyDeviceToDevice, s);
        const cudaError_t e2 = cudaStreamSynchronize(s);
        W->barrier();
        resume();
        return e != cudaSuccess ? e : e2;
    }
};

Xport *make_emu_xport(EmuWorld *w, int rank) { return new EmuXport(w, rank); }

}  // namespace rs

struct rs_emu_world {
    rs::EmuWorld w;
};

namespace rs {
EmuWorld *emu_world_of(rs_emu_world *w) { return w ? &w->w : nullptr; }
int emu_world_size(EmuWorld *w) { return w->world; }
}  // namespace rs

extern "C" rs_status rs_emu_world_create(rs_emu_world **out, int32_t world) {
    if (!out || world < 1 || world > rs::kEmuMaxWorld) return RS_EINVAL;
    rs_emu_world *e = new rs_emu_world();
    e->w.world = world;
    e->w.ptr.assign(world, nullptr);
    *out = e;
    return RS_OK;
}

extern "C" void rs_emu_world_destroy(rs_emu_world *w) { delete w; }

extern "C" rs_status rs_emu_world_serial(rs_emu_world *w, int32_t on) {
    if (!w) return RS_EINVAL;
    std::lock_guard<std::mutex> lk(w->w.mu);
    w->w.serial = on != 0;
    w->w.token = 0;
    return RS_OK;
}

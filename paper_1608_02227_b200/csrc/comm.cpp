// Collectives for the row-sharded path: NCCL, or the in-process local group (see comm.h).
#include "comm.h"

#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <mutex>
#include <vector>

namespace cr {

struct LocalGroup {
    int world;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    struct Slot {
        const void *send = nullptr;
        void *recv = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr;
        double *scratch = nullptr;   // allreduce result staging
        size_t cap = 0;              // doubles
    };
    std::vector<Slot> slot;
    explicit LocalGroup(int w) : world(w), slot(w) {}

    // host rendezvous of all ranks; false after a 120 s timeout (a rank died): the group is broken
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) return false;
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

constexpr size_t kScratch = 64;

LocalGroup *local_group_create(int world) {
    if (world < 1 || world > kLocalMaxWorld) return nullptr;
    return new LocalGroup(world);
}

void local_group_destroy(LocalGroup *g) {
    if (!g) return;
    for (auto &s : g->slot) {
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.done) cudaEventDestroy(s.done);
        if (s.scratch) cudaFree(s.scratch);
    }
    delete g;
}

int local_group_world(const LocalGroup *g) { return g ? g->world : 0; }

namespace {

thread_local char g_err[256];

const char *cuda_err(const char *what, cudaError_t e) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return g_err;
}

#define LG_CK(call)                                          \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_err(#call, e_);   \
    } while (0)

// Phase 1 of a local collective: publish pointers, mark this stream's prior work, meet, and
// make this stream wait for every rank's prior work.
const char *local_enter(LocalGroup *g, int r, const void *send, void *recv, cudaStream_t s) {
    auto &me = g->slot[r];
    if (!me.ready) {
        LG_CK(cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming));
        LG_CK(cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming));
    }
    me.send = send;
    me.recv = recv;
    LG_CK(cudaEventRecord(me.ready, s));
    if (!g->barrier()) return "local group: a rank did not arrive (timeout)";
    for (int p = 0; p < g->world; ++p)
        if (p != r) LG_CK(cudaStreamWaitEvent(s, g->slot[p].ready, 0));
    return nullptr;
}

// Phase 2: mark this rank's reads done, meet, wait for every rank's reads (so no rank
// overwrites a buffer a peer still reads).
const char *local_leave(LocalGroup *g, int r, cudaStream_t s) {
    LG_CK(cudaEventRecord(g->slot[r].done, s));
    if (!g->barrier()) return "local group: a rank did not arrive (timeout)";
    for (int p = 0; p < g->world; ++p)
        if (p != r) LG_CK(cudaStreamWaitEvent(s, g->slot[p].done, 0));
    if (!g->barrier()) return "local group: a rank did not arrive (timeout)";
    return nullptr;
}

const char *nccl_err(const char *what, ncclResult_t r) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, ncclGetErrorString(r));
    return g_err;
}

}  // namespace

const char *comm_allgather(Comm &c, void *recv, size_t count, int esize, cudaStream_t s) {
    char *rb = static_cast<char *>(recv);
    if (!c.local) {
        ncclResult_t r = ncclAllGather(rb + (size_t)c.rank * count * esize, rb, count,
                                       esize == 8 ? ncclFloat64 : ncclFloat32, c.nccl, s);
        return r == ncclSuccess ? nullptr : nccl_err("ncclAllGather", r);
    }
    LocalGroup *g = c.local;
    if (const char *e = local_enter(g, c.rank, nullptr, recv, s)) return e;
    for (int p = 0; p < g->world; ++p) {
        if (p == c.rank) continue;
        const size_t off = (size_t)p * count * esize;
        LG_CK(cudaMemcpyAsync(rb + off, static_cast<const char *>(g->slot[p].recv) + off, count * esize,
                              cudaMemcpyDeviceToDevice, s));
    }
    return local_leave(g, c.rank, s);
}

const char *comm_reduce_scatter_f64(Comm &c, const double *send, double *recv, size_t count, cudaStream_t s) {
    if (!c.local) {
        ncclResult_t r = ncclReduceScatter(send, recv, count, ncclFloat64, ncclSum, c.nccl, s);
        return r == ncclSuccess ? nullptr : nccl_err("ncclReduceScatter", r);
    }
    LocalGroup *g = c.local;
    if (const char *e = local_enter(g, c.rank, send, recv, s)) return e;
    SrcPtrs src{};
    for (int p = 0; p < g->world; ++p) src.p[p] = static_cast<const double *>(g->slot[p].send);
    LG_CK(launch_combine(src, g->world, (int64_t)c.rank * (int64_t)count, (int64_t)count, recv, COLL_SUM, s));
    return local_leave(g, c.rank, s);
}

const char *comm_allreduce_f64(Comm &c, double *buf, size_t count, CollOp op, cudaStream_t s) {
    if (!c.local) {
        ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat64, op == COLL_MAX ? ncclMax : ncclSum, c.nccl, s);
        return r == ncclSuccess ? nullptr : nccl_err("ncclAllReduce", r);
    }
    LocalGroup *g = c.local;
    auto &me = g->slot[c.rank];
    if (me.cap < count) {                                   // grow this rank's staging buffer
        if (me.scratch) LG_CK(cudaFree(me.scratch));
        me.cap = count > kScratch ? count : kScratch;
        LG_CK(cudaMalloc(&me.scratch, me.cap * sizeof(double)));
    }
    if (const char *e = local_enter(g, c.rank, buf, buf, s)) return e;
    SrcPtrs src{};
    for (int p = 0; p < g->world; ++p) src.p[p] = static_cast<const double *>(g->slot[p].send);
    double *scr = g->slot[c.rank].scratch;
    LG_CK(launch_combine(src, g->world, 0, (int64_t)count, scr, op, s));
    if (const char *e = local_leave(g, c.rank, s)) return e;     // every rank has read every buf
    LG_CK(cudaMemcpyAsync(buf, scr, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return nullptr;
}

}  // namespace cr

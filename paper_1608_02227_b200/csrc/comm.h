// Collectives of the row-sharded path: NCCL between processes (one GPU each),
// or an in-process "local group" that lets world > 1 contexts share ONE GPU for testing the
// sharded arithmetic end to end.  The local group never makes kernels wait on one another:
// ranks are host threads, each with its own stream; a collective is a host rendezvous plus
// cross-stream event dependencies and plain copies / a fixed-order sum kernel.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <nccl.h>

namespace cr {

struct LocalGroup;

enum CollOp { COLL_SUM = 0, COLL_MAX = 1 };

struct Comm {
    ncclComm_t nccl = nullptr;
    LocalGroup *local = nullptr;
    int rank = 0, world = 1;
};

LocalGroup *local_group_create(int world);
void local_group_destroy(LocalGroup *g);
int local_group_world(const LocalGroup *g);

// All return nullptr on success, else a static / thread-local error string.
// In-place all-gather: rank r's `count` elements live at recv + r * count * esize.
const char *comm_allgather(Comm &c, void *recv, size_t count, int esize, cudaStream_t s);
// recv[k] = sum_p send_p[rank * count + k]   (send holds world * count doubles)
const char *comm_reduce_scatter_f64(Comm &c, const double *send, double *recv, size_t count, cudaStream_t s);
// buf[k] = op_p buf_p[k], in place
const char *comm_allreduce_f64(Comm &c, double *buf, size_t count, CollOp op, cudaStream_t s);

// fixed-order (p = 0 .. P-1) combine of P device arrays (kernels/comm.cu)
constexpr int kLocalMaxWorld = 16;
struct SrcPtrs {
    const double *p[kLocalMaxWorld];
};
cudaError_t launch_combine(const SrcPtrs &src, int P, int64_t off, int64_t count, double *dst, int op, cudaStream_t s);

}  // namespace cr

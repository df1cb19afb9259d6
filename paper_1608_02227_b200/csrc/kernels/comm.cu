// Fixed-order combine of P same-device arrays for the in-process local group (comm.h).
#include <cuda_runtime.h>
#include <cstdint>
#include "../comm.h"

namespace cr {
namespace {
__global__ void combine_kernel(const SrcPtrs src, int P, int64_t off, int64_t count, double *dst, int op) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        double v = src.p[0][off + k];
        for (int q = 1; q < P; ++q) {
            const double w = src.p[q][off + k];
            v = op == COLL_MAX ? fmax(v, w) : v + w;
        }
        dst[k] = v;
    }
}
}  // namespace

cudaError_t launch_combine(const SrcPtrs &src, int P, int64_t off, int64_t count, double *dst, int op, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const int64_t nb = (count + 255) / 256;
    combine_kernel<<<(unsigned)(nb < 1024 ? nb : 1024), 256, 0, s>>>(src, P, off, count, dst, op);
    return cudaGetLastError();
}
}  // namespace cr

// Max-affine estimator of a fitted (y, xi): f_hat(z) = max_i y_i + xi_i^T (z - x_i)
//                                                              = max_i (y_i - a_i) + xi_i^T z,
// a_i = xi_i^T x_i (the prologue's a).  fp64, CUDA cores: 64 queries x 64 rows per tile, thread
// = 4 queries x 4 rows, running max over the rows of this CTA's row split; a second kernel takes
// the max over splits (order-independent: deterministic).
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"

namespace cr {
namespace {
constexpr int QB = 64, RB = 64;

__global__ void __launch_bounds__(256) predict_kernel(const PredictParams p) {
    extern __shared__ double psm[];
    double *zs = psm;                        // [n][QB]
    double *xs = zs + (size_t)p.n * QB;      // [n][RB]
    double *bs = xs + (size_t)p.n * RB;      // [RB]
    double *red = bs + RB;                   // [16][QB]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t q0 = (int64_t)blockIdx.x * QB;
    for (int e = threadIdx.x; e < p.n * QB; e += blockDim.x) {
        const int d = e / QB, qq = e % QB;
        zs[e] = q0 + qq < p.M ? p.Z[(q0 + qq) * p.n + d] : 0.0;
    }
    double best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const int64_t nrt = (p.Ns + RB - 1) / RB;
    const int64_t rt0 = nrt * blockIdx.y / gridDim.y, rt1 = nrt * (blockIdx.y + 1) / gridDim.y;
    for (int64_t rt = rt0; rt < rt1; ++rt) {
        const int64_t i0 = rt * RB;
        __syncthreads();
        for (int e = threadIdx.x; e < p.n * RB; e += blockDim.x) {
            const int d = e / RB, ii = e % RB;
            xs[e] = i0 + ii < p.Ns ? p.Xi[(i0 + ii) * p.n + d] : 0.0;
        }
        for (int ii = threadIdx.x; ii < RB; ii += blockDim.x)
            bs[ii] = i0 + ii < p.Ns ? p.y[p.row0 + i0 + ii] - p.a[i0 + ii] : -INFINITY;
        __syncthreads();
        double acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = bs[ty * 4 + r];
        for (int d = 0; d < p.n; ++d) {
            double xv[4], zv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) xv[r] = xs[d * RB + ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) zv[c] = zs[d * QB + tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fma(xv[r], zv[c], acc[r][c]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) best[c] = fmax(best[c], acc[r][c]);
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c) red[ty * QB + tx * 4 + c] = best[c];
    __syncthreads();
    if (threadIdx.x < QB && q0 + threadIdx.x < p.M) {
        double m = -INFINITY;
        for (int t = 0; t < 16; ++t) m = fmax(m, red[t * QB + threadIdx.x]);
        p.part[(int64_t)blockIdx.y * p.M + q0 + threadIdx.x] = m;
    }
}

__global__ void predict_max_kernel(const double *part, int splits, int64_t M, double *out) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    double v = -INFINITY;
    for (int s = 0; s < splits; ++s) v = fmax(v, part[s * M + m]);
    out[m] = v;
}
}  // namespace

int predict_splits(int64_t M, int64_t Ns, int nsm) {
    const int64_t qblocks = (M + QB - 1) / QB, rtiles = (Ns + RB - 1) / RB;
    int64_t s = (2 * (int64_t)nsm + qblocks - 1) / qblocks;      // ~2 waves of CTAs
    if (s > rtiles) s = rtiles;
    if (s < 1) s = 1;
    if (s > 1024) s = 1024;
    return (int)s;
}

cudaError_t launch_predict(const PredictParams &p, cudaStream_t s) {
    if (p.M <= 0) return cudaSuccess;
    const size_t smem = sizeof(double) * ((size_t)p.n * (QB + RB) + RB + 16 * QB);
    cudaError_t e = cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((p.M + QB - 1) / QB), (unsigned)p.splits);
    predict_kernel<<<grid, 256, smem, s>>>(p);
    predict_max_kernel<<<(unsigned)((p.M + 255) / 256), 256, 0, s>>>(p.part, p.splits, p.M, p.out);
    return cudaGetLastError();
}
}  // namespace cr

// Probe: CUDA-core FMA throughput, fp64 vs fp32, on this B200 (8 independent chains per thread).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == (T)1.2345) out[0] = s;
}
int main() {
    void *out; cudaMalloc(&out, 8);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = nsm * 8, threads = 256;
    for (int t = 0; t < 2; ++t) {
        float ms;
        if (t == 0) { fma_loop<double><<<blocks, threads>>>((double *)out, 10, 0.999, 0.001); cudaEventRecord(e0);
                      fma_loop<double><<<blocks, threads>>>((double *)out, iters, 0.999, 0.001); }
        else { fma_loop<float><<<blocks, threads>>>((float *)out, 10, 0.999f, 0.001f); cudaEventRecord(e0);
               fma_loop<float><<<blocks, threads>>>((float *)out, iters, 0.999f, 0.001f); }
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 8 * (double)iters * blocks * threads;
        printf("%s FMA: %.2f TFLOP/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", t ? "fp32" : "fp64", fl / ms / 1e9,
               fl / 2 / (ms * 1e-3) / nsm / 1.965e9);
    }
    return 0;
}

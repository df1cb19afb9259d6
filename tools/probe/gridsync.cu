// Probe: cost of cooperative-groups grid.sync() and of a hand-rolled atomic grid barrier on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void cg_sync(int K, int *out) {
    cg::grid_group g = cg::this_grid();
    for (int k = 0; k < K; ++k) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = K;
}
// sense-reversing barrier: one atomic per CTA, thread 0 spins on a generation word
__device__ __forceinline__ void bar_sync(unsigned *count, volatile unsigned *gen, unsigned nb, unsigned &mygen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned g0 = mygen;
        if (atomicAdd(count, 1u) == nb - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned *)gen, 1u);
        } else {
            while (*gen == g0) __nanosleep(20);
        }
        mygen = g0 + 1;
        __threadfence();
    }
    __syncthreads();
}
__global__ void my_sync(int K, unsigned *count, unsigned *gen, int *out) {
    unsigned mygen = *((volatile unsigned *)gen);
    for (int k = 0; k < K; ++k) bar_sync(count, gen, gridDim.x, mygen);
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = K;
}
int main() {
    int *out; unsigned *cnt, *gen;
    cudaMalloc(&out, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int G : {1, 16, 74, 143, 148}) {
        int K = 2000;
        void *args[] = {&K, &out};
        cudaLaunchCooperativeKernel((void *)cg_sync, G, 256, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)cg_sync, G, 256, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        void *args2[] = {&K, &cnt, &gen, &out};
        cudaLaunchCooperativeKernel((void *)my_sync, G, 256, args2, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)my_sync, G, 256, args2, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        printf("G=%3d  cg grid.sync %.3f us   atomic barrier %.3f us   (%s)\n", G, 1e3 * ms / K, 1e3 * ms2 / K,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

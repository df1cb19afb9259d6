// Probe: which smem-descriptor encoding makes tcgen05.mma kind::tf32 read a B operand stored
// MN-major with no swizzle (core matrix = 8 K-rows x 16 B = 4 MN-contiguous elements).
// D[128 x NN] = A[128 x 8] (TMEM) * B^T, B[NN x 8] given as an image [j(K)][d(MN)] in core
// matrices: byte ((d/4)*4 + j/8)*128 + (j%8)*16 + (d%4)*4 (the pass's X_J image with 32 j).
// Small integers: every product and sum is exact.  Prints mismatches per variant.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_1608_02227_b200/csrc/kernels/sm100.cuh"
using namespace cr::sm100;

template <int NN>
__global__ void probe(const float *img, const float *A, float *D, uint32_t lbo, uint32_t sbo, uint32_t layout,
                      int bmaj, int jj) {
    __shared__ __align__(1024) float sB[NN * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < NN * 32; i += blockDim.x) sB[i] = img[i];
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tbase, 256);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tbase;
    // A row r = threadIdx.x: 8 tf32 at TMEM columns 128..135
    {
        uint32_t a[8];
        for (int k = 0; k < 8; ++k) a[k] = __float_as_uint(A[threadIdx.x * 8 + k]);
        tmem_st8(t + ((uint32_t)(warp * 32) << 16) + 128, a);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint64_t d = smem_desc_u32(smem_u32(sB) + (bmaj ? jj * 128 : jj * 2 * lbo), lbo, sbo, layout);
        mma_tf32_ts_warp(t, t + 128, d, idesc_tf32(128, NN, 0, bmaj), 0);
        mma_commit_warp(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < NN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + c0, r);
        tmem_wait_ld();
        for (int e = 0; e < 16; ++e) D[threadIdx.x * NN + c0 + e] = __uint_as_float(r[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(t, 256);
}

template <int NN>
int run(uint32_t lbo, uint32_t sbo, uint32_t layout, int bmaj, int jj, const char *name, int kimg = 0) {
    std::vector<float> X(32 * NN), img(NN * 32), A(128 * 8), D(128 * NN);
    for (int j = 0; j < 32; ++j)
        for (int d = 0; d < NN; ++d) X[j * NN + d] = (float)(((j * 7 + d * 3) % 11) - 5);
    for (int j = 0; j < 32; ++j)
        for (int d = 0; d < NN; ++d) {
            if (kimg) img[((j / 4) * (NN / 8) + d / 8) * 32 + (d % 8) * 4 + (j % 4)] = X[j * NN + d];
            else img[((d / 4) * 4 + j / 8) * 32 + (j % 8) * 4 + (d % 4)] = X[j * NN + d];
        }
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 8; ++k) A[r * 8 + k] = (float)(((r * 5 + k * 13) % 9) - 4);
    float *dI, *dA, *dD;
    cudaMalloc(&dI, img.size() * 4); cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dI, img.data(), img.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    probe<NN><<<1, 128>>>(dI, dA, dD, lbo, sbo, layout, bmaj, jj);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
        for (int d = 0; d < NN; ++d) {
            float s = 0;
            for (int k = 0; k < 8; ++k) s += A[r * 8 + k] * X[(jj * 8 + k) * NN + d];
            if (s != D[r * NN + d]) ++bad;
        }
    printf("%-34s NN=%d jj=%d lbo=%u sbo=%u layout=%u bmaj=%d: %s mismatches=%d / %d\n", name, NN, jj, lbo, sbo,
           layout, bmaj, cudaGetErrorString(e), bad, 128 * NN);
    cudaFree(dI); cudaFree(dA); cudaFree(dD);
    return bad;
}

int main() {
    run<32>(32 * 16, 128, 0, 0, 0, "CONTROL K-major [d][j] image", 1);
    run<32>(32 * 16, 128, 0, 0, 1, "CONTROL K-major [d][j] image", 1);
    run<48>(48 * 16, 128, 0, 0, 2, "CONTROL K-major [d][j] image", 1);
    run<32>(128, 512, 0, 1, 0, "MN none LBO=K-grp SBO=MN-chunk");
    run<32>(512, 128, 0, 1, 0, "MN none LBO=MN-chunk SBO=K-grp");
    run<32>(128, 512, 0, 1, 1, "MN none LBO=K-grp SBO=MN-chunk");
    run<32>(512, 128, 0, 1, 1, "MN none LBO=MN-chunk SBO=K-grp");
    run<48>(128, 512, 0, 1, 2, "MN none LBO=K-grp SBO=MN-chunk");
    run<48>(512, 128, 0, 1, 2, "MN none LBO=MN-chunk SBO=K-grp");
    run<16>(128, 512, 0, 1, 3, "MN none LBO=K-grp SBO=MN-chunk");
    run<16>(512, 128, 0, 1, 3, "MN none LBO=MN-chunk SBO=K-grp");
    return 0;
}

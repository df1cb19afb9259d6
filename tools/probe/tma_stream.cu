// Probe: HBM throughput of the fused pass's data movement alone (no math): per 128 x 32 fp32
// tile, load Theta^{k-1} and Theta^{k-2} tiles and store one tile back, persistent CTAs over
// contiguous tile ranges, S-slot ring.  Two Theta layouts:
//   mode 0: row-major [rows][ldT], 2-D TMA boxes 32 cols x 128 rows (128 B per row)  (current)
//   mode 1: tile-major, each 16 KB tile contiguous, 1-D bulk copies                 (candidate)
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1608_02227_b200/csrc/kernels/sm100.cuh"
using namespace cr::sm100;

constexpr int TB = 16384;
struct Bars { uint64_t full[8], empty[8]; };

__device__ __forceinline__ void bulk_store(void *g, const void *s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2,
                                                        const float *A, float *B, int nCB, int64_t T, int S, int mode,
                                                        const float *Ximg, int xbytes) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    Bars *bar = reinterpret_cast<Bars *>(sm + (size_t)S * 2 * TB + (xbytes ? 2 * 24576 : 0));
    uint8_t *xs = sm + (size_t)S * 2 * TB;
    const int64_t t0 = blockIdx.x * T / gridDim.x, t1 = (blockIdx.x + 1) * T / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&bar->full[s], 1); mbar_init(&bar->empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        int s = 0, ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&bar->empty[s], ph ^ 1);
            uint8_t *st = sm + (size_t)s * 2 * TB;
            mbar_arrive_expect_tx(&bar->full[s], 2 * TB + xbytes);
            const int rb = (int)(t / nCB), cb = (int)(t % nCB);
            if (xbytes)   // emulate the pass's per-column-tile X images (L2-resident, evict-last)
                bulk_load(xs + (s & 1) * 24576, Ximg + (size_t)cb * (xbytes / 4), xbytes, &bar->full[s], policy_evict_last());
            if (mode == 0) {
                tma_load_2d(st, &m1, cb * 32, rb * 128, &bar->full[s], pol);
                tma_load_2d(st + TB, &m2, cb * 32, rb * 128, &bar->full[s], pol);
            } else {
                bulk_load(st, A + t * 4096, TB, &bar->full[s], pol);
                bulk_load(st + TB, B + t * 4096, TB, &bar->full[s], pol);
            }
            if (++s == S) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        int s = 0, ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&bar->full[s], ph);
            uint8_t *st = sm + (size_t)s * 2 * TB;
            const int rb = (int)(t / nCB), cb = (int)(t % nCB);
            if (mode == 0) tma_store_2d(&m2, cb * 32, rb * 128, st + TB, pol);
            else bulk_store(B + t * 4096, st + TB, TB);
            bulk_commit();
            bulk_wait_read<0>();
            mbar_arrive(&bar->empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
        }
        bulk_wait<0>();
    }
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                          const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const int64_t N = argc > 1 ? atoll(argv[1]) : 16384;
    const int64_t ldT = N, rows = N;
    const int nCB = (int)(N / 32);
    const int64_t T = (rows / 128) * nCB;
    const int xbytes = argc > 2 ? atoi(argv[2]) : 0;
    float *A, *B, *Xi;
    cudaMalloc(&Xi, (size_t)(N / 32) * (xbytes > 0 ? xbytes : 4));
    cudaMemset(Xi, 0, (size_t)(N / 32) * (xbytes > 0 ? xbytes : 4));
    cudaMalloc(&A, rows * ldT * 4);
    cudaMalloc(&B, rows * ldT * 4);
    cudaMemset(A, 0, rows * ldT * 4);
    cudaMemset(B, 0, rows * ldT * 4);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = (EncFn)fp;
    CUtensorMap m1, m2;
    const cuuint64_t dims[2] = {(cuuint64_t)ldT, (cuuint64_t)rows};
    const cuuint64_t str[1] = {(cuuint64_t)ldT * 4};
    const cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    printf("X image bytes per tile: %d\n", xbytes);
    for (int mode = 1; mode < 2; ++mode)
        for (int S = 2; S <= 6; ++S) {
            const int smem = S * 2 * TB + 2048 + (xbytes ? 2 * 24576 : 0);
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int g : {nsm, 2 * nsm}) {
                if (g == 2 * nsm && S > 3) continue;
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                for (int w = 0; w < 3; ++w) stream_kernel<<<g, 128, smem>>>(m1, m2, A, B, nCB, T, S, mode, Xi, xbytes);
                float best = 1e9;
                for (int r = 0; r < 10; ++r) {
                    cudaEventRecord(e0);
                    stream_kernel<<<g, 128, smem>>>(m1, m2, A, B, nCB, T, S, mode, Xi, xbytes);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("mode %d (%s) S=%d grid=%d: %.3f ms  %.0f GB/s  err=%s\n", mode, mode ? "tile-major bulk" : "row-major 2D TMA",
                       S, g, best, 12.0 * rows * ldT / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}

// Fused pair pass on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32), sm_100a.
//
// Same mathematics as pass_simt.cu (Steps 2 and 4 of P-APG Fig. 2, plus the
// sums Step 1 of the next iteration needs), organised like a flash-attention forward:
//
//   GEMM1  S'  = Xi'_I X_J^T          M=128 rows i, N=32 cols j, K=n   (A = Xi' in TMEM)
//   epilogue   Theta^k = (Theta^{k-1} + beta (Theta^{k-1} - Theta^{k-2}) + S' - y'_j - b'_i)_+
//   GEMM2  P_I += Theta^k_IJ [X | 1]_J M=128 rows i, N=n+1, K=32 cols j (A = Theta^k in TMEM)
//   column sums of Theta^k on CUDA cores (warp butterfly), per (row block, column tile)
//
// Both GEMMs use 3xTF32 (hi*hi + hi*lo + lo*hi, hi = fp32 with the low 13 mantissa bits
// cleared) so products carry ~fp32 accuracy.  Theta^{k-1}, Theta^{k-2} tiles arrive by TMA
// (128B-swizzled 128x32 boxes), Theta^k leaves by TMA store from the same smem slot; the
// row accumulator lives in TMEM and is flushed to fp64 (global, per CTA run slot) every
// `window` tiles.  Warp roles: 0 = TMA producer, 1 = MMA issuer (+ TMEM owner),
// 2..5 = epilogue (one TMEM lane quarter each).  Persistent: CTA g owns tiles
// [g T / G, (g+1) T / G) of the row-major (row block, column tile) order, like the SIMT pass.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"
#include "sm100.cuh"

namespace cr {
namespace {

using namespace sm100;

constexpr int TBM = kTcBM;      // 128 rows per tile (TMEM lanes)
constexpr int TBN = kTcBN;      // 32 columns per tile
constexpr int NTHR = 192;       // 6 warps
constexpr uint32_t TILE_BYTES = TBM * TBN * 4;     // 16 KB
constexpr uint32_t PANEL_BYTES = TBN * 128;        // 4 KB: 32 rows j x 32 fp32 (128 B)

struct __align__(8) TcBarriers {
    uint64_t full[kTcMaxStages], empty[kTcMaxStages];
    uint64_t d1_full[2], d1_empty[2], at_full[2], at_empty[2];
    uint64_t d2_full, d2_empty, xi_full;
    uint32_t tmem_base;
};

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void __launch_bounds__(NTHR, 1)
pass_tc_kernel(const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmB2, const TcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    const uint32_t stage_bytes = p.stage_bytes;
    TcBarriers *bar = reinterpret_cast<TcBarriers *>(smem + (size_t)S * stage_bytes);
    float *colS = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(bar) + sizeof(TcBarriers) + 8);  // [2][4][32]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = (int64_t)blockIdx.x * p.T / p.G, t1 = (int64_t)(blockIdx.x + 1) * p.T / p.G;
    if (t0 >= t1) return;
    const int nCB = p.nCB;
    const int NK = p.NK, NP2 = p.NP2, NPAN = p.NPAN;
    const uint32_t xpan_bytes = (uint32_t)NPAN * PANEL_BYTES;

    auto stage_ptr = [&](int s) { return smem + (size_t)s * stage_bytes; };
    // stage image: [B1 16K][B2 16K][Xhi NPAN*4K][Xlo NPAN*4K][y' 128B]
    auto run_start = [&](int64_t t) { return t == t0 || (t % nCB) == 0; };
    auto flush_after = [&](int64_t t) {
        if (t + 1 == t1 || ((t + 1) % nCB) == 0) return true;
        const int64_t rs = (t / nCB) * nCB > t0 ? (t / nCB) * nCB : t0;
        return ((t - rs + 1) % p.window) == 0;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&bar->full[s], 1); mbar_init(&bar->empty[s], 2); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar->d1_full[b], 1); mbar_init(&bar->d1_empty[b], 4);
            mbar_init(&bar->at_full[b], 4); mbar_init(&bar->at_empty[b], 1);
        }
        mbar_init(&bar->d2_full, 1);
        mbar_init(&bar->d2_empty, 4);
        mbar_init(&bar->xi_full, 4);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bar->tmem_base, 512);
    if (warp == 0 && lane == 0) { prefetch_tmap(&tmB1); prefetch_tmap(&tmB2); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;
    // TMEM column map
    const uint32_t c_d1 = 0, c_at = 64, c_d2 = 192, c_xi = 192 + (uint32_t)NP2;

    if (warp == 0) {
        // ============================================================ TMA producer
        if (lane == 0) {
            const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
            for (int64_t t = t0; t < t1; ++t) {
                const int64_t u = t - t0;
                const int s = (int)(u % S);
                mbar_wait(&bar->empty[s], (uint32_t)(((u / S) & 1) ^ 1));
                const int64_t rb = t / nCB, cb = t % nCB;
                uint8_t *st = stage_ptr(s);
                mbar_arrive_expect_tx(&bar->full[s], 2 * TILE_BYTES + 2 * xpan_bytes + TBN * 4);
                tma_load_2d(st, &tmB1, (int)(cb * TBN), (int)(rb * TBM), &bar->full[s], pol_stream);
                tma_load_2d(st + TILE_BYTES, &tmB2, (int)(cb * TBN), (int)(rb * TBM), &bar->full[s], pol_stream);
                bulk_load(st + 2 * TILE_BYTES, p.xhi_img + (size_t)cb * xpan_bytes / 4, xpan_bytes, &bar->full[s], pol_keep);
                bulk_load(st + 2 * TILE_BYTES + xpan_bytes, p.xlo_img + (size_t)cb * xpan_bytes / 4, xpan_bytes,
                          &bar->full[s], pol_keep);
                bulk_load(st + 2 * TILE_BYTES + 2 * xpan_bytes, p.yv + cb * TBN, TBN * 4, &bar->full[s], pol_keep);
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer
        if (lane == 0) {
            const uint32_t id1 = idesc_tf32(TBM, TBN, 0, 0);   // A K-major (TMEM), B K-major (X tile, k inner)
            const uint32_t id2 = idesc_tf32(TBM, NP2, 0, 1);   // A K-major (TMEM), B MN-major (X tile, d inner)
            int64_t run = 0, flushes = 0;
            bool window_start = true;
            auto gemm1 = [&](int64_t t) {
                const int64_t u = t - t0;
                const int s = (int)(u % S), b = (int)(u & 1);
                mbar_wait(&bar->full[s], (uint32_t)((u / S) & 1));
                mbar_wait(&bar->d1_empty[b], (uint32_t)(((u >> 1) & 1) ^ 1));
                tc_fence_after();
                const uint8_t *xh = stage_ptr(s) + 2 * TILE_BYTES, *xl = xh + xpan_bytes;
                const uint32_t d = tmem + c_d1 + (uint32_t)b * TBN;
                uint32_t acc = 0;
                for (int pass = 0; pass < 3; ++pass) {
                    const uint8_t *xb = pass == 1 ? xl : xh;
                    const uint32_t a_col = c_xi + (pass == 2 ? (uint32_t)NK : 0u);
                    for (int kk = 0; kk < NK / 8; ++kk) {
                        // K-major SW128 B: panel kk/4, 32-byte step kk%4 inside the 128-B row
                        const uint64_t bd = smem_desc(xb + (kk >> 2) * PANEL_BYTES + (kk & 3) * 32, 16, 1024);
                        mma_tf32_ts(d, tmem + a_col + (uint32_t)kk * 8, bd, id1, acc);
                        acc = 1;
                    }
                }
                mma_commit(&bar->d1_full[b]);
            };
            mbar_wait(&bar->xi_full, 0);
            tc_fence_after();
            gemm1(t0);
            for (int64_t t = t0; t < t1; ++t) {
                const int64_t u = t - t0;
                const bool next_same_run = (t + 1 < t1) && !run_start(t + 1);
                if (next_same_run) gemm1(t + 1);
                const int s = (int)(u % S), a = (int)(u & 1);
                mbar_wait(&bar->at_full[a], (uint32_t)((u >> 1) & 1));
                if (window_start && flushes > 0) mbar_wait(&bar->d2_empty, (uint32_t)((flushes - 1) & 1));
                tc_fence_after();
                const uint8_t *xh = stage_ptr(s) + 2 * TILE_BYTES, *xl = xh + xpan_bytes;
                uint32_t acc = window_start ? 0u : 1u;
                for (int pass = 0; pass < 3; ++pass) {
                    const uint8_t *xb = pass == 1 ? xl : xh;
                    const uint32_t a_col = c_at + (uint32_t)a * 64 + (pass == 2 ? 32u : 0u);
                    for (int jj = 0; jj < TBN / 8; ++jj) {
                        // MN-major SW128 B: rows j = 8 jj .. 8 jj + 7 (one swizzle atom along K),
                        // 32-wide d panels LBO = PANEL_BYTES apart
                        const uint64_t bd = smem_desc(xb + jj * 1024, PANEL_BYTES, 1024);
                        mma_tf32_ts(tmem + c_d2, tmem + a_col + (uint32_t)jj * 8, bd, id2, acc);
                        acc = 1;
                    }
                }
                mma_commit(&bar->at_empty[a]);
                mma_commit(&bar->empty[s]);
                window_start = false;
                if (flush_after(t)) {
                    mma_commit(&bar->d2_full);
                    ++flushes;
                    window_start = true;
                }
                if (t + 1 < t1 && !next_same_run) {
                    ++run;
                    mbar_wait(&bar->xi_full, (uint32_t)(run & 1));
                    tc_fence_after();
                    gemm1(t + 1);
                }
            }
        }
    } else {
        // ============================================================ epilogue (4 warps)
        const int q = warp & 3;                       // TMEM lane quarter
        const int r = q * 32 + lane;                  // row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float beta = (float)((p.ts[0] - 1.0) / p.ts[1]);   // beta_{k-1} = (t_{k-1}-1)/t_k
        const double beta64 = (p.ts[0] - 1.0) / p.ts[1];
        (void)beta64;
        const bool store_thread = (threadIdx.x == 64);
        int slot = p.cta_slot0[blockIdx.x];
        bool first_flush = true;
        int64_t flushes = 0, run = 0;
        float bi = 0.f;
        int64_t prev_s = -1;

        auto load_xi = [&](int64_t rb) {
            // Xi' row r of row block rb into TMEM (hi and lo columns), b'_i into a register
            const int64_t lr = rb * TBM + r;
            const float *src = p.XiR + lr * NK;
            bi = p.bv[lr];
            for (int k0 = 0; k0 < NK; k0 += 8) {
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float x = src[k0 + e];
                    const float h = tf32_hi(x);
                    hi[e] = __float_as_uint(h);
                    lo[e] = __float_as_uint(x - h);
                }
                tmem_st8(tmem + lane_off + c_xi + (uint32_t)k0, hi);
                tmem_st8(tmem + lane_off + c_xi + (uint32_t)(NK + k0), lo);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->xi_full);
        };

        load_xi(t0 / nCB);
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t u = t - t0;
            const int s = (int)(u % S), b = (int)(u & 1);
            const int64_t rb = t / nCB, cb = t % nCB;
            if (t != t0 && run_start(t)) { ++run; load_xi(rb); }

            // ---- S' = Xi' X^T from TMEM
            mbar_wait(&bar->d1_full[b], (uint32_t)((u >> 1) & 1));
            tc_fence_after();
            uint32_t sv[32];
            {
                uint32_t a0[16], a1[16];
                tmem_ld16(tmem + lane_off + c_d1 + (uint32_t)b * TBN, a0);
                tmem_ld16(tmem + lane_off + c_d1 + (uint32_t)b * TBN + 16, a1);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) { sv[e] = a0[e]; sv[16 + e] = a1[e]; }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->d1_empty[b]);

            // ---- Theta tiles landed?
            mbar_wait(&bar->full[s], (uint32_t)((u / S) & 1));
            uint8_t *st = stage_ptr(s);
            const float *yt = reinterpret_cast<const float *>(st + 2 * TILE_BYTES + 2 * xpan_bytes);
            uint8_t *rowB1 = st + r * 128, *rowB2 = st + TILE_BYTES + r * 128;
            const int64_t lr = rb * TBM + r, gr = p.row0 + lr;
            float th[32];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int off = ((k ^ (r & 7)) << 4);
                const float4 v1 = *reinterpret_cast<const float4 *>(rowB1 + off);
                const float4 v2 = *reinterpret_cast<const float4 *>(rowB2 + off);
                const float4 yv4 = *reinterpret_cast<const float4 *>(yt + 4 * k);
                const float b1[4] = {v1.x, v1.y, v1.z, v1.w}, b2[4] = {v2.x, v2.y, v2.z, v2.w};
                const float yj[4] = {yv4.x, yv4.y, yv4.z, yv4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = 4 * k + e;
                    const int64_t j = cb * TBN + c;
                    const float acc = __uint_as_float(sv[c]) - (yj[e] + bi);   // -(C eta)_ij / L
                    // theta~ + acc with one rounding of (b1 + acc) recovered exactly (TwoSum)
                    const float dd = b1[e] - b2[e];
                    const float sm = b1[e] + acc;
                    const float bb = sm - b1[e];
                    const float er = (b1[e] - (sm - bb)) + (acc - bb);
                    const float v = fmaf(beta, dd, sm) + er;
                    const bool ok = (lr < p.Ns) && (j < p.N) && (j != gr);
                    th[c] = (ok && v > 0.f) ? v : 0.f;              // ( . )_+ (Step 2), mask
                }
            }
            // ---- Theta^k (hi = raw, lo = remainder) into TMEM as GEMM2's A operand
            mbar_wait(&bar->at_empty[b], (uint32_t)(((u >> 1) & 1) ^ 1));
            tc_fence_after();
            {
                uint32_t h[16], l[16];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const float x = th[16 * half + e];
                        h[e] = __float_as_uint(x);
                        l[e] = __float_as_uint(x - tf32_hi(x));
                    }
                    tmem_st16(tmem + lane_off + c_at + (uint32_t)b * 64 + 16 * half, h);
                    tmem_st16(tmem + lane_off + c_at + (uint32_t)b * 64 + 32 + 16 * half, l);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->at_full[b]);

            // ---- Theta^k into the B2 slot (in place) for the TMA store
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int off = ((k ^ (r & 7)) << 4);
                *reinterpret_cast<float4 *>(rowB2 + off) = make_float4(th[4 * k], th[4 * k + 1], th[4 * k + 2], th[4 * k + 3]);
            }
            // ---- column sums over this warp's 32 rows (butterfly transpose-reduce)
            {
                float v16[16];
                const bool up16 = lane & 16;
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float send = up16 ? th[c] : th[c + 16];
                    const float keep = up16 ? th[c + 16] : th[c];
                    v16[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
                float v8[8];
                const bool up8 = lane & 8;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float send = up8 ? v16[c] : v16[c + 8];
                    const float keep = up8 ? v16[c + 8] : v16[c];
                    v8[c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                }
                float v4[4];
                const bool up4 = lane & 4;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float send = up4 ? v8[c] : v8[c + 4];
                    const float keep = up4 ? v8[c + 4] : v8[c];
                    v4[c] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
                float v2[2];
                const bool up2 = lane & 2;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const float send = up2 ? v4[c] : v4[c + 2];
                    const float keep = up2 ? v4[c + 2] : v4[c];
                    v2[c] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                }
                const bool up1 = lane & 1;
                const float send = up1 ? v2[0] : v2[1];
                const float keep = up1 ? v2[1] : v2[0];
                const float csum = keep + __shfl_xor_sync(0xffffffffu, send, 1);   // column = lane
                colS[((u & 1) * 4 + q) * 32 + lane] = csum;
            }
            fence_proxy_async_smem();
            named_barrier(1, 128);
            if (store_thread) {
                tma_store_2d(&tmB2, (int)(cb * TBN), (int)(rb * TBM), st + TILE_BYTES, policy_evict_first());
                bulk_commit();
                bulk_wait_read<1>();                      // store of the previous tile has read its slot
                if (prev_s >= 0) mbar_arrive(&bar->empty[prev_s]);
                prev_s = s;
            }
            if (q == 0) {
                const float *cs = colS + (u & 1) * 4 * 32;
                const float c4 = (cs[lane] + cs[32 + lane]) + (cs[64 + lane] + cs[96 + lane]);
                p.colpart[rb * p.ldT + cb * TBN + lane] = c4;
            }
            // ---- row accumulator flush (fp64, per CTA run slot)
            if (flush_after(t)) {
                mbar_wait(&bar->d2_full, (uint32_t)(flushes & 1));
                tc_fence_after();
                double *dst = p.rowpart + ((int64_t)slot * TBM + r) * NP2;
                for (int d0 = 0; d0 < NP2; d0 += 16) {
                    uint32_t a[16];
                    tmem_ld16(tmem + lane_off + c_d2 + (uint32_t)d0, a);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const double v = (double)__uint_as_float(a[e]);
                        if (first_flush) dst[d0 + e] = v;
                        else atomicAdd(dst + d0 + e, v);          // exclusive owner: ordered, deterministic
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar->d2_empty);
                ++flushes;
                first_flush = false;
                if (t + 1 == t1 || ((t + 1) % nCB) == 0) { ++slot; first_flush = true; }
            }
        }
        if (store_thread) bulk_wait<0>();
        (void)run;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_pass_tc(const CUtensorMap &tmB1, const CUtensorMap &tmB2, const TcParams &p, cudaStream_t s) {
    pass_tc_kernel<<<p.G, NTHR, p.smem_bytes, s>>>(tmB1, tmB2, p);
    return cudaGetLastError();
}

cudaError_t pass_tc_prepare(int smem_bytes) {
    return cudaFuncSetAttribute(pass_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

size_t tc_barrier_bytes() { return sizeof(TcBarriers) + 8 + 2 * 4 * 32 * 4; }

// X-hat images for the TC pass: per 32-column tile, NPAN panels of [32 rows j][32 d] fp32,
// 128-B rows with the SW128 chunk swizzle (chunk' = chunk ^ (j & 7)); hi = tf32 truncation,
// lo = remainder; column d = n holds 1 (row sums), d > n and j >= N hold 0.
__global__ void tc_xhat_kernel(const double *X64, int64_t N, int n, int NPAN, int nCB, float *hi, float *lo) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;     // one element (j, d)
    const int64_t total = (int64_t)nCB * TBN * NPAN * 32;
    if (e >= total) return;
    const int d = (int)(e % (NPAN * 32));
    const int64_t j = e / (NPAN * 32);
    const int64_t cb = j / TBN;
    const int jj = (int)(j % TBN);
    float x = 0.f;
    if (j < N) x = d < n ? (float)X64[j * n + d] : (d == n ? 1.f : 0.f);
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    const int pan = d / 32, dd = d % 32;
    const int64_t byte = cb * (int64_t)NPAN * PANEL_BYTES + pan * PANEL_BYTES + jj * 128 +
                         (((dd >> 2) ^ (jj & 7)) << 4) + (dd & 3) * 4;
    hi[byte / 4] = h;
    lo[byte / 4] = x - h;
}

cudaError_t launch_tc_xhat(const double *X64, int64_t N, int n, int NPAN, int nCB, float *hi, float *lo,
                           cudaStream_t s) {
    const int64_t total = (int64_t)nCB * TBN * NPAN * 32;
    tc_xhat_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(X64, N, n, NPAN, nCB, hi, lo);
    return cudaGetLastError();
}

}  // namespace cr

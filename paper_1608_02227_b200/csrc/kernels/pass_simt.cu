// Fused pair pass on CUDA cores (SIMT), sm_100a.
//
// One launch = Steps 2 and 4 of P-APG Fig. 2 for every pair (i, j) of
// this shard, plus the sums that Step 1 of the NEXT iteration needs:
//
//   theta~_ij = B1_ij + beta (B1_ij - B2_ij)                  (Step 4 of the previous iteration)
//   Theta^k_ij = ( theta~_ij - (C eta)_ij / L )_+             (Step 2), diagonal masked
//   (C eta)_ij / L = y'_j + b'_i - xi'_i . x_j,   y' = y/L, b' = (a - y)/L, xi' = xi/L
//   r_i += Theta^k_ij,  c_j += Theta^k_ij,  (Theta X)_i += Theta^k_ij x_j
//
// B1 holds Theta^{k-1}, B2 holds Theta^{k-2}; Theta^k is written over B2 (12 B/pair fp32).
// Structure per 64x64 tile (256 threads):
//   S-phase  : thread owns 4 rows x 4 cols; depth-NB register-blocked outer product from
//              smem (xi'^T tile, X^T tile); epilogue forms Theta^k, stores it (16-B
//              streaming stores), transposes it into smem, and column-reduces it.
//   P-phase  : Theta^k tile (smem) x [X | 1] tile (smem) -> per-thread 4x4 blocks of the
//              row accumulators (Theta X, r), K split across thread groups.
// Work: tiles are linearised row-major over (row block, column tile); CTA g owns the
// contiguous range [g T / G, (g+1) T / G) (stream-K style, every CTA moves the same bytes).
// Row accumulators are flushed to fp64 every kFlush tiles and written per (CTA, row-block
// run) slot; column partials per (row block, column tile).  A separate reduce kernel sums
// both in a fixed order (deterministic).
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"

namespace cr {
namespace {

constexpr int BM = kBM, BN = kBN, NT = kThreads;
constexpr int kFlush = 8;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 4 consecutive elements, streaming (evict-first) global access
__device__ __forceinline__ void ld4cs(const float *p, float (&o)[4]) {
    float4 t = __ldcs(reinterpret_cast<const float4 *>(p));
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
}
__device__ __forceinline__ void ld4cs(const double *p, double (&o)[4]) {
    double2 a = __ldcs(reinterpret_cast<const double2 *>(p));
    double2 b = __ldcs(reinterpret_cast<const double2 *>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
__device__ __forceinline__ void st4cs(float *p, const float (&v)[4]) {
    __stcs(reinterpret_cast<float4 *>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void st4cs(double *p, const double (&v)[4]) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(v[0], v[1]));
    __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(v[2], v[3]));
}
// 4 consecutive elements from shared memory
__device__ __forceinline__ void lds4(const float *p, float (&o)[4]) {
    float4 t = *reinterpret_cast<const float4 *>(p);
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
}
__device__ __forceinline__ void lds4(const double *p, double (&o)[4]) {
    double2 a = reinterpret_cast<const double2 *>(p)[0];
    double2 b = reinterpret_cast<const double2 *>(p)[1];
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
__device__ __forceinline__ void sts4(float *p, float a, float b, float c, float d) {
    *reinterpret_cast<float4 *>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void sts4(double *p, double a, double b, double c, double d) {
    reinterpret_cast<double2 *>(p)[0] = make_double2(a, b);
    reinterpret_cast<double2 *>(p)[1] = make_double2(c, d);
}
__device__ __forceinline__ float fmax0(float v) { return fmaxf(v, 0.0f); }
__device__ __forceinline__ double fmax0(double v) { return fmax(v, 0.0); }

template <typename T, int NB, int NBP>
struct Smem {
    static constexpr int NOB = 4 * NBP;                      // 4x4 output blocks of the P-GEMM
    static constexpr int PB = (NOB + NT - 1) / NT;           // blocks per thread
    static constexpr int KS0 = NOB >= NT ? 1 : NT / NOB;
    static constexpr int KS = KS0 >= 8 ? 8 : KS0 >= 4 ? 4 : KS0 >= 2 ? 2 : 1;
    // byte offsets
    static constexpr size_t o_xi = 0;                                  // [NB][BM]
    static constexpr size_t o_b = o_xi + sizeof(T) * NB * BM;          // [BM]
    static constexpr size_t o_x = o_b + sizeof(T) * BM;                // [2][NB][BN]
    static constexpr size_t o_xh = o_x + sizeof(T) * 2 * NB * BN;      // [2][BN][NBP]
    static constexpr size_t o_y = o_xh + sizeof(T) * 2 * BN * NBP;     // [2][BN]
    static constexpr size_t o_th = o_y + sizeof(T) * 2 * BN;           // [BN][BM] swizzled
    static constexpr size_t o_col = o_th + sizeof(T) * BN * BM;        // [8][BN]
    static constexpr size_t o_pd = (o_col + sizeof(T) * 8 * BN + 15) / 16 * 16;  // [KS*NOB or NOB][16] fp64
    static constexpr size_t bytes = o_pd + sizeof(double) * 16 * (PB > 1 ? PB * NT : NT);
};

// fp64: one CTA per SM so the register-blocked 4x4 fp64 tiles and row accumulators fit in
// registers (capped at 128 for 2 CTAs, ptxas spilled ~1 KB per thread)
template <typename T, int NB>
constexpr int simt_min_blocks() { return sizeof(T) == 8 ? 1 : 2; }

template <typename T, int NB, int NBP, int MODE>
__global__ void __launch_bounds__(NT, simt_min_blocks<T, NB>()) pass_simt_kernel(const PassParams p) {
    using S = Smem<T, NB, NBP>;
    constexpr int NOB = S::NOB, PB = S::PB, KS = S::KS;
    extern __shared__ __align__(16) unsigned char smem[];
    T *xiS = reinterpret_cast<T *>(smem + S::o_xi);
    T *bS = reinterpret_cast<T *>(smem + S::o_b);
    T *xS = reinterpret_cast<T *>(smem + S::o_x);
    T *xhS = reinterpret_cast<T *>(smem + S::o_xh);
    T *yS = reinterpret_cast<T *>(smem + S::o_y);
    T *thS = reinterpret_cast<T *>(smem + S::o_th);
    T *colS = reinterpret_cast<T *>(smem + S::o_col);
    double *Pd = reinterpret_cast<double *>(smem + S::o_pd);

    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31, warp = tid >> 5;
    pdl_wait();
    pdl_trigger();
    const int64_t t0 = (int64_t)blockIdx.x * p.T / p.G;
    const int64_t t1 = (int64_t)(blockIdx.x + 1) * p.T / p.G;
    if (t0 >= t1) return;

    const T *B1 = static_cast<const T *>(p.B1);
    const T *B2 = static_cast<const T *>(p.B2);
    T *Bout = static_cast<T *>(p.Bout);
    const T *XT = static_cast<const T *>(p.XT);
    const T *Xh = static_cast<const T *>(p.Xh);
    const T *XiT = static_cast<const T *>(p.XiT);
    const T *bv = static_cast<const T *>(p.bv);
    const T *yv = static_cast<const T *>(p.yv);
    T *colpart = static_cast<T *>(p.colpart);
    const int64_t ldT = p.ldT;

    double beta64 = 0.0;
    if (MODE == MODE_STEP) beta64 = (p.ts[0] - 1.0) / p.ts[1];   // beta_{k-1} = (t_{k-1}-1)/t_k

    // X-tile loader (cp.async): X^T tile [NB][BN], [X|1] tile [BN][NBP], y' tile [BN]
    auto load_xtile = [&](int64_t cb, int buf) {
        constexpr int EPC = 16 / sizeof(T);            // elements per 16-byte chunk
        constexpr int CX = NB * BN / EPC, CH = BN * NBP / EPC, CY = BN / EPC;
        T *xd = xS + buf * NB * BN, *hd = xhS + buf * BN * NBP, *yd = yS + buf * BN;
        for (int c = tid; c < CX + CH + CY; c += NT) {
            if (c < CX) {
                int k = c / (BN / EPC), q = c % (BN / EPC);
                cp_async16(xd + k * BN + q * EPC, XT + (int64_t)k * ldT + cb * BN + q * EPC);
            } else if (c < CX + CH) {
                int q = c - CX;
                cp_async16(hd + q * EPC, Xh + cb * BN * NBP + (int64_t)q * EPC);
            } else {
                int q = c - CX - CH;
                cp_async16(yd + q * EPC, yv + cb * BN + q * EPC);
            }
        }
        cp_async_commit();
    };
    // Theta tile loads for this thread's 4x4 block
    auto load_theta = [&](int64_t t, T (&b1)[4][4], T (&b2)[4][4]) {
        int64_t rb = t / p.nCB, cb = t % p.nCB;
        // tile-major buffers hold nCBt * 32 columns (<= the 64-column grid): beyond is zero
        const bool in = !p.tiled || cb * BN + tx * 4 < (int64_t)p.nCBt * 32;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (in) {
                const int64_t o = theta_off(rb * BM + ty * 4 + r, cb * BN + tx * 4, ldT, p.tiled, p.nCBt);
                ld4cs(B1 + o, b1[r]);
                if (MODE == MODE_STEP) ld4cs(B2 + o, b2[r]);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) { b1[r][c] = T(0); b2[r][c] = T(0); }
            }
        }
    };

    float pacc_f[PB][16];      // fp32 (or fp64 when T = double) row accumulators
    T pacc[PB][16];
    (void)pacc_f;
    int slot = p.cta_slot0[blockIdx.x];
    double dacc[4] = {0.0, 0.0, 0.0, 0.0};     // adaptive step: sum_j (Theta^k - theta~)^2 of the 4 rows
    int64_t cur_rb = -1;
    int since_flush = 0;

    auto flush_to_pd = [&]() {
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            int idx = (PB > 1) ? (q * NT + tid) : tid;
            if (idx < (PB > 1 ? NOB : NOB * KS)) {
#pragma unroll
                for (int e = 0; e < 16; ++e) Pd[idx * 16 + e] += (double)pacc[q][e];
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) pacc[q][e] = T(0);
        }
    };
    auto zero_pd = [&]() {
        const int tot = 16 * (PB > 1 ? PB * NT : NT);
        for (int e = tid; e < tot; e += NT) Pd[e] = 0.0;
    };
    // write the run's row partials (sum over K-split groups) to slot
    auto write_run = [&](int64_t rb) {
        flush_to_pd();
        __syncthreads();
        double *dst = p.rowpart + (int64_t)slot * BM * NBP;
        for (int o = tid; o < BM * NBP; o += NT) {
            int i = o / NBP, d = o % NBP;
            int ob = (d >> 2) * 16 + (i >> 2), e = (i & 3) * 4 + (d & 3);
            double s = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) s += Pd[(ks * NOB + ob) * 16 + e];
            dst[o] = s;
        }
        if (MODE == MODE_STEP && p.adapt) {
            __syncthreads();                     // column dcol of the slot rows written above
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double v = dacc[r];
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);   // over tx
                if (tx == 0) dst[(ty * 4 + r) * NBP + p.dcol] = v;
                dacc[r] = 0.0;
            }
        }
        ++slot;
        (void)rb;
    };

    T cb1[4][4], cb2[4][4];
    load_theta(t0, cb1, cb2);
    load_xtile(t0 % p.nCB, 0);

    for (int64_t t = t0; t < t1; ++t) {
        const int64_t rb = t / p.nCB, cb = t % p.nCB;
        const int buf = (int)((t - t0) & 1);
        __syncthreads();                                   // previous tile fully consumed
        if (rb != cur_rb) {
            if (cur_rb >= 0) { write_run(cur_rb); __syncthreads(); }
            // this row block's xi' (k-major) and b'
            for (int e = tid; e < NB * BM; e += NT) {
                int k = e / BM, i = e % BM;
                xiS[k * BM + i] = XiT[(int64_t)k * p.Rp + rb * BM + i];
            }
            for (int i = tid; i < BM; i += NT) bS[i] = bv[rb * BM + i];
            zero_pd();
#pragma unroll
            for (int q = 0; q < PB; ++q)
#pragma unroll
                for (int e = 0; e < 16; ++e) pacc[q][e] = T(0);
            cur_rb = rb;
            since_flush = 0;
        }
        // prefetch next tile (X data into the other buffer, Theta into registers)
        T nb1[4][4], nb2[4][4];
        if (t + 1 < t1) {
            load_xtile((t + 1) % p.nCB, buf ^ 1);
            load_theta(t + 1, nb1, nb2);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();                                   // X tile (buf) and xi' visible

        const T *xs = xS + buf * NB * BN;
        const T *xh = xhS + buf * BN * NBP;
        const T *ys = yS + buf * BN;

        // ---------------- S-phase: Theta^k for the thread's 4x4 block -----------------
        T th[4][4];
        const int64_t lr0 = rb * BM + ty * 4;               // local row of r = 0
        const int64_t gj0 = cb * BN + tx * 4;               // global column of c = 0
        if (MODE == MODE_STEP) {
            T yj[4], bi[4];
            lds4(ys + tx * 4, yj);
            lds4(bS + ty * 4, bi);
            T acc[4][4];                                     // -> -(C eta)_ij / L
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = -(yj[c] + bi[r]);
#pragma unroll 4
            for (int k = 0; k < NB; ++k) {
                T xv[4], xj[4];
                lds4(xiS + k * BM + ty * 4, xv);
                lds4(xs + k * BN + tx * 4, xj);
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = fma(xv[r], xj[c], acc[r][c]);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t lr = lr0 + r, gr = p.row0 + lr;
                const int64_t bs = p.nbar > 1 ? gr - gr % p.nbar : gr;   // first row of gr's block
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int64_t gj = gj0 + c;
                    // dualized pairs only: cross-block (Assumption 1; K = N: j != i)
                    const bool ok = (lr < p.Ns) && (gj < p.N) && (gj < bs || gj >= bs + p.nbar);
                    // theta~ (Step 4 of the previous iteration) - (C eta)/L, combined in fp64 so
                    // the stored value carries one rounding
                    const double b1 = (double)cb1[r][c];
                    const double v = fma(beta64, b1 - (double)cb2[r][c], b1) + (double)acc[r][c];
                    th[r][c] = ok ? T(fmax(v, 0.0)) : T(0);           // ( . )_+  (Step 2)
                    if (p.adapt) {                                     // D = Theta^k - theta~
                        const double d = ((double)th[r][c] - b1) - beta64 * (b1 - (double)cb2[r][c]);
                        dacc[r] = fma(d, d, dacc[r]);
                    }
                }
                if (!p.tiled || gj0 < (int64_t)p.nCBt * 32) st4cs(Bout + theta_off(lr, gj0, ldT, p.tiled, p.nCBt), th[r]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) th[r][c] = cb1[r][c];
        }
        // transpose into smem (swizzled 16-B slots) and column-reduce
        {
            const int sw = tx & 7;                           // == ((j >> 2) & 7) for j = 4 tx + c
            T cs[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sts4(thS + (tx * 4 + c) * BM + ((ty ^ sw) * 4), th[0][c], th[1][c], th[2][c], th[3][c]);
                cs[c] = (th[0][c] + th[1][c]) + (th[2][c] + th[3][c]);
                cs[c] += __shfl_xor_sync(0xffffffffu, cs[c], 16);
            }
            if (lane < 16) sts4(colS + warp * BN + tx * 4, cs[0], cs[1], cs[2], cs[3]);
        }
        __syncthreads();

        // ---------------- P-phase: row accumulators += Theta^k tile x [X | 1] -------------
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int ob = (PB > 1) ? (q * NT + tid) : (tid % NOB);
            const int ks = (PB > 1) ? 0 : (tid / NOB);
            if ((PB > 1 && ob < NOB) || (PB == 1 && ks < KS)) {
                const int pi = ob & 15, pd = ob >> 4;
                const int j0 = ks * (BN / KS);
#pragma unroll 4
                for (int jj = 0; jj < BN / KS; ++jj) {
                    const int j = j0 + jj;
                    T tv[4], xv[4];
                    lds4(thS + j * BM + ((pi ^ ((j >> 2) & 7)) * 4), tv);
                    lds4(xh + j * NBP + pd * 4, xv);
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                        for (int dd = 0; dd < 4; ++dd) pacc[q][rr * 4 + dd] = fma(tv[rr], xv[dd], pacc[q][rr * 4 + dd]);
                }
            }
        }
        if (tid < BN) {
            T s = T(0);
#pragma unroll
            for (int w = 0; w < 8; ++w) s += colS[w * BN + tid];
            colpart[rb * ldT + cb * BN + tid] = s;
        }
        if (++since_flush == kFlush) { flush_to_pd(); since_flush = 0; }

        if (t + 1 < t1) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) { cb1[r][c] = nb1[r][c]; cb2[r][c] = nb2[r][c]; }
        }
    }
    __syncthreads();
    write_run(cur_rb);
}

template <typename T, int NB, int MODE>
cudaError_t launch_one(const PassParams &p, cudaStream_t s) {
    constexpr int NBP = NB + 4;
    using S = Smem<T, NB, NBP>;
    // dynamic-smem attribute is set once by pass_simt_config (not per launch: graph capture)
    cudaError_t e = pdl_launch(pass_simt_kernel<T, NB, NBP, MODE>, dim3(p.G), dim3(NT), S::bytes, s, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int NB>
cudaError_t config_one(int *smem, int *bps) {
    constexpr int NBP = NB + 4;
    using S = Smem<T, NB, NBP>;
    auto kern = pass_simt_kernel<T, NB, NBP, MODE_STEP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(pass_simt_kernel<T, NB, NBP, MODE_SUMS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
    if (e != cudaSuccess) return e;
    *smem = (int)S::bytes;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, kern, NT, S::bytes);
}

#define CR_NB_LIST(X) X(4) X(8) X(12) X(16) X(20) X(24) X(32) X(40) X(48) X(64) X(80)

}  // namespace

int simt_bucket(int n) {
    static const int b[] = {4, 8, 12, 16, 20, 24, 32, 40, 48, 64, 80};
    for (int v : b)
        if (n <= v) return v;
    return 0;
}

cudaError_t launch_pass_simt(const PassParams &p, int fp64, int NB, int mode, cudaStream_t s) {
#define CR_CASE(V)                                                                              \
    case V:                                                                                     \
        if (fp64) return V > 24 ? cudaErrorInvalidValue                                         \
                                : (mode == MODE_STEP ? launch_one<double, (V > 24 ? 4 : V), MODE_STEP>(p, s) \
                                                     : launch_one<double, (V > 24 ? 4 : V), MODE_SUMS>(p, s)); \
        return mode == MODE_STEP ? launch_one<float, V, MODE_STEP>(p, s)                        \
                                 : launch_one<float, V, MODE_SUMS>(p, s);
    switch (NB) {
        CR_NB_LIST(CR_CASE)
        default: return cudaErrorInvalidValue;
    }
#undef CR_CASE
}

cudaError_t pass_simt_config(int fp64, int NB, int *smem, int *bps) {
#define CR_CASE(V) \
    case V: return fp64 ? (V > 24 ? cudaErrorInvalidValue : config_one<double, (V > 24 ? 4 : V)>(smem, bps)) \
                        : config_one<float, V>(smem, bps);
    switch (NB) {
        CR_NB_LIST(CR_CASE)
        default: return cudaErrorInvalidValue;
    }
#undef CR_CASE
}

}  // namespace cr

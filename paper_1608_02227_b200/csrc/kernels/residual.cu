// Residual pass of cr_primal: the diagnostics of eta(Theta) (Theorem 1)
//
//   R_ij = (C eta)_ij = y_j - y_i + xi_i^T (x_i - x_j) = (y_j + (a_i - y_i)) - xi_i . x_j,  a_i = xi_i . x_i
//   gap = sum_{i != j} Theta_ij R_ij,   v2 = sum (R_ij)_-^2,   vmax = max (-R_ij)_+
//
// in fp64 (the diagnostics are compared with the fp64 oracle to 1e-4 relative, and the max
// violation is a small difference of O(|xi||x|) terms).  The pass is an fp64 rank-n contraction
// S = Xi X^T with a reduction epilogue: N^2 n DFMA against one 4-byte read of Theta per pair, so it
// is bound by the fp64 FMA pipe (64 DFMA / clk / SM), not by HBM.  Layout for that bound:
//   * CTA tile 128 rows (i) x 64 columns (j), 256 threads = 8 warps in a 4 x 2 grid, 2 CTAs per SM,
//     each warp a 32 x 32 block of 4 x 4 fp64 tensor-core tiles (mma.sync m8n8k4 .f64: 256 FMA per
//     instruction).  A CUDA-core DFMA version (8 x 8 or 4 x 8 register tiles) left the fp64 pipe
//     41% busy with "wait" (fixed-latency issue) the top stall: the issue rate, not the pipe,
//     was the limit.  Operand rows are padded (LDA, LDB) so a fragment load is conflict-free.
//   * Both operands k-major in global memory (X^T prepared once in cr_init, Xi^T by a transpose
//     before the pass), moved in chunks of KC features by cp.async into a shared ring; the
//     chunk sequence runs across tiles, so the next tile's first chunks load under this tile's
//     last ones.  Features beyond n are zero-filled (cp.async src-size 0).
//   * Theta (fp32) for the tile is staged into a shared image together with the tile's second
//     chunk (16 KB per 128 x 32 tile-major tile, or 128 row segments of 256 B), so its HBM
//     latency overlaps the tile's remaining chunks; fp64 Theta (small problems) is read from
//     global memory in the epilogue.
//   * Persistent CTAs (one per SM) walk tiles blockIdx.x, +gridDim.x, ... in a fixed order; the
//     per-thread sums and the final block tree are fixed-order, so results are bitwise repeatable.
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"

namespace cr {
namespace {

// KC = 16 features per chunk with a 2-stage ring (one barrier per 16 features: ncu showed the
// per-chunk barrier as the third stall at KC = 8); rows padded to 136 doubles so a fragment
// load's four k-rows fall in bank halves {0, 1} / {2, 3} (two wavefronts, the minimum for 256 B)
// (KC = 8 with 3 stages when n is not a multiple of 16: C4's n = 40 would otherwise run 20% zero
// features)
// Two CTAs of 8 warps per SM, CTA tile 128 x 64: one CTA's epilogue and barriers overlap the
// other's tensor work (with one 16-warp CTA per SM every warp reached the epilogue and every
// chunk barrier together).  Operand rows padded: LDA = 136, LDB = 72 doubles.
constexpr int RBM = 128, RBN = 64, RTH = 256, LDA = 136, LDB = 72;
template <int KC> struct ResCfg {
    static constexpr int STAGES = KC == 16 ? 2 : 3;
    static constexpr int A_BYTES = KC * LDA * 8, B_BYTES = KC * LDB * 8;   // padded rows
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
};
constexpr int TH_BYTES = RBM * RBN * 4;                              // fp32 Theta tile, 32 KB
constexpr int VEC_BYTES = (RBN + 2 * RBM) * 8;                       // y_j, a_i, y_i
constexpr int TBUF_BYTES = TH_BYTES + VEC_BYTES;

__device__ __forceinline__ void cp16(void *smem, const void *gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;                                    // 0: zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp8(void *smem, const void *gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <typename T, int KC>
__global__ void __launch_bounds__(RTH, 2) residual2_kernel(const ResidualParams p) {
    constexpr int STAGES = ResCfg<KC>::STAGES, A_BYTES = ResCfg<KC>::A_BYTES, STAGE_BYTES = ResCfg<KC>::STAGE_BYTES;
    extern __shared__ __align__(16) uint8_t rsm[];
    uint8_t *stages = rsm;                                   // [STAGES][A | B]
    uint8_t *tbuf = rsm + STAGES * STAGE_BYTES;              // Theta tile | y_j | a_i | y_i (one buffer)
    __shared__ double red[3][RTH];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, wr = warp >> 1, wc = warp & 1;   // warp block (wr, wc): 4 x 2
    const int fg = lane >> 2, ft = lane & 3;                    // mma fragment group / thread in group
    const int nrb = (int)((p.Ns + RBM - 1) / RBM), ncb = (int)((p.N + RBN - 1) / RBN);
    const int ntiles = nrb * ncb;                             // < 2^31 (N <= 2^22 rows / columns)
    const int G = gridDim.x;
    const int my = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;   // tiles of this CTA
    // chunks per tile (zero chunks pad small n); the tile's Theta is staged with chunk STAGES - 1,
    // the first one issued after the previous tile's epilogue has passed its barrier
    constexpr int KTH = STAGES - 1;
    const int nCk = max((p.nP + KC - 1) / KC, KTH + 1);
    const bool stage_theta = sizeof(T) == 4;

    // Loads of one chunk (tile it of this CTA at (rb, cb), feature chunk kc) into ring stage st;
    // the tile's first chunk also brings its Theta tile and vectors into tbuf[it & 1].  Cursors
    // advance incrementally: no 64-bit division in the loop.
    struct Cur { int it, kc, st, rb, cb; };
    auto locate = [&](Cur &c) {
        const int t = (int)blockIdx.x + c.it * G;
        c.rb = t / ncb;
        c.cb = t - c.rb * ncb;
    };
    auto advance = [&](Cur &c) {
        if (++c.st == STAGES) c.st = 0;
        if (++c.kc == nCk) { c.kc = 0; ++c.it; if (c.it < my) locate(c); }
    };
    auto issue = [&](const Cur &c) {
        if (c.it < my) {
            const int64_t i0 = (int64_t)c.rb * RBM, j0 = (int64_t)c.cb * RBN;
            uint8_t *st = stages + c.st * STAGE_BYTES;
            double *As = reinterpret_cast<double *>(st), *Bs = reinterpret_cast<double *>(st + A_BYTES);
            // A: Xi^T rows k0.., columns i0..i0+127 (KC x 1 KB); B: X^T, columns j0..j0+63 (KC x 512 B)
#pragma unroll
            for (int e = 0; e < KC * 64 / RTH; ++e) {
                const int f = tid + e * RTH;                // KC x 64 pieces of 16 B
                const int kk = f >> 6, q = f & 63;
                const int k = c.kc * KC + kk;
                const bool ok = k < p.nP;
                cp16(As + kk * LDA + q * 2, p.XiT + (ok ? (int64_t)k * p.Rp + i0 + q * 2 : 0), ok);
            }
#pragma unroll
            for (int e = 0; e < KC * 32 / RTH; ++e) {
                const int f = tid + e * RTH;                // KC x 32 pieces of 16 B
                const int kk = f >> 5, q = f & 31;
                const int k = c.kc * KC + kk;
                const bool ok = k < p.nP;
                cp16(Bs + kk * LDB + q * 2, p.XT + (ok ? (int64_t)k * p.ldX + j0 + q * 2 : 0), ok);
            }
            if (c.kc == KTH) {
                // the tile's Theta and vectors into the single tile buffer: chunk KTH is issued
                // in iteration (tile start), after the barrier that follows the previous tile's
                // epilogue; consumed after chunk nCk - 1 >= KTH
                uint8_t *tb = tbuf;
                if (stage_theta) {
                    const float *Th = static_cast<const float *>(p.Theta);
                    if (p.tiled) {
                        // two 128 x 32 tiles of 16 KB (tile-major, swizzled image kept as is)
                        const int64_t tbase = ((i0 >> 7) * p.nCBt) << 12;
#pragma unroll
                        for (int e = 0; e < 2048 / RTH; ++e) {
                            const int f = tid + e * RTH;    // 2048 pieces
                            const int q = f >> 10, w = f & 1023;
                            const int tcb = c.cb * 2 + q;
                            const bool ok = tcb < p.nCBt;
                            const float *src = Th + (ok ? tbase + ((int64_t)tcb << 12) + w * 4 : 0);
                            cp16(tb + q * 16384 + w * 16, src, ok);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 2048 / RTH; ++e) {
                            const int f = tid + e * RTH;    // 128 rows x 16 pieces
                            const int r = f >> 4, w = f & 15;
                            cp16(tb + r * 256 + w * 16, Th + (i0 + r) * p.ldT + j0 + w * 4, true);
                        }
                    }
                }
                double *v = reinterpret_cast<double *>(tb + TH_BYTES);
                if (tid < RBN) {
                    const int64_t j = j0 + tid;
                    cp8(v + tid, p.y64 + (j < p.N ? j : 0), j < p.N);
                }
                if (tid < RBM) {
                    const int64_t i = i0 + tid;
                    cp8(v + RBN + tid, p.a64 + (i < p.Ns ? i : 0), i < p.Ns);
                    cp8(v + RBN + RBM + tid, p.y64 + (i < p.Ns ? p.row0 + i : 0), i < p.Ns);
                }
            }
        }
        cp_commit();                                        // (possibly empty group: uniform accounting)
    };

    double gap = 0.0, v2 = 0.0, vmax = 0.0;
    double acc[4][4][2];                                     // [row tile][col tile][2 cols]
    Cur cc{0, 0, 0, 0, 0}, ci{0, 0, 0, 0, 0};
    if (my > 0) { locate(cc); locate(ci); }
    for (int g = 0; g < STAGES - 1; ++g) { issue(ci); advance(ci); }
    for (; cc.it < my; advance(cc)) {
        if (cc.kc == 0) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        }
        cp_wait<STAGES - 2>();
        __syncthreads();
        issue(ci);
        advance(ci);
        const uint8_t *st = stages + cc.st * STAGE_BYTES;
        // fragments (m8n8k4, .row A / .col B): A[fg][ft] = Xi_{i0+fg}[k0+ft], B[ft][fg] = x_{j0+fg}[k0+ft]
        const double *As = reinterpret_cast<const double *>(st) + ft * LDA + wr * 32 + fg;
        const double *Bs = reinterpret_cast<const double *>(st + A_BYTES) + ft * LDB + wc * 32 + fg;
#pragma unroll
        for (int k4 = 0; k4 < KC / 4; ++k4) {
            double a[4], b[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) a[mt] = As[k4 * 4 * LDA + mt * 8];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) b[nt] = Bs[k4 * 4 * LDB + nt * 8];
            // m16n8k4 (sm_90+): rows fg and fg + 8 of a 16-row tile = the m8 sub-tiles 2 mp, 2 mp + 1
            // (a0 = A[fg][ft], a1 = A[fg + 8][ft]; c0, c1 / c2, c3 = rows fg / fg + 8): half the
            // instructions of m8n8k4 for the same fragments
#pragma unroll
            for (int mp = 0; mp < 2; ++mp)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
                                 "{%0,%1,%2,%3};"
                                 : "+d"(acc[2 * mp][nt][0]), "+d"(acc[2 * mp][nt][1]), "+d"(acc[2 * mp + 1][nt][0]),
                                   "+d"(acc[2 * mp + 1][nt][1])
                                 : "d"(a[2 * mp]), "d"(a[2 * mp + 1]), "d"(b[nt]));
        }
        if (cc.kc == nCk - 1) {
            // ---- epilogue of the tile: R = (y_j + (a_i - y_i)) - xi_i . x_j over the thread's 32 pairs
            // (accumulator [mt][nt][c] = pair (wr*32 + mt*8 + fg, wc*32 + nt*8 + 2 ft + c))
            const int64_t i0 = (int64_t)cc.rb * RBM, j0 = (int64_t)cc.cb * RBN;
            const uint8_t *tb = tbuf;
            const double *v = reinterpret_cast<const double *>(tb + TH_BYTES);
            const float *Ts = reinterpret_cast<const float *>(tb);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int il = wr * 32 + mt * 8 + fg;
                const int64_t i = i0 + il;
                if (i >= p.Ns) continue;
                const double ab = v[RBN + il] - v[RBN + RBM + il];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int jj = nt * 8 + 2 * ft + c;             // column within the 32-wide tc tile wc
                        const int jl = wc * 32 + jj;
                        const int64_t j = j0 + jl;
                        if (j >= p.N || p.row0 + i == j) continue;
                        const double R = (v[jl] + ab) - acc[mt][nt][c];
                        double th;
                        if (stage_theta) {
                            th = p.tiled ? (double)Ts[wc * 4096 + il * 32 + (((jj >> 2) ^ (il & 7)) << 2) + (jj & 3)]
                                         : (double)Ts[il * RBN + jl];
                        } else {
                            th = (double)static_cast<const T *>(p.Theta)[theta_off(i, j, p.ldT, p.tiled, p.nCBt)];
                        }
                        gap = fma(th, R, gap);
                        if (R < 0.0) {
                            v2 = fma(R, R, v2);
                            vmax = fmax(vmax, -R);
                        }
                    }
                }
            }
        }
    }
    cp_wait<0>();
    red[0][tid] = gap;
    red[1][tid] = v2;
    red[2][tid] = vmax;
    __syncthreads();
    for (int s = RTH / 2; s > 0; s >>= 1) {
        if (tid < s) {
            red[0][tid] += red[0][tid + s];
            red[1][tid] += red[1][tid + s];
            red[2][tid] = fmax(red[2][tid], red[2][tid + s]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        p.statpart[blockIdx.x * 8 + 4] = red[0][0];
        p.statpart[blockIdx.x * 8 + 5] = red[1][0];
        p.statpart[blockIdx.x * 8 + 6] = red[2][0];
        p.statpart[blockIdx.x * 8 + 7] = (isfinite(red[0][0]) && isfinite(red[1][0])) ? 0.0 : 1.0;
    }
}

// dst[k][i] = src[i][k] for k < n, 0 for n <= k < nP; i < rows (zero for rows <= i < ld)
__global__ void transpose_pad_kernel(const double *src, int64_t rows, int n, int nP, int64_t ld, double *dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)nP * ld) return;
    const int64_t k = e / ld, i = e - k * ld;
    dst[e] = (i < rows && k < n) ? src[i * n + k] : 0.0;
}

}  // namespace

size_t residual_smem_bytes() {
    const size_t a = (size_t)ResCfg<16>::STAGES * ResCfg<16>::STAGE_BYTES, b = (size_t)ResCfg<8>::STAGES * ResCfg<8>::STAGE_BYTES;
    return (a > b ? a : b) + (size_t)TBUF_BYTES;
}

cudaError_t launch_transpose_pad(const double *src, int64_t rows, int n, int nP, int64_t ld, double *dst,
                                 cudaStream_t s) {
    const int64_t total = (int64_t)nP * ld;
    if (total == 0) return cudaSuccess;
    transpose_pad_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(src, rows, n, nP, ld, dst);
    return cudaGetLastError();
}

cudaError_t launch_residual(const ResidualParams &p, int fp64, cudaStream_t s, int *nb_out) {
    // Xi^T for this call (the prologue wrote Xi64 [Rp][n])
    cudaError_t e = launch_transpose_pad(p.Xi64, p.Ns, p.n, p.nP, p.Rp, const_cast<double *>(p.XiT), s);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = ((p.Ns + RBM - 1) / RBM) * ((p.N + RBN - 1) / RBN);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int cap = 2 * sms < kStatBlocks ? 2 * sms : kStatBlocks;   // two CTAs per SM
    const int nb = (int)(ntiles < cap ? (ntiles > 0 ? ntiles : 1) : cap);
    const int smem = (int)residual_smem_bytes();
    const bool k16 = p.nP % 16 == 0;
#define CR_RES(T, K)                                                                                 \
    do {                                                                                             \
        e = cudaFuncSetAttribute(residual2_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        if (e != cudaSuccess) return e;                                                              \
        residual2_kernel<T, K><<<nb, RTH, smem, s>>>(p);                                             \
    } while (0)
    if (fp64) {
        if (k16) CR_RES(double, 16); else CR_RES(double, 8);
    } else {
        if (k16) CR_RES(float, 16); else CR_RES(float, 8);
    }
#undef CR_RES
    if (nb_out) *nb_out = nb;
    return cudaGetLastError();
}

}  // namespace cr

// SMEM-resident multi-iteration solver for small N (C1, C2 shapes): one cooperative launch runs
// K P-APG iterations (Fig. 2) with both state matrices held in shared memory.
//
// CTA g owns the rows [g R, min(N, (g+1) R)) of Theta^{k-1} and Theta^{k-2} (all N columns)
// for the whole launch, so Theta never touches HBM between iterations; row sums r_i and
// (Theta X)_i are CTA-local, only the column sums c_j cross CTAs.  Per iteration:
//   A  Step 1 for own rows from S~ = S^{k-1} + beta (S^{k-1} - S^{k-2}):
//      y_i = ybar_i + c~_i - r~_i, xi_i = (r~_i x_i - P~_i)/gamma, a_i = xi_i . x_i; y_i -> global
//   -- grid sync --
//   B  Steps 2 + 4 for own rows x all columns, Theta^k written over Theta^{k-2} in
//      smem (theta~ formed on the fly, fp64 combine, one rounding to storage); then column
//      partials (thread per column, rows in order) -> global, r_i^k and P_i^k (warp per row)
//   -- grid sync --
//   C  c_i^k = sum_g cpart[g][i] for own rows (fixed order); Step 3; roles rotate.
// Two grid syncs per iteration; every reduction has a fixed order (bitwise reproducible).
// At the end the state (Theta rows, sums of both iterates, t) is written back to the workspace
// exactly as K graph-replayed iterations of the streaming path would leave it.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"

namespace cg = cooperative_groups;

namespace cr {
namespace {

constexpr int RT = 512;         // threads per CTA (16 warps: latency hiding at 1 CTA per SM)
constexpr int NW = RT / 32;
constexpr int kB2Chunks = 8;    // small-N B2: column chunks per row

template <typename T, int NMAX>
__global__ void __launch_bounds__(RT, 1) resident_kernel(const ResidentParams p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char rsm_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t N = p.N;
    const int n = p.n, R = p.R, ldS = p.ldS;
    const int64_t row0 = (int64_t)blockIdx.x * R;
    const int64_t rem = N - row0;
    const int rows = rem <= 0 ? 0 : (rem < R ? (int)rem : R);
    const bool multi = gridDim.x > 1;
    // ---- shared memory carve-up
    // X and xi are padded to NMAX features with zeros, so the hot loops run to the compile-time
    // NMAX without per-feature branches
    // (X and xi in the storage precision T: the products of the pass are formed in T, as in the
    // streaming SIMT pass; the combine and every sum across lanes / CTAs are fp64)
    double *ys = reinterpret_cast<double *>(rsm_raw);          // [N]        y of all rows
    double *as = ys + N;                                        // [R]        a_i - y_i
    double *r1 = as + R, *r2 = r1 + R, *c1 = r2 + R, *c2 = c1 + R;   // sums of Theta^{k-1}, ^{k-2}
    double *P1 = c2 + R, *P2 = P1 + (size_t)R * n;
    // B1 row groups: with N < RT, H column copies of the thread set split the rows (H N <= RT)
    int H = 1;
    while (H < 16 && 2 * H * N <= RT) H *= 2;
    double *cph = P2 + (size_t)R * n;                           // [H][N]     column partials (H > 1)
    // small N: B2 runs over (row, column chunk) pairs; their partial records
    double *b2s = cph + (N < RT ? RT : 0);                      // [R][kB2Chunks][1 + NMAX] (N < RT)
    T *xT = reinterpret_cast<T *>(b2s + (N < RT ? (size_t)R * kB2Chunks * (1 + NMAX) : 0));   // [NMAX][N]
    T *xis = xT + (size_t)N * NMAX;                             // [R][NMAX]  xi of own rows
    T *thA = xis + (size_t)R * NMAX;                            // [R][ldS] Theta^{k-1}
    T *thB = thA + (size_t)R * ldS;                             // [R][ldS] Theta^{k-2} -> Theta^k
    const T *gA = static_cast<const T *>(p.TA);
    const T *gB = static_cast<const T *>(p.TB);

    // ---- load the state
    for (int i = 0; i < rows; ++i)
        for (int64_t j = threadIdx.x; j < N; j += RT) {
            thA[(size_t)i * ldS + j] = gA[(row0 + i) * p.ldT + j];
            thB[(size_t)i * ldS + j] = gB[(row0 + i) * p.ldT + j];
        }
    for (int64_t j = threadIdx.x; j < N; j += RT)
        for (int d = 0; d < NMAX; ++d) xT[(size_t)d * N + j] = d < n ? T(p.X64[j * n + d]) : T(0);
    for (int e = threadIdx.x; e < R * NMAX; e += RT) xis[e] = T(0);
    for (int i = threadIdx.x; i < rows; i += RT) {
        r1[i] = p.rA[row0 + i]; c1[i] = p.cA[row0 + i];
        r2[i] = p.rB[row0 + i]; c2[i] = p.cB[row0 + i];
    }
    for (int e = threadIdx.x; e < rows * n; e += RT) {
        P1[e] = p.PA[row0 * n + e];
        P2[e] = p.PB[row0 * n + e];
    }
    double t_prev = p.ts->t_prev, t_cur = p.ts->t_cur;
    const double invL = 1.0 / p.L, invG = 1.0 / p.gamma;
    __syncthreads();

#define RS_TRACE(ev)                                                                          \
    do {                                                                                      \
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && it < 16) p.trace[it * 8 + (ev)] = clock64(); \
    } while (0)
    for (int64_t it = 0; it < p.K; ++it) {
        RS_TRACE(0);
        const double beta = (t_prev - 1.0) / t_cur;             // beta_{k-1} = (t_{k-1} - 1)/t_k
        // ---------------- A: Step 1 for own rows (thread per row, n <= 32)
        for (int i = threadIdx.x; i < rows; i += RT) {
            const int64_t gi = row0 + i;
            const double rt = r1[i] + beta * (r1[i] - r2[i]);
            const double ct = c1[i] + beta * (c1[i] - c2[i]);
            const double y = p.ybar[gi] + ct - rt;
            double a = 0.0;
            const double *x = p.X64 + gi * n;
            for (int d = 0; d < n; ++d) {
                const double Pt = P1[i * n + d] + beta * (P1[i * n + d] - P2[i * n + d]);
                const double xd = x[d];
                const double xi = (rt * xd - Pt) * invG;
                xis[i * NMAX + d] = T(xi * invL);               // xi / L: the pass operand
                a = fma(xi, xd, a);
                if (it + 1 == p.K) p.Xi64[gi * n + d] = xi;
            }
            as[i] = a - y;
            if (multi) p.yg[gi] = y;
            else ys[gi] = y;
            p.a64[gi] = a;                                      // eta^k outputs (cr_get_eta)
            p.y64[gi] = y;
        }
        RS_TRACE(1);
        if (multi) {
            grid.sync();
            RS_TRACE(2);
            for (int64_t j = threadIdx.x; j < N; j += RT) ys[j] = p.yg[j];
        }
        __syncthreads();
        RS_TRACE(3);
        // ---------------- B1: Steps 2 + 4, thread per column j (x_j in registers), own rows in
        // groups of 4 (independent dot products); column partial of the CTA's rows in order.
        // Small N (H > 1): thread (h, j) takes rows h, h + H, ...; the H partials are combined
        // in h order (fixed: bitwise reproducible)
        for (int64_t t = threadIdx.x; t < (H > 1 ? (int64_t)H * N : N); t += RT) {
            const int64_t j = H > 1 ? t % N : t;
            const int h = H > 1 ? (int)(t / N) : 0;
            T x[NMAX];     // storage precision for the dot products (fp32 configs: as the streaming
                           // SIMT pass does), fp64 for the combine
#pragma unroll
            for (int d = 0; d < NMAX; ++d) x[d] = xT[(size_t)d * N + j];
            const double yj = ys[j];
            double cs = 0.0;
            for (int i0 = h; i0 < rows; i0 += 4 * H) {
                T s[4] = {T(0), T(0), T(0), T(0)};
                int iq[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) iq[q] = min(i0 + q * H, rows - 1);
#pragma unroll
                for (int d = 0; d < NMAX; ++d) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) s[q] = fma(xis[iq[q] * NMAX + d], x[d], s[q]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = i0 + q * H;
                    if (i < rows) {
                        // (C eta)_ij / L = (y_j - y_i + a_i)/L - (xi_i / L) . x_j
                        const double RL = (yj + as[i]) * invL - (double)s[q];
                        const double b1 = (double)thA[(size_t)i * ldS + j];
                        const double v = fma(beta, b1 - (double)thB[(size_t)i * ldS + j], b1) - RL;
                        const T th = (row0 + i == j) ? T(0) : T(fmax(v, 0.0));    // ( . )_+, diag
                        thB[(size_t)i * ldS + j] = th;
                        cs += (double)th;
                    }
                }
            }
            if (H > 1) cph[(size_t)h * N + j] = cs;
            else if (multi) p.cpart[(int64_t)blockIdx.x * N + j] = cs;
            else ys[j] = cs;                                    // single CTA: c directly (y consumed)
        }
        if (H > 1) {
            __syncthreads();
            for (int64_t j = threadIdx.x; j < N; j += RT) {
                double cs = 0.0;
                for (int h = 0; h < H; ++h) cs += cph[(size_t)h * N + j];
                if (multi) p.cpart[(int64_t)blockIdx.x * N + j] = cs;
                else ys[j] = cs;
            }
        }
        __syncthreads();
        RS_TRACE(4);
        // ---------------- B2: r_i^k and (Theta^k X)_i
        if (N < RT) {
            // small N: thread per (row, column chunk), chunks combined in order (fixed)
            for (int t = threadIdx.x; t < rows * kB2Chunks; t += RT) {
                const int i = t / kB2Chunks, ch = t % kB2Chunks;
                const int64_t ja = N * ch / kB2Chunks, jb = N * (ch + 1) / kB2Chunks;
                T racc_t = T(0), pacc_t[NMAX];
#pragma unroll
                for (int d = 0; d < NMAX; ++d) pacc_t[d] = T(0);
                const T *row = thB + (size_t)i * ldS;
                for (int64_t j = ja; j < jb; ++j) {
                    const T th = row[j];
                    racc_t += th;
#pragma unroll
                    for (int d = 0; d < NMAX; ++d) pacc_t[d] = fma(th, xT[(size_t)d * N + j], pacc_t[d]);
                }
                double *rec = b2s + (size_t)t * (1 + NMAX);
                rec[0] = (double)racc_t;
#pragma unroll
                for (int d = 0; d < NMAX; ++d) rec[1 + d] = (double)pacc_t[d];
            }
            __syncthreads();
            for (int e = threadIdx.x; e < rows * (1 + n); e += RT) {
                const int i = e / (1 + n), d = e % (1 + n);          // d = 0: r, d >= 1: (Theta X)_{d-1}
                double v = 0.0;
                for (int ch = 0; ch < kB2Chunks; ++ch) v += b2s[((size_t)i * kB2Chunks + ch) * (1 + NMAX) + d];
                if (d == 0) { r2[i] = r1[i]; r1[i] = v; }
                else { P2[i * n + d - 1] = P1[i * n + d - 1]; P1[i * n + d - 1] = v; }
            }
        } else
        // warp per row, lanes over j (d independent)
        for (int i = warp; i < rows; i += NW) {
            // per-lane sums in the storage precision (fp32 within a lane's <= N/32 terms, as the
            // streaming pass sums within a tile), fp64 across lanes
            T racc_t = T(0), pacc_t[NMAX];
#pragma unroll
            for (int d = 0; d < NMAX; ++d) pacc_t[d] = T(0);
            const T *row = thB + (size_t)i * ldS;
            for (int64_t j = lane; j < N; j += 32) {
                const T th = row[j];
                racc_t += th;
#pragma unroll
                for (int d = 0; d < NMAX; ++d) pacc_t[d] = fma(th, xT[(size_t)d * N + j], pacc_t[d]);
            }
            double racc = (double)racc_t, pacc[NMAX];
#pragma unroll
            for (int d = 0; d < NMAX; ++d) pacc[d] = (double)pacc_t[d];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                racc += __shfl_xor_sync(0xffffffffu, racc, o);
#pragma unroll
                for (int d = 0; d < NMAX; ++d) pacc[d] += __shfl_xor_sync(0xffffffffu, pacc[d], o);
            }
            // roll the sums: S^{k-2} <- S^{k-1}, S^{k-1} <- S^k (c in phase C)
            if (lane == 0) { r2[i] = r1[i]; r1[i] = racc; }
#pragma unroll
            for (int d = 0; d < NMAX; ++d)
                if (d < n && lane == d) { P2[i * n + d] = P1[i * n + d]; P1[i * n + d] = pacc[d]; }
        }
        RS_TRACE(5);
        if (multi) grid.sync();
        else __syncthreads();
        RS_TRACE(6);
        // ---------------- C: column sums of own rows (warp per row, lanes over CTAs), Step 3
        for (int i = warp; i < rows; i += NW) {
            double s = 0.0;
            if (multi) {
                // all of a lane's loads in flight before the fixed-order sum
                double v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int g = lane + 32 * q;
                    v[q] = g < (int)gridDim.x ? p.cpart[(int64_t)g * N + row0 + i] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) s += v[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            } else {
                s = ys[row0 + i];
            }
            if (lane == 0) { c2[i] = c1[i]; c1[i] = s; }
        }
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t_cur * t_cur)) / 2.0;   // Step 3
        t_prev = t_cur;
        t_cur = tn;
        T *tmp = thA; thA = thB; thB = tmp;                     // Theta^k is Theta^{k-1} next
        __syncthreads();
    }
    // ---- write the state back: Theta^k replaced Theta^{k-2} K times, so after K iterations the
    // buffer roles flipped K times; sums likewise
    T *oA = static_cast<T *>((p.K & 1) ? p.TB : p.TA);         // receives Theta^k
    T *oB = static_cast<T *>((p.K & 1) ? p.TA : p.TB);         // receives Theta^{k-1}
    double *orA = (p.K & 1) ? p.rB : p.rA, *ocA = (p.K & 1) ? p.cB : p.cA, *oPA = (p.K & 1) ? p.PB : p.PA;
    double *orB = (p.K & 1) ? p.rA : p.rB, *ocB = (p.K & 1) ? p.cA : p.cB, *oPB = (p.K & 1) ? p.PA : p.PB;
    for (int i = 0; i < rows; ++i)
        for (int64_t j = threadIdx.x; j < N; j += RT) {
            oA[(row0 + i) * p.ldT + j] = thA[(size_t)i * ldS + j];
            oB[(row0 + i) * p.ldT + j] = thB[(size_t)i * ldS + j];
        }
    for (int i = threadIdx.x; i < rows; i += RT) {
        orA[row0 + i] = r1[i]; ocA[row0 + i] = c1[i];
        orB[row0 + i] = r2[i]; ocB[row0 + i] = c2[i];
    }
    for (int e = threadIdx.x; e < rows * n; e += RT) {
        oPA[row0 * n + e] = P1[e];
        oPB[row0 * n + e] = P2[e];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ts->t_prev = t_prev;
        p.ts->t_cur = t_cur;
    }
}

template <typename T, int NMAX>
size_t smem_of(const ResidentParams &p) {
    return sizeof(double) * ((size_t)p.N + 2 * (size_t)p.R * (size_t)p.n + 5 * (size_t)p.R + (p.N < RT ? RT : 0) +
                             (p.N < RT ? (size_t)p.R * kB2Chunks * (1 + NMAX) : 0)) +
           sizeof(T) * ((size_t)p.N * NMAX + (size_t)p.R * NMAX + 2 * (size_t)p.R * p.ldS) + 16;
}

template <typename T, int NMAX>
cudaError_t launch_t(const ResidentParams &p, cudaStream_t s) {
    const size_t smem = smem_of<T, NMAX>(p);
    cudaError_t e = cudaFuncSetAttribute(resident_kernel<T, NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ResidentParams q = p;
    void *args[] = {&q};
    return cudaLaunchCooperativeKernel((const void *)resident_kernel<T, NMAX>, dim3(p.G), dim3(RT), args, smem, s);
}

}  // namespace

int resident_bucket(int n) { return n <= 2 ? 2 : n <= 4 ? 4 : n <= 8 ? 8 : n <= 12 ? 12 : n <= 16 ? 16 : n <= 24 ? 24 : n <= 32 ? 32 : 0; }

size_t resident_smem_bytes(const ResidentParams &p, int fp64) {
    switch (resident_bucket(p.n)) {
#define CR_CASE(V) case V: return fp64 ? smem_of<double, V>(p) : smem_of<float, V>(p);
        CR_CASE(2) CR_CASE(4) CR_CASE(8) CR_CASE(12) CR_CASE(16) CR_CASE(24) CR_CASE(32)
#undef CR_CASE
        default: return (size_t)1 << 40;
    }
}

cudaError_t launch_resident(const ResidentParams &p, int fp64, cudaStream_t s) {
    if (p.K <= 0) return cudaSuccess;
    switch (resident_bucket(p.n)) {
#define CR_CASE(V) case V: return fp64 ? launch_t<double, V>(p, s) : launch_t<float, V>(p, s);
        CR_CASE(2) CR_CASE(4) CR_CASE(8) CR_CASE(12) CR_CASE(16) CR_CASE(24) CR_CASE(32)
#undef CR_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace cr

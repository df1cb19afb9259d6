// Step 1 of P-APG for a general partition K < N (Section 2.1): per block of nbar
// points, the G-norm projection of the closed-form point eta0 = (y0, xi0) onto the block's
// intra-block constraints (Eq. (subgradient_split)),
//     min 1/2 ||y - y0||^2 + gamma/2 ||xi - xi0||^2   s.t.   y_l' - y_l + xi_l . (x_l - x_l') >= 0,
// by a primal-dual interior-point method (Mehrotra predictor-corrector) whose normal equations
// M = G + A^T D A are block arrowhead (Eq. (arrowhead)) and are solved through the
// y-block Schur complement S = M00 - sum_l M0l Mll^{-1} M0l^T (the closed form of Theorem
// "cholesky-block-arrowhead" P:660-700 with F0 the Cholesky factor of S -- see DESIGN.md R20).
// One CTA per block, fp64; X and S in shared memory, the per-constraint vectors and the Mll
// Cholesky factors in a per-block global scratch (L1/L2-resident).
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include "../cr_internal.h"

namespace cr {
namespace {

constexpr int IT = 512;
constexpr int TY = IT / 16;           // rows of the 16-wide thread grid (Cholesky update, S tiles)
constexpr int kMaxNbar = 128;         // == kIpmMaxNbar
constexpr double kRho = 1.0;          // multiplier-method penalty of the polish (G-scaled problem)
constexpr int kPolishRounds = 6;
constexpr int kPolishIters = 60;
constexpr int kRhoAttempts = 3;       // rho = 1, 10, 100

__device__ __forceinline__ double block_reduce(double v, double *sh, bool is_max) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = IT / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            sh[threadIdx.x] = is_max ? fmax(sh[threadIdx.x], sh[threadIdx.x + s]) : sh[threadIdx.x] + sh[threadIdx.x + s];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

struct Blk {
    int nb, n;            // points in the block, features
    double gamma;
    const double *Xs;     // smem [nb][n]
    double *S;            // smem [nb][nb] Schur complement / its Cholesky factor (lower)
    double *Mll;          // smem [G][n][n]
    double *Z;            // smem [G][n][nb]
    double *Lf;           // global [nb][n][n] Cholesky factors of Mll
    double *D;            // global [m] lambda / s
    double *red;          // smem [IT] reduction scratch
    double *Drow;         // smem [G][nb] row l of D (factor)
    int G;                // points factored concurrently (one warp each)
    // pair p = (l, l') -> p = l (nb - 1) + l' - [l' > l]
    __device__ int pid(int l, int lp) const { return l * (nb - 1) + lp - (lp > l ? 1 : 0); }
    __device__ double delta(int l, int lp, int d) const { return Xs[l * n + d] - Xs[lp * n + d]; }
};

// out_p = (A v)_p = v_y[l'] - v_y[l] + v_xi[l] . (x_l - x_l')   for all pairs (threads over p)
__device__ void apply_A(const Blk &B, const double *vy, const double *vxi, double *out) {
    const int m = B.nb * (B.nb - 1);
    for (int p = threadIdx.x; p < m; p += IT) {
        const int l = p / (B.nb - 1), q = p % (B.nb - 1), lp = q + (q >= l ? 1 : 0);
        double s = vy[lp] - vy[l];
        for (int d = 0; d < B.n; ++d) s += vxi[l * B.n + d] * B.delta(l, lp, d);
        out[p] = s;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int NW = IT / 32;
constexpr int kMaxPerLane = (kMaxNbar + 31) / 32;   // pairs (l, .) handled per lane

// (A^T w): y part [nb], xi part [nb][n].  Warp per point k, lanes over its partners o:
//   (A^T w)_y[k]  = sum_o w(o,k) - w(k,o)          (+1 on y_l' of pair (o,k), -1 on y_l of (k,o))
//   (A^T w)_xi[k] = sum_o w(k,o) (x_k - x_o)
__device__ void apply_AT(const Blk &B, const double *w, double *oy, double *oxi) {
    const int lane = threadIdx.x & 31, nb = B.nb;
    for (int k = threadIdx.x >> 5; k < nb; k += NW) {
        double wk[kMaxPerLane];
        double sy = 0.0;
#pragma unroll
        for (int q = 0; q < kMaxPerLane; ++q) {
            const int o = lane + 32 * q;
            wk[q] = 0.0;
            if (o < nb && o != k) {
                wk[q] = w[B.pid(k, o)];
                sy += w[B.pid(o, k)] - wk[q];
            }
        }
        sy = warp_sum(sy);
        if (lane == 0) oy[k] = sy;
        for (int d = 0; d < B.n; ++d) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < kMaxPerLane; ++q) {
                const int o = lane + 32 * q;
                if (o < nb) v += wk[q] * B.delta(k, o, d);       // wk = 0 at o == k
            }
            v = warp_sum(v);
            if (lane == 0) oxi[k * B.n + d] = v;
        }
    }
}

// Cholesky (lower, in place) of the k x k smem matrix A (row-major, lda); right-looking, the
// trailing update on a 16-wide thread grid.  Pivots are floored at 1e-15 of the largest diagonal
// entry (the Schur complement of a late interior-point iteration can lose definiteness to
// rounding; the polish removes the effect).  Only the lower triangle is read or written.
__device__ void chol(double *A, int k, int lda, double *red) {
    double dm = 0.0;
    for (int j = threadIdx.x; j < k; j += IT) dm = fmax(dm, A[j * lda + j]);
    const double floor_ = fmax(block_reduce(dm, red, true) * 1e-15, 1e-300);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    for (int j = 0; j < k; ++j) {
        const double djj = sqrt(fmax(A[j * lda + j], floor_));
        __syncthreads();                                    // everyone has read A[j][j]
        const double rj = 1.0 / djj;
        if (threadIdx.x == 0) A[j * lda + j] = rj;           // the factor's diagonal is stored inverted
        for (int i = j + 1 + threadIdx.x; i < k; i += IT) A[i * lda + j] *= rj;
        __syncthreads();
        for (int i = j + 1 + ty; i < k; i += TY) {
            const double aij = A[i * lda + j];
            for (int c = j + 1 + tx; c <= i; c += 16) A[i * lda + c] -= aij * A[c * lda + j];
        }
        __syncthreads();
    }
}

// Same for a small k x k matrix by ONE warp (lanes over rows); no block barrier.
__device__ void chol_warp(double *A, int k, int lda) {
    const int lane = threadIdx.x & 31;
    double dm = 0.0;
    for (int j = lane; j < k; j += 32) dm = fmax(dm, A[j * lda + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    const double floor_ = fmax(dm * 1e-15, 1e-300);
    for (int j = 0; j < k; ++j) {
        const double djj = sqrt(fmax(A[j * lda + j], floor_));
        __syncwarp();
        const double rj = 1.0 / djj;
        if (lane == 0) A[j * lda + j] = rj;                  // the factor's diagonal is stored inverted
        for (int i = j + 1 + lane; i < k; i += 32) A[i * lda + j] *= rj;
        __syncwarp();
        for (int i = j + 1 + lane; i < k; i += 32) {
            const double aij = A[i * lda + j];
            for (int c = j + 1; c <= i; ++c) A[i * lda + c] -= aij * A[c * lda + j];
        }
        __syncwarp();
    }
}

// in place: v <- (L L^T)^{-1} v, L the k x k lower factor (row-major, ld k, diagonal stored inverted); one warp,
// column-oriented substitutions (lanes over the rows below / above the pivot)
__device__ void chol_solve_warp(const double *Lm, int k, double *v) {
    const int lane = threadIdx.x & 31;
    for (int c = 0; c < k; ++c) {
        if (lane == 0) v[c] *= Lm[c * k + c];
        __syncwarp();
        const double vc = v[c];
        for (int i = c + 1 + lane; i < k; i += 32) v[i] -= Lm[i * k + c] * vc;
        __syncwarp();
    }
    for (int c = k - 1; c >= 0; --c) {
        if (lane == 0) v[c] *= Lm[c * k + c];
        __syncwarp();
        const double vc = v[c];
        for (int i = lane; i < c; i += 32) v[i] -= Lm[c * k + i] * vc;
        __syncwarp();
    }
}

// in place: v <- (L L^T)^{-1} v for the k x k factor in smem (row-major, ld k, diagonal stored
// inverted), v in smem; the whole block: 32-row diagonal blocks by warp 0 in registers (shuffle
// broadcast), the off-diagonal updates by all threads.
__device__ void chol_solve_block(const double *Lm, int k, double *v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int kb = 0; kb < k; kb += 32) {                  // forward: L y = v
        const int bs = min(32, k - kb);
        if (warp == 0) {
            double x = lane < bs ? v[kb + lane] : 0.0;
            for (int c = 0; c < bs; ++c) {
                if (lane == c) x *= Lm[(kb + c) * k + kb + c];
                const double yc = __shfl_sync(0xffffffffu, x, c);
                if (lane > c && lane < bs) x -= Lm[(kb + lane) * k + kb + c] * yc;
            }
            if (lane < bs) v[kb + lane] = x;
        }
        __syncthreads();
        for (int i = kb + bs + threadIdx.x; i < k; i += IT) {
            double s = 0.0;
            for (int c = 0; c < bs; ++c) s += Lm[i * k + kb + c] * v[kb + c];
            v[i] -= s;
        }
        __syncthreads();
    }
    for (int kb = ((k - 1) / 32) * 32; kb >= 0; kb -= 32) {   // backward: L^T x = y
        const int bs = min(32, k - kb);
        if (warp == 0) {
            double x = lane < bs ? v[kb + lane] : 0.0;
            for (int c = bs - 1; c >= 0; --c) {
                if (lane == c) x *= Lm[(kb + c) * k + kb + c];
                const double xc = __shfl_sync(0xffffffffu, x, c);
                if (lane < c) x -= Lm[(kb + c) * k + kb + lane] * xc;
            }
            if (lane < bs) v[kb + lane] = x;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kb; i += IT) {
            double s = 0.0;
            for (int c = 0; c < bs; ++c) s += Lm[(kb + c) * k + i] * v[kb + c];
            v[i] -= s;
        }
        __syncthreads();
    }
}

// Form the Schur complement S and the Mll factors for the current D (= lambda / s).
__device__ void factor(const Blk &B) {
    const int nb = B.nb, n = B.n, lane = threadIdx.x & 31;
    // M00 = I + sum_p D_p (e_l' - e_l)(e_l' - e_l)^T: a weighted graph Laplacian plus I
    for (int e = threadIdx.x; e < nb * nb; e += IT) {
        const int i = e / nb, j = e % nb;
        if (i != j) B.S[e] = -(B.D[B.pid(i, j)] + B.D[B.pid(j, i)]);
    }
    __syncthreads();
    for (int i = threadIdx.x >> 5; i < nb; i += NW) {
        double v = 0.0;
        for (int j = lane; j < nb; j += 32)
            if (j != i) v -= B.S[i * nb + j];
        v = warp_sum(v);
        if (lane == 0) B.S[i * nb + i] = 1.0 + v;
    }
    // Per point l (independent across l): Mll = gamma I + sum_l' D_ll' delta delta^T, its
    // Cholesky factor Lll (kept in Lf), and Z_l = Lll^{-1} M0l^T (n x nb), M0l^T's column l' =
    // D_ll' delta_ll' (l' != l), column l = -(sum of the others).  G points at a time (smem Drow /
    // Mll / Z per point), every phase spread over the whole block; then S -= sum_l Z_l^T Z_l.
    const int G = B.G, warp = threadIdx.x >> 5;
    const int nlow = n * (n + 1) / 2;
    for (int l0 = 0; l0 < nb; l0 += G) {
        const int gw = min(G, nb - l0);
        for (int e = threadIdx.x; e < gw * nb; e += IT) {
            const int g = e / nb, lp = e % nb, l = l0 + g;
            B.Drow[g * nb + lp] = lp == l ? 0.0 : B.D[B.pid(l, lp)];
        }
        __syncthreads();
        // Mll (lower triangle) and the unscaled M0l^T panels
        for (int e = threadIdx.x; e < gw * nlow; e += IT) {
            const int g = e / nlow, t = e % nlow, l = l0 + g;
            int d = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
            while (d * (d + 1) / 2 > t) --d;
            while ((d + 1) * (d + 2) / 2 <= t) ++d;
            const int f = t - d * (d + 1) / 2;
            const double *Dr = B.Drow + g * nb;
            double v = d == f ? B.gamma : 0.0;
            for (int lp = 0; lp < nb; ++lp) v += Dr[lp] * B.delta(l, lp, d) * B.delta(l, lp, f);
            B.Mll[g * n * n + d * n + f] = v;
        }
        for (int e = threadIdx.x; e < gw * n * nb; e += IT) {
            const int g = e / (n * nb), r = e % (n * nb), d = r / nb, lp = r % nb;
            B.Z[(size_t)g * n * nb + r] = B.Drow[g * nb + lp] * B.delta(l0 + g, lp, d);   // Drow[l] = 0
        }
        __syncthreads();
        for (int gd = warp; gd < gw * n; gd += NW) {                 // column l of M0l^T
            const int g = gd / n, d = gd % n;
            double *zr = B.Z + (size_t)g * n * nb + d * nb;
            double v = 0.0;
            for (int lp = lane; lp < nb; lp += 32) v -= zr[lp];
            v = warp_sum(v);
            if (lane == 0) zr[l0 + g] = v;
        }
        for (int g = warp; g < gw; g += NW) chol_warp(B.Mll + g * n * n, n, n);
        __syncthreads();
        // Z_l <- Lll^{-1} M0l^T (forward substitution, threads over the (point, column) pairs)
        for (int e = threadIdx.x; e < gw * nb; e += IT) {
            const int g = e / nb, lp = e % nb;
            const double *Ml = B.Mll + g * n * n;
            double *zc = B.Z + (size_t)g * n * nb + lp;
            for (int d = 0; d < n; ++d) {
                double s = zc[d * nb];
                for (int c = 0; c < d; ++c) s -= Ml[d * n + c] * zc[c * nb];
                zc[d * nb] = s * Ml[d * n + d];
            }
        }
        for (int e = threadIdx.x; e < gw * n * n; e += IT) B.Lf[(size_t)l0 * n * n + e] = B.Mll[e];
        __syncthreads();
        // S -= sum_w Z_w^T Z_w on the lower triangle: 4 x 4 register tiles on a 16 x TY thread grid
        const int K = gw * n;
        const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
        for (int i0 = 4 * ty; i0 < nb; i0 += 4 * TY)
            for (int j0 = 4 * tx; j0 <= i0; j0 += 64) {
                double acc[4][4] = {};
                for (int kk = 0; kk < K; ++kk) {
                    const double *zr = B.Z + (size_t)(kk / n) * n * nb + (kk % n) * nb;
                    double zi[4], zj[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        zi[q] = i0 + q < nb ? zr[i0 + q] : 0.0;
                        zj[q] = j0 + q < nb ? zr[j0 + q] : 0.0;
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[a][b] = fma(zi[a], zj[b], acc[a][b]);
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (i0 + a < nb && j0 + b <= i0 + a) B.S[(i0 + a) * nb + j0 + b] -= acc[a][b];
            }
        __syncthreads();
    }
    chol(B.S, nb, nb, B.red);
}

// Solve M [dy; dxi] = [by; bxi] with the factors (Schur complement form); by, bxi overwritten
// by the solution.  Scratch t [nb][n] (global).  Warp per point for the block-diagonal parts,
// each warp staging its Lll and right-hand side in its private smem (the factor's Mll / Z
// areas) so the substitution chains run from shared memory.
__device__ void solve(const Blk &B, double *by, double *bxi, double *t) {
    const int nb = B.nb, n = B.n, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp (Lll, rhs) staging areas carved from the factor's contiguous Mll + Z panels
    const int Ws = min(NW, (int)(((size_t)B.G * ((size_t)n * n + (size_t)n * nb)) / ((size_t)n * n + n)));
    const bool has = warp < Ws;
    double *Mw = B.Mll + (size_t)warp * (n * n + n), *vw = Mw + n * n;
    // t_l = Mll^{-1} b_l
    if (has)
        for (int l = warp; l < nb; l += Ws) {
            for (int e = lane; e < n * n; e += 32) Mw[e] = B.Lf[(size_t)l * n * n + e];
            for (int d = lane; d < n; d += 32) vw[d] = bxi[l * n + d];
            __syncwarp();
            chol_solve_warp(Mw, n, vw);
            for (int d = lane; d < n; d += 32) t[l * n + d] = vw[d];
            __syncwarp();
        }
    __syncthreads();
    // by <- by - sum_l M0l t_l ; (M0l t_l)[k] = D_lk delta_lk . t_l (l != k), [k] = -sum_l D_kl delta_kl . t_k
    for (int k = warp; k < nb; k += NW) {
        double s = 0.0;
        for (int l = lane; l < nb; l += 32) {
            if (l == k) continue;
            double dk = 0.0, dl = 0.0;
            for (int d = 0; d < n; ++d) {
                dk += B.delta(l, k, d) * t[l * n + d];
                dl += B.delta(k, l, d) * t[k * n + d];
            }
            s += B.D[B.pid(l, k)] * dk - B.D[B.pid(k, l)] * dl;
        }
        s = warp_sum(s);
        if (lane == 0) by[k] -= s;
    }
    __syncthreads();
    {
        double *v = B.Drow;                               // [>= nb] smem
        for (int k = threadIdx.x; k < nb; k += IT) v[k] = by[k];
        __syncthreads();
        chol_solve_block(B.S, nb, v);
        for (int k = threadIdx.x; k < nb; k += IT) by[k] = v[k];
    }
    __syncthreads();
    // dxi_l = Mll^{-1} (b_l - M0l^T dy);  (M0l^T dy)_d = sum_l' D_ll' delta_d (dy_l' - dy_l)
    if (has)
        for (int l = warp; l < nb; l += Ws) {
            double wv[kMaxPerLane];
            const double byl = by[l];
#pragma unroll
            for (int q = 0; q < kMaxPerLane; ++q) {
                const int lp = lane + 32 * q;
                wv[q] = (lp < nb && lp != l) ? B.D[B.pid(l, lp)] * (by[lp] - byl) : 0.0;
            }
            for (int e = lane; e < n * n; e += 32) Mw[e] = B.Lf[(size_t)l * n * n + e];
            for (int d = 0; d < n; ++d) {
                double v = 0.0;
#pragma unroll
                for (int q = 0; q < kMaxPerLane; ++q) {
                    const int lp = lane + 32 * q;
                    if (lp < nb) v += wv[q] * B.delta(l, lp, d);
                }
                v = warp_sum(v);
                if (lane == 0) vw[d] = bxi[l * n + d] - v;
            }
            __syncwarp();
            chol_solve_warp(Mw, n, vw);
            for (int d = lane; d < n; d += 32) bxi[l * n + d] = vw[d];
            __syncwarp();
        }
    __syncthreads();
}

__global__ void __launch_bounds__(IT, 1) block_ipm_kernel(const BlockIpmParams p) {
    extern __shared__ double bsm[];
    // optional phase timing (thread 0, clock64): [0] factor, [1] solve, [2] A, [3] A^T, [4] total
    // and call counts (factorizations, solves, A / A^T products) for the work model
    unsigned long long pt[5] = {0, 0, 0, 0, 0}, pt0 = 0;
    unsigned cnt[4] = {0, 0, 0, 0};
    const unsigned long long tk0 = clock64();
#define PROF_BEGIN() do { if (p.prof && threadIdx.x == 0) pt0 = clock64(); } while (0)
#define PROF_END(c) do { ++cnt[c]; if (p.prof && threadIdx.x == 0) pt[c] += clock64() - pt0; } while (0)
    __shared__ double red[IT];
    const int nb = p.nbar, n = p.n, m = nb * (nb - 1);
    const int64_t blk = blockIdx.x;
    const int64_t row0 = blk * nb;                               // local rows of this block
    const int G = p.lgroup;
    double *Xs = bsm, *S = Xs + nb * n, *Mll = S + nb * nb, *Z = Mll + G * n * n, *Drow = Z + G * n * nb;
    double *g = p.scratch + (size_t)blk * p.scratch_per_block;
    const int ne = nb * (n + 1);
    double *s = g, *lam = s + m, *D = lam + m, *a = D + m, *dsa = a + m, *dla = dsa + m, *w = dla + m;
    double *eta = w + m, *eta0 = eta + ne, *rhs = eta0 + ne, *ds = rhs + ne, *tv = ds + ne;
    double *Lf = tv + ne;
    double *wact = Lf + (size_t)nb * n * n, *wla = wact + m, *wflag = wla + m;   // warm start (persists)
    // the last settled polish's factorization: [0] valid, [1] rho, [2] gamma, [3..) the Schur factor
    // S (its Mll factors are still in Lf unless a factorization ran since)
    double *fsave = wflag + 1;
    for (int e = threadIdx.x; e < nb * n; e += IT) Xs[e] = p.X64[(p.row0 + row0) * n + e];
    for (int k = threadIdx.x; k < nb; k += IT) {
        eta0[k] = p.y64[p.row0 + row0 + k];
        eta[k] = eta0[k];
    }
    for (int e = threadIdx.x; e < nb * n; e += IT) {
        eta0[nb + e] = p.Xi64[row0 * n + e];
        eta[nb + e] = eta0[nb + e];
    }
    __syncthreads();
    Blk B{nb, n, p.gamma, Xs, S, Mll, Z, Lf, D, red, Drow, G};
    double *ey = eta, *exi = eta + nb, *ry = rhs, *rxi = rhs + nb;
    // sc: the data scale of this projection (thresholds below are relative to it)
    PROF_BEGIN(); apply_A(B, ey, exi, a); PROF_END(2);
    __syncthreads();
    double amax = 0.0;
    for (int q = threadIdx.x; q < m; q += IT) amax = fmax(amax, fabs(a[q]));
    amax = block_reduce(amax, red, true);
    const double sc = fmax(1.0, amax);
    // ---- polish: solve the equality-constrained projection on a guessed active set exactly by
    // the method of multipliers, (G + rho A_a^T A_a) eta = G eta0 + A_a^T la, la <- la - rho A_a eta,
    // adding violated / dropping negative-multiplier constraints between rounds (a primal
    // active-set correction); settles only at a KKT point of the projection.  Active flags in
    // dla, multipliers in dsa (set by the caller); eta is overwritten only on success.
    bool polished = false;
    int rounds = 0, mult_iters = 0;
    double rho_last = 0.0;
    // reuse: the warm start's active set is exactly the one the saved factorization was made for
    // (a settled polish ends on an unchanged active set), so with the same rho and gamma the
    // first round needs no factorization
    auto polish = [&](bool reuse) {
        int a0 = 0;
        if (reuse) a0 = fsave[1] == 10.0 * kRho ? 1 : (fsave[1] == 100.0 * kRho ? 2 : 0);
        for (int round = 0; round < kPolishRounds && !polished; ++round) {
            rounds = round + 1;
            double lmax = 0.0;
            // penalty rho = kRho, escalated x10 (refactor) while the multiplier iteration stalls
            for (int attempt = round == 0 ? a0 : 0; attempt < kRhoAttempts; ++attempt) {
                const double rho = kRho * (attempt == 0 ? 1.0 : attempt == 1 ? 10.0 : 100.0);
                rho_last = rho;
                for (int q = threadIdx.x; q < m; q += IT) D[q] = rho * dla[q];
                if (reuse && round == 0 && attempt == a0) {
                    for (int e = threadIdx.x; e < nb * nb; e += IT) S[e] = fsave[3 + e];
                    __syncthreads();
                } else {
                    __syncthreads();
                    if (threadIdx.x == 0) fsave[0] = 0.0;                // Lf is about to change
                    PROF_BEGIN(); factor(B); PROF_END(0);
                }
                bool conv = false;
                for (int r = 0; r < kPolishIters; ++r) {
                    PROF_BEGIN(); apply_AT(B, dsa, ry, rxi); PROF_END(3);
                    __syncthreads();
                    for (int k = threadIdx.x; k < ne; k += IT) rhs[k] += (k < nb ? 1.0 : p.gamma) * eta0[k];
                    __syncthreads();
                    PROF_BEGIN(); solve(B, ry, rxi, tv); PROF_END(1);
                    PROF_BEGIN(); apply_A(B, ry, rxi, a); PROF_END(2);
                    __syncthreads();
                    double cm = 0.0, lm = 0.0;
                    for (int q = threadIdx.x; q < m; q += IT)
                        if (dla[q] != 0.0) {
                            dsa[q] -= rho * a[q];
                            cm = fmax(cm, fabs(a[q]));
                            lm = fmax(lm, fabs(dsa[q]));
                        }
                    cm = block_reduce(cm, red, true);
                    lmax = block_reduce(lm, red, true);
                    mult_iters = max(mult_iters, r + 1);
                    if (cm <= 1e-13 * sc) { conv = true; break; }
                }
                if (conv) break;
            }
            // a = A eta of the last solve (all pairs): violated inactive / negative active constraints
            int changed = 0;
            for (int q = threadIdx.x; q < m; q += IT) {
                if (dla[q] == 0.0 && a[q] < -1e-12 * sc) { dla[q] = 1.0; changed = 1; }
                else if (dla[q] != 0.0 && dsa[q] < -1e-14 * fmax(1.0, lmax)) { dla[q] = 0.0; dsa[q] = 0.0; changed = 1; }
                if (dsa[q] < 0.0) dsa[q] = 0.0;
            }
            changed = __syncthreads_or(changed);
            if (!changed) {
                polished = true;
                for (int k = threadIdx.x; k < ne; k += IT) eta[k] = rhs[k];
            }
            __syncthreads();
        }
    };
    // 1) warm start: the previous Step 1's active set and multipliers (blocks move little between
    //    P-APG iterations), verified by the polish itself
    const bool warm = p.warm && wflag[0] != 0.0;
    if (warm) {
        const bool reuse = fsave[0] != 0.0 && fsave[2] == p.gamma &&
                           (fsave[1] == kRho || fsave[1] == 10.0 * kRho || fsave[1] == 100.0 * kRho);
        for (int q = threadIdx.x; q < m; q += IT) { dla[q] = wact[q]; dsa[q] = wla[q]; }
        __syncthreads();
        polish(reuse);
    }
    // 2) otherwise the interior point method from s = max(A eta0, 0) + sc, lambda = sc / 100, then
    //    the polish from its active set {lambda > s}
    int it = 0;
    bool ipm_ok = true;
    if (!polished) {
        rounds = 0;
        if (warm) {                                       // the failed polish left A eta in a
            PROF_BEGIN(); apply_A(B, ey, exi, a); PROF_END(2);
            __syncthreads();
        }
        for (int q = threadIdx.x; q < m; q += IT) {
            s[q] = fmax(a[q], 0.0) + sc;
            lam[q] = sc * 1e-2;
        }
        __syncthreads();
        for (; it < p.max_iter; ++it) {
            // residuals: r_p = A eta - s (in a), r_d = G (eta - eta0) - A^T lambda (in rhs, negated below)
            PROF_BEGIN(); apply_A(B, ey, exi, a); PROF_END(2);
            PROF_BEGIN(); apply_AT(B, lam, ry, rxi); PROF_END(3);
            __syncthreads();
            double mu = 0.0, cmax = 0.0, rp = 0.0, rdn = 0.0;
            for (int q = threadIdx.x; q < m; q += IT) {
                a[q] -= s[q];
                mu += s[q] * lam[q];
                cmax = fmax(cmax, s[q] * lam[q]);
                rp = fmax(rp, fabs(a[q]));
                D[q] = lam[q] / s[q];
            }
            for (int k = threadIdx.x; k < nb * (n + 1); k += IT) {
                const double gk = k < nb ? 1.0 : p.gamma;
                const double rd = gk * (eta[k] - eta0[k]) - rhs[k];
                rhs[k] = rd;                                  // r_d
                rdn = fmax(rdn, fabs(rd));
            }
            mu = block_reduce(mu, red, false) / m;
            cmax = block_reduce(cmax, red, true);
            rp = block_reduce(rp, red, true);
            rdn = block_reduce(rdn, red, true);
            if (!isfinite(mu) || !isfinite(rdn) || !isfinite(rp)) { it = p.max_iter; break; }
            if (cmax <= p.tol * sc * sc && rp <= p.tol * sc && rdn <= p.tol * sc) break;
            PROF_BEGIN(); factor(B); PROF_END(0);
            // ---- predictor: w = -lambda - D r_p ; rhs_aff = -r_d + A^T w
            for (int q = threadIdx.x; q < m; q += IT) w[q] = -lam[q] - D[q] * a[q];
            __syncthreads();
            PROF_BEGIN(); apply_AT(B, w, tv, tv + nb); PROF_END(3);
            __syncthreads();
            for (int k = threadIdx.x; k < nb * (n + 1); k += IT) ds[k] = -rhs[k] + tv[k];
            __syncthreads();
            PROF_BEGIN(); solve(B, ds, ds + nb, tv); PROF_END(1);                        // ds[0 .. nb (n+1)) = d eta_aff
            PROF_BEGIN(); apply_A(B, ds, ds + nb, dsa); PROF_END(2);                     // A d eta
            __syncthreads();
            double ap = 1.0, ad = 1.0;
            for (int q = threadIdx.x; q < m; q += IT) {
                dsa[q] += a[q];                               // ds_aff = A d eta + r_p
                dla[q] = w[q] - D[q] * (dsa[q] - a[q]);       // dl_aff = w - D A d eta
                if (dsa[q] < 0) ap = fmin(ap, -s[q] / dsa[q]);
                if (dla[q] < 0) ad = fmin(ad, -lam[q] / dla[q]);
            }
            ap = -block_reduce(-ap, red, true);
            ad = -block_reduce(-ad, red, true);
            double mua = 0.0;
            for (int q = threadIdx.x; q < m; q += IT) mua += (s[q] + ap * dsa[q]) * (lam[q] + ad * dla[q]);
            mua = block_reduce(mua, red, false) / m;
            const double sigma = fmin(1.0, pow(mua / mu, 3.0));
            // ---- corrector: w = -lambda + sigma mu / s - D r_p - ds_aff dl_aff / s
            for (int q = threadIdx.x; q < m; q += IT) w[q] = -lam[q] + (sigma * mu - dsa[q] * dla[q]) / s[q] - D[q] * a[q];
            __syncthreads();
            PROF_BEGIN(); apply_AT(B, w, tv, tv + nb); PROF_END(3);
            __syncthreads();
            for (int k = threadIdx.x; k < nb * (n + 1); k += IT) ds[k] = -rhs[k] + tv[k];
            __syncthreads();
            PROF_BEGIN(); solve(B, ds, ds + nb, tv); PROF_END(1);
            PROF_BEGIN(); apply_A(B, ds, ds + nb, dsa); PROF_END(2);
            __syncthreads();
            ap = 1.0;
            ad = 1.0;
            for (int q = threadIdx.x; q < m; q += IT) {
                const double dsq = dsa[q] + a[q];
                const double dlq = w[q] - D[q] * dsa[q];
                dsa[q] = dsq;
                dla[q] = dlq;
                if (dsq < 0) ap = fmin(ap, -s[q] / dsq);
                if (dlq < 0) ad = fmin(ad, -lam[q] / dlq);
            }
            ap = fmin(1.0, 0.995 * (-block_reduce(-ap, red, true)));
            ad = fmin(1.0, 0.995 * (-block_reduce(-ad, red, true)));
            for (int q = threadIdx.x; q < m; q += IT) {
                s[q] += ap * dsa[q];
                lam[q] += ad * dla[q];
            }
            for (int k = threadIdx.x; k < nb * (n + 1); k += IT) eta[k] += ap * ds[k];
            __syncthreads();
        }

        ipm_ok = it < p.max_iter;
        if (ipm_ok) {
            for (int q = threadIdx.x; q < m; q += IT) {
                const bool act = lam[q] > s[q];
                dla[q] = act ? 1.0 : 0.0;
                dsa[q] = act ? lam[q] : 0.0;
            }
            __syncthreads();
            polish(false);
        }
    }
    if (polished && p.warm) {
        for (int q = threadIdx.x; q < m; q += IT) { wact[q] = dla[q]; wla[q] = dsa[q]; }
        // smem S / Lf hold the factorization of the final (unchanged) active set at rho_last
        for (int e = threadIdx.x; e < nb * nb; e += IT) fsave[3 + e] = S[e];
        __syncthreads();
        if (threadIdx.x == 0) {
            wflag[0] = 1.0;
            fsave[1] = rho_last;
            fsave[2] = p.gamma;
            fsave[0] = 1.0;
        }
    } else if (threadIdx.x == 0) {
        fsave[0] = 0.0;
    }
    for (int k = threadIdx.x; k < nb; k += IT) p.y64[p.row0 + row0 + k] = eta[k];
    for (int e = threadIdx.x; e < nb * n; e += IT) p.Xi64[row0 * n + e] = eta[nb + e];
    if (p.prof && threadIdx.x == 0) {
        pt[4] = clock64() - tk0;
        for (int c = 0; c < 5; ++c) p.prof[8 * blk + c] = pt[c];
    }
    if (threadIdx.x == 0) {
        // [0] IPM iterations, [1] polish rounds, [2] max multiplier iterations in a round,
        // [3] status: 0 ok, 1 IPM failed (limit / non-finite), 2 polish did not settle,
        // [4] 1 if the warm start settled (no IPM run)
        p.iters[8 * blk + 0] = it;
        p.iters[8 * blk + 1] = rounds;
        p.iters[8 * blk + 2] = mult_iters;
        p.iters[8 * blk + 3] = !ipm_ok ? 1 : (!polished ? 2 : 0);
        p.iters[8 * blk + 4] = (warm && it == 0 && polished) ? 1 : 0;
        p.work[3 * blk + 0] += cnt[0];                   // cumulative since cr_init
        p.work[3 * blk + 1] += cnt[1];
        p.work[3 * blk + 2] += cnt[2] + cnt[3];
    }
}

}  // namespace

int block_ipm_group(int nbar, int n, size_t smem_max) {
    const size_t fixed = 8 * ((size_t)nbar * n + (size_t)nbar * nbar);
    const size_t per = 8 * ((size_t)n * n + (size_t)n * nbar + nbar);
    if (fixed + per > smem_max) return 0;
    return (int)std::min<size_t>(NW, (smem_max - fixed) / per);
}

size_t block_ipm_smem(int nbar, int n, int G) {
    return 8 * ((size_t)nbar * n + (size_t)nbar * nbar + (size_t)G * ((size_t)n * n + (size_t)n * nbar + nbar));
}

size_t block_ipm_scratch_per_block(int nbar, int n) {
    const size_t m = (size_t)nbar * (nbar - 1);
    return 7 * m + 5 * (size_t)nbar * (n + 1) + (size_t)nbar * n * n + 2 * m + 1 + 3 + (size_t)nbar * nbar;
}

cudaError_t block_ipm_prepare(int smem) {
    return cudaFuncSetAttribute(block_ipm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

cudaError_t launch_block_ipm(const BlockIpmParams &p, cudaStream_t s) {
    if (p.nblocks <= 0) return cudaSuccess;
    block_ipm_kernel<<<(unsigned)p.nblocks, IT, (size_t)p.smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace cr

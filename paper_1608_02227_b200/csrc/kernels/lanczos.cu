// L_gamma = sigma_max(C)^2 / gamma (Eq. (lischitz)) on the device: the same plain
// Lanczos as csrc/lanczos.cpp (three-term recurrence, no re-orthogonalisation, identical
// splitmix64 start vector), with the structured O(N n^2) product of C^T C (see lanczos.cpp for
// the derivation) and every reduction in a fixed order (deterministic: all ranks agree).
// The host keeps the tridiagonal (alpha, beta) and the Ritz bisection.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>
#include "../cr_internal.h"

namespace cr {
namespace {

constexpr int LB = 256;

// fixed-order block reduction of one value per thread (blockDim = LB)
__device__ __forceinline__ double block_sum(double v, double *sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = LB / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// S2[d][e] = sum_l X[l][d] X[l][e] (one block per (d, e)); s[d] = sum_l X[l][d] (e == n slot)
__global__ void __launch_bounds__(LB) lz_gram_kernel(const double *X, int64_t N, int n, double *S2, double *s) {
    __shared__ double sh[LB];
    const int d = blockIdx.x / (n + 1), e = blockIdx.x % (n + 1);
    double acc = 0.0;
    for (int64_t l = threadIdx.x; l < N; l += LB) acc += X[l * n + d] * (e < n ? X[l * n + e] : 1.0);
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        if (e < n) S2[(size_t)d * n + e] = acc;
        else s[d] = acc;
    }
}

constexpr int LQ = 4;                 // feature slots per lane: n <= 128
constexpr int LW = LB / 32;           // warps per block
constexpr int LROWS = 64;             // rows per block in the per-row kernels

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// per-block partials of Y = sum y, Sa = sum a, Sxi[d] = sum xi_d, w[d] = sum y x_d; a_k = xi_k.x_k.
// Warp per row (lanes over d, coalesced), rows [b LROWS, (b+1) LROWS) of block b, warp w taking
// rows w, w + LW, ...; warps combined in order.  part layout per block: [Y, Sa, Sxi[0..n), w[0..n)]
__global__ void __launch_bounds__(LB) lz_sums_kernel(const double *X, int64_t N, int n, const double *v, double *a,
                                                     double *part) {
    __shared__ double sh[LW][2 + 2 * 32 * LQ];
    const double *y = v, *xi = v + N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double Y = 0.0, Sa = 0.0, Sx[LQ], W[LQ];
#pragma unroll
    for (int q = 0; q < LQ; ++q) { Sx[q] = 0.0; W[q] = 0.0; }
    const int64_t r0 = (int64_t)blockIdx.x * LROWS, r1 = min(N, r0 + LROWS);
    for (int64_t k = r0 + warp; k < r1; k += LW) {
        const double yk = y[k];
        double ak = 0.0;
#pragma unroll
        for (int q = 0; q < LQ; ++q) {
            const int d = lane + 32 * q;
            if (d < n) {
                const double xv = X[k * n + d], xiv = xi[k * n + d];
                ak += xiv * xv;
                Sx[q] += xiv;
                W[q] += yk * xv;
            }
        }
        ak = warp_sum(ak);
        if (lane == 0) a[k] = ak;
        Y += yk;
        Sa += ak;
    }
    if (lane == 0) { sh[warp][0] = Y; sh[warp][1] = Sa; }
#pragma unroll
    for (int q = 0; q < LQ; ++q) {
        const int d = lane + 32 * q;
        if (d < n) { sh[warp][2 + d] = Sx[q]; sh[warp][2 + n + d] = W[q]; }
    }
    __syncthreads();
    double *out = part + (size_t)blockIdx.x * (2 + 2 * n);
    for (int qq = threadIdx.x; qq < 2 + 2 * n; qq += LB) {
        double r = 0.0;
        for (int w = 0; w < LW; ++w) r += sh[w][qq];
        out[qq] = r;
    }
}

// fixed-order sum of the block partials -> tot [2 + 2n]: one block per output value, threads
// over the partials (strided), then a fixed tree
__global__ void __launch_bounds__(LB) lz_sums_final_kernel(const double *part, int nb, int n, double *tot) {
    __shared__ double sh[LB];
    const int q = blockIdx.x;
    double r = 0.0;
    for (int b = threadIdx.x; b < nb; b += LB) r += part[(size_t)b * (2 + 2 * n) + q];
    r = block_sum(r, sh);
    if (threadIdx.x == 0) tot[q] = r;
}

// out = C^T C v (lanczos.cpp CtC::apply), warp per LR rows (lanes over d); S2 is symmetric, so
// lane d reads S2[e][d] (coalesced) for t_d = sum_e S2[d][e] xi_k[e], each S2 element serving
// the warp's LR rows
constexpr int LR = 4;
__global__ void __launch_bounds__(LB) lz_apply_kernel(const double *X, int64_t N, int n, const double *S2,
                                                      const double *s, const double *v, const double *a,
                                                      const double *tot, double *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k0 = ((int64_t)blockIdx.x * LW + warp) * LR;
    if (k0 >= N) return;
    const double *y = v, *xi = v + N;
    const double Y = tot[0], Sa = tot[1];
    const double *Sxi = tot + 2, *w = tot + 2 + n;
    const double Nd = (double)N;
    double xik[LR][LQ], t[LR][LQ], sd[LQ];
#pragma unroll
    for (int q = 0; q < LQ; ++q) {
        const int d = lane + 32 * q;
        sd[q] = d < n ? s[d] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < LR; ++r) {
        const int64_t k = k0 + r;
#pragma unroll
        for (int q = 0; q < LQ; ++q) {
            const int d = lane + 32 * q;
            xik[r][q] = (k < N && d < n) ? xi[k * n + d] : 0.0;
            t[r][q] = 0.0;
        }
    }
#pragma unroll
    for (int qe = 0; qe < LQ; ++qe) {
        if (32 * qe >= n) break;
        for (int src = 0; src < 32; ++src) {
            const int e = 32 * qe + src;
            if (e >= n) break;
            double xe[LR];
#pragma unroll
            for (int r = 0; r < LR; ++r) xe[r] = __shfl_sync(0xffffffffu, xik[r][qe], src);
            const double *row = S2 + (size_t)e * n;
#pragma unroll
            for (int q = 0; q < LQ; ++q) {
                const int d = lane + 32 * q;
                if (d < n) {
                    const double sv = row[d];
#pragma unroll
                    for (int r = 0; r < LR; ++r) t[r][q] += sv * xe[r];
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < LR; ++r) {
        const int64_t k = k0 + r;
        if (k >= N) break;
        double xk[LQ], xs = 0.0, sx = 0.0;
#pragma unroll
        for (int q = 0; q < LQ; ++q) {
            const int d = lane + 32 * q;
            xk[q] = d < n ? X[k * n + d] : 0.0;
            xs += xik[r][q] * sd[q];
            sx += (d < n ? Sxi[d] : 0.0) * xk[q];
        }
        xs = warp_sum(xs);
        sx = warp_sum(sx);
        const double yk = y[k], ak = a[k];
        const double rho = Y - Nd * yk + Nd * ak - xs;
        if (lane == 0) out[k] = 2.0 * Nd * yk - 2.0 * Y + Sa - sx - Nd * ak + xs;
        double *ok = out + N + k * n;
#pragma unroll
        for (int q = 0; q < LQ; ++q) {
            const int d = lane + 32 * q;
            if (d < n) ok[d] = xk[q] * rho - w[d] + (yk - ak) * sd[q] + t[r][q];
        }
    }
}

// per-block partial of dot(a, b)
__global__ void __launch_bounds__(LB) lz_dot_kernel(const double *a, const double *b, int64_t m, double *part) {
    __shared__ double sh[LB];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < m; i += (int64_t)gridDim.x * LB) acc += a[i] * b[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// w -= alpha v + beta vprev, per-block partial of |w|^2
__global__ void __launch_bounds__(LB) lz_update_kernel(double *w, const double *v, const double *vprev, int64_t m,
                                                       const double *alpha, const double *beta_prev, double *part) {
    __shared__ double sh[LB];
    const double al = *alpha, bp = *beta_prev;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < m; i += (int64_t)gridDim.x * LB) {
        const double t = w[i] - (al * v[i] + bp * vprev[i]);
        w[i] = t;
        acc += t * t;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// fixed-order sum of nb partials (one block of LB threads: strided partial sums, then a tree)
__global__ void __launch_bounds__(LB) lz_final_kernel(const double *part, int nb, double *dst, int take_sqrt) {
    __shared__ double sh[LB];
    double r = 0.0;
    for (int b = threadIdx.x; b < nb; b += LB) r += part[b];
    r = block_sum(r, sh);
    if (threadIdx.x == 0) *dst = take_sqrt ? sqrt(r) : r;
}

// vprev <- v, v <- w / b
__global__ void lz_shift_kernel(double *v, double *vprev, const double *w, int64_t m, const double *b) {
    const double inv_b = 1.0 / *b;
    for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < m; i += (int64_t)gridDim.x * LB) {
        vprev[i] = v[i];
        v[i] = w[i] * inv_b;
    }
}

// Start vector on the device: the host Lanczos's splitmix64 sequence (value i = mix(seed + (i+1)
// golden), counter-based, so every entry is computed independently), then unit-normalized with
// the fixed-order device reductions (the norm's summation order differs from the host loop's, so
// L agrees with the host Lanczos to rounding, not bit for bit).  Generating and copying the 5.3M
// entries of C5's start vector on the host cost ~25 ms of cr_init.
__global__ void lz_start_kernel(double *v, int64_t m, uint64_t seed) {
    for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < m; i += (int64_t)gridDim.x * LB) {
        uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
}
__global__ void lz_scale_kernel(double *v, int64_t m, const double *nrm) {
    const double inv = 1.0 / *nrm;
    for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < m; i += (int64_t)gridDim.x * LB) v[i] *= inv;
}

}  // namespace

// sigma_max(C)^2 by device Lanczos.  X: device [N][n] fp64.  Scratch is stream-ordered
// (cudaMallocAsync).  The start vector is generated on the device (lz_start_kernel).  Returns < 0 on
// a CUDA error (then *err holds it).
double sigma_max_sq_lanczos_device(int64_t N, int n, const double *X, double tol, int max_iter, cudaStream_t st,
                                   cudaError_t *err, void *scratch, size_t scratch_bytes) {
    const int64_t m = N * (int64_t)(n + 1);
    const int nbk = (int)((N + LROWS - 1) / LROWS);           // lz_sums blocks
    const int nba = (int)((N + (int64_t)LW * LR - 1) / ((int64_t)LW * LR));   // lz_apply blocks (warp per LR rows)
    const int nbv = (int)std::min<int64_t>((m + LB - 1) / LB, 1024);
    const int itmax = (int)std::min<int64_t>(max_iter, m);
    double *S2 = nullptr, *s = nullptr, *v = nullptr, *vp = nullptr, *w = nullptr, *a = nullptr, *part = nullptr,
           *tot = nullptr, *ab = nullptr;
    auto ok = [&](cudaError_t e) { if (e != cudaSuccess && *err == cudaSuccess) *err = e; return e == cudaSuccess; };
    *err = cudaSuccess;
    const size_t npart = std::max<size_t>((size_t)nbk * (2 + 2 * n), (size_t)nbv);
    // the caller's scratch when it is large enough (cr_init passes the not-yet-used Theta
    // buffers: no allocation in the init path), else stream-ordered allocations
    const size_t nS2 = (size_t)n * n + n, nv = 3 * (size_t)m, na = (size_t)N, ntot = 2 + 2 * (size_t)n,
                 nab = 2 * (size_t)itmax + 1;
    const size_t need = sizeof(double) * (nS2 + nv + na + npart + ntot + nab);
    const bool own = !(scratch && scratch_bytes >= need);
    if (!own) {
        double *q = static_cast<double *>(scratch);
        S2 = q; q += nS2;
        v = q; q += nv;
        a = q; q += na;
        part = q; q += npart;
        tot = q; q += ntot;
        ab = q;
    } else {
        ok(cudaMallocAsync(&S2, sizeof(double) * nS2, st));
        ok(cudaMallocAsync(&v, sizeof(double) * nv, st));
        ok(cudaMallocAsync(&a, sizeof(double) * na, st));
        ok(cudaMallocAsync(&part, sizeof(double) * npart, st));
        ok(cudaMallocAsync(&tot, sizeof(double) * ntot, st));
        ok(cudaMallocAsync(&ab, sizeof(double) * nab, st));   // alpha[it], beta[it], 0
    }
    double result = -1.0;
    if (*err == cudaSuccess) {
        s = S2 + (size_t)n * n;
        vp = v + m;
        w = vp + m;
        double *al_d = ab, *be_d = ab + itmax, *zero_d = ab + 2 * itmax;
        lz_start_kernel<<<nbv, LB, 0, st>>>(v, m, 0x1608022270000001ull);
        lz_dot_kernel<<<nbv, LB, 0, st>>>(v, v, m, part);
        lz_final_kernel<<<1, LB, 0, st>>>(part, nbv, tot, 1);
        lz_scale_kernel<<<nbv, LB, 0, st>>>(v, m, tot);
        ok(cudaMemsetAsync(vp, 0, sizeof(double) * m, st));
        ok(cudaMemsetAsync(zero_d, 0, sizeof(double), st));
        lz_gram_kernel<<<n * (n + 1), LB, 0, st>>>(X, N, n, S2, s);
        ok(cudaGetLastError());
        // The recurrence runs on the device in chunks of kChunk iterations (alpha, beta kept in
        // device memory); after each chunk the host replays the stopping logic of the host
        // Lanczos iteration by iteration on the copied (alpha, beta), so L is the same as
        // stepping with a host round trip per iteration (iterations past the stop are unused).
        constexpr int kChunk = 8;
        std::vector<double> al, be, hab(2 * (size_t)itmax);
        double prev = 0.0;
        int stable = 0, it = 0, done = 0;
        bool stop = false;
        while (!stop && it < itmax && *err == cudaSuccess) {
            const int end = std::min(itmax, it + kChunk);
            for (; it < end; ++it) {
                lz_sums_kernel<<<nbk, LB, 0, st>>>(X, N, n, v, a, part);
                lz_sums_final_kernel<<<2 + 2 * n, LB, 0, st>>>(part, nbk, n, tot);
                lz_apply_kernel<<<nba, LB, 0, st>>>(X, N, n, S2, s, v, a, tot, w);
                lz_dot_kernel<<<nbv, LB, 0, st>>>(w, v, m, part);
                lz_final_kernel<<<1, LB, 0, st>>>(part, nbv, al_d + it, 0);
                lz_update_kernel<<<nbv, LB, 0, st>>>(w, v, vp, m, al_d + it, it > 0 ? be_d + it - 1 : zero_d, part);
                lz_final_kernel<<<1, LB, 0, st>>>(part, nbv, be_d + it, 1);
                lz_shift_kernel<<<nbv, LB, 0, st>>>(v, vp, w, m, be_d + it);
            }
            ok(cudaGetLastError());
            ok(cudaMemcpyAsync(hab.data(), al_d, sizeof(double) * it, cudaMemcpyDeviceToHost, st));
            ok(cudaMemcpyAsync(hab.data() + itmax, be_d, sizeof(double) * it, cudaMemcpyDeviceToHost, st));
            ok(cudaStreamSynchronize(st));
            for (; done < it && !stop; ++done) {
                al.push_back(hab[done]);
                const double theta = lanczos_max_ritz(al.data(), be.data(), (int)al.size());
                result = theta;
                if (done > 2 && std::fabs(theta - prev) <= tol * std::fabs(theta)) {
                    if (++stable >= 3) { stop = true; break; }
                } else {
                    stable = 0;
                }
                prev = theta;
                const double b = hab[itmax + done];
                if (b <= 1e-14 * std::fabs(theta)) { stop = true; break; }
                be.push_back(b);
            }
        }
    }
    if (own) {
        cudaFreeAsync(S2, st);
        cudaFreeAsync(v, st);
        cudaFreeAsync(a, st);
        cudaFreeAsync(part, st);
        cudaFreeAsync(tot, st);
        cudaFreeAsync(ab, st);
    }
    ok(cudaStreamSynchronize(st));
    return *err == cudaSuccess ? result : -1.0;
}

}  // namespace cr

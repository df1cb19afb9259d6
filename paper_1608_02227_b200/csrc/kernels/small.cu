// O(N n) kernels around the fused pass (the residual pass of cr_primal is kernels/residual.cu).
//
//   prologue   : Step 1 of Fig. 2 in closed form at K = N, from the linear sums
//                S = (r, c, Theta X) of Theta^{k-1} and Theta^{k-2}:
//                  S~ = S^{k-1} + beta_{k-1} (S^{k-1} - S^{k-2})      (Step 4 is linear)
//                  y_i  = ybar_i + c~_i - r~_i                          (A1^T theta, Def. A1A2)
//                  xi_i = (r~_i x_i - (Theta~ X)_i) / gamma             (A2^T theta / gamma)
//                  a_i  = xi_i . x_i
//                all in fp64; writes the storage-precision operands of the pass
//                (y' = y s, b' = (a - y) s, xi' = xi s with s = 1/L) and fp64 masters.
//   reduce     : fixed-order fp64 sums of the pass's row / column partials -> S^k; t update.
//   stats      : finalize of the prologue and residual partials.

#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include "../cr_internal.h"

namespace cr {
namespace {

// CR_FLAG_P2P all-gather of y': one row's value to every rank's receive array (peer stores) ...
template <typename T>
__device__ __forceinline__ void p2p_ypush_row(void *const *yrecv, int W, int64_t gi, T v) {
    for (int q = 0; q < W; ++q) static_cast<T *>(yrecv[q])[gi] = v;
}
// ... and, once per CTA after its rows, the row count to every rank's arrival counter
__device__ __forceinline__ void p2p_ysignal(unsigned long long *const *yflag, int W, int rank, unsigned long long cnt) {
    __threadfence_system();
    for (int q = 0; q < W; ++q) atomicAdd_system(yflag[q] + rank, cnt);
}

// One warp per row (grid-stride), lanes over the n features: coalesced fp64 reads of the
// sums, coalesced writes of xi; a_i by a fixed-order warp reduction.  Per-block partials of
// |u|^2, u.ybar, |xi|^2 and a nonfinite flag go to statpart (fixed order: deterministic).
// Latency: the row's static inputs (x_i, ybar_i) and the sums of Theta^{k-2} (written three
// launches back) are loaded before the programmatic-dependency wait, and each warp keeps the
// next row's loads in flight while it computes the current one.
// kPQ feature chunks of 32 per lane: n <= 32 kPQ (instantiated for 1, 2, 3: cr_max_dim 80)
template <int kPQ>
struct ProRow {
    double r1, r2, c1, c2, yb;
    double P1[kPQ], P2[kPQ], x[kPQ];
};

template <typename T, int kPQ>
__global__ void __launch_bounds__(256, kPQ == 1 ? 3 : 2) prologue_kernel(const SmallParams p) {
    __shared__ double red[4][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = p.n;
    const int64_t stride = (int64_t)gridDim.x * 8;
    int64_t i = (int64_t)blockIdx.x * 8 + warp;
    double u2 = 0.0, uy = 0.0, xi2 = 0.0, bad = 0.0;
    T *XiT = static_cast<T *>(p.XiT);
    auto load_static = [&](int64_t r, ProRow<kPQ> &d) {          // inputs final before this launch
        const int64_t gr = p.row0 + r;
        d.yb = p.ybar[gr];
        if (!p.from_eta) { d.r2 = p.r2[r]; d.c2 = p.c2[r]; }
#pragma unroll
        for (int q = 0; q < kPQ; ++q) {
            const int dd = lane + 32 * q;
            d.x[q] = dd < n ? p.X64[gr * n + dd] : 0.0;
            d.P2[q] = (!p.from_eta && dd < n) ? p.P2[r * n + dd] : 0.0;
        }
    };
    auto load_fresh = [&](int64_t r, ProRow<kPQ> &d) {           // written by the preceding reduce
        if (p.from_eta) {
            d.r1 = p.y64[p.row0 + r];
#pragma unroll
            for (int q = 0; q < kPQ; ++q) {
                const int dd = lane + 32 * q;
                d.P1[q] = dd < n ? p.Xi64[r * n + dd] : 0.0;
            }
            return;
        }
        d.r1 = p.r1[r];
        d.c1 = p.c1[r];
#pragma unroll
        for (int q = 0; q < kPQ; ++q) {
            const int dd = lane + 32 * q;
            d.P1[q] = dd < n ? p.P1[r * n + dd] : 0.0;
        }
    };
    ProRow<kPQ> cur, nxt;
    unsigned rows_pushed = 0;                               // (lane 0: rows sent over peer memory)
    if (i < p.Ns) load_static(i, cur);
    pdl_wait();
    pdl_trigger();
    const double beta = p.use_beta ? (p.ts->t_prev - 1.0) / p.ts->t_cur : 0.0;
    const double scale = p.s_dev ? 1.0 / *p.s_dev : p.scale;
    if (i < p.Ns) load_fresh(i, cur);
    for (; i < p.Ns; i += stride) {
        const int64_t in = i + stride;
        if (in < p.Ns) { load_static(in, nxt); load_fresh(in, nxt); }     // next row in flight
        const int64_t gi = p.row0 + i;
        double rt = 0.0, y, u;
        if (p.from_eta) {                               // projected Step-1 point (partition K < N)
            y = cur.r1;
            u = y - cur.yb;
        } else {
            rt = cur.r1 + beta * (cur.r1 - cur.r2);
            const double ct = cur.c1 + beta * (cur.c1 - cur.c2);
            u = ct - rt;                                // (A1^T theta~)_i
            y = cur.yb + u;
        }
        double a = 0.0, q2 = 0.0;
#pragma unroll
        for (int q = 0; q < kPQ; ++q) {
            const int d = lane + 32 * q;
            if (d >= n) continue;
            double xi;
            if (p.from_eta) {
                xi = cur.P1[q];
            } else {
                const double Pt = cur.P1[q] + beta * (cur.P1[q] - cur.P2[q]);
                xi = (rt * cur.x[q] - Pt) / p.gamma;    // (A2^T theta~)_i / gamma
                p.Xi64[i * n + d] = xi;
            }
            if (XiT) XiT[(int64_t)d * p.Rp + i] = T(xi * scale);
            if (p.XiR) p.XiR[i * p.NK + d] = (float)(xi * scale);
            a += xi * cur.x[q];
            q2 += xi * xi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            q2 += __shfl_xor_sync(0xffffffffu, q2, o);
        }
        if (lane == 0) {
            if (!p.from_eta) p.y64[gi] = y;
            p.a64[i] = a;
            static_cast<T *>(p.yv)[gi] = T(y * scale);
            if (p.p2p_push) {
                p2p_ypush_row<T>(p.p2p_yrecv, p.p2p_W, gi, T(y * scale));
                ++rows_pushed;
            }
            static_cast<T *>(p.bv)[i] = T((a - y) * scale);
            u2 += u * u;
            uy += u * cur.yb;
            xi2 += q2;
            bad += (isfinite(y) && isfinite(a)) ? 0.0 : 1.0;
        }
        cur = nxt;
    }
    __shared__ unsigned pushed[8];
    if (lane == 0) { red[0][warp] = u2; red[1][warp] = uy; red[2][warp] = xi2; red[3][warp] = bad; pushed[warp] = rows_pushed; }
    __syncthreads();
    if (p.p2p_push && threadIdx.x == 0) {
        unsigned long long cnt = 0;
        for (int w = 0; w < 8; ++w) cnt += pushed[w];
        if (cnt) p2p_ysignal(p.p2p_yflag, p.p2p_W, p.p2p_rank, cnt);
    }
    if (threadIdx.x < 4 && p.statpart) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
        p.statpart[blockIdx.x * 8 + threadIdx.x] = t;
    }
}

// Blocks [0, ncolb): column sums, 128 (fp32 partials, float4 per lane) or 32 (fp64) columns per
// block, 8 warps splitting the row-block range
// (fixed chunks, combined in order).  Remaining blocks: one warp per row, lanes over d <= n (+1),
// summing that row's run slots in a fixed order.  Every pass rewrites every column of the slots
// it owns, so the partials are read-only here.
// Column j's sum of this rank's partials: into c_out (NCCL / local reduce-scatter follows), or
// straight into its owner's receive slab over peer memory (CR_FLAG_P2P).
__device__ __forceinline__ void col_store(const ReduceParams &p, int64_t j, double v) {
    if (p.p2p_recv) {
        const int64_t q = j / p.p2p_S;
        p.p2p_recv[q][p.p2p_rank * p.p2p_S + (j - q * p.p2p_S)] = v;
    } else {
        p.c_out[j] = v;
    }
}

// One column block (128 columns of fp32 partials / 32 of fp64): fixed-order sums; with P2P the
// block then releases its arrival to the owner (system scope: the owner is another GPU).
template <typename Tc>
__device__ void colsum_block(const ReduceParams &p, int64_t cb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb0 = (int)((int64_t)p.nRB * warp / 8), rb1 = (int)((int64_t)p.nRB * (warp + 1) / 8);
    if constexpr (sizeof(Tc) == 4) {
        // fp32 partials: 128 columns per block, a float4 of 4 columns per lane, 4 row blocks
        // of loads in flight per lane
        __shared__ double cs4[8][128];
        const int64_t j = (int64_t)cb * 128 + 4 * lane;      // ldT % 4 == 0: in bounds
        const float *cp = static_cast<const float *>(p.colpart);
        double s[4] = {0.0, 0.0, 0.0, 0.0};
        if (j < p.N) {
            int rb = rb0;
            for (; rb + 4 <= rb1; rb += 4) {
                float4 v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const float4 *>(cp + (int64_t)(rb + k) * p.ldT + j);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    s[0] += (double)v[k].x; s[1] += (double)v[k].y; s[2] += (double)v[k].z; s[3] += (double)v[k].w;
                }
            }
            for (; rb < rb1; ++rb) {
                const float4 v = *reinterpret_cast<const float4 *>(cp + (int64_t)rb * p.ldT + j);
                s[0] += (double)v.x; s[1] += (double)v.y; s[2] += (double)v.z; s[3] += (double)v.w;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cs4[warp][4 * lane + q] = s[q];
        __syncthreads();
        if (threadIdx.x < 128) {
            const int64_t jj = (int64_t)cb * 128 + threadIdx.x;
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += cs4[w][threadIdx.x];
            if (jj < p.N) col_store(p, jj, t);
        }
    } else {
        __shared__ double cs[8][32];
        const int64_t j = (int64_t)cb * 32 + lane;
        const Tc *cp = static_cast<const Tc *>(p.colpart);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (j < p.N) {
            int rb = rb0;
            for (; rb + 4 <= rb1; rb += 4) {
                s0 += (double)cp[(int64_t)rb * p.ldT + j];
                s1 += (double)cp[(int64_t)(rb + 1) * p.ldT + j];
                s2 += (double)cp[(int64_t)(rb + 2) * p.ldT + j];
                s3 += (double)cp[(int64_t)(rb + 3) * p.ldT + j];
            }
            for (; rb < rb1; ++rb) s0 += (double)cp[(int64_t)rb * p.ldT + j];
        }
        cs[warp][lane] = (s0 + s1) + (s2 + s3);
        __syncthreads();
        if (warp == 0 && j < p.N) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += cs[w][lane];
            col_store(p, j, t);
        }
    }
    if (p.p2p_recv) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t q = cb * (sizeof(Tc) == 4 ? 128 : 32) / p.p2p_S;
            __threadfence_system();
            atomicAdd_system(p.p2p_flag[q] + p.p2p_rank, 1ULL);
        }
    }
}

__device__ __forceinline__ void reduce_row(const ReduceParams &p, int i, int lane);

template <typename Tc>
__global__ void __launch_bounds__(256, 4) reduce_kernel(const ReduceParams p, int ncolb) {
    pdl_wait();
    pdl_trigger();
    if ((int)blockIdx.x < ncolb) {
        colsum_block<Tc>(p, blockIdx.x);
    } else {
        // one warp per row, lanes over d <= n (32-bit index math: Ns < 2^31)
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int i = (int)(blockIdx.x - ncolb) * 8 + warp;
        if (i < p.Ns) reduce_row(p, i, lane);
    }
    if (p.advance_t && blockIdx.x == 0 && threadIdx.x == 0) {
        const double t = p.ts->t_cur;
        p.ts->t_prev = t;
        p.ts->t_cur = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;   // Step 3
    }
    if (p.yepoch && blockIdx.x == 0 && threadIdx.x == 0) *p.yepoch += 1;
}

// Row partial sums of one row (warp, lanes over d): the reduce's row half, shared by
// reduce_kernel and reduce_prologue_kernel (identical fixed order).
__device__ __forceinline__ void reduce_row(const ReduceParams &p, int i, int lane) {
    const int rb = i / p.rbm, ii = i - rb * p.rbm;
    const int e0 = p.rb_ptr[rb], ns = p.rb_ptr[rb + 1] - e0;
    const double *rp = p.rowpart;
    for (int base = 0; base < ns; base += 32) {
        const int m = min(32, ns - base);
        const int *ids = p.rb_slots + e0 + base;
        // virtual columns: d < n -> Theta X, d = n -> r, d = n + 1 -> ||D||^2 (adaptive)
        const int dmax = p.n + (p.dcol0 >= 0 ? 1 : 0);
        for (int d = lane; d <= dmax; d += 32) {
            const int col = d < p.n ? d : (d == p.n ? p.rcol0 : p.dcol0);
            const int col2 = d < p.n ? -1 : (d == p.n ? p.rcol1 : p.dcol1);
            const bool two = col2 >= 0;
            double *out = d < p.n ? p.P + (int64_t)i * p.n + d : (d == p.n ? p.r + i : p.dsq + i);
            double s = base == 0 ? 0.0 : *out;
            for (int q0 = 0; q0 < m; q0 += 4) {
                double v[4], w[4];
                const double *rows[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {           // 4 independent loads in flight
                    const bool ok = q0 + k < m;
                    const int sl = ok ? ids[q0 + k] : 0;
                    rows[k] = rp + ((int64_t)sl * p.rbm + ii) * p.NBP;
                    v[k] = ok ? rows[k][col] : 0.0;
                    w[k] = (ok && two) ? rows[k][col2] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (q0 + k < m) {
                        s += v[k];
                        if (two) s += w[k];
                    }
                }
            }
            *out = s;
        }
    }
}

// reduce (iteration k) + prologue (iteration k+1) for 32 rows per block, fp32 storage, one rank.
//   phase A: c_i for the block's 32 columns (= its rows): warp w sums row blocks
//            [nRB w / 8, nRB (w+1) / 8) of the fp32 column partials in order, lane = column, the
//            8 warp sums combined in warp order -- reduce_kernel's colsum_block order per column;
//            r_i, (Theta X)_i from the row-partial slots (reduce_row).
//   phase B: prologue_kernel's per-row Step 1 at theta~^{k+1} from S^k (phase A, read back after
//            the block barrier) and S^{k-1}.
// beta_k = (t_k - 1) / t_{k+1} is formed from t_k read at the start; the last block to arrive
// (after every block has read t_k) stores t_prev = t_k, t_cur = t_{k+1} (Step 3).
// RPB rows per block (32 or 8): the block's critical path is RPB / 8 row reductions + RPB / 8
// row prologues per warp, so small problems (few blocks) take RPB = 8 for more, shorter blocks
template <int kPQ, int RPB>
__global__ void __launch_bounds__(256) reduce_prologue_kernel(const ReduceParams rd, const SmallParams p) {
    constexpr int RPW = RPB / 8;                 // rows per warp
    __shared__ double cs[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = p.n;
    const int64_t i0 = (int64_t)blockIdx.x * RPB;
    // static inputs of the warp's 4 rows (final before this launch: X, ybar, S^{k-1})
    ProRow<kPQ> row[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int64_t r = i0 + warp * RPW + q;
        if (r < p.Ns) {
            row[q].yb = p.ybar[p.row0 + r];
            row[q].r2 = p.r2[r];
            row[q].c2 = p.c2[r];
#pragma unroll
            for (int qq = 0; qq < kPQ; ++qq) {
                const int dd = lane + 32 * qq;
                row[q].x[qq] = dd < n ? p.X64[(p.row0 + r) * n + dd] : 0.0;
                row[q].P2[qq] = dd < n ? p.P2[r * n + dd] : 0.0;
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    const double tk = p.ts->t_cur;
    const double tn = (1.0 + sqrt(1.0 + 4.0 * tk * tk)) / 2.0;   // Step 3
    const double beta = (tk - 1.0) / tn;                         // beta_k = (t_k - 1) / t_{k+1}
    // ---- phase A: column sums of the block's 32 columns, row sums of its 32 rows
    {
        const int rb0 = (int)((int64_t)rd.nRB * warp / 8), rb1 = (int)((int64_t)rd.nRB * (warp + 1) / 8);
        const int64_t j = i0 + lane;
        const float *cp = static_cast<const float *>(rd.colpart);
        double s = 0.0;
        if (lane < RPB && j < rd.N) {
            int rb = rb0;
            for (; rb + 4 <= rb1; rb += 4) {
                float v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = cp[(int64_t)(rb + k) * rd.ldT + j];
#pragma unroll
                for (int k = 0; k < 4; ++k) s += (double)v[k];
            }
            for (; rb < rb1; ++rb) s += (double)cp[(int64_t)rb * rd.ldT + j];
        }
        cs[warp][lane] = s;
    }
#pragma unroll 1
    for (int q = 0; q < RPW; ++q) {
        const int64_t r = i0 + warp * RPW + q;
        if (r < p.Ns) reduce_row(rd, (int)r, lane);
    }
    __syncthreads();
    if (warp == 0 && lane < RPB && i0 + lane < rd.N) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += cs[w][lane];
        rd.c_out[i0 + lane] = t;
    }
    __syncthreads();
    // ---- phase B: Step 1 for the warp's rows
    const double scale = p.scale;
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int64_t i = i0 + warp * RPW + q;
        if (i >= p.Ns) continue;
        ProRow<kPQ> &cur = row[q];
        cur.r1 = p.r1[i];
        cur.c1 = p.c1[i];
#pragma unroll
        for (int qq = 0; qq < kPQ; ++qq) {
            const int dd = lane + 32 * qq;
            cur.P1[qq] = dd < n ? p.P1[i * n + dd] : 0.0;
        }
        const int64_t gi = p.row0 + i;
        const double rt = cur.r1 + beta * (cur.r1 - cur.r2);
        const double ct = cur.c1 + beta * (cur.c1 - cur.c2);
        const double u = ct - rt;                                // (A1^T theta~)_i
        const double y = cur.yb + u;
        double a = 0.0;
#pragma unroll
        for (int qq = 0; qq < kPQ; ++qq) {
            const int d = lane + 32 * qq;
            if (d >= n) continue;
            const double Pt = cur.P1[qq] + beta * (cur.P1[qq] - cur.P2[qq]);
            const double xi = (rt * cur.x[qq] - Pt) / p.gamma;  // (A2^T theta~)_i / gamma
            p.Xi64[i * n + d] = xi;
            if (p.XiT) static_cast<float *>(p.XiT)[(int64_t)d * p.Rp + i] = (float)(xi * scale);
            if (p.XiR) p.XiR[i * p.NK + d] = (float)(xi * scale);
            a += xi * cur.x[qq];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) {
            p.y64[gi] = y;
            p.a64[i] = a;
            static_cast<float *>(p.yv)[gi] = (float)(y * scale);
            static_cast<float *>(p.bv)[i] = (float)((a - y) * scale);
        }
    }
    // ---- Step 3 by the last block (every block has read t_k by now)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long prev = atomicAdd(&p.ts->fuse_cnt, 1ULL);
        if (prev == gridDim.x - 1) {
            p.ts->t_prev = tk;
            p.ts->t_cur = tn;
            p.ts->fuse_cnt = 0ULL;
        }
    }
}

// Adaptive step check in quadratic form: one warp per row, lanes over d.
//   Dr = r_O - (r_A + beta (r_A - r_B)), Dc likewise, DP_d likewise  (sums of D = Theta^k - theta~)
//   q_i = (Dc_i - Dr_i)^2 + sum_d (Dr_i x_id - DP_id)^2 / gamma       ((A1^T D)_i^2 + |(A2^T D)_i|^2/gamma)
// Per-block partials of Q = sum q_i and ||D||^2 = sum dsq_i to statpart (fixed order).
__global__ void __launch_bounds__(256) adapt_check_kernel(const AdaptParams p) {
    __shared__ double red[2][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double beta = (p.ts->t_prev - 1.0) / p.ts->t_cur;
    double Q = 0.0, D2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < p.Ns; i += (int64_t)gridDim.x * 8) {
        const double dr = p.rO[i] - (p.rA[i] + beta * (p.rA[i] - p.rB[i]));
        const double dc = p.cO[i] - (p.cA[i] + beta * (p.cA[i] - p.cB[i]));
        const double *x = p.X64 + (p.row0 + i) * p.n;
        double q = 0.0;
        for (int d = lane; d < p.n; d += 32) {
            const int64_t e = i * p.n + d;
            const double dP = p.PO[e] - (p.PA[e] + beta * (p.PA[e] - p.PB[e]));
            const double a2 = dr * x[d] - dP;
            q += a2 * a2;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) {
            const double a1 = dc - dr;
            Q += a1 * a1 + q / p.gamma;
            D2 += p.dsq[i];
        }
    }
    if (lane == 0) { red[0][warp] = Q; red[1][warp] = D2; }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
        p.statpart[blockIdx.x * 8 + threadIdx.x] = t;
    }
}

// Accept / retry: the trial at s = ad[STRY] passes iff Q <= s ||D||^2 (the quadratic
// form of Eq. (adaptive-check), R15; a non-finite trial fails).  Accept: s_k = s,
// Step 3, next iteration starts at l = 0 with s_{k} / ups.  Reject: l += 1, s *= ups.
__global__ void adapt_decide_kernel(DevScalars *ts, cudaGraphConditionalHandle cond, int has_cond) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double *ad = ts->ad;
    if (ad[AD_ERR] != 0.0) {                // an earlier iteration exhausted its trials: the
        if (has_cond) cudaGraphSetConditional(cond, 0u);   // context is poisoned, change nothing
        return;
    }
    const double Q = ts->stats[8], D = ts->stats[9], s = ad[AD_STRY];
    const bool ok = isfinite(Q) && isfinite(D) && Q <= s * D;
    bool more;
    if (ok) {
        const double t = ts->t_cur;
        ts->t_prev = t;
        ts->t_cur = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        ad[AD_S] = s;
        ad[AD_TLAST] = ad[AD_L] + 1.0;
        ad[AD_TTOT] += ad[AD_L] + 1.0;
        ad[AD_L] = 0.0;
        // next iteration's first trial: s_{k-1} ups^(l-1) at l = 0, or s_{k-1} (monotone)
        ad[AD_STRY] = ad[AD_MONO] != 0.0 ? s : s * pow(ad[AD_UPS], -1.0);
        more = false;
    } else {
        ad[AD_L] += 1.0;
        // formed afresh from s_{k-1}, as the oracle does
        ad[AD_STRY] = ad[AD_S] * pow(ad[AD_UPS], ad[AD_L] - (ad[AD_MONO] != 0.0 ? 0.0 : 1.0));
        more = ad[AD_L] < ad[AD_MAX];
        if (!more) ad[AD_ERR] = 1.0;
    }
    if (has_cond) cudaGraphSetConditional(cond, more ? 1u : 0u);
}

// Fixed-order block reductions for the finalize kernels (256 threads: strided partial sums in
// a fixed assignment, then a fixed tree)
__device__ __forceinline__ double fin_sum(double v, double *sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}
__device__ __forceinline__ double fin_max(double v, double *sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + st]);
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) adapt_finalize_kernel(const double *part, int nb, DevScalars *ts) {
    __shared__ double sh[256];
    double q = 0.0, d = 0.0;
    for (int b = threadIdx.x; b < nb; b += 256) { q += part[b * 8]; d += part[b * 8 + 1]; }
    q = fin_sum(q, sh);
    d = fin_sum(d, sh);
    if (threadIdx.x == 0) {
        ts->stats[8] = q;
        ts->stats[9] = d;
    }
}

__global__ void __launch_bounds__(256) stats_finalize_kernel(const double *pro, int nb_pro, const double *res,
                                                             int nb_res, DevScalars *ts) {
    __shared__ double sh[256];
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nb_pro; b += 256)
        for (int q = 0; q < 4; ++q) s[q] += pro[b * 8 + q];
    for (int b = threadIdx.x; b < nb_res; b += 256) {
        s[4] += res[b * 8 + 4];
        s[5] += res[b * 8 + 5];
        s[6] = fmax(s[6], res[b * 8 + 6]);
        s[7] += res[b * 8 + 7];
    }
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = q == 6 ? fin_max(s[q], sh) : fin_sum(s[q], sh);
    if (threadIdx.x == 0)
        for (int q = 0; q < 8; ++q) ts->stats[q] = r[q];
}

template <typename T>
__global__ void fill_inputs_kernel(const double *X64, int64_t N, int n, int NB, int NBP, int64_t ldT,
                                   T *XT, T *Xh) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ldT) return;
    for (int k = 0; k < NB; ++k) XT[(int64_t)k * ldT + j] = (j < N && k < n) ? T(X64[j * n + k]) : T(0);
    for (int d = 0; d < NBP; ++d)
        Xh[j * NBP + d] = (j < N && d < n) ? T(X64[j * n + d]) : ((j < N && d == n) ? T(1) : T(0));
}

template <typename T>
__global__ void convert_rows_kernel(const double *src, int64_t rows, int64_t N, int64_t ldT, T *dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * ldT) return;
    const int64_t i = e / ldT, j = e % ldT;
    dst[e] = j < N ? T(src[i * N + j]) : T(0);
}

template <typename T>
__global__ void unconvert_rows_kernel(const T *src, int64_t rows, int64_t N, int64_t ldT, double *dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * N) return;
    const int64_t i = e / N, j = e % N;
    dst[e] = (double)src[i * ldT + j];
}

inline unsigned nblk(int64_t work, int bs) { return (unsigned)((work + bs - 1) / bs); }

// Receiving side of the y' all-gather (one CTA): acquire each source's rows for this epoch
// (source r sends min(S, N - r S) rows per epoch), then copy all N rows into yv.
template <typename T>
__device__ void p2p_ygather_block(const T *yrecv, unsigned long long *flag, unsigned long long *epoch, int W,
                                  int64_t N, int64_t S, T *yv) {
    if (threadIdx.x == 0) {
        const unsigned long long e = *epoch + 1;
        for (int r = 0; r < W; ++r) {
            const int64_t rows = max((int64_t)0, min(S, N - (int64_t)r * S));
            const unsigned long long target = e * (unsigned long long)rows;
            unsigned long long v;
            while (true) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + r) : "memory");
                if (v >= target) break;
                __nanosleep(64);
            }
        }
        *epoch = e;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) yv[j] = yrecv[j];
}

template <typename T>
__global__ void __launch_bounds__(1024) p2p_ygather_kernel(const P2PYGather g) {
    pdl_wait();
    p2p_ygather_block<T>(static_cast<const T *>(g.yrecv), g.flag, g.epoch, g.W, g.N, g.S, static_cast<T *>(g.yv));
}

// y' self-test: blocks [0, W nbp) push rank (b / nbp)'s rows (256 per block), the last W blocks
// receive.  Cooperative launch: all resident.
struct P2PYEmu {
    int W;
    int64_t N, S, nbp;
    const float *y;
    float *out;                              // [W][N]
    void *const *yrecv;
    unsigned long long *const *yflag;
    unsigned long long *epoch;               // [W]
};

__global__ void __launch_bounds__(256) p2p_yemulate_kernel(const P2PYEmu em) {
    const int64_t b = blockIdx.x;
    if (b < em.W * em.nbp) {
        const int r = (int)(b / em.nbp);
        const int64_t r0 = (int64_t)r * em.S, r1 = min(em.N, r0 + em.S);
        const int64_t gi = r0 + (b % em.nbp) * 256 + threadIdx.x;
        __shared__ unsigned cnt;
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        if (gi < r1) {
            p2p_ypush_row<float>(em.yrecv, em.W, gi, em.y[gi]);
            atomicAdd(&cnt, 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0 && cnt) p2p_ysignal(em.yflag, em.W, r, cnt);
    } else {
        const int q = (int)(b - em.W * em.nbp);
        p2p_ygather_block<float>(static_cast<const float *>(em.yrecv[q]), em.yflag[q], em.epoch + q, em.W, em.N, em.S,
                                 em.out + (int64_t)q * em.N);
    }
}

// Owner side of the peer-memory reduce-scatter (one CTA): acquire every source's arrivals for
// this epoch, then sum the W contributions in rank order.
__device__ void p2p_gather_block(const double *slab, unsigned long long *flag, unsigned long long *epoch, int W,
                                 int64_t S, int64_t Ns, int64_t nblk, double *c_out) {
    __shared__ unsigned long long target;
    if (threadIdx.x == 0) {
        const unsigned long long e = *epoch + 1;
        target = e * (unsigned long long)nblk;
        for (int r = 0; r < W; ++r) {
            unsigned long long v;
            while (true) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + r) : "memory");
                if (v >= target) break;
                __nanosleep(64);
            }
        }
        *epoch = e;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < Ns; i += blockDim.x) {
        double t = 0.0;
        for (int r = 0; r < W; ++r) t += slab[(int64_t)r * S + i];
        c_out[i] = t;
    }
}

__global__ void __launch_bounds__(1024) p2p_gather_kernel(const P2PGather g) {
    pdl_wait();
    p2p_gather_block(g.slab, g.flag, g.epoch, g.W, g.S, g.Ns, g.nblk, g.c_out);
}

// Self-test kernel: blocks [0, W ncolb) are rank (b / ncolb)'s column-sum blocks pushing into
// the owners' slabs; the last W blocks are the owners gathering.  A cooperative launch, so all
// blocks are resident and the owners' waits always see their sources run.
constexpr int kP2PMaxWorld = kP2PTab;
struct P2PEmu {
    int W, nRB;
    int64_t N, S, ncolb, ldT;
    const float *colpart[kP2PMaxWorld];
    double *c_out[kP2PMaxWorld];
    unsigned long long *epoch[kP2PMaxWorld];
    double *const *recv;
    unsigned long long *const *flag;
};

__global__ void __launch_bounds__(256) p2p_emulate_kernel(const P2PEmu em) {
    const int64_t b = blockIdx.x;
    if (b < em.W * em.ncolb) {
        const int r = (int)(b / em.ncolb);
        ReduceParams p{};
        p.N = em.N;
        p.ldT = em.ldT;
        p.nRB = em.nRB;
        p.colpart = em.colpart[r];
        p.p2p_recv = em.recv;
        p.p2p_flag = em.flag;
        p.p2p_rank = r;
        p.p2p_S = em.S;
        colsum_block<float>(p, b % em.ncolb);
    } else {
        const int q = (int)(b - em.W * em.ncolb);
        const int64_t Ns = min(em.S, em.N - q * em.S);
        const int64_t nblk = (Ns + 127) / 128;
        p2p_gather_block(em.recv[q], em.flag[q], em.epoch[q], em.W, em.S, Ns, nblk, em.c_out[q]);
    }
}

}  // namespace

// One resident wave: the grid-stride loop keeps two rows in flight per warp, so more CTAs than
// fit at once only add waves of latency.
template <typename T, int Q>
int prologue_wave() {
    static int wave = 0;                       // per instantiation; the device does not change
    if (wave == 0) {
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, prologue_kernel<T, Q>, 256, 0);
        wave = std::max(1, nsm * std::max(occ, 1));
    }
    return wave;
}

cudaError_t launch_prologue(const SmallParams &p, int fp64, cudaStream_t s, int *nb_out) {
    int64_t nb = (p.Ns + 7) / 8;
    if (nb < 1) nb = 1;
    const int q = (p.n + 31) / 32;
    const int wave = q <= 1 ? (fp64 ? prologue_wave<double, 1>() : prologue_wave<float, 1>())
                   : q == 2 ? (fp64 ? prologue_wave<double, 2>() : prologue_wave<float, 2>())
                            : (fp64 ? prologue_wave<double, 3>() : prologue_wave<float, 3>());
    if (nb > wave) nb = wave;
    if (nb > kStatBlocks) nb = kStatBlocks;
    cudaError_t e;
    if (q <= 1)
        e = fp64 ? pdl_launch(prologue_kernel<double, 1>, dim3((unsigned)nb), dim3(256), 0, s, p)
                 : pdl_launch(prologue_kernel<float, 1>, dim3((unsigned)nb), dim3(256), 0, s, p);
    else if (q == 2)
        e = fp64 ? pdl_launch(prologue_kernel<double, 2>, dim3((unsigned)nb), dim3(256), 0, s, p)
                 : pdl_launch(prologue_kernel<float, 2>, dim3((unsigned)nb), dim3(256), 0, s, p);
    else if (q == 3)
        e = fp64 ? pdl_launch(prologue_kernel<double, 3>, dim3((unsigned)nb), dim3(256), 0, s, p)
                 : pdl_launch(prologue_kernel<float, 3>, dim3((unsigned)nb), dim3(256), 0, s, p);
    else
        return cudaErrorInvalidValue;
    if (e != cudaSuccess) return e;
    if (nb_out) *nb_out = (int)nb;
    return cudaGetLastError();
}

int reduce_col_block(int fp64) { return fp64 ? 32 : 128; }

cudaError_t launch_p2p_ygather(const P2PYGather &g, int fp64, cudaStream_t s) {
    if (fp64) p2p_ygather_kernel<double><<<1, 1024, 0, s>>>(g);
    else p2p_ygather_kernel<float><<<1, 1024, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t p2p_selftest_y(int W, int64_t N, const float *y, float *out, cudaStream_t s) {
    if (W < 1 || W > kP2PTab || N < 1) return cudaErrorInvalidValue;
    const int64_t S = shard_rows(N, W, 1), nbp = (S + 255) / 256;
    char *buf = nullptr;
    const size_t yb = (sizeof(float) * (size_t)N + 255) / 256 * 256, fb = sizeof(unsigned long long) * (size_t)W;
    const size_t per = (yb + fb + 255) / 256 * 256;     // y' receive, then the (8-B aligned) flags
    cudaError_t e = cudaMallocAsync(&buf, per * W + sizeof(void *) * 2 * kP2PTab + sizeof(unsigned long long) * W, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(buf, 0, per * W + sizeof(void *) * 2 * kP2PTab + sizeof(unsigned long long) * W, s);
    void *tab[2 * kP2PTab] = {};
    for (int q = 0; q < W; ++q) {
        tab[q] = buf + per * q;
        tab[kP2PTab + q] = buf + per * q + yb;
    }
    void **dtab = reinterpret_cast<void **>(buf + per * W);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dtab, tab, sizeof tab, cudaMemcpyHostToDevice, s);
    P2PYEmu em{};
    em.W = W;
    em.N = N;
    em.S = S;
    em.nbp = nbp;
    em.y = y;
    em.out = out;
    em.yrecv = dtab;
    em.yflag = reinterpret_cast<unsigned long long *const *>(dtab + kP2PTab);
    em.epoch = reinterpret_cast<unsigned long long *>(dtab + 2 * kP2PTab);
    if (e == cudaSuccess) {
        void *args[] = {&em};
        e = cudaLaunchCooperativeKernel((const void *)p2p_yemulate_kernel, dim3((unsigned)(W * nbp + W)), dim3(256),
                                        args, 0, s);
    }
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaFreeAsync(buf, s);
    return e != cudaSuccess ? e : e2;
}

cudaError_t launch_p2p_gather(const P2PGather &g, cudaStream_t s) {
    p2p_gather_kernel<<<1, 1024, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t p2p_selftest(int W, int64_t N, int nRB, const float *colpart, int64_t ldT, double *c, cudaStream_t s) {
    if (W < 1 || W > kP2PMaxWorld || N < 1) return cudaErrorInvalidValue;
    const int64_t S = shard_rows(N, W, 1);
    if (S % 128) return cudaErrorInvalidValue;                 // column blocks may not straddle owners
    const int64_t ncolb = (N + 127) / 128;
    // per virtual rank: a receive slab [W][S] + flags [W] + epoch, one allocation
    const size_t per = (size_t)W * S + W + 1;
    double *buf = nullptr;
    cudaError_t e = cudaMallocAsync(&buf, sizeof(double) * per * W + sizeof(void *) * 2 * kP2PMaxWorld, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(buf, 0, sizeof(double) * per * W, s);
    P2PEmu em{};
    em.W = W;
    em.N = N;
    em.S = S;
    em.ncolb = ncolb;
    double *hr[kP2PMaxWorld];
    unsigned long long *hf[kP2PMaxWorld];
    for (int q = 0; q < W; ++q) {
        hr[q] = buf + per * q;
        hf[q] = reinterpret_cast<unsigned long long *>(hr[q] + (size_t)W * S);
        em.epoch[q] = hf[q] + W;
        em.colpart[q] = colpart + (size_t)q * nRB * ldT;
        em.c_out[q] = c + q * S;
    }
    double **tab = reinterpret_cast<double **>(buf + per * W);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tab, hr, sizeof(void *) * W, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(tab + kP2PMaxWorld, hf, sizeof(void *) * W, cudaMemcpyHostToDevice, s);
    em.recv = tab;
    em.flag = reinterpret_cast<unsigned long long *const *>(tab + kP2PMaxWorld);
    em.nRB = nRB;
    em.ldT = ldT;
    if (e == cudaSuccess) {
        void *args[] = {&em};
        e = cudaLaunchCooperativeKernel((const void *)p2p_emulate_kernel, dim3((unsigned)(W * ncolb + W)), dim3(256),
                                        args, 0, s);
    }
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaFreeAsync(buf, s);
    return e != cudaSuccess ? e : e2;
}

cudaError_t launch_reduce(const ReduceParams &p, int fp64, cudaStream_t s) {
    const int ncolb = (int)((p.N + (fp64 ? 31 : 127)) / (fp64 ? 32 : 128));
    const int64_t nrowb = (p.Ns + 7) / 8;
    const unsigned nb = (unsigned)(ncolb + nrowb);
    cudaError_t e = fp64 ? pdl_launch(reduce_kernel<double>, dim3(nb), dim3(256), 0, s, p, ncolb)
                         : pdl_launch(reduce_kernel<float>, dim3(nb), dim3(256), 0, s, p, ncolb);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_reduce_prologue(const ReduceParams &rd, const SmallParams &pr, cudaStream_t s) {
    if (!rd.advance_t || rd.p2p_recv || pr.p2p_push || pr.statpart || pr.s_dev || pr.from_eta || !pr.use_beta)
        return cudaErrorInvalidValue;
    // 32 rows per block once that still gives >= 4 blocks per SM-sized wave (148 SMs), else 8
    int rpb = pr.Ns >= 32 * 4 * 148 ? 32 : 8;
    if (const char *e = std::getenv("CR_FUSE_RPB")) rpb = std::atoi(e) == 32 ? 32 : 8;
    const unsigned nb = (unsigned)std::max<int64_t>(1, (pr.Ns + rpb - 1) / rpb);
    const int q = (pr.n + 31) / 32;
#define CR_RP(Q) (rpb == 32 ? pdl_launch(reduce_prologue_kernel<Q, 32>, dim3(nb), dim3(256), 0, s, rd, pr) \
                            : pdl_launch(reduce_prologue_kernel<Q, 8>, dim3(nb), dim3(256), 0, s, rd, pr))
    if (q <= 1) return CR_RP(1);
    if (q == 2) return CR_RP(2);
    if (q == 3) return CR_RP(3);
#undef CR_RP
    return cudaErrorInvalidValue;
}

cudaError_t launch_adapt_check(const AdaptParams &p, cudaStream_t s) {
    int64_t nb = (p.Ns + 7) / 8;
    if (nb < 1) nb = 1;
    if (nb > kStatBlocks) nb = kStatBlocks;
    adapt_check_kernel<<<(unsigned)nb, 256, 0, s>>>(p);
    adapt_finalize_kernel<<<1, 256, 0, s>>>(p.statpart, (int)nb, p.ts);
    return cudaGetLastError();
}

cudaError_t launch_adapt_decide(DevScalars *ts, unsigned long long cond, int has_cond, cudaStream_t s) {
    adapt_decide_kernel<<<1, 32, 0, s>>>(ts, (cudaGraphConditionalHandle)cond, has_cond);
    return cudaGetLastError();
}


cudaError_t launch_stats_finalize(const double *pro, int nb_pro, const double *res, int nb_res,
                                  DevScalars *ts, cudaStream_t s) {
    stats_finalize_kernel<<<1, 256, 0, s>>>(pro, nb_pro, res, nb_res, ts);
    return cudaGetLastError();
}

cudaError_t launch_fill_inputs(const double *X64, int64_t N, int n, int NB, int NBP, int64_t ldT,
                               int fp64, void *XT, void *Xh, cudaStream_t s) {
    const unsigned nb = nblk(ldT, 256);
    if (fp64) fill_inputs_kernel<double><<<nb, 256, 0, s>>>(X64, N, n, NB, NBP, ldT, (double *)XT, (double *)Xh);
    else fill_inputs_kernel<float><<<nb, 256, 0, s>>>(X64, N, n, NB, NBP, ldT, (float *)XT, (float *)Xh);
    return cudaGetLastError();
}

cudaError_t launch_convert_rows(const double *src, int64_t rows, int64_t N, int64_t ldT, int fp64,
                                void *dst, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const unsigned nb = nblk(rows * ldT, 256);
    if (fp64) convert_rows_kernel<double><<<nb, 256, 0, s>>>(src, rows, N, ldT, (double *)dst);
    else convert_rows_kernel<float><<<nb, 256, 0, s>>>(src, rows, N, ldT, (float *)dst);
    return cudaGetLastError();
}

cudaError_t launch_unconvert_rows(const void *src, int64_t rows, int64_t N, int64_t ldT, int fp64,
                                  double *dst, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const unsigned nb = nblk(rows * N, 256);
    if (fp64) unconvert_rows_kernel<double><<<nb, 256, 0, s>>>((const double *)src, rows, N, ldT, dst);
    else unconvert_rows_kernel<float><<<nb, 256, 0, s>>>((const float *)src, rows, N, ldT, dst);
    return cudaGetLastError();
}

}  // namespace cr

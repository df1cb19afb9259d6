// Internal declarations shared by the host orchestration (cr_api.cpp) and the
// CUDA kernels.  Not part of the ABI (include/cr.h is).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <utility>

namespace cr {

// Programmatic dependent launch (PDL) for the per-iteration kernel chain: a kernel launched with
// pdl_launch may be scheduled while its predecessor drains; it calls pdl_wait() before touching
// the predecessor's outputs (griddepcontrol.wait: all prerequisite grids complete, memory
// visible) and pdl_trigger() once its own dependents may launch.  CR_NO_PDL=1 disables it.
bool pdl_enabled();
// CR_TC_TRACE buffer: [5 roles][256 tiles][8 events] clock64 of CTA 0, then per CTA
// [entry, predecessor complete, exit, tiles] (globaltimer ns)
constexpr int kTraceTile = 5 * 256 * 8, kTraceWords = kTraceTile + 4 * 1024;
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

constexpr int kBM = 64;           // SIMT fused-pass tile rows
constexpr int kBN = 64;           // SIMT fused-pass tile columns
constexpr int kThreads = 256;     // SIMT fused-pass CTA size
constexpr int kGMax = 4096;       // upper bound on fused-pass CTAs (slot table sizing)
constexpr int kRowAlign = 128;    // Theta rows allocated per shard rounded to this
constexpr int kColAlign = 256;    // Theta row pitch (elements) rounded to this
constexpr int kStatBlocks = 1024; // max CTAs of the stats/residual kernels
constexpr int kTcBM = 128;        // tensor-core pass tile rows (TMEM lanes)
constexpr int kTcBN = 32;         // tensor-core pass tile columns
constexpr int kTcMaxStages = 6;
constexpr int64_t kIpmMaxNbar = 128;         // partition block size limit (block_ipm smem: S, X, Z)
constexpr size_t kIpmMaxSmem = 220 * 1024;
constexpr int kIpmMaxIter = 100;             // interior-point iterations per projection
constexpr double kIpmTol = 1e-9;             // relative residuals / max complementarity (then the polish)
constexpr int kP2PTab = 8;                   // CR_FLAG_P2P: largest world (pointer table size)
constexpr int64_t kLanczosHostMax = 1 << 14;   // N (n + 1) at or below: L by the host Lanczos in cr_init
constexpr int64_t kResidentMaxN = 4096;   // SMEM-resident small-N solver: eligible sizes
constexpr int kResidentMaxCTAs = 256;

// Rows per shard (include/cr.h, cr_shard_rows): ceil(N / world), rounded up to the 128-column
// block of the column-sum / peer-memory exchange when world > 1 and every rank keeps >= 1 row
// (all-pairs only: a partition needs S % nbar == 0 instead).
inline int64_t shard_rows(int64_t N, int world, int64_t nbar) {
    const int64_t S = (N + world - 1) / world;
    if (world <= 1 || nbar > 1) return S;
    const int64_t Sp = (S + 127) / 128 * 128;
    return (int64_t)(world - 1) * Sp < N ? Sp : S;
}

// Element (i, j) of a Theta buffer (local row i, column j), in elements from the buffer base.
//   row-major (SIMT configs): i * ldT + j
//   tile-major (tensor-core configs): 128 x 32 tiles of 16 KB, each contiguous, tiles in
//   row-block-major order (nCBt tiles per row block); inside a tile row r (128 B) the 16-B chunk
//   q = (j % 32) / 4 sits at position q ^ (r % 8) -- exactly the 128-B-swizzled shared-memory
//   image of the tile, so one 16-KB bulk copy moves a tile between HBM and the pass's smem.
__host__ __device__ inline int64_t theta_off(int64_t i, int64_t j, int64_t ldT, int tiled, int nCBt) {
    if (!tiled) return i * ldT + j;
    const int64_t rb = i >> 7, cb = j >> 5;
    const int r = (int)(i & 127), c = (int)(j & 31);
    return ((rb * nCBt + cb) << 12) + (r << 5) + ((((c >> 2) ^ (r & 7))) << 2) + (c & 3);
}

// n-buckets compiled for the SIMT pass (S-GEMM depth NB; P-GEMM width NBP = NB + 4).
int simt_bucket(int n);           // smallest compiled NB >= n, or 0 if none

// Device scalar block (fp64), lives in the workspace.
struct DevScalars {
    double t_prev;      // t_{k-1}
    double t_cur;       // t_k
    double stats[16];   // finalized diagnostics (see stats kernels); [8], [9]: adaptive Q, ||D||^2
    // adaptive step rule state (device-resident so a CUDA-graph WHILE loop can run the trials):
    // [0] s_{k-1}  [1] s of the next trial  [2] ups  [3] trials of the last iteration
    // [4] trials in total  [5] l of the next trial  [6] max trials  [7] error (no l passed)
    // [8] variant: 0 the paper's s_{k-1} ups^(l-1), 1 monotone backtracking s_{k-1} ups^l
    double ad[10];
    unsigned long long fuse_cnt;   // reduce_prologue_kernel: arrivals of this launch (the last block
                                   // advances t and resets it to 0)
};
enum AdaptSlots { AD_S = 0, AD_STRY = 1, AD_UPS = 2, AD_TLAST = 3, AD_TTOT = 4, AD_L = 5, AD_MAX = 6, AD_ERR = 7,
                  AD_MONO = 8 };

struct PassParams {
    const void *B1;        // Theta^{k-1} (read)
    void *B2;              // Theta^{k-2} (read)
    void *Bout;            // Theta^k (MODE_STEP): B2 (in place) or a third buffer (adaptive step)
    int tiled, nCBt;       // Theta layout (theta_off)
    int adapt;             // 1: row partial column n+1 receives sum_j (Theta^k - theta~)^2
    int dcol;              // that column (n + 1 < NBP)
    int64_t ldT;           // row pitch of Theta, XT, colpart (elements)
    int64_t N, Ns, row0;   // global size, shard rows, first global row of the shard
    int64_t nbar;          // partition block size (Assumption 1): Theta_ij = 0 when i / nbar == j / nbar
    int nRB, nCB;          // tile grid (row blocks of kBM, column tiles of kBN)
    int64_t T;             // nRB * nCB
    int G;                 // CTAs
    const void *XT;        // [NB][ldT]   x_j[k] (k-major), zero padded
    const void *Xh;        // [ldT][NBP]  x_j[d], 1 at d = n, zero padded
    const void *XiT;       // [NB][Rp]    xi_i[k] * scale (k-major)
    const void *bv;        // [Rp]        (a_i - y_i) * scale
    const void *yv;        // [>= ldT]    y_j * scale (all columns, gathered)
    int64_t Rp;            // allocated rows
    void *colpart;         // [nRB][ldT] column partial sums (acc type)
    double *rowpart;       // [slots][kBM][NBP] row partials (r at d = n, Theta X at d < n)
    const int *cta_slot0;  // [G] first row-partial slot of each CTA
    const double *ts;      // DevScalars* (t_prev, t_cur) -> beta
};

enum PassMode { MODE_STEP = 0, MODE_SUMS = 1 };

// SIMT fused pass (kernels/pass_simt.cu).
cudaError_t launch_pass_simt(const PassParams &p, int prec_fp64, int NB, int mode, cudaStream_t s);
cudaError_t pass_simt_config(int prec_fp64, int NB, int *smem_bytes, int *blocks_per_sm);

struct SmallParams {
    int64_t N, Ns, row0, Rp, ldT;
    int n, NB, NBP;
    double gamma, scale;
    const double *X64;     // [N][n]
    const double *ybar;    // [N]
    // sums slots (r, c, P) for S^{k-1} (s1) and S^{k-2} (s2)
    const double *r1, *c1, *P1, *r2, *c2, *P2;
    double *y64;           // [>= N] y of eta (all rows after gather)
    double *Xi64;          // [Rp][n]
    double *a64;           // [Rp]
    void *yv, *bv, *XiT;   // storage-precision copies for the pass
    double *statpart;      // [kStatBlocks][8] per-CTA partials
    DevScalars *ts;
    int use_beta;          // 1: beta from ts (Step 1 at theta~^k); 0: beta = 0 (eta(Theta^k))
    const double *s_dev;   // non-null: scale = 1 / *s_dev (the adaptive trial's s, device-resident)
    float *XiR;            // optional [Rp][NK] row-major xi * scale (tensor-core pass operand)
    int NK;
    int from_eta;          // 1: take (y, xi) from y64 / Xi64 (after the block projections) instead of
                           //    the closed form; refreshes a64, the pass operands and the stat partials
    // CR_FLAG_P2P all-gather of y': with p2p_push, every row's y' also goes to each rank q's
    // receive array p2p_yrecv[q][global row] (peer stores), and each CTA then adds its row count to
    // p2p_yflag[q][p2p_rank] (system-scope release)
    void *const *p2p_yrecv;
    unsigned long long *const *p2p_yflag;
    int p2p_rank, p2p_W, p2p_push;
};

cudaError_t launch_prologue(const SmallParams &p, int prec_fp64, cudaStream_t s, int *nblocks_out);

struct ReduceParams {
    int64_t N, Ns, Rp, ldT;
    int n, NBP, nRB, rbm;  // rbm: rows per row block of the pass that wrote the partials
    int rcol0, rcol1;      // slot-row columns holding row-sum partials (rcol1 < 0: none)
    const void *colpart;   // [nRB][ldT]
    const double *rowpart; // [slots][kBM][NBP]
    const int *rb_ptr;     // [nRB + 1]
    const int *rb_slots;   // row-partial slot list per row block (CTA order)
    int dcol0, dcol1;      // slot-row columns holding ||Theta^k - theta~||^2 partials (-1: none)
    double *dsq;           // [Rp] per-row ||Theta^k - theta~||^2 (when dcol0 >= 0)
    double *r, *P;         // this shard's rows
    double *c_out;         // column sums for all N columns (shard partial)
    DevScalars *ts;
    int advance_t;         // 1: t_prev <- t_cur, t_cur <- (1 + sqrt(1 + 4 t^2)) / 2
    unsigned long long *yepoch;   // non-null: ++*yepoch (the pass consumed this epoch's peer y')
    // Peer-memory reduce-scatter (CR_FLAG_P2P): non-null -> column j's partial goes straight to
    // its owner q = j / S, at p2p_recv[q][p2p_rank * S + j - q S] (NVLink peer store), and each
    // column block then bumps p2p_flag[q][p2p_rank] with a system-scope release (S % block = 0)
    double *const *p2p_recv;
    unsigned long long *const *p2p_flag;
    int p2p_rank;
    int64_t p2p_S;
};

cudaError_t launch_reduce(const ReduceParams &p, int prec_fp64, cudaStream_t s);

// reduce of iteration k fused with the prologue of iteration k+1 (one rank, fp32 storage,
// constant step): a block owns 32 rows i, and column i's sum is c_i, so the block needs only its
// own columns' partials -- no grid-wide dependency between the two halves.  Same arithmetic and
// summation order as reduce_kernel followed by prologue_kernel (bitwise identical results);
// Step 3 (t update) by the last block to finish.  rd.advance_t must be 1.
cudaError_t launch_reduce_prologue(const ReduceParams &rd, const SmallParams &pr, cudaStream_t s);
int reduce_col_block(int prec_fp64);   // columns per column-sum CTA (128 fp32 partials, 32 fp64)

// Owner side of the peer-memory reduce-scatter: one CTA waits (acquire, system scope) until
// every source rank's column blocks for this epoch have landed in the local slab, then sums
// the W contributions in rank order (deterministic) into c_out.
struct P2PGather {
    const double *slab;          // [W][S] this rank's receive slab
    unsigned long long *flag;    // [W]    arrivals per source (monotonic)
    unsigned long long *epoch;   // [1]    gathers completed (this rank)
    int W;
    int64_t S, Ns, nblk;         // nblk: column blocks each source sends per epoch
    double *c_out;               // [Ns]
};
cudaError_t launch_p2p_gather(const P2PGather &g, cudaStream_t s);
// Receiving side of the y' all-gather: acquire every source's rows for this epoch, then copy the
// receive array (all N rows) into the pass operand yv.
struct P2PYGather {
    const void *yrecv;           // [N] storage precision, written by every rank's prologue
    unsigned long long *flag;    // [W] rows received per source (monotonic)
    unsigned long long *epoch;   // [1]
    int W;
    int64_t N, S;
    void *yv;                    // [>= N] storage precision
};
cudaError_t launch_p2p_ygather(const P2PYGather &g, int prec_fp64, cudaStream_t s);
// Self-test of the y' all-gather protocol: W virtual ranks' row pushes and receivers in ONE
// cooperative launch; out[q][j] = rank q's gathered y'_j.
cudaError_t p2p_selftest_y(int W, int64_t N, const float *y_dev /* [N] */, float *out_dev /* [W][N] */,
                           cudaStream_t s);
// Self-test: W virtual ranks' column sums + reduce-scatter in ONE cooperative launch on one
// GPU (push blocks and owner blocks co-resident, so the owners' waits cannot deadlock).
cudaError_t p2p_selftest(int W, int64_t N, int nRB, const float *colpart_dev /* [W][nRB][ldT] */, int64_t ldT,
                         double *c_dev /* [N] */, cudaStream_t s);

// Adaptive step: Eq. (adaptive-check) in its quadratic form (R15),
//   Q = ||A1^T D||^2 + ||A2^T D||^2 / gamma   vs   s ||D||^2,   D = Theta^k - theta~^k,
// from the sums of Theta^{k-1} (A), Theta^{k-2} (B), Theta^k (O) and the per-row ||D||^2.
struct AdaptParams {
    int64_t Ns, row0;
    int n;
    double gamma;
    const double *X64;
    const double *rA, *cA, *PA, *rB, *cB, *PB, *rO, *cO, *PO;
    const double *dsq;
    double *statpart;      // [kStatBlocks][8]: Q at 0, ||D||^2 at 1
    DevScalars *ts;        // beta from (t_prev, t_cur); results to stats[8], stats[9]
};
cudaError_t launch_adapt_check(const AdaptParams &p, cudaStream_t s);
// Accept / retry after the check (ts->ad, Step 3 on acceptance).  cond != 0: also drive the
// enclosing CUDA-graph WHILE node (0 = leave the trial loop).
cudaError_t launch_adapt_decide(DevScalars *ts, unsigned long long cond, int has_cond, cudaStream_t s);

struct ResidualParams {
    const void *Theta;     // storage precision, layout theta_off(tiled, nCBt)
    int64_t ldT, N, Ns, row0, Rp;
    int tiled, nCBt;
    int n, nP;             // features; nP = n rounded up to 8 (k-major operand rows)
    const double *X64, *y64, *Xi64, *a64;
    const double *XT;      // [nP][ldX] x_j[k], k-major, zero padded (cr_init)
    int64_t ldX;
    double *XiT;           // [nP][Rp] xi_i[k], k-major (written by launch_residual from Xi64)
    double *statpart;      // [kStatBlocks][8]
};

// kernels/residual.cu: the fp64 residual pass of cr_primal (transposes Xi64 into XiT first)
cudaError_t launch_residual(const ResidualParams &p, int prec_fp64, cudaStream_t s, int *nblocks_out);
size_t residual_smem_bytes();
// dst[k][i] = src[i][k] (k < n; zero for n <= k < nP and rows <= i < ld)
cudaError_t launch_transpose_pad(const double *src, int64_t rows, int n, int nP, int64_t ld, double *dst,
                                 cudaStream_t s);

// Sum the per-CTA partials: prologue partials (nb_pro blocks: |u|^2, u.ybar, |xi|^2,
// nonfinite) and residual partials (nb_res blocks: gap, sum R_-^2, max -R, nonfinite)
// into ts->stats[0..7] (rank-local).
cudaError_t launch_stats_finalize(const double *pro, int nb_pro, const double *res, int nb_res,
                                  DevScalars *ts, cudaStream_t s);

struct TcParams {
    const float *B1, *B2;            // Theta^{k-1}, Theta^{k-2} (tile-major, theta_off)
    float *Bout;                     // Theta^k
    int64_t N, Ns, row0, ldT, T;
    int G, nCB, NK, NP2, stages, window;
    int g1stages, g2stages;          // X_J / X_J^T image ring slots
    int g1passes;                    // GEMM1 passes: 3 = Xi_hi X_hi + Xi_hi X_lo + Xi_lo X_hi;
                                     // 2 = without Xi_hi X_lo (the X_J ring then holds X_hi only)
    int g1f16;                       // 1: GEMM1 in kind::f16 (hi / lo halves of 11 bits each, like tf32,
                                     //    at twice the rate and half the X_J image); Xi' rows scaled by
                                     //    2^e_i, X by 2^xexp into the fp16 range, D1 scaled back exactly
    int xexp;                        // the X scale exponent of the f16 images
    // CR_FLAG_P2P y' all-gather fused into the pass (SURVEY §8(e) fix 1): yv is this rank's receive
    // array (global row order); before the first tile of owner q's columns the producer acquires
    // (system scope) yflag[q] >= (*yepoch + 1) * rows_q; the CTAs sweep their columns starting at
    // column tile rot (this rank's own columns, whose y' is local), so the peers' pushes overlap
    // the first tiles.  yflag == nullptr: yv already holds every row (NCCL / one rank).
    const unsigned long long *yflag;
    const unsigned long long *yepoch;
    int W, rot;
    int64_t S;
    int n;                           // features (Xi' entries k >= n are treated as 0)
    int adapt;                       // 1: also accumulate ||Theta^k - theta~||^2 per row (adaptive step)
    int poll_ns;                     // producer back-off when no ring slot is free (ns)
    int theta_l2;                    // 1: Theta loads/stores with the evict-normal L2 policy (state ~ L2 size)
    int64_t nbar;                    // partition block size (1: all pairs dualized)
    int smem_bytes;
    const float *g1_hi, *g1_lo;      // [nCB][NK * 32]  X_J  tiles (K-major interleave), tf32 hi / lo
    const float *g2_hi, *g2_lo;      // [nCB][NP2 * 32] X_J^T tiles (K-major interleave), tf32 hi / lo
    const float *yv;                 // y * scale, gathered
    const float *XiR;                // [Rp][NK] xi * scale
    const float *bv;                 // [Rp] (a - y) * scale
    float *colpart;                  // [nRB128][ldT]
    double *rowpart;                 // [slots][128][NP2 + 4]: Theta X | r (wg 0, 1) | ||D||^2 (wg 0, 1)
    const int *cta_slot0;
    unsigned long long *trace;       // debug: clock64 timeline of CTA 0 + per-CTA globaltimer records (nullptr = off)
    int g1_runahead;                 // 1: GEMM1 does not wait for the tile's Theta (needs X_J, Xi' only)
    unsigned long long *check;       // CR_TC_CHECK: first ring-protocol violation (nullptr = checks off),
                                     // (code << 56) | (CTA << 32) | tile; see tc_check_code
    const double *ts;
};

// tcgen05 fused pass (kernels/pass_tc.cu).
cudaError_t launch_pass_tc(const TcParams &p, cudaStream_t s);
cudaError_t pass_tc_prepare(int NK, int smem_bytes);
size_t tc_barrier_bytes();
cudaError_t launch_tc_images(const double *X64, int64_t N, int n, int NK, int NP2, int nCB, float *g1h, float *g1l,
                             float *g2h, float *g2l, int g1f16, int xexp, cudaStream_t s);

// SMEM-resident multi-iteration solver for small N (kernels/resident.cu): K constant-step
// iterations in one cooperative launch, row-major Theta buffers (SIMT layout), world == 1.
struct ResidentParams {
    int64_t N, ldT, K;
    int n, R, ldS, G;           // rows per CTA, smem row pitch, CTAs
    void *TA, *TB;              // Theta^{k-1}, Theta^{k-2} (global, row-major)
    double *rA, *cA, *PA, *rB, *cB, *PB;
    const double *X64, *ybar;
    double gamma, L;
    DevScalars *ts;
    double *yg;                 // [N] y of the current Step 1 (all rows)
    double *y64, *a64, *Xi64;   // eta of the last Step 1 (cr_get_eta)
    double *cpart;              // [G][N]
    unsigned long long *trace;  // debug: clock64 per phase of CTA 0, first 16 iterations (nullptr = off)
};
size_t resident_smem_bytes(const ResidentParams &p, int fp64);
cudaError_t launch_resident(const ResidentParams &p, int fp64, cudaStream_t s);

// sigma_max(C)^2 (Eq. (lischitz)): host Lanczos helpers (lanczos.cpp) and the device
// Lanczos (kernels/lanczos.cu, X device fp64 [N][n]; < 0 and *err set on a CUDA error).
double lanczos_max_ritz(const double *al, const double *be, int m);
void lanczos_start(int64_t N, int n, double *v);
double sigma_max_sq_lanczos_device(int64_t N, int n, const double *X, double tol, int max_iter, cudaStream_t st,
                                   cudaError_t *err, void *scratch = nullptr, size_t scratch_bytes = 0);

// Max-affine estimator f_hat(z) = max_i (y_i - a_i) + xi_i . z over this shard's rows
// (kernels/predict.cu); fp64.
struct PredictParams {
    const double *Z;       // [M][n] queries (device)
    int64_t M, Ns, row0;
    int n, splits;
    const double *y;       // [>= row0 + Ns] (global rows)
    const double *a;       // [Ns] xi_i . x_i
    const double *Xi;      // [Ns][n]
    double *part;          // [splits][M]
    double *out;           // [M]
};
int predict_splits(int64_t M, int64_t Ns, int nsm);
cudaError_t launch_predict(const PredictParams &p, cudaStream_t s);

// Step 1 for a partition K < N (kernels/block_ipm.cu): per block of nbar rows, the G-norm
// projection of (y64, Xi64) onto the intra-block constraints, in place, by a primal-dual
// interior-point method; one CTA per block, fp64.
struct BlockIpmParams {
    int nbar, n, max_iter;
    int64_t nblocks, row0;          // blocks of this shard; first global row of the shard
    double gamma, tol;
    const double *X64;              // [N][n] (global rows)
    double *y64;                    // [>= row0 + Ns] (global rows)
    double *Xi64;                   // [Rp][n] (shard rows)
    double *scratch;                // [nblocks][scratch_per_block]
    size_t scratch_per_block;
    int *iters;                     // [nblocks][8] IPM iterations, polish rounds, multiplier iterations,
                                    // status, warm start settled
    int warm;                       // 1: try the previous projection's active set first
    int smem;                       // dynamic shared memory bytes
    int lgroup;                     // points factored concurrently (block_ipm_group)
    unsigned long long *prof;       // optional [nblocks][8] clock64 phase totals (CR_IPM_PROF)
    unsigned long long *work;       // [nblocks][3] cumulative factorizations, solves, A / A^T products
};
size_t block_ipm_scratch_per_block(int nbar, int n);   // doubles
int block_ipm_group(int nbar, int n, size_t smem_max);  // 0: does not fit
size_t block_ipm_smem(int nbar, int n, int G);
cudaError_t launch_block_ipm(const BlockIpmParams &p, cudaStream_t s);
cudaError_t block_ipm_prepare(int smem);

// Column-major helpers for initialisation.
cudaError_t launch_fill_inputs(const double *X64, int64_t N, int n, int NB, int NBP, int64_t ldT,
                               int prec_fp64, void *XT, void *Xh, cudaStream_t s);
cudaError_t launch_convert_rows(const double *src, int64_t rows, int64_t N, int64_t ldT,
                                int prec_fp64, void *dst, cudaStream_t s);   // double -> storage
cudaError_t launch_unconvert_rows(const void *src, int64_t rows, int64_t N, int64_t ldT,
                                  int prec_fp64, double *dst, cudaStream_t s); // storage -> double

}  // namespace cr

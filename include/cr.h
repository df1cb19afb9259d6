/*
 * cr.h -- C ABI of libcr: the B200 (sm_100a) hot path of Aybat & Wang,
 * "A Parallelizable Dual Smoothing Method for Large Scale Convex Regression
 * Problems" (arXiv 1608.02227).  Citations "P:n" are lines of PAPER.md.
 *
 * Problem (Eq. (regularize)): given observations {(x_l, ybar_l)}
 * (Eq. (data)) and gamma > 0,
 *     min 1/2 ||y - ybar||^2 + gamma/2 ||xi||^2
 *     s.t. y_j - y_i + xi_i^T (x_i - x_j) >= 0   for all i != j   (Eq. (original)).
 * Every pair constraint is dualized (the paper's partition with K = N
 * singleton blocks, Assumption 1 P:138-143 relaxed as in DESIGN.md), so the
 * dual variable theta (Eq. (dual-problem)) is a dense nonnegative
 * N x N matrix Theta, Theta[i][j] <-> pair (l1, l2) = (i, j) in the
 * lexicographic row order of P:101-102 (packed index i(N-1) + j - [j > i]),
 * Theta[i][i] == 0.
 *
 * One call of cr_dual_step() is one iteration of the constant-step P-APG
 * method, Fig. 2:
 *   Step 1 eta^k = argmin L(eta, theta~^k): at K = N in closed form,
 *          y = ybar + c - r,  xi_i = (r_i x_i - (Theta X)_i) / gamma,
 *          r/c the row/column sums of theta~^k (Def. A1A2);
 *   Step 2 Theta^k = (theta~^k - (1/L) C eta^k)_+ ,
 *          (C eta)_ij = y_j - y_i + xi_i^T (x_i - x_j);
 *   Steps 3-4 t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2,
 *          theta~^{k+1} = Theta^k + (t_k - 1)/t_{k+1} (Theta^k - Theta^{k-1}).
 * theta~ is never stored: the fused pass reads Theta^{k-1} and Theta^{k-2}
 * and writes Theta^k over Theta^{k-2} (12 B per pair in fp32).
 *
 * Conventions
 *   - Host arrays are row-major double unless stated; they are copied, never
 *     retained.  Device workspace is owned by the caller (e.g. a torch tensor)
 *     and must outlive the context; it must be 256-byte aligned.
 *   - Every call enqueues on cfg.stream; calls that return host data
 *     synchronize that stream.
 *   - Every call returns cr_status; nothing is thrown across the ABI.
 *     CR_ERR_INVALID_ARG / CR_ERR_STATE leave the context usable (except an exhausted
 *     adaptive iteration, see cr_set_step_rule);
 *     CR_ERR_CUDA / CR_ERR_NCCL / CR_ERR_OOM poison it (only cr_destroy,
 *     cr_last_error are then allowed).  cr_last_error() holds the message.
 *   - Multi-GPU: one process per GPU; rank p owns the contiguous row block
 *     [p*S, min(N,(p+1)*S)), S = cr_shard_rows(N, world, nbar), of both Theta buffers.
 *     Per iteration ranks exchange an all-gather of y and a reduce-scatter of
 *     the column sums (NCCL); X and ybar are replicated.
 *   - Not thread-safe per context.
 */
#ifndef CR_H_
#define CR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CR_ABI_VERSION 1

typedef enum {
    CR_OK = 0,
    CR_ERR_INVALID_ARG = 1,  /* bad argument; context (if any) unchanged and usable       */
    CR_ERR_CUDA = 2,         /* CUDA runtime/launch error; context poisoned                */
    CR_ERR_NCCL = 3,         /* NCCL error; context poisoned                               */
    CR_ERR_OOM = 4,          /* workspace too small / host allocation failed               */
    CR_ERR_STATE = 5,        /* call not allowed in the current state (e.g. poisoned ctx)  */
    CR_ERR_UNSUPPORTED = 6   /* configuration not built into this library (e.g. n too big) */
} cr_status;

typedef enum {
    CR_FP32 = 0,   /* Theta, X, eta copies stored and combined in fp32; sums combined in fp64 */
    CR_FP64 = 1    /* everything fp64 (BASELINE config C1)                                     */
} cr_precision;

typedef enum {
    CR_KERNEL_AUTO = 0,  /* library picks (tensor-core pass when built and n large enough) */
    CR_KERNEL_SIMT = 1,  /* CUDA-core fused pass                                           */
    CR_KERNEL_TC = 2     /* tcgen05 (3xTF32) fused pass, fp32 only                         */
} cr_kernel;

/* Step rule of Step 2 (P:387 / P:400-407). */
typedef enum {
    CR_STEP_CONSTANT = 0,  /* step 1/L_gamma, Fig. 2 as printed                                  */
    CR_STEP_ADAPTIVE = 1,  /* step 1/s_k, s_k = s_{k-1} ups^(l_k - 1), l_k >= 0 the smallest
                              integer passing Eq. (adaptive-check); s_0 = L_gamma.
                              The step may grow every iteration; on the paper's own Section-4
                              workload at N = 2400 this diverges (R18)              */
    CR_STEP_BACKTRACK = 2  /* not in the paper: the monotone variant s_k = s_{k-1} ups^(l_k),
                              same check -- steps never grow (Beck-Teboulle backtracking, whose
                              O(1/k^2) rate holds with L -> max s_k); start below L via s_prev */
} cr_step_rule;

/* cr_config.flags */
#define CR_FLAG_P2P 2       /* multi-GPU (NCCL mode): the per-iteration exchanges over NVLink peer
                               memory instead of NCCL.  y' all-gather: the prologue stores each
                               row's y' into every rank's receive array and releases a per-source
                               row counter; a one-CTA acquire kernel copies it into the pass
                               operand.  Column-sum reduce-scatter: the reduce kernel
                               stores each column sum straight into its owner rank's receive slab
                               (CUDA IPC, mapped once in cr_init over the NCCL communicator) and
                               releases a per-source arrival counter (system scope); the owner's
                               gather kernel acquires the W counters and sums the slabs in rank
                               order.  Requires world <= 8 and shard rows S % 128 == 0 (32 for
                               fp64); CR_ERR_UNSUPPORTED otherwise.  Verified on one GPU through
                               cr_selftest_p2p / cr_selftest_p2p_allgather (all ranks in one
                               cooperative launch) and a 1-rank communicator (CR_FORCE_NCCL);
                               not yet run across GPUs.                                          */
#define CR_FLAG_ADAPTIVE 1  /* reserve a third Theta buffer + sums slot so cr_set_step_rule can
                               select CR_STEP_ADAPTIVE (a rejected trial must not overwrite
                               Theta^{k-2}); +1 Theta matrix of workspace                       */

typedef struct cr_ctx cr_ctx;
typedef struct cr_group cr_group;   /* in-process group of world contexts sharing one GPU */

typedef struct {
    int64_t N;                  /* observations, N >= 2                                       */
    int32_t n;                  /* dimension, 1 <= n <= cr_max_dim()                          */
    const double *X;            /* HOST, N x n row-major (rows xbar_l); copied          */
    const double *ybar;         /* HOST, N; copied                                      */
    double gamma;               /* Tikhonov weight gamma > 0 (Eq. (regularize))          */
    double L;                   /* > 0: step constant used as given; 0: L = sigma_max(C)^2/gamma
                                   by Lanczos (Eq. (lischitz); requires gamma <= 1)      */
    cr_precision prec;
    cr_kernel kernel;
    int32_t rank, world;        /* world >= 1, 0 <= rank < world                               */
    const void *nccl_unique_id; /* world > 1: 128-byte ncclUniqueId, identical on all ranks    */
    int32_t device;             /* CUDA device ordinal                                        */
    void *stream;               /* cudaStream_t to enqueue on (NULL = legacy default stream)   */
    void *workspace;            /* DEVICE memory, >= cr_workspace_size(...) bytes, caller-owned */
    size_t workspace_bytes;
    int32_t flags;              /* CR_FLAG_* (0: constant step only)                           */
    cr_group *local_group;      /* world > 1 without NCCL: all ranks are contexts of ONE process
                                   (one host thread each, same or different GPUs) joined by
                                   cr_local_group_create(world); NULL -> NCCL via nccl_unique_id */
    int64_t nbar;               /* partition block size Nbar (Assumption 1): 0 or 1 =
                                   every pair dualized (K = N, the paper's experiments); > 1 = K =
                                   N / Nbar blocks of consecutive rows, only cross-block pairs
                                   dualized, Step 1 = per-block G-norm projections (Eq.
                                   (subgradient_split) P:184-187) by an fp64 interior-point kernel.
                                   Requires N % Nbar == 0, Nbar <= 128, shard rows % Nbar == 0,
                                   no CR_FLAG_ADAPTIVE; else CR_ERR_UNSUPPORTED                  */
} cr_config;

/* Diagnostics of eta(Theta^k) (Theorem 1 semantics) reported per P:951 / P:1106. */
typedef struct {
    int64_t k;             /* iterations completed                                            */
    double t_k;            /* momentum scalar t_{k+1} that the next iteration will use          */
    double g;              /* dual value g_gamma(Theta^k) (Eq. (g_gamma))                 */
    double r_gamma;        /* primal objective of eta(Theta^k) (Eq. (regularize))         */
    double gap;            /* <Theta^k, C eta(Theta^k)>  ("duality gap")                 */
    double max_violation;  /* max_{i != j} (-(C eta)_ij)_+                                      */
    double infeas_norm;    /* ||(A1 y + A2 xi)_-||_2 / sqrt(N^2 - N)                 */
    int32_t nonfinite;     /* 1 if a NaN/Inf was seen in the reported quantities               */
} cr_step_stats;

typedef struct {
    int32_t report_every;  /* evaluate the test every m iterations (m >= 1)                    */
    double infeas_tol;     /* stop when infeas_norm <= infeas_tol (paper: 1e-1) ...    */
    double gap_tol;        /* ... and |gap| / (N^2 - N) <= gap_tol (paper: 5e-7)       */
} cr_stop;

typedef struct {
    int64_t iters;         /* iterations run by this call                                     */
    int32_t converged;     /* 1 if the stop test fired                                         */
    cr_step_stats last;    /* stats at exit (only when stop != NULL)                           */
} cr_report;

/* Bytes of device workspace cr_init needs for this shape / rank / flags (0 if unsupported). */
size_t cr_workspace_size(int64_t N, int32_t n, cr_precision prec, cr_kernel kernel,
                         int32_t rank, int32_t world, int32_t flags);

/* Same with a partition block size (cr_config.nbar; 0 or 1 = all pairs). */
size_t cr_workspace_size_ex(int64_t N, int32_t n, cr_precision prec, cr_kernel kernel,
                            int32_t rank, int32_t world, int32_t flags, int64_t nbar);

/* Largest n this library was built for. */
int32_t cr_max_dim(void);

/* Debug: the first ring-protocol violation the tensor-core pass recorded since cr_init, when the
 * context was created with CR_TC_CHECK=1 in the environment (0 = none, or checks off; ~0 on a CUDA
 * error).  Layout: (code << 56) | (CTA << 32) | tile index; codes: 1/2/3 Theta slot seen by the
 * epilogue / GEMM1 / storer holds another tile, 4/5 X_J / X_J^T slot, 6 Theta^k A operand,
 * 7 Xi' run.  With CR_TC_G1_RUNAHEAD=1, GEMM1 no longer waits for the tile's Theta.  Synchronizes. */
uint64_t cr_tc_check_word(cr_ctx *ctx);

/* Rows S of each rank's shard (rank p owns [p*S, min(N, (p+1)*S))): ceil(N/world), rounded up to
 * a multiple of 128 when world > 1, nbar <= 1 and every rank still owns at least one row (so the
 * peer-memory column-sum exchange, whose 128-column blocks must not straddle owners, covers
 * shapes like N = 4000 at 2/4/8 ranks); a partition (nbar > 1) keeps ceil(N/world), which must
 * be a multiple of nbar.  0 for N < 1 or world < 1.  Host-only; no device needed. */
int64_t cr_shard_rows(int64_t N, int32_t world, int64_t nbar);

/* In-process group for world > 1 contexts driven by `world` host threads of one process
 * (tests run the row-sharded path on one GPU this way).  Its collectives are host rendezvous
 * of the rank threads plus cross-stream event dependencies, copies and a fixed-order sum
 * kernel -- no kernel ever waits on another.  CUDA graphs are not used by contexts in a local
 * group.  A rank that does not arrive within 120 s breaks the group (CR_ERR_NCCL).
 * 1 <= world <= 16.  Destroy after all member contexts. */
cr_status cr_local_group_create(int32_t world, cr_group **out);
void cr_local_group_destroy(cr_group *g);

/* world > 1 bootstrap: write a fresh 128-byte ncclUniqueId into out (host memory).  Rank 0
 * calls this and broadcasts the bytes to the other ranks (e.g. over torch.distributed). */
cr_status cr_nccl_get_unique_id(void *out);

/* Validate cfg, copy X/ybar to the device, compute L if cfg->L == 0 (Lanczos, host fp64),
 * initialise the NCCL communicator (world > 1), set Theta^0 = 0, t_1 = 1.
 * On success *out owns the context; on failure *out = NULL. */
cr_status cr_init(const cr_config *cfg, cr_ctx **out);

/* Load a full APG state: Theta^{k-1} and Theta^{k-2} (HOST, this rank's rows x N, zero
 * diagonal; NULL means all-zero) and the scalars t_{k-1}, t_k, so that the next
 * cr_dual_step forms theta~^k = Theta^{k-1} + (t_{k-1}-1)/t_k (Theta^{k-1} - Theta^{k-2}).
 * The paper's start is (Theta^0, Theta^0, 1, 1).  Values are rounded to the
 * storage precision.  Negative or non-finite entries: CR_ERR_INVALID_ARG. */
cr_status cr_set_theta(cr_ctx *ctx, const double *theta_km1, const double *theta_km2,
                       double t_km1, double t_k);

/* Read back the state: Theta^k, Theta^{k-1} (HOST, rows x N each, either may be NULL)
 * and t_k, t_{k+1} -- exactly the arguments cr_set_theta takes to continue. */
cr_status cr_get_theta(cr_ctx *ctx, double *theta_k, double *theta_km1, double *t_k,
                       double *t_kp1);

/* Read rows [row0, row0 + nrows) (local to this rank) of Theta^k (which = 0) or
 * Theta^{k-1} (which = 1) into HOST out (nrows x N). */
cr_status cr_get_theta_rows(cr_ctx *ctx, int32_t which, int64_t row0, int64_t nrows,
                            double *out);

/* One P-APG iteration (Fig. 2).  If out != NULL, also evaluates eta(Theta^k) and the
 * diagnostics (one extra read-only pass over Theta^k) and synchronizes. */
cr_status cr_dual_step(cr_ctx *ctx, cr_step_stats *out);

/* Run up to max_iters iterations (CUDA-graph replay).  stop == NULL: exactly max_iters,
 * no synchronisation.  Otherwise evaluates the paper's stopping pair every
 * stop->report_every iterations and returns early when both hold. */
cr_status cr_solve(cr_ctx *ctx, int64_t max_iters, const cr_stop *stop, cr_report *out);

/* Final estimator eta(Theta^k) (Theorem 1): y (HOST, all N) and xi (HOST, this
 * rank's rows x n), either may be NULL; optional diagnostics.  Synchronizes. */
cr_status cr_primal(cr_ctx *ctx, double *y, double *xi, cr_step_stats *out);

/* eta^k = Step-1 minimizer of the most recent iteration (eta(theta~^k)), or of the most
 * recent cr_primal: y (HOST, all N), xi (HOST, this rank's rows x n). */
cr_status cr_get_eta(cr_ctx *ctx, double *y, double *xi);

/* The linear sums of Theta^k (which = 0) or Theta^{k-1} (which = 1) that Step 1 of the next
 * iteration combines (Def. A1A2: A1^T theta = c - r, A2^T theta = r x - Theta X):
 * r (HOST, this rank's rows), c (HOST, this rank's rows; column sums over ALL rows of all
 * ranks), P (HOST, rows x n, Theta X).  Any pointer may be NULL.  Synchronizes. */
cr_status cr_get_sums(cr_ctx *ctx, int32_t which, double *r, double *c, double *P);

/* Select the step rule for subsequent cr_dual_step / cr_solve calls.
 *   CR_STEP_CONSTANT: 1/L (upsilon, s_prev ignored).
 *   CR_STEP_ADAPTIVE (needs CR_FLAG_ADAPTIVE at cr_init, else CR_ERR_STATE): growth factor
 *     upsilon > 1 (the paper leaves it open; 2 is the usual choice), s_prev = s_{k-1} the
 *     next iteration starts from (0 -> L_gamma, the paper's s_0).  Each iteration
 *     evaluates trials l = 0, 1, ... : a prologue + fused pass + reduce writing the trial
 *     Theta^k into the spare buffer, and the check of Eq. (adaptive-check) evaluated as
 *         ||A1^T D||^2 + ||A2^T D||^2 / gamma <= s ||D||^2,   D = Theta^k - theta~^k,
 *     which is the same inequality because g_gamma is quadratic at K = N (R15);
 *     one host synchronisation per trial (a trial whose Theta^k overflows the storage
 *     precision counts as failing).  An iteration whose 64 trials all fail returns
 *     CR_ERR_STATE and POISONS the context (t_k was not advanced and the spare buffer holds a
 *     rejected trial, so no valid iterate remains; cr_solve reports it at its next stop test or
 *     at its end, the failed iteration's successors being no-ops on the device).
 * Errors: CR_ERR_INVALID_ARG for a bad rule / upsilon / s_prev (context unchanged). */
cr_status cr_set_step_rule(cr_ctx *ctx, cr_step_rule rule, double upsilon, double s_prev);

/* s_k of the last accepted step (L for the constant rule), trials l_k + 1 of the last
 * adaptive iteration and the total number of adaptive trials; any pointer may be NULL. */
cr_status cr_step_info(cr_ctx *ctx, double *s_k, int64_t *trials_last, int64_t *trials_total);

/* Self-test of the CR_FLAG_P2P protocol on the current device: `world` virtual ranks, each with
 * nrb rows of fp32 column partials (HOST colpart[world][nrb][N], the fused pass's layout), run
 * the production column-sum blocks (push into the owners' slabs + release) and owner gathers
 * (acquire + rank-order sum) in ONE cooperative launch; c (HOST, N) receives every owner's
 * slice = the column sums over all ranks and rows.  1 <= world <= 8, cr_shard_rows(N, world, 1)
 * % 128 == 0 (else CR_ERR_UNSUPPORTED); CR_ERR_CUDA on a CUDA error. */
cr_status cr_selftest_p2p(int32_t world, int64_t N, int32_t nrb, const float *colpart, double *c);

/* Self-test of the CR_FLAG_P2P y' all-gather on the current device: `world` virtual ranks each
 * push their rows [r S, min(N, (r+1) S)) of y (HOST, N) to every rank's receive array with
 * per-CTA release counters (the prologue's code path) and each rank acquires all and copies
 * them out, in ONE cooperative launch; out (HOST, world x N) = every rank's gathered vector. */
cr_status cr_selftest_p2p_allgather(int32_t world, int64_t N, const float *y, float *out);

/* Partition diagnostics (cr_config.nbar) of the block projections of this rank's LAST Step 1. */
typedef struct {
    int64_t nbar;                  /* block size in use (1: K = N, nothing below is set)          */
    int64_t blocks;                /* blocks of this rank                                         */
    int32_t ipm_iters_max;         /* interior-point iterations (limit 100)                       */
    int32_t polish_rounds_max;     /* active-set rounds of the polish (limit 6)                   */
    int32_t multiplier_iters_max;  /* multiplier iterations per penalty (limit 60; rho 1, 10, 100) */
    int64_t failed_blocks;         /* blocks whose IPM did not meet its tolerance (relative
                                      residuals and max complementarity 1e-9, 100 iterations)    */
    int64_t unpolished_blocks;     /* blocks whose polish did not settle: they keep the IPM point
                                      (feasible to ~1e-9 relative, not exact)                     */
    int64_t warm_blocks;           /* blocks solved from the previous Step 1's active set and
                                      multipliers alone (exact; no interior-point run;
                                      CR_IPM_COLD=1 in the environment disables the warm start)   */
    int64_t factorizations;        /* cumulative since cr_init, summed over this rank's blocks:   */
    int64_t solves;                /*   normal-matrix factorizations, solves with them, and       */
    int64_t products;              /*   A / A^T products (the work model of DESIGN.md §9)         */
    double timed_ms;               /* summed duration of the block-projection launches of the
                                      last pass-timing window (cr_set_pass_timing / cr_pass_timing) */
    int64_t timed_launches;
} cr_partition_stats;

/* Synchronizes.  CR_ERR_STATE (and *out filled) if failed_blocks > 0. */
cr_status cr_partition_info(cr_ctx *ctx, cr_partition_stats *out);

/* Change the Tikhonov weight (Eq. (regularize)) of the problem being solved and restart
 * Fig. 2 at the current iterate: theta^0 := Theta^k, theta~^1 = theta^0, t_1 = 1.
 * L > 0 is used as given; L == 0 uses sigma_max(C)^2 / gamma with the sigma_max(C)^2 this
 * context holds (= L * gamma of cr_init; Eq. (lischitz), valid for gamma <= 1).  Under
 * the adaptive rule s is reset to the new L.  Errors: CR_ERR_INVALID_ARG. */
cr_status cr_set_gamma(cr_ctx *ctx, double gamma, double L);

/* Continuation over gamma (Section 2.4.1).  Outer stages t = 1..stages:
 *   eps_t = eps0 / beta^t,  gamma_t = kappa_gamma * eps_t  (must lie in (0, 1]),
 *   theta^(t) = P-APG on the gamma_t problem started from theta^(t-1) (cr_set_gamma(gamma_t, 0)
 *   then cr_solve), theta^(0) = the context's current Theta^k (0 after cr_init),
 * each stage running iters[t-1] iterations (HOST array of `stages` budgets, the K_t of P:580,
 * which the paper bounds a priori but leaves to the user), or iters_per_stage when iters is
 * NULL, ending early when `stop` (nullable) holds -- the stopping pair of P:1106, as in cr_solve.
 * The step rule in force (cr_set_step_rule) is used inside the stages. */
typedef struct {
    double eps0;              /* eps_0 > 0                                   */
    double beta;              /* beta > 1                                    */
    double kappa_gamma;       /* kappa_gamma > 0                             */
    int32_t stages;           /* T >= 1                                      */
    const int64_t *iters;     /* HOST [stages] or NULL                       */
    int64_t iters_per_stage;  /* used when iters == NULL (>= 0)              */
    const cr_stop *stop;      /* nullable                                    */
} cr_cont;

typedef struct {
    int32_t stages_run;
    int64_t iters_total;
    double gamma_last, L_last;
    cr_step_stats last;       /* diagnostics of eta(Theta) on the gamma_last problem */
} cr_cont_report;

cr_status cr_continuation(cr_ctx *ctx, const cr_cont *params, cr_cont_report *out);

/* The fitted estimator at query points: with (y, xi) = eta(Theta^k) (Theorem 1,
 * P:243), f_hat(z) = max_i  y_i + xi_i^T (z - x_i), the max-affine function the pair
 * constraints certify (it interpolates y when every constraint holds).  Z: HOST, M x n
 * row-major; out: HOST, M.  fp64 on the device; with world > 1 each rank maximises over its
 * rows and the ranks all-reduce (max), so every rank returns the full result.  Synchronizes.
 * Errors: CR_ERR_INVALID_ARG (M < 0, NULL pointers with M > 0, non-finite Z). */
cr_status cr_predict(cr_ctx *ctx, const double *Z, int64_t M, double *out);

/* Step constant in use (L_gamma of the current gamma). */
double cr_lipschitz(const cr_ctx *ctx);

/* Host-only: L = sigma_max(C)^2 / gamma by fp64 Lanczos on the structured C^T C
 * (Eq. (lischitz); Lemma 4 P:476 bounds it).  No device needed. */
cr_status cr_lipschitz_host(int64_t N, int32_t n, const double *X, double gamma, double *L_out);

/* Kernel-level accounting: number of kernels this context launched (all calls). */
int64_t cr_launch_count(const cr_ctx *ctx);

/* Per-launch timing of the fused pair pass: when on, CUDA events bracket every pass
 * launch on the context stream.  cr_pass_timing synchronizes and returns the summed
 * pass time (ms) and number of timed launches since the last reset. */
cr_status cr_set_pass_timing(cr_ctx *ctx, int32_t on);
cr_status cr_pass_timing(cr_ctx *ctx, double *total_ms, int64_t *launches);

/* Which fused-pass kernel the context uses (CR_KERNEL_SIMT or CR_KERNEL_TC). */
cr_kernel cr_active_kernel(const cr_ctx *ctx);

const char *cr_last_error(const cr_ctx *ctx);
const char *cr_status_string(cr_status s);
void cr_destroy(cr_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CR_H_ */

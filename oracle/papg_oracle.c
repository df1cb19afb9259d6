/*
 * oracle/papg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of the constant-step
 * P-APG iteration of Aybat & Wang (arXiv 1608.02227), Fig. 2
 * (P:377-397), with every pair constraint dualized (partition K = N singleton
 * blocks, so Q = R^{N(n+1)} and C = [A1 A2], Def. C).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header or
 * constant with the CUDA path (paper_1608_02227_b200/), and never reads it.
 *
 * Notation:
 *   X      N x n row-major, rows xbar_l
 *   ybar   N
 *   Theta  dense N x N row-major; Theta[i][j] is the multiplier of the pair
 *          constraint (l1,l2)=(i,j):  y_j - y_i + xi_i^T (x_i - x_j) >= 0
 *          (Eq. (original), row order P:101-102).  Theta[i][i] == 0.
 *   L      step constant, Eq. (lischitz), passed in by the caller.
 *
 * Step 1 at K = N has no constraints, so its minimizer is the
 * stationary point of Eq. (g_gamma) P:365:
 *     y  = ybar + A1^T theta,   gamma * xi = A2^T theta,
 * with A1, A2 from Def. A1A2:
 *     (A1^T theta)_l = sum_{i != l} Theta[i][l] - sum_{j != l} Theta[l][j]
 *     (A2^T theta)_l = sum_{j != l} Theta[l][j] (x_l - x_j)
 * Step 2:  Theta^k = ( Theta~^k - (1/L) C eta^k )_+ ,
 *     (C eta)_{ij} = y_j - y_i + xi_i^T (x_i - x_j).
 * Steps 3-4: t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2,
 *     Theta~^{k+1} = Theta^k + ((t_k - 1)/t_{k+1}) (Theta^k - Theta^{k-1}).
 *
 * Summation order: fixed (row blocks of ORACLE_RB rows summed in increasing
 * order), so results do not depend on the OpenMP thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_RB 256

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Step 1 closed form at K = N:  y = ybar + A1^T theta,
 * xi_l = (1/gamma) sum_{j != l} Theta[l][j] (x_l - x_j)   ("direct form"). */
static int step1(int64_t N, int n, const double *X, const double *ybar, double gamma,
                 const double *T, double *y, double *xi)
{
    int64_t nb = (N + ORACLE_RB - 1) / ORACLE_RB;
    double *colpart = (double *)calloc((size_t)(nb * N), sizeof(double));
    double *rowsum = (double *)calloc((size_t)N, sizeof(double));
    if (!colpart || !rowsum) { free(colpart); free(rowsum); return 1; }

    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        double *cp = colpart + b * N;
        int64_t i1 = (b + 1) * ORACLE_RB < N ? (b + 1) * ORACLE_RB : N;
        for (int64_t i = b * ORACLE_RB; i < i1; ++i) {
            const double *Ti = T + i * N;
            const double *xi_ = X + i * n;
            double r = 0.0;
            double *xii = xi + i * n;
            for (int d = 0; d < n; ++d) xii[d] = 0.0;
            for (int64_t j = 0; j < N; ++j) {
                if (j == i) continue;
                double t = Ti[j];
                r += t;
                cp[j] += t;
                const double *xj = X + j * n;
                for (int d = 0; d < n; ++d) xii[d] += t * (xi_[d] - xj[d]);
            }
            rowsum[i] = r;
            for (int d = 0; d < n; ++d) xii[d] /= gamma;
        }
    }
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < N; ++j) {
        double c = 0.0;
        for (int64_t b = 0; b < nb; ++b) c += colpart[b * N + j];
        y[j] = ybar[j] + (c - rowsum[j]);
    }
    free(colpart);
    free(rowsum);
    return 0;
}

/* (C eta)_{ij} = y_j - y_i + xi_i^T (x_i - x_j)   (Eq. (original), Def. A1A2). */
static inline double pair_residual(int n, const double *X, const double *y, const double *xi,
                                   int64_t i, int64_t j)
{
    const double *xi_i = xi + i * n, *x_i = X + i * n, *x_j = X + j * n;
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += xi_i[d] * (x_i[d] - x_j[d]);
    return y[j] - y[i] + s;
}

/* eta(Theta): Step-1 formulas on a given multiplier matrix (Theorem 1). */
int oracle_eta(int64_t N, int n, const double *X, const double *ybar, double gamma,
               const double *T, double *y, double *xi, int nthreads)
{
    set_threads(nthreads);
    return step1(N, n, X, ybar, gamma, T, y, xi);
}

/*
 * K iterations of P-APG (Fig. 2).  State in/out:
 *   Tprev : theta^{k-1}        (at k = 1: theta^0)
 *   Tt    : theta~^k           (at k = 1: theta~^1 = theta^0)
 *   t     : t_k                (at k = 1: t_1 = 1)
 * After the call: Tprev = theta^{k+K-1}, Tt = theta~^{k+K}, *t = t_{k+K}.
 * y_out/xi_out (nullable) receive eta^{k+K-1} = Step 1 of the last iteration.
 */
int oracle_papg(int64_t N, int n, const double *X, const double *ybar, double gamma, double L,
                int64_t K, double *Tprev, double *Tt, double *t, double *y_out, double *xi_out,
                int nthreads)
{
    set_threads(nthreads);
    double *y = (double *)malloc((size_t)N * sizeof(double));
    double *xi = (double *)malloc((size_t)(N * n) * sizeof(double));
    if (!y || !xi) { free(y); free(xi); return 1; }
    for (int64_t k = 0; k < K; ++k) {
        /* Step 1: eta^k = argmin L(eta, theta~^k). */
        if (step1(N, n, X, ybar, gamma, Tt, y, xi)) { free(y); free(xi); return 1; }
        /* Step 3. */
        double tk = *t;
        double tn = (1.0 + sqrt(1.0 + 4.0 * tk * tk)) / 2.0;
        double beta = (tk - 1.0) / tn;
        /* Step 2 and Step 4, element by element. */
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < N; ++i) {
            double *Tti = Tt + i * N, *Tpi = Tprev + i * N;
            for (int64_t j = 0; j < N; ++j) {
                double tnew = 0.0;                       /* no constraint for l1 == l2 */
                if (j != i) {
                    double R = pair_residual(n, X, y, xi, i, j);
                    double v = Tti[j] - R / L;
                    tnew = v > 0.0 ? v : 0.0;            /* ( . )_+ */
                }
                Tti[j] = tnew + beta * (tnew - Tpi[j]);
                Tpi[j] = tnew;
            }
        }
        *t = tn;
    }
    if (y_out) memcpy(y_out, y, (size_t)N * sizeof(double));
    if (xi_out) memcpy(xi_out, xi, (size_t)(N * n) * sizeof(double));
    free(y);
    free(xi);
    return 0;
}

/*
 * Primal quality of eta = (y, xi) against multipliers Theta, as reported in
 * PAPER.md §4:
 *   stats[0] r_gamma = 1/2 ||y - ybar||^2 + gamma/2 ||xi||^2      (Eq. (regularize))
 *   stats[1] g       = r_gamma - <theta, C eta>                    (Eq. (g_gamma) P:365 at its
 *                                                                   minimizer, i.e. g_gamma(theta)
 *                                                                   when eta = eta(theta))
 *   stats[2] gap     = <theta, C eta>                              ("duality gap")
 *   stats[3] max_{i != j} ( -(C eta)_{ij} )_+                      (max constraint violation)
 *   stats[4] ||(A1 y + A2 xi)_-||_2 / sqrt(N^2 - N)                (normalized infeasibility)
 */
int oracle_stats(int64_t N, int n, const double *X, const double *ybar, double gamma,
                 const double *T, const double *y, const double *xi, double *stats, int nthreads)
{
    set_threads(nthreads);
    int64_t nb = (N + ORACLE_RB - 1) / ORACLE_RB;
    double *gp = (double *)calloc((size_t)nb, sizeof(double));
    double *vp = (double *)calloc((size_t)nb, sizeof(double));
    double *mp = (double *)calloc((size_t)nb, sizeof(double));
    if (!gp || !vp || !mp) { free(gp); free(vp); free(mp); return 1; }
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        int64_t i1 = (b + 1) * ORACLE_RB < N ? (b + 1) * ORACLE_RB : N;
        double g = 0.0, v = 0.0, m = 0.0;
        for (int64_t i = b * ORACLE_RB; i < i1; ++i)
            for (int64_t j = 0; j < N; ++j) {
                if (j == i) continue;
                double R = pair_residual(n, X, y, xi, i, j);
                if (T) g += T[i * N + j] * R;
                if (R < 0.0) { v += R * R; if (-R > m) m = -R; }
            }
        gp[b] = g; vp[b] = v; mp[b] = m;
    }
    double gap = 0.0, viol2 = 0.0, maxv = 0.0;
    for (int64_t b = 0; b < nb; ++b) { gap += gp[b]; viol2 += vp[b]; if (mp[b] > maxv) maxv = mp[b]; }
    double ry = 0.0, rx = 0.0;
    for (int64_t i = 0; i < N; ++i) { double u = y[i] - ybar[i]; ry += u * u; }
    for (int64_t i = 0; i < N * n; ++i) rx += xi[i] * xi[i];
    double rg = 0.5 * ry + 0.5 * gamma * rx;
    stats[0] = rg;
    stats[1] = rg - gap;
    stats[2] = gap;
    stats[3] = maxv;
    stats[4] = sqrt(viol2) / sqrt((double)N * (double)N - (double)N);
    free(gp); free(vp); free(mp);
    return 0;
}

/*
 * Step 2 for a subset of rows, given eta^k = (y, xi) for all rows and
 * the rows of theta~^k:  out[r][j] = ( Tt_rows[r][j] - (C eta)_{i_r j} / L )_+ ,
 * out[r][i_r] = 0.  Used by full-size sampled parity tests.
 */
int oracle_project_rows(int64_t N, int n, const double *X, const double *y, const double *xi,
                        double L, const int64_t *rows, int64_t nrows, const double *Tt_rows,
                        double *out, int nthreads)
{
    set_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        for (int64_t j = 0; j < N; ++j) {
            double tnew = 0.0;
            if (j != i) {
                double v = Tt_rows[r * N + j] - pair_residual(n, X, y, xi, i, j) / L;
                tnew = v > 0.0 ? v : 0.0;
            }
            out[r * N + j] = tnew;
        }
    }
    return 0;
}

/*
 * g_gamma(theta) at its Step-1 minimizer (Eq. (g_gamma)):
 *     g(theta) = 1/2 ||y - ybar||^2 + gamma/2 ||xi||^2 - <theta, C eta(theta)>,
 * with eta(theta) = (y, xi) from step1().  Pair terms summed in row-block order.
 */
static int dual_value(int64_t N, int n, const double *X, const double *ybar, double gamma,
                      const double *T, const double *y, const double *xi, double *g_out)
{
    int64_t nb = (N + ORACLE_RB - 1) / ORACLE_RB;
    double *gp = (double *)calloc((size_t)nb, sizeof(double));
    if (!gp) return 1;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        int64_t i1 = (b + 1) * ORACLE_RB < N ? (b + 1) * ORACLE_RB : N;
        double s = 0.0;
        for (int64_t i = b * ORACLE_RB; i < i1; ++i)
            for (int64_t j = 0; j < N; ++j)
                if (j != i) s += T[i * N + j] * pair_residual(n, X, y, xi, i, j);
        gp[b] = s;
    }
    double tc = 0.0, ry = 0.0, rx = 0.0;
    for (int64_t b = 0; b < nb; ++b) tc += gp[b];
    for (int64_t i = 0; i < N; ++i) { double u = y[i] - ybar[i]; ry += u * u; }
    for (int64_t i = 0; i < N * n; ++i) rx += xi[i] * xi[i];
    *g_out = 0.5 * ry + 0.5 * gamma * rx - tc;
    free(gp);
    return 0;
}

/*
 * K iterations of P-APG with the paper's adaptive step rule ("PAPG_A"):
 * Step 2 uses 1/s_k instead of 1/L_gamma, where s_k = s_{k-1} * ups^(l_k - 1) and l_k >= 0
 * is the smallest integer for which Eq. (adaptive-check) holds:
 *     g(theta^k) >= g(theta~^k) + <grad g(theta~^k), theta^k - theta~^k>
 *                   - (s_k/2) ||theta^k - theta~^k||^2,
 * grad g(theta~^k) = -C eta^k (Eq. (dual gradient) P:370), theta^k = (theta~^k - C eta^k / s_k)_+.
 * Steps 1, 3, 4 as in oracle_papg.  s_0 = L_gamma is the caller's initial *s.
 * State in/out as oracle_papg plus *s = s_{k-1} (in) / s_{k+K-1} (out).
 * trials[k] (nullable) = l_k + 1 (number of Step-2 evaluations), s_hist[k] (nullable) = s_k.
 * max_trials bounds l_k + 1 (returns 2 if exceeded).
 * backtrack != 0 selects the monotone variant s_k = s_{k-1} ups^(l_k) (not in the paper; see
 * DESIGN.md R18): with it the accepted s_k never decrease.
 */
int oracle_papg_adaptive(int64_t N, int n, const double *X, const double *ybar, double gamma, double ups,
                         int64_t K, double *Tprev, double *Tt, double *t, double *s, int64_t *trials,
                         double *s_hist, double *y_out, double *xi_out, int max_trials, int backtrack,
                         int nthreads)
{
    set_threads(nthreads);
    double *y = (double *)malloc((size_t)N * sizeof(double));
    double *xi = (double *)malloc((size_t)(N * n) * sizeof(double));
    double *y2 = (double *)malloc((size_t)N * sizeof(double));
    double *xi2 = (double *)malloc((size_t)(N * n) * sizeof(double));
    double *Tn = (double *)malloc((size_t)(N * N) * sizeof(double));
    int64_t nb = (N + ORACLE_RB - 1) / ORACLE_RB;
    double *lp = (double *)calloc((size_t)nb, sizeof(double));
    double *qp = (double *)calloc((size_t)nb, sizeof(double));
    int rc = 0;
    if (!y || !xi || !y2 || !xi2 || !Tn || !lp || !qp) { rc = 1; goto done; }
    for (int64_t k = 0; k < K; ++k) {
        /* Step 1 at theta~^k and g(theta~^k). */
        double g_t;
        if (step1(N, n, X, ybar, gamma, Tt, y, xi) || dual_value(N, n, X, ybar, gamma, Tt, y, xi, &g_t)) {
            rc = 1; goto done;
        }
        const double s_prev = *s;
        double s_k = 0.0;
        int l;
        for (l = 0; l < max_trials; ++l) {
            /* paper's rule: s_k = s_{k-1} ups^(l-1) (a step may grow); backtrack != 0: the monotone
               variant s_k = s_{k-1} ups^l (steps never grow; Beck & Teboulle's backtracking) */
            s_k = s_prev * pow(ups, backtrack ? (double)l : (double)l - 1.0);
            /* Step 2 with step 1/s_k; <grad g(theta~), D> = -sum R D, ||D||^2. */
            #pragma omp parallel for schedule(dynamic, 1)
            for (int64_t b = 0; b < nb; ++b) {
                int64_t i1 = (b + 1) * ORACLE_RB < N ? (b + 1) * ORACLE_RB : N;
                double lin = 0.0, sq = 0.0;
                for (int64_t i = b * ORACLE_RB; i < i1; ++i)
                    for (int64_t j = 0; j < N; ++j) {
                        double tnew = 0.0, R = 0.0;
                        if (j != i) {
                            R = pair_residual(n, X, y, xi, i, j);
                            double v = Tt[i * N + j] - R / s_k;
                            tnew = v > 0.0 ? v : 0.0;
                        }
                        Tn[i * N + j] = tnew;
                        double D = tnew - Tt[i * N + j];
                        lin += -R * D;
                        sq += D * D;
                    }
                lp[b] = lin;
                qp[b] = sq;
            }
            double lin = 0.0, sq = 0.0;
            for (int64_t b = 0; b < nb; ++b) { lin += lp[b]; sq += qp[b]; }
            double g_new;
            if (step1(N, n, X, ybar, gamma, Tn, y2, xi2) ||
                dual_value(N, n, X, ybar, gamma, Tn, y2, xi2, &g_new)) { rc = 1; goto done; }
            if (g_new >= g_t + lin - 0.5 * s_k * sq) break;      /* Eq. (adaptive-check) */
        }
        if (l == max_trials) { rc = 2; goto done; }
        if (trials) trials[k] = l + 1;
        if (s_hist) s_hist[k] = s_k;
        *s = s_k;
        /* Steps 3-4. */
        double tk = *t;
        double tn = (1.0 + sqrt(1.0 + 4.0 * tk * tk)) / 2.0;
        double beta = (tk - 1.0) / tn;
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < N * N; ++e) {
            double tnew = Tn[e];
            Tt[e] = tnew + beta * (tnew - Tprev[e]);
            Tprev[e] = tnew;
        }
        *t = tn;
    }
    if (y_out) memcpy(y_out, y, (size_t)N * sizeof(double));
    if (xi_out) memcpy(xi_out, xi, (size_t)(N * n) * sizeof(double));
done:
    free(y); free(xi); free(y2); free(xi2); free(Tn); free(lp); free(qp);
    return rc;
}

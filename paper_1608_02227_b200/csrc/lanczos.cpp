// L_gamma = sigma_max(C)^2 / gamma  (Eq. (lischitz)), host fp64.
//
// sigma_max(C)^2 = lambda_max(C^T C), C = [A1 A2] (all pairs dualized).  C^T C is never
// formed: for an input vector v = (y, xi) the product uses the pair residual
// z_kl = y_l - y_k + a_k - xi_k^T x_l  (a_k = xi_k^T x_k; z_kk = 0 so sums may include l = k)
// and its row / column sums in O(N n^2) instead of O(N^2 n):
//   rho_k          = sum_l z_kl = Y - N y_k + N a_k - xi_k^T s
//   (A1^T z)_k     = sum_m z_mk - rho_k
//                  = 2N y_k - 2Y + sum a - (sum_m xi_m)^T x_k - N a_k + xi_k^T s
//   (A2^T z)_k     = sum_l z_kl (x_k - x_l) = x_k rho_k - w + (y_k - a_k) s + S2 xi_k
// with Y = sum y, s = sum x_l, w = X^T y, S2 = X^T X   (rows of A1, A2 from Def. A1A2).
// The extreme eigenvalue is found by plain Lanczos (three-term recurrence, no
// re-orthogonalisation: loss of orthogonality only duplicates converged Ritz values), with
// the largest Ritz value of the tridiagonal T_m computed by Sturm-sequence bisection.
// Start vector: deterministic splitmix64 hash, so every rank gets the same L.
#include <cmath>
#include <cstdint>
#include <vector>
#include <algorithm>

namespace cr {
namespace {

struct CtC {
    int64_t N;
    int n;
    const double *X;
    std::vector<double> s, S2;
    CtC(int64_t N_, int n_, const double *X_) : N(N_), n(n_), X(X_), s(n_, 0.0), S2((size_t)n_ * n_, 0.0) {
        for (int64_t l = 0; l < N; ++l)
            for (int d = 0; d < n; ++d) s[d] += X[l * n + d];
        #pragma omp parallel for if ((int64_t)N * n * n > (1 << 20))   // small problems: no thread wake-ups
        for (int d = 0; d < n; ++d)
            for (int e = 0; e < n; ++e) {
                double acc = 0.0;
                for (int64_t l = 0; l < N; ++l) acc += X[l * n + d] * X[l * n + e];
                S2[(size_t)d * n + e] = acc;
            }
    }
    void apply(const double *v, double *out) const {
        const double *y = v, *xi = v + N;
        double Y = 0.0, Sa = 0.0;
        std::vector<double> a(N), Sxi(n, 0.0), w(n, 0.0);
        for (int64_t k = 0; k < N; ++k) {
            double ak = 0.0;
            for (int d = 0; d < n; ++d) ak += xi[k * n + d] * X[k * n + d];
            a[k] = ak;
            Y += y[k];
            Sa += ak;
            for (int d = 0; d < n; ++d) { Sxi[d] += xi[k * n + d]; w[d] += y[k] * X[k * n + d]; }
        }
        const double Nd = (double)N;
        #pragma omp parallel for schedule(static) if ((int64_t)N * n * n > (1 << 20))
        for (int64_t k = 0; k < N; ++k) {
            const double *xk = X + k * n, *xik = xi + k * n;
            double xs = 0.0, sx = 0.0;
            for (int d = 0; d < n; ++d) { xs += xik[d] * s[d]; sx += Sxi[d] * xk[d]; }
            const double rho = Y - Nd * y[k] + Nd * a[k] - xs;
            out[k] = 2.0 * Nd * y[k] - 2.0 * Y + Sa - sx - Nd * a[k] + xs;
            double *ok = out + N + k * n;
            for (int d = 0; d < n; ++d) {
                double t = 0.0;
                const double *row = S2.data() + (size_t)d * n;
                for (int e = 0; e < n; ++e) t += row[e] * xik[e];
                ok[d] = xk[d] * rho - w[d] + (y[k] - a[k]) * s[d] + t;
            }
        }
    }
};

// number of eigenvalues of the symmetric tridiagonal (alpha, beta) that are < x
int sturm_count(const std::vector<double> &al, const std::vector<double> &be, double x) {
    int cnt = 0;
    double q = al[0] - x;
    if (q < 0) ++cnt;
    for (size_t i = 1; i < al.size(); ++i) {
        double qq = q != 0.0 ? q : 1e-300;
        q = al[i] - x - be[i - 1] * be[i - 1] / qq;
        if (q < 0) ++cnt;
    }
    return cnt;
}

double max_ritz(const std::vector<double> &al, const std::vector<double> &be) {
    double lo = al[0], hi = al[0];
    for (size_t i = 0; i < al.size(); ++i) {
        double r = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i + 1 < al.size() ? std::fabs(be[i]) : 0.0);
        lo = std::min(lo, al[i] - r);
        hi = std::max(hi, al[i] + r);
    }
    const int m = (int)al.size();
    for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::fabs(hi)); ++it) {
        double mid = 0.5 * (lo + hi);
        if (sturm_count(al, be, mid) < m) lo = mid;   // some eigenvalue >= mid
        else hi = mid;
    }
    return 0.5 * (lo + hi);
}

uint64_t splitmix(uint64_t &x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace

// Largest Ritz value of the tridiagonal (al[0..m), be[0..m-1)) (shared with the device Lanczos).
double lanczos_max_ritz(const double *al, const double *be, int m) {
    return max_ritz(std::vector<double>(al, al + m), std::vector<double>(be, be + std::max(0, m - 1)));
}

// The deterministic unit start vector (splitmix64 hash; every rank gets the same one).
void lanczos_start(int64_t N, int n, double *v) {
    const int64_t dim = N * (int64_t)(n + 1);
    uint64_t seed = 0x1608022270000001ull;
    double nrm = 0.0;
    for (int64_t i = 0; i < dim; ++i) {
        v[i] = (double)(splitmix(seed) >> 11) * (1.0 / 9007199254740992.0) - 0.5;
        nrm += v[i] * v[i];
    }
    nrm = std::sqrt(nrm);
    for (int64_t i = 0; i < dim; ++i) v[i] /= nrm;
}

// Returns lambda_max(C^T C) (= sigma_max(C)^2); negative on failure.
double sigma_max_sq_lanczos(int64_t N, int n, const double *X, double tol, int max_iter) {
    const int64_t dim = N * (int64_t)(n + 1);
    CtC op(N, n, X);
    std::vector<double> v(dim), vprev(dim, 0.0), w(dim);
    lanczos_start(N, n, v.data());
    std::vector<double> al, be;
    double prev = 0.0, bprev = 0.0;
    int stable = 0;
    for (int it = 0; it < std::min<int64_t>(max_iter, dim); ++it) {
        op.apply(v.data(), w.data());
        double a = 0.0;
        for (int64_t i = 0; i < dim; ++i) a += w[i] * v[i];
        double b = 0.0;
        for (int64_t i = 0; i < dim; ++i) {
            w[i] -= a * v[i] + bprev * vprev[i];
            b += w[i] * w[i];
        }
        b = std::sqrt(b);
        al.push_back(a);
        const double theta = max_ritz(al, be);
        if (it > 2 && std::fabs(theta - prev) <= tol * std::fabs(theta)) {
            if (++stable >= 3) return theta;
        } else {
            stable = 0;
        }
        prev = theta;
        if (b <= 1e-14 * std::fabs(theta)) return theta;   // invariant subspace found
        be.push_back(b);
        for (int64_t i = 0; i < dim; ++i) {
            vprev[i] = v[i];
            v[i] = w[i] / b;
        }
        bprev = b;
    }
    return al.empty() ? -1.0 : prev;
}

}  // namespace cr

// Real eigen-decomposition of the interior second-derivative block
// K = D2[1..q][1..q] of the Chebyshev-Lobatto collocation matrix (real,
// nonsymmetric, real distinct negative eigenvalues), used by the
// tensor-product leaf inverse of the constant-coefficient store:
//     (c2 (K (+) K) - sigma)^{-1} = (V (x) V) diag(1/(c2(l_i + l_j) - sigma)) (V^-1 (x) V^-1)
// Hessenberg reduction + shifted QR (Givens) for the eigenvalues, inverse
// iteration for the eigenvectors, Gauss-Jordan for V^-1.  q <= 30.
#include <algorithm>
#include <cmath>
#include <vector>

#include "rexp_internal.hpp"

namespace rexp {
namespace {

using Mat = std::vector<double>;  // row-major n x n

void hessenberg(int n, Mat& A) {
    for (int k = 0; k < n - 2; ++k) {
        double alpha = 0.0;
        for (int i = k + 1; i < n; ++i) alpha += A[i * n + k] * A[i * n + k];
        alpha = std::sqrt(alpha);
        if (alpha == 0.0) continue;
        if (A[(k + 1) * n + k] > 0) alpha = -alpha;
        std::vector<double> v(n, 0.0);
        v[k + 1] = A[(k + 1) * n + k] - alpha;
        for (int i = k + 2; i < n; ++i) v[i] = A[i * n + k];
        double vv = 0.0;
        for (int i = k + 1; i < n; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        // A = H A H, H = I - 2 v v^T / vv
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = k + 1; i < n; ++i) s += v[i] * A[i * n + j];
            s *= 2.0 / vv;
            for (int i = k + 1; i < n; ++i) A[i * n + j] -= s * v[i];
        }
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = k + 1; j < n; ++j) s += A[i * n + j] * v[j];
            s *= 2.0 / vv;
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= s * v[j];
        }
    }
}

// eigenvalues of an upper Hessenberg matrix with real spectrum
bool hqr_real(int n, Mat H, std::vector<double>& lam) {
    lam.assign(n, 0.0);
    int hi = n - 1;
    int iter = 0;
    while (hi >= 0) {
        if (hi == 0) {
            lam[0] = H[0];
            break;
        }
        // deflation check
        int l = hi;
        while (l > 0) {
            const double s = std::fabs(H[(l - 1) * n + l - 1]) + std::fabs(H[l * n + l]);
            if (std::fabs(H[l * n + l - 1]) <= 1e-15 * s) break;
            --l;
        }
        if (l == hi) {
            lam[hi] = H[hi * n + hi];
            --hi;
            iter = 0;
            continue;
        }
        if (++iter > 500) return false;
        // Wilkinson shift from the trailing 2x2
        const double a = H[(hi - 1) * n + hi - 1], b = H[(hi - 1) * n + hi], c = H[hi * n + hi - 1], d = H[hi * n + hi];
        const double tr = a + d, det = a * d - b * c;
        double disc = tr * tr / 4.0 - det;
        double mu;
        if (disc >= 0.0) {
            const double r1 = tr / 2.0 + std::sqrt(disc), r2 = tr / 2.0 - std::sqrt(disc);
            mu = std::fabs(r1 - d) < std::fabs(r2 - d) ? r1 : r2;
        } else {
            mu = tr / 2.0;
        }
        if (iter % 11 == 10) mu += 1e-3 * std::fabs(mu) + 1e-3;  // exceptional shift
        // QR step on the active block [l, hi] with Givens rotations
        for (int i = l; i <= hi; ++i) H[i * n + i] -= mu;
        std::vector<double> cs(hi - l), sn(hi - l);
        for (int k = l; k < hi; ++k) {
            const double x = H[k * n + k], y = H[(k + 1) * n + k];
            const double r = std::hypot(x, y);
            const double cc = r == 0.0 ? 1.0 : x / r, ss = r == 0.0 ? 0.0 : y / r;
            cs[k - l] = cc;
            sn[k - l] = ss;
            for (int j = k; j < n; ++j) {
                const double t1 = H[k * n + j], t2 = H[(k + 1) * n + j];
                H[k * n + j] = cc * t1 + ss * t2;
                H[(k + 1) * n + j] = -ss * t1 + cc * t2;
            }
        }
        for (int k = l; k < hi; ++k) {
            const double cc = cs[k - l], ss = sn[k - l];
            for (int i = 0; i <= std::min(hi, k + 2); ++i) {
                const double t1 = H[i * n + k], t2 = H[i * n + k + 1];
                H[i * n + k] = cc * t1 + ss * t2;
                H[i * n + k + 1] = -ss * t1 + cc * t2;
            }
        }
        for (int i = l; i <= hi; ++i) H[i * n + i] += mu;
    }
    return true;
}

bool solve_lu(int n, Mat A, std::vector<double>& b) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
        if (A[p * n + k] == 0.0) return false;
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
            std::swap(b[k], b[p]);
        }
        for (int i = k + 1; i < n; ++i) {
            const double f = A[i * n + k] / A[k * n + k];
            for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
            b[i] -= f * b[k];
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        double s = b[k];
        for (int j = k + 1; j < n; ++j) s -= A[k * n + j] * b[j];
        b[k] = s / A[k * n + k];
    }
    return true;
}

}  // namespace

// K row-major q x q -> lam[q], V (columns = eigenvectors, row-major), Vinv; returns REXP_OK
int real_eig(int q, const std::vector<double>& K, std::vector<double>& lam, std::vector<double>& V,
             std::vector<double>& Vinv) {
    Mat H = K;
    hessenberg(q, H);
    if (!hqr_real(q, H, lam)) {
        set_error("eig: QR iteration did not converge");
        return REXP_ESINGULAR;
    }
    std::sort(lam.begin(), lam.end());
    V.assign(q * q, 0.0);
    double knorm = 0.0;
    for (double v : K) knorm = std::max(knorm, std::fabs(v));
    for (int e = 0; e < q; ++e) {
        std::vector<double> x(q);
        for (int i = 0; i < q; ++i) x[i] = 1.0 + 0.37 * i - 0.011 * i * i;
        const double shift = lam[e] + 1e-10 * (std::fabs(lam[e]) + 1.0);
        for (int it = 0; it < 3; ++it) {
            Mat A = K;
            for (int i = 0; i < q; ++i) A[i * q + i] -= shift;
            if (!solve_lu(q, A, x)) {
                set_error("eig: inverse iteration singular");
                return REXP_ESINGULAR;
            }
            double nr = 0.0;
            for (double v : x) nr += v * v;
            nr = std::sqrt(nr);
            for (double& v : x) v /= nr;
        }
        // Rayleigh-type refinement of lambda: lam = x^T K x / x^T x
        double num = 0.0;
        for (int i = 0; i < q; ++i) {
            double s = 0.0;
            for (int j = 0; j < q; ++j) s += K[i * q + j] * x[j];
            num += x[i] * s;
        }
        lam[e] = num;
        for (int i = 0; i < q; ++i) V[i * q + e] = x[i];
    }
    // K centro-symmetric (the interior block of a Chebyshev D2 is): its eigenvectors are even or
    // odd under i -> q-1-i.  Inverse iteration returns them with a parity defect of ~1e-12; project
    // each onto its parity so that V, and V^-1 computed from it below, are parity-symmetric to
    // rounding - the parity-split leaf GEMMs (leaf_gemm.cuh) rely on e_1 = -Pi e_0, a1^ = Pi a0^
    {
        double asym = 0.0;
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j)
                asym = std::max(asym, std::fabs(K[i * q + j] - K[(q - 1 - i) * q + (q - 1 - j)]));
        if (asym <= 1e-12 * knorm) {
            for (int e = 0; e < q; ++e) {
                double dp = 0.0, dm = 0.0;
                for (int i = 0; i < q; ++i) {
                    dp += std::fabs(V[i * q + e] - V[(q - 1 - i) * q + e]);
                    dm += std::fabs(V[i * q + e] + V[(q - 1 - i) * q + e]);
                }
                const double par = dp <= dm ? 1.0 : -1.0;
                double nr = 0.0;
                for (int i = 0; i < (q + 1) / 2; ++i) {
                    const double v = 0.5 * (V[i * q + e] + par * V[(q - 1 - i) * q + e]);
                    V[i * q + e] = v;
                    V[(q - 1 - i) * q + e] = par * v;
                }
                for (int i = 0; i < q; ++i) nr += V[i * q + e] * V[i * q + e];
                nr = std::sqrt(nr);
                for (int i = 0; i < q; ++i) V[i * q + e] /= nr;
            }
        }
    }
    // residual check ||K V - V L|| / ||K||
    double res = 0.0;
    for (int i = 0; i < q; ++i)
        for (int e = 0; e < q; ++e) {
            double s = 0.0;
            for (int j = 0; j < q; ++j) s += K[i * q + j] * V[j * q + e];
            res = std::max(res, std::fabs(s - lam[e] * V[i * q + e]));
        }
    if (res > 1e-9 * knorm) {
        set_error("eig: residual too large");
        return REXP_ESINGULAR;
    }
    // V^-1 by Gauss-Jordan
    Mat A = V, I(q * q, 0.0);
    for (int i = 0; i < q; ++i) I[i * q + i] = 1.0;
    for (int k = 0; k < q; ++k) {
        int p = k;
        for (int i = k + 1; i < q; ++i)
            if (std::fabs(A[i * q + k]) > std::fabs(A[p * q + k])) p = i;
        if (A[p * q + k] == 0.0) {
            set_error("eig: singular eigenvector matrix");
            return REXP_ESINGULAR;
        }
        for (int j = 0; j < q; ++j) {
            std::swap(A[k * q + j], A[p * q + j]);
            std::swap(I[k * q + j], I[p * q + j]);
        }
        const double d = A[k * q + k];
        for (int j = 0; j < q; ++j) {
            A[k * q + j] /= d;
            I[k * q + j] /= d;
        }
        for (int i = 0; i < q; ++i) {
            if (i == k) continue;
            const double f = A[i * q + k];
            if (f == 0.0) continue;
            for (int j = 0; j < q; ++j) {
                A[i * q + j] -= f * A[k * q + j];
                I[i * q + j] -= f * I[k * q + j];
            }
        }
    }
    Vinv = I;
    return REXP_OK;
}

}  // namespace rexp

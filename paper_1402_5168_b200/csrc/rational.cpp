// Rational approximation of e^{iy}: Gaussian sums (§3.1), the Table-1
// rational approximation of the Gaussian (§3.2) and the stability filter
// S(iy) R(iy) written as one proper rational function (§3.3).
// DESIGN.md readings R1-R6 apply; the construction is restated here from the
// paper (it shares no code with oracle/).
#include <cmath>

#include "rexp_internal.hpp"

namespace rexp {
namespace {

constexpr double kPi = 3.14159265358979323846;

// PAPER.md Table 1 (lines 705-751): mu and a_j, j = -11..11.
constexpr int kL = 11;
constexpr double kMu = -4.315321510875024;
constexpr double kA[2 * kL + 1][2] = {
    {-1.0845749544592896e-7, 2.77075431662228e-8},
    {1.858753344202957e-8, -9.105375434750162e-7},
    {3.6743713227243024e-6, 7.073284346322969e-7},
    {-2.7990058083347696e-6, 0.0000112564827639346},
    {0.000014918577548849352, -0.0000316278486761932},
    {-0.0010751767283285608, -0.00047282220513073084},
    {0.003816465653840016, 0.017839810396560574},
    {0.12124105653274578, -0.12327042473830248},
    {-0.9774980792734348, -0.1877130220537587},
    {1.3432866123333178, 3.2034715228495942},
    {4.072408546157305, -6.123755543580666},
    {-9.442699917778205, 0.0},
    {4.072408620272648, 6.123755841848161},
    {1.3432860877712938, -3.2034712658530275},
    {-0.9774985292598916, 0.18771238018072134},
    {0.1212417070363373, 0.12326987628935386},
    {0.0038169724770333343, -0.017839242222443888},
    {-0.0010756025812659208, 0.0004731874917343858},
    {0.000014713754789095218, 0.000031358475831136815},
    {-2.659323898804944e-6, -0.000011341571201752273},
    {3.6970377676364553e-6, -6.517457477594937e-7},
    {3.883933649142257e-9, 9.128496023863376e-7},
    {-1.0816457995911385e-7, -2.954309729192276e-8},
};

// Reading R2: even part of the table, a~_j = (a_j + conj(a_{-j}))/2.
std::vector<cd> table_even() {
    std::vector<cd> a(2 * kL + 1);
    for (int j = -kL; j <= kL; ++j) {
        cd aj(kA[j + kL][0], kA[j + kL][1]);
        cd amj(kA[-j + kL][0], kA[-j + kL][1]);
        a[j + kL] = 0.5 * (aj + std::conj(amj));
    }
    return a;
}

// psihat_h(xi) = h exp(-4 pi^2 h^2 xi^2)  (Fourier transform of psi_h, e^{-2 pi i x xi}).
double psihat(double xi, double h) { return h * std::exp(-4.0 * kPi * kPi * h * h * xi * xi); }

// Partial fractions of sum_{m=-M}^{M} c_m psi_h(x + m h) in y = 2 pi x (§3 composition):
//   poles alpha+_n = -2 pi h (mu + i n), alpha-_n = 2 pi h (mu - i n), n = -(M+L)..(M+L)
//   residues b+_n = pi h sum_{m+j=n} c_m a_j,  b-_n = -pi h sum_{m+j=n} c_m conj(a_j)
void compose(double h, const std::vector<cd>& c, std::vector<cd>& poles, std::vector<cd>& res) {
    const std::vector<cd> a = table_even();
    const int M = (static_cast<int>(c.size()) - 1) / 2;
    const int K = M + kL;
    poles.clear();
    res.clear();
    std::vector<cd> C(2 * K + 1), Dn(2 * K + 1);
    for (int n = -K; n <= K; ++n) {
        cd sC = 0.0, sD = 0.0;
        const int jlo = std::max(-kL, n - M), jhi = std::min(kL, n + M);  // reading R3
        for (int j = jlo; j <= jhi; ++j) {
            sC += c[n - j + M] * a[j + kL];
            sD += c[n - j + M] * std::conj(a[j + kL]);
        }
        C[n + K] = sC;
        Dn[n + K] = sD;
    }
    for (int n = -K; n <= K; ++n) {
        poles.push_back(-2.0 * kPi * h * cd(kMu, static_cast<double>(n)));
        res.push_back(kPi * h * C[n + K]);
    }
    for (int n = -K; n <= K; ++n) {
        poles.push_back(2.0 * kPi * h * cd(kMu, -static_cast<double>(n)));
        res.push_back(-kPi * h * Dn[n + K]);
    }
}

}  // namespace

cd rational_eval(const std::vector<cd>& poles, const std::vector<cd>& res, cd z) {
    cd s = 0.0;
    for (size_t k = 0; k < poles.size(); ++k) s += res[k] / (z - poles[k]);
    return s;
}

int build_exp_approx(double A, double delta, RationalApprox& out) {
    if (!(A > 0.0) || !(delta > 0.0)) {
        set_error("build_exp_approx: need tau*Lambda > 0 and delta > 0");
        return REXP_EINVAL;
    }
    // Reading R5: h = 0.17, hS = 2.5 h, M0 = ceil(X/hS) + c, M = ceil(M0 hS / h),
    // X = A/(2 pi); the margin c grows from 8 until both checks below pass.
    const double X = A / (2.0 * kPi);
    const double h = 0.17, hS = 2.5 * h;
    double err = 0.0, mx = 0.0;
    for (int margin = 8; margin <= 16; ++margin) {
        const int M0 = static_cast<int>(std::ceil(X / hS)) + margin;
        const int M = static_cast<int>(std::ceil(M0 * hS / h - 1e-9));
        // R_gauss: c_m = (h/psihat_h(1)) e^{-2 pi i m h}
        std::vector<cd> c(2 * M + 1);
        for (int m = -M; m <= M; ++m)
            c[m + M] = (h / psihat(1.0, h)) * std::exp(cd(0.0, -2.0 * kPi * m * h));
        // S ~ chi: unit coefficients (Eq. "partition of unity-1")
        std::vector<cd> cS(2 * M0 + 1, cd(1.0, 0.0));
        std::vector<cd> pR, rR, pS, rS;
        compose(h, c, pR, rR);
        compose(hS, cS, pS, rS);
        // product S*R as a proper rational function (reading R6)
        double gap = 1e300;
        for (auto& a : pS)
            for (auto& b : pR) gap = std::min(gap, std::abs(a - b));
        if (gap < 1e-8) {
            set_error("build_exp_approx: pole collision between filter and approximant");
            return REXP_EACCURACY;
        }
        out.poles.clear();
        out.res.clear();
        for (size_t k = 0; k < pS.size(); ++k) {
            out.poles.push_back(pS[k]);
            out.res.push_back(rS[k] * rational_eval(pR, rR, pS[k]));
        }
        for (size_t k = 0; k < pR.size(); ++k) {
            out.poles.push_back(pR[k]);
            out.res.push_back(rR[k] * rational_eval(pS, rS, pR[k]));
        }
        out.h = h;
        out.hS = hS;
        out.M = M;
        out.M0 = M0;
        // verification by dense sampling (paper's own style, Figs. 3-5)
        err = 0.0;
        mx = 0.0;
        const int nin = static_cast<int>(2 * A * 32) + 1;
        for (int k = 0; k < nin; ++k) {
            const double y = -A + 2.0 * A * k / (nin - 1);
            const cd v = rational_eval(out.poles, out.res, cd(0.0, y));
            err = std::max(err, std::abs(v - std::exp(cd(0.0, y))));
            mx = std::max(mx, std::abs(v));
        }
        const double Y = 4 * A + 60;
        const int nfar = static_cast<int>(8 * A * 32) + 1;
        for (int k = 0; k < nfar; ++k) {
            const double y = -Y + 2.0 * Y * k / (nfar - 1);
            mx = std::max(mx, std::abs(rational_eval(out.poles, out.res, cd(0.0, y))));
        }
        for (int k = 0; k < 400; ++k) {
            const double y = std::pow(10.0, 7.0 * k / 399.0);
            mx = std::max(mx, std::abs(rational_eval(out.poles, out.res, cd(0.0, y))));
            mx = std::max(mx, std::abs(rational_eval(out.poles, out.res, cd(0.0, -y))));
        }
        if (err <= delta && mx <= 1.0 + delta) break;
    }
    out.err = err;
    out.maxmod = mx;
    if (err > delta) {
        set_error("rational approximation error " + std::to_string(err) + " exceeds delta");
        return REXP_EACCURACY;
    }
    if (mx > 1.0 + delta) {
        set_error("|R(iy)| exceeds 1 + delta: " + std::to_string(mx));
        return REXP_EACCURACY;
    }
    return REXP_OK;
}

}  // namespace rexp

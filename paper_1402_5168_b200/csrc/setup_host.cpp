// Build stage (§1.3, §2.3): pole tables for the
// elliptic reformulations (§2.1) and the host factorization of every shifted
// collocation system into the merge-tree solution operators.
//
// For one half pole with elliptic shift sigma(x) the HPS recurrences are
// (leaf tau with interior I, boundary B; merge of alpha|beta along interface 3):
//   leaf:   S = -A_II^{-1} A_IB,   T = N_B + N_I S          (DtN, outward normal)
//   merge:  X = (T^a_33 + T^b_33)^{-1},  S = -X [T^a_3,ext | T^b_3,ext],
//           Y = [T^a_ext,3 ; T^b_ext,3],  T = blockdiag(T^c_ext,ext) + Y S
//   root:   periodic closure  s = -(P^T T P)^{-1} P^T h   (P duplicates seams)
// The apply then runs  w = A_II^{-1} f, h = N_I w (leaves), w3 = -X(h^a_3 + h^b_3),
// h = h^c_ext + Y w3 (up), u3 = S u_ext + w3, u_I = S_leaf u_B + w (down).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>

#include "rexp_internal.hpp"

namespace rexp {

// ---------------------------------------------------------------------------
// pole tables
// ---------------------------------------------------------------------------
void build_pole_tables(const Problem& P, const RationalApprox& ra, PoleTables& pt) {
    pt = PoleTables();
    const double tau = P.tau;
    for (size_t k = 0; k < ra.poles.size(); ++k) {
        const cd a = ra.poles[k];
        double w;
        if (a.imag() > 0.0)
            w = 2.0;
        else if (a.imag() == 0.0)
            w = 1.0;
        else
            continue;
        pt.full_index.push_back(static_cast<int32_t>(k));
        pt.alpha.push_back(a);
        pt.b.push_back(ra.res[k]);
        pt.omega.push_back(w);
        pt.beta.push_back(a / tau);
    }
    const size_t nh = pt.alpha.size();
    if (P.model == REXP_MODEL_RSW) {
        const double f = P.f;
        pt.nF = 3;  // eta0, div v0, curl v0 = d_x v02 - d_y v01
        pt.nE = 3;  // sums of b' eta, b' p eta, b' q eta
        double Ps = 0.0, Qs = 0.0;
        for (size_t m = 0; m < nh; ++m) {
            const cd be = pt.beta[m];
            const cd k2 = be * be + f * f;
            const cd pp = be / k2, qq = -f / k2;       // A_beta = p I + q J
            const cd bp = pt.b[m] / tau;               // (tau L - alpha)^{-1} = (1/tau)(L - beta)^{-1}
            pt.shift.push_back(k2);
            pt.cF.push_back(k2 / be);                  // (k^2/beta) eta0
            pt.cF.push_back(cd(1.0, 0.0));             // (k^2/beta) p div v0
            pt.cF.push_back(-f / be);                  // (k^2/beta) q curl v0
            const double w = pt.omega[m];
            pt.dE.push_back(w * bp);
            pt.dE.push_back(w * bp * pp);
            pt.dE.push_back(w * bp * qq);
            Ps += w * (bp * pp).real();
            Qs += w * (bp * qq).real();
        }
        pt.scal = {Ps, Qs};
    } else {
        pt.nF = 2;  // v0/kappa, d_x w0 + d_y z0
        pt.nE = 2;  // sums of b' v, b'/beta v
        double B1 = 0.0;
        for (size_t m = 0; m < nh; ++m) {
            const cd be = pt.beta[m];
            const cd bp = pt.b[m] / tau;
            pt.shift.push_back(be * be);               // sigma(x) = beta^2 / kappa(x)
            pt.cF.push_back(be);
            pt.cF.push_back(cd(1.0, 0.0));
            const double w = pt.omega[m];
            pt.dE.push_back(w * bp);
            pt.dE.push_back(w * bp / be);
            B1 += w * (bp / be).real();
        }
        pt.scal = {B1};
    }
}

// ---------------------------------------------------------------------------
// small dense complex kernels (row-major)
// ---------------------------------------------------------------------------
namespace {

// C[m x n] = alpha * A[m x k] B[k x n] + beta * C
void zgemm(int m, int n, int k, cd alpha, const cd* A, const cd* B, cd beta, cd* C) {
    std::vector<double> acc(2 * static_cast<size_t>(n));
    for (int i = 0; i < m; ++i) {
        std::fill(acc.begin(), acc.end(), 0.0);
        double* ac = acc.data();
        for (int l = 0; l < k; ++l) {
            const double ar = A[static_cast<size_t>(i) * k + l].real();
            const double ai = A[static_cast<size_t>(i) * k + l].imag();
            if (ar == 0.0 && ai == 0.0) continue;
            const double* b = reinterpret_cast<const double*>(B + static_cast<size_t>(l) * n);
            for (int j = 0; j < n; ++j) {
                const double br = b[2 * j], bi = b[2 * j + 1];
                ac[2 * j] += ar * br - ai * bi;
                ac[2 * j + 1] += ar * bi + ai * br;
            }
        }
        cd* c = C + static_cast<size_t>(i) * n;
        for (int j = 0; j < n; ++j) {
            const cd v(ac[2 * j], ac[2 * j + 1]);
            c[j] = (beta == cd(0.0) ? cd(0.0) : beta * c[j]) + alpha * v;
        }
    }
}

// In-place inverse by Gauss-Jordan elimination with partial pivoting.
bool zinverse(int n, cd* A) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int pr = k;
        double best = std::abs(A[static_cast<size_t>(k) * n + k]);
        for (int r = k + 1; r < n; ++r) {
            const double v = std::abs(A[static_cast<size_t>(r) * n + k]);
            if (v > best) { best = v; pr = r; }
        }
        if (!(best > 0.0)) return false;
        piv[k] = pr;
        if (pr != k)
            for (int c = 0; c < n; ++c) std::swap(A[static_cast<size_t>(k) * n + c], A[static_cast<size_t>(pr) * n + c]);
        const cd d = 1.0 / A[static_cast<size_t>(k) * n + k];
        A[static_cast<size_t>(k) * n + k] = 1.0;
        for (int c = 0; c < n; ++c) A[static_cast<size_t>(k) * n + c] *= d;
        for (int r = 0; r < n; ++r) {
            if (r == k) continue;
            const cd fr = A[static_cast<size_t>(r) * n + k];
            if (fr == cd(0.0)) continue;
            A[static_cast<size_t>(r) * n + k] = 0.0;
            const double fre = fr.real(), fim = fr.imag();
            double* rowr = reinterpret_cast<double*>(A + static_cast<size_t>(r) * n);
            const double* rowk = reinterpret_cast<const double*>(A + static_cast<size_t>(k) * n);
            for (int c = 0; c < n; ++c) {
                const double kr = rowk[2 * c], ki = rowk[2 * c + 1];
                rowr[2 * c] -= fre * kr - fim * ki;
                rowr[2 * c + 1] -= fre * ki + fim * kr;
            }
        }
    }
    for (int k = n - 1; k >= 0; --k)
        if (piv[k] != k)
            for (int r = 0; r < n; ++r) std::swap(A[static_cast<size_t>(r) * n + k], A[static_cast<size_t>(r) * n + piv[k]]);
    return true;
}

// store row-major (rows x cols) as column-major into dst
// M (rows x cols, row-major) <- Vb^-1 M Vb with Vb = blockdiag(V) over q-row and
// q-column segments (rows, cols multiples of q)
void conj_edge_basis(std::vector<cd>& M, int rows, int cols, int q, const std::vector<double>& V,
                     const std::vector<double>& Vi) {
    std::vector<cd> tmp(static_cast<size_t>(q));
    for (int c = 0; c < cols; ++c)
        for (int s0 = 0; s0 < rows; s0 += q) {
            for (int a = 0; a < q; ++a) {
                cd acc = 0.0;
                for (int b = 0; b < q; ++b) acc += Vi[static_cast<size_t>(a) * q + b] * M[static_cast<size_t>(s0 + b) * cols + c];
                tmp[a] = acc;
            }
            for (int a = 0; a < q; ++a) M[static_cast<size_t>(s0 + a) * cols + c] = tmp[a];
        }
    for (int r = 0; r < rows; ++r)
        for (int s0 = 0; s0 < cols; s0 += q) {
            cd* row = M.data() + static_cast<size_t>(r) * cols + s0;
            for (int a = 0; a < q; ++a) {
                cd acc = 0.0;
                for (int b = 0; b < q; ++b) acc += row[b] * V[static_cast<size_t>(b) * q + a];
                tmp[a] = acc;
            }
            for (int a = 0; a < q; ++a) row[a] = tmp[a];
        }
}

void store_colmajor(const cd* src, int rows, int cols, cd* dst) {
    for (int c = 0; c < cols; ++c)
        for (int r = 0; r < rows; ++r) dst[static_cast<size_t>(c) * rows + r] = src[static_cast<size_t>(r) * cols + c];
}

struct LeafGeom {
    int p, q, q2, nb;
    double c1, c2;  // 2/H, (2/H)^2
    std::vector<cd> AIB;  // q2 x nb (row-major), sigma-independent
    std::vector<cd> NB;   // nb x nb
    std::vector<cd> NI;   // nb x q2
    std::vector<double> K;  // q2 x q2 Laplacian part of A_II (sigma-independent)
};

LeafGeom make_leaf_geom(const Cheb& ch, int n) {
    LeafGeom g;
    g.p = ch.p;
    g.q = ch.p - 2;
    g.q2 = g.q * g.q;
    g.nb = 4 * g.q;
    const double H = 1.0 / n;
    g.c1 = 2.0 / H;
    g.c2 = g.c1 * g.c1;
    const int p = g.p, q = g.q, q2 = g.q2, nb = g.nb;
    g.AIB.assign(static_cast<size_t>(q2) * nb, 0.0);
    g.K.assign(static_cast<size_t>(q2) * q2, 0.0);
    const double* D = ch.D.data();
    const double* D2 = ch.D2.data();
    auto I = [q](int i, int j) { return (j - 1) * q + (i - 1); };
    for (int j = 1; j <= q; ++j)
        for (int i = 1; i <= q; ++i) {
            const int r = I(i, j);
            for (int k = 0; k < p; ++k) {
                const double vx = g.c2 * D2[i * p + k];  // node (k, j)
                if (k == 0) g.AIB[static_cast<size_t>(r) * nb + 3 * q + (j - 1)] += vx;
                else if (k == p - 1) g.AIB[static_cast<size_t>(r) * nb + q + (j - 1)] += vx;
                else g.K[static_cast<size_t>(r) * q2 + I(k, j)] += vx;
                const double vy = g.c2 * D2[j * p + k];  // node (i, k)
                if (k == 0) g.AIB[static_cast<size_t>(r) * nb + (i - 1)] += vy;
                else if (k == p - 1) g.AIB[static_cast<size_t>(r) * nb + 2 * q + (i - 1)] += vy;
                else g.K[static_cast<size_t>(r) * q2 + I(i, k)] += vy;
            }
        }
    g.NB.assign(static_cast<size_t>(nb) * nb, 0.0);
    g.NI.assign(static_cast<size_t>(nb) * q2, 0.0);
    for (int i = 1; i <= q; ++i) {  // bottom (i,0): -c1 sum_k D[0,k] u(i,k)
        const int b = i - 1;
        for (int k = 0; k < p; ++k) {
            const double v = -g.c1 * D[0 * p + k];
            if (k == 0) g.NB[static_cast<size_t>(b) * nb + (i - 1)] += v;
            else if (k == p - 1) g.NB[static_cast<size_t>(b) * nb + 2 * q + (i - 1)] += v;
            else g.NI[static_cast<size_t>(b) * q2 + I(i, k)] += v;
        }
    }
    for (int j = 1; j <= q; ++j) {  // right (p-1,j): +c1 sum_k D[p-1,k] u(k,j)
        const int b = q + j - 1;
        for (int k = 0; k < p; ++k) {
            const double v = g.c1 * D[(p - 1) * p + k];
            if (k == 0) g.NB[static_cast<size_t>(b) * nb + 3 * q + (j - 1)] += v;
            else if (k == p - 1) g.NB[static_cast<size_t>(b) * nb + q + (j - 1)] += v;
            else g.NI[static_cast<size_t>(b) * q2 + I(k, j)] += v;
        }
    }
    for (int i = 1; i <= q; ++i) {  // top (i,p-1): +c1 sum_k D[p-1,k] u(i,k)
        const int b = 2 * q + i - 1;
        for (int k = 0; k < p; ++k) {
            const double v = g.c1 * D[(p - 1) * p + k];
            if (k == 0) g.NB[static_cast<size_t>(b) * nb + (i - 1)] += v;
            else if (k == p - 1) g.NB[static_cast<size_t>(b) * nb + 2 * q + (i - 1)] += v;
            else g.NI[static_cast<size_t>(b) * q2 + I(i, k)] += v;
        }
    }
    for (int j = 1; j <= q; ++j) {  // left (0,j): -c1 sum_k D[0,k] u(k,j)
        const int b = 3 * q + j - 1;
        for (int k = 0; k < p; ++k) {
            const double v = -g.c1 * D[0 * p + k];
            if (k == 0) g.NB[static_cast<size_t>(b) * nb + 3 * q + (j - 1)] += v;
            else if (k == p - 1) g.NB[static_cast<size_t>(b) * nb + q + (j - 1)] += v;
            else g.NI[static_cast<size_t>(b) * q2 + I(k, j)] += v;
        }
    }
    return g;
}

struct Ctx {
    const Problem* P;
    const Tree* T;
    const PoleTables* pt;
    LeafGeom lg;
    bool shared;
    bool root_fourier;
    // spectral edge basis (shared RSW store with the spectral leaf path): every
    // stored edge operator is conjugated by Vb = blockdiag(V) over its q-node
    // segments, K = D2[1..q][1..q] = V diag(l) V^-1 (DESIGN.md §6 "edge basis")
    bool edge_basis;
    std::vector<double> V, Vi;   // q x q row-major

    int h0;
    std::vector<HostLevelOps>* ops;
};

// factor one half pole; returns REXP_OK or error code
int factor_one(const Ctx& C, int hidx) {
    const Tree& T = *C.T;
    const LeafGeom& g = C.lg;
    const int q2 = g.q2, nb = g.nb;
    const int slot = hidx - C.h0;
    const cd s = C.pt->shift[hidx];
    const int nleaf_f = C.shared ? 1 : T.nelem;
    std::vector<HostLevelOps>& ops = *C.ops;

    // ---- leaves ----
    std::vector<std::vector<cd>> Tchild(nleaf_f);
    std::vector<cd> A(static_cast<size_t>(q2) * q2), S(static_cast<size_t>(q2) * nb);
    for (int e = 0; e < nleaf_f; ++e) {
        for (size_t k = 0; k < A.size(); ++k) A[k] = g.K[k];
        for (int r = 0; r < q2; ++r) {
            double gx = 1.0;
            if (C.P->model == REXP_MODEL_WAVE) {
                const int i = r % g.q + 1, j = r / g.q + 1;
                const int64_t gi = T.elem_g[static_cast<size_t>(e) * g.p * g.p + j * g.p + i];
                gx = 1.0 / C.P->kappa[gi];
            }
            A[static_cast<size_t>(r) * q2 + r] -= s * gx;
        }
        if (!zinverse(q2, A.data())) {
            set_error("singular leaf operator (half pole " + std::to_string(hidx) + ")");
            return REXP_ESINGULAR;
        }
        zgemm(q2, nb, q2, cd(-1.0), A.data(), g.AIB.data(), cd(0.0), S.data());
        std::vector<cd> Tl(g.NB);
        zgemm(nb, nb, q2, cd(1.0), g.NI.data(), S.data(), cd(1.0), Tl.data());
        Tchild[e] = std::move(Tl);
        HostLevelOps& L0 = ops[0];
        const size_t base0 = (static_cast<size_t>(slot) * L0.nodes_stored + e);
        store_colmajor(A.data(), q2, q2, L0.m[0].data() + base0 * q2 * q2);
        store_colmajor(S.data(), q2, nb, L0.m[1].data() + base0 * q2 * nb);
    }

    // ---- merges ----
    for (size_t li = 0; li < T.levels.size(); ++li) {
        const MergeLevel& L = T.levels[li];
        const int nn = C.shared ? 1 : L.nodes;
        const int n3 = L.n3, ne = L.next, nc = L.nchild;
        std::vector<std::vector<cd>> Tpar(nn);
        HostLevelOps& LO = ops[li + 1];
        std::vector<cd> X(static_cast<size_t>(n3) * n3), Tc3(static_cast<size_t>(n3) * ne),
            Sm(static_cast<size_t>(n3) * ne), Y(static_cast<size_t>(ne) * n3);
        for (int node = 0; node < nn; ++node) {
            // children of this node (shared mode: the representative child 0 of each kind)
            int ca, cb;
            if (C.shared) {
                ca = 0;
                cb = 0;
            } else {
                ca = L.ia3[static_cast<size_t>(node) * n3] / nc;
                cb = L.ib3[static_cast<size_t>(node) * n3] / nc;
            }
            const cd* Ta = Tchild[ca].data();
            const cd* Tb = Tchild[cb].data();
            for (int r = 0; r < n3; ++r)
                for (int c = 0; c < n3; ++c)
                    X[static_cast<size_t>(r) * n3 + c] =
                        Ta[static_cast<size_t>(L.ia3_pos[r]) * nc + L.ia3_pos[c]] +
                        Tb[static_cast<size_t>(L.ib3_pos[r]) * nc + L.ib3_pos[c]];
            if (!zinverse(n3, X.data())) {
                set_error("singular merge operator (half pole " + std::to_string(hidx) + ")");
                return REXP_ESINGULAR;
            }
            for (int k = 0; k < n3 * n3; ++k) X[k] = -X[k];  // Xneg
            const size_t ob = static_cast<size_t>(node) * ne;  // node 0 in shared mode is representative
            for (int r = 0; r < ne; ++r) {
                const bool isb = L.ext_is_b[ob + r] != 0;
                const int pos = L.ext_pos[ob + r];
                const cd* Tc = isb ? Tb : Ta;
                const std::vector<int32_t>& i3 = isb ? L.ib3_pos : L.ia3_pos;
                for (int t = 0; t < n3; ++t) {
                    Tc3[static_cast<size_t>(t) * ne + r] = Tc[static_cast<size_t>(i3[t]) * nc + pos];
                    Y[static_cast<size_t>(r) * n3 + t] = Tc[static_cast<size_t>(pos) * nc + i3[t]];
                }
            }
            zgemm(n3, ne, n3, cd(1.0), X.data(), Tc3.data(), cd(0.0), Sm.data());  // S = Xneg Tc3
            std::vector<cd> Tp(static_cast<size_t>(ne) * ne, cd(0.0));
            for (int r = 0; r < ne; ++r) {
                const bool isb = L.ext_is_b[ob + r] != 0;
                const int pr = L.ext_pos[ob + r];
                const cd* Tc = isb ? Tb : Ta;
                for (int c2 = 0; c2 < ne; ++c2)
                    if ((L.ext_is_b[ob + c2] != 0) == isb)
                        Tp[static_cast<size_t>(r) * ne + c2] = Tc[static_cast<size_t>(pr) * nc + L.ext_pos[ob + c2]];
            }
            zgemm(ne, ne, n3, cd(1.0), Y.data(), Sm.data(), cd(1.0), Tp.data());
            Tpar[node] = std::move(Tp);
            const size_t base = static_cast<size_t>(slot) * LO.nodes_stored + node;
            if (C.edge_basis) {   // stored copies only: T above used the nodal operators
                const int q = T.q;
                conj_edge_basis(X, n3, n3, q, C.V, C.Vi);
                conj_edge_basis(Y, ne, n3, q, C.V, C.Vi);
                conj_edge_basis(Sm, n3, ne, q, C.V, C.Vi);
            }
            store_colmajor(X.data(), n3, n3, LO.m[0].data() + base * n3 * n3);
            store_colmajor(Y.data(), ne, n3, LO.m[1].data() + base * ne * n3);
            store_colmajor(Sm.data(), n3, ne, LO.m[2].data() + base * n3 * ne);
        }
        Tchild.swap(Tpar);
    }

    // ---- root closure: the two cylinders merged across both horizontal seams ----
    //   X = -(T^a_33 + T^b_33)^{-1},  s = X (h^a_3 + h^b_3)  (no exterior left)
    {
        const int ns = T.ns;
        const int nbc = T.levels.back().next;   // cylinder boundary size
        const cd* Ta = Tchild[0].data();
        const cd* Tb = Tchild[C.shared ? 0 : 1].data();
        std::vector<cd> M(static_cast<size_t>(ns) * ns);
        for (int a = 0; a < ns; ++a)
            for (int b = 0; b < ns; ++b) {
                const int a1 = T.root_pos1[a], b1 = T.root_pos1[b];
                const int a2 = T.root_pos2[a] - nbc, b2 = T.root_pos2[b] - nbc;
                M[static_cast<size_t>(a) * ns + b] = Ta[static_cast<size_t>(a1) * nbc + b1] +
                                                     Tb[static_cast<size_t>(a2) * nbc + b2];
            }
        HostLevelOps& LR = ops.back();
        if (C.root_fourier) {
            // Translation invariance along x (shared store): seam index s = (sigma, e, i)
            // = sigma*n*q + e*q + i, and M[(sigma,e,i),(sigma',e',i')] depends on e - e'
            // only, so M is block circulant:  C_d = M[(., e'+d, .), (., e', .)]
            // (averaged over e'),  M^_k = sum_d C_d w^{-kd},  w = exp(2 pi i / n),
            // and X^_k = -(M^_k)^{-1}   (DESIGN.md §6 "Fourier root").
            const int n = T.n, q = T.q, r2q = 2 * q, nq = n * q;
            auto sidx = [&](int sg, int e, int i) { return sg * nq + ((e % n + n) % n) * q + i; };
            std::vector<cd> Cd(static_cast<size_t>(n) * r2q * r2q, cd(0.0));
            for (int d = 0; d < n; ++d)
                for (int ep = 0; ep < n; ++ep)
                    for (int sg = 0; sg < 2; ++sg)
                        for (int i = 0; i < q; ++i)
                            for (int sg2 = 0; sg2 < 2; ++sg2)
                                for (int i2 = 0; i2 < q; ++i2)
                                    Cd[(static_cast<size_t>(d) * r2q + sg * q + i) * r2q + sg2 * q + i2] +=
                                        M[static_cast<size_t>(sidx(sg, ep + d, i)) * ns + sidx(sg2, ep, i2)] /
                                        static_cast<double>(n);
            constexpr double kPi = 3.14159265358979323846;
            std::vector<cd> Mk(static_cast<size_t>(r2q) * r2q);
            for (int k = 0; k < n; ++k) {
                std::fill(Mk.begin(), Mk.end(), cd(0.0));
                for (int d = 0; d < n; ++d) {
                    const double ang = -2.0 * kPi * static_cast<double>((static_cast<long long>(k) * d) % n) / n;
                    const cd w(std::cos(ang), std::sin(ang));
                    for (int e = 0; e < r2q * r2q; ++e) Mk[e] += Cd[static_cast<size_t>(d) * r2q * r2q + e] * w;
                }
                if (!zinverse(r2q, Mk.data())) {
                    set_error("singular periodic closure block (half pole " + std::to_string(hidx) + ")");
                    return REXP_ESINGULAR;
                }
                for (auto& v : Mk) v = -v;
                if (C.edge_basis) conj_edge_basis(Mk, r2q, r2q, q, C.V, C.Vi);
                store_colmajor(Mk.data(), r2q, r2q,
                               LR.m[1].data() + (static_cast<size_t>(slot) * n + k) * r2q * r2q);
            }
        } else {
            if (!zinverse(ns, M.data())) {
                set_error("singular periodic closure (half pole " + std::to_string(hidx) + ")");
                return REXP_ESINGULAR;
            }
            for (auto& v : M) v = -v;
            store_colmajor(M.data(), ns, ns, LR.m[0].data() + static_cast<size_t>(slot) * ns * ns);
        }
    }
    return REXP_OK;
}

}  // namespace

int factor_host(const Problem& P, const Tree& T, const PoleTables& pt, int h0, int h1, bool shared,
                int nthreads, std::vector<HostLevelOps>& ops, bool root_fourier, bool edge_basis) {
    const int nh = h1 - h0;
    const Cheb ch = make_cheb(T.p);
    root_fourier = root_fourier && shared;
    Ctx C{&P, &T, &pt, make_leaf_geom(ch, T.n), shared, root_fourier, edge_basis && root_fourier, {}, {}, h0, &ops};
    if (C.edge_basis) {
        const int q = T.q;
        std::vector<double> K(static_cast<size_t>(q) * q), lam;
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j) K[static_cast<size_t>(i) * q + j] = ch.D2[(i + 1) * T.p + (j + 1)];
        const int rc = real_eig(q, K, lam, C.V, C.Vi);
        if (rc != REXP_OK) return rc;
    }
    const int q2 = C.lg.q2, nb = C.lg.nb;
    // allocate
    ops.assign(T.levels.size() + 2, HostLevelOps());
    {
        HostLevelOps& L0 = ops[0];
        L0.nmat = 2;
        L0.nodes_stored = shared ? 1 : T.nelem;
        L0.rows[0] = q2; L0.cols[0] = q2;
        L0.rows[1] = q2; L0.cols[1] = nb;
        for (int k = 0; k < 2; ++k)
            L0.m[k].resize(static_cast<size_t>(nh) * L0.nodes_stored * L0.rows[k] * L0.cols[k]);
    }
    for (size_t li = 0; li < T.levels.size(); ++li) {
        const MergeLevel& L = T.levels[li];
        HostLevelOps& LO = ops[li + 1];
        LO.nmat = 3;
        LO.nodes_stored = shared ? 1 : L.nodes;
        LO.rows[0] = L.n3; LO.cols[0] = L.n3;
        LO.rows[1] = L.next; LO.cols[1] = L.n3;
        LO.rows[2] = L.n3; LO.cols[2] = L.next;
        for (int k = 0; k < 3; ++k)
            LO.m[k].resize(static_cast<size_t>(nh) * LO.nodes_stored * LO.rows[k] * LO.cols[k]);
    }
    {
        HostLevelOps& LR = ops.back();
        LR.nmat = 1;
        LR.nodes_stored = 1;
        if (root_fourier) {   // n Fourier blocks of (2q x 2q)
            LR.rows[1] = 2 * T.q; LR.cols[1] = 2 * T.q * T.n;
            LR.m[1].resize(static_cast<size_t>(nh) * T.n * 4 * T.q * T.q);
        } else {
            LR.rows[0] = T.ns; LR.cols[0] = T.ns;
            LR.m[0].resize(static_cast<size_t>(nh) * T.ns * T.ns);
        }
    }
    if (nthreads <= 0) nthreads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    nthreads = std::min(nthreads, std::max(1, nh));
    std::atomic<int> next(h0);
    std::atomic<int> status(REXP_OK);
    auto work = [&]() {
        for (;;) {
            const int k = next.fetch_add(1);
            if (k >= h1 || status.load() != REXP_OK) break;
            const int rc = factor_one(C, k);
            if (rc != REXP_OK) status.store(rc);
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(work);
    for (auto& t : th) t.join();
    return status.load();
}

}  // namespace rexp

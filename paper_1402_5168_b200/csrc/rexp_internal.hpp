// Internal declarations of the rexp library (host side).
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rexp.h"

namespace rexp {

using cd = std::complex<double>;

void set_error(const std::string& msg);

// ---------------------------------------------------------------------------
// Rational approximation (§3)
// ---------------------------------------------------------------------------
struct RationalApprox {
    std::vector<cd> poles;   // all poles, order [S+ , S-, R+, R-], each n = -K..K
    std::vector<cd> res;     // residues b_m
    double err = 0.0;        // sampled sup |R(iy) - e^{iy}| on |y| <= A
    double maxmod = 0.0;     // sampled sup |R(iy)|
    double h = 0.0, hS = 0.0;
    int M = 0, M0 = 0;
};

// Builds R = S * R_gauss for the interval |y| <= A; returns REXP_OK or error code.
int build_exp_approx(double A, double delta, RationalApprox& out);
cd rational_eval(const std::vector<cd>& poles, const std::vector<cd>& res, cd z);

// ---------------------------------------------------------------------------
// Spectral-element mesh + HPS merge tree (§2.2-2.3)
// ---------------------------------------------------------------------------
struct Cheb {
    int p = 0;
    std::vector<double> t;     // Chebyshev-Lobatto points, ascending
    std::vector<double> D;     // p x p row-major, D[i*p+k] = l_k'(t_i)
    std::vector<double> D2;    // D*D
    std::vector<double> Dw;    // (p-2) x p row-major edge-tangential stencil (reading R8)
};
Cheb make_cheb(int p);
std::vector<double> lagrange_diff(const std::vector<double>& t);

// one merge level of the tree (parents at this level)
struct MergeLevel {
    int dir = 0;                 // 0: merge in x (left|right), 1: merge in y (bottom|top)
    int a = 0, b = 0;            // parent box size in elements
    int nbx = 0, nby = 0;        // parent boxes per direction
    int nodes = 0;               // nbx * nby
    int n3 = 0;                  // interface size
    int next = 0;                // parent boundary size
    int nchild = 0;              // child boundary size
    int child_nodes = 0;
    // per parent node (node-major)
    std::vector<int32_t> ia3, ib3;   // [nodes][n3]   flat index into child h: child*nchild + pos
    std::vector<int32_t> ext;        // [nodes][next] flat index into child h
    std::vector<int32_t> ext_is_b;   // [nodes][next] 1 if from child beta (setup helper)
    std::vector<int32_t> ext_pos;    // [nodes][next] position inside that child's boundary
    std::vector<int32_t> ia3_pos, ib3_pos; // [n3] positions inside alpha/beta boundary (node-independent)
    std::vector<int32_t> gext;       // [nodes][next] global edge index of parent boundary nodes
    std::vector<int32_t> g3;         // [nodes][n3]   global edge index of interface nodes
};

struct Tree {
    int n = 0, p = 0, q = 0;
    int64_t NI = 0, NV = 0, NH = 0, N = 0, NE = 0;
    int nelem = 0;
    std::vector<int32_t> leaf_gB;    // [nelem][4q] global edge index of leaf boundary nodes
    std::vector<MergeLevel> levels;  // merge levels, bottom-up
    int ns = 0;                      // root seam unknowns = 2 n q
    std::vector<int32_t> root_pos1, root_pos2;  // [ns] positions in root boundary
    std::vector<int32_t> root_gs;               // [ns] global edge index of seam nodes
    // element-local (i,j) -> global index (-1 corner), [nelem][p*p] (j*p+i)
    std::vector<int32_t> elem_g;
    std::vector<double> x, y;        // node coordinates
};
int build_tree(int n, int p, Tree& T);

// ---------------------------------------------------------------------------
// Host operator store (column-major complex matrices)
// ---------------------------------------------------------------------------
struct HostLevelOps {
    int rows[3] = {0, 0, 0}, cols[3] = {0, 0, 0};
    int nmat = 0;                      // matrices per level per half-pole (1 leaf: 2, merge: 3, root: 1)
    int nodes_stored = 0;              // 1 (shared) or nodes
    std::vector<cd> m[3];              // [half][node_stored][rows*cols], column-major
};

struct Problem {
    int model = REXP_MODEL_RSW;
    int n = 0, p = 0;
    double f = 0.0;
    std::vector<double> kappa;         // WAVE: at all N global nodes
    double tau = 0, delta = 0, Lambda = 0;
};

struct PoleTables {
    // half poles (Im alpha >= 0), in construction order
    std::vector<int32_t> full_index;   // index into RationalApprox::poles
    std::vector<cd> alpha, b;          // alpha_m, b_m
    std::vector<double> omega;         // 2 (Im > 0) or 1 (real pole)
    std::vector<cd> beta;              // alpha / tau
    std::vector<cd> shift;             // elliptic shift scale s_m: sigma(x) = s_m * g(x)
    int nF = 0;                        // pole-independent RHS fields
    std::vector<cd> cF;                // [half][nF]  RHS coefficients
    int nE = 0;                        // pole sums
    std::vector<cd> dE;                // [half][nE]  omega_m-weighted, b_m/tau folded in
    std::vector<double> scal;          // host-side post scalars (RSW: P, Q ; WAVE: B1)
};
void build_pole_tables(const Problem& P, const RationalApprox& ra, PoleTables& pt);

// real eigen-decomposition of a q x q matrix with real spectrum (eig.cpp)
int real_eig(int q, const std::vector<double>& K, std::vector<double>& lam, std::vector<double>& V,
             std::vector<double>& Vinv);

// Host HPS factorization of half poles [h0, h1) into ops (levels: 0 leaf, 1..L merges, L+1 root)
// root_fourier (shared store only): the periodic closure as n Fourier blocks
// (ops.back().m[1], [half][n][2q x 2q]) instead of the dense ns x ns inverse (m[0])
int factor_host(const Problem& P, const Tree& T, const PoleTables& pt, int h0, int h1,
                bool shared, int nthreads, std::vector<HostLevelOps>& ops, bool root_fourier = false,
                bool edge_basis = false);
// edge_basis (with root_fourier): stored merge / root operators act on edge
// data in the spectral basis V^-1 u of every q-node edge segment

}  // namespace rexp

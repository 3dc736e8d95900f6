// Spectral (tensor-product) leaf solves for the constant-coefficient (shared) store.
//
// On a leaf the interior collocation operator is a Kronecker sum
//     A_II = c2 (I (x) K + K (x) I) - sigma_m,   K = D2[1..q][1..q],  c2 = (2/H)^2
// (§2.2 collocation; interior index (i, j), i fastest).  With
// K = V diag(l) V^-1 (real, kappa(V) ~ 1.6 for q <= 16):
//     A_II^{-1} T = V W V^T,   W = (V^-1 T V^-T) ./ (c2 (l_i + l_j) - sigma_m).
// Everything pole-dependent is elementwise in the spectral basis, so the
// O(q^3) transforms are hoisted out of the pole loop:
//   * RHS fields:   G_f = V^-1 F_f V^-T once per step (k_spec_pre_fused), and
//                   V^-1 (sum_f c_mf F_f) V^-T = sum_f c_mf G_f;
//   * boundary:     A_IB u_B is a sum of four outer products a (x) u_side, so
//                   V^-1 (A_IB u_B) V^-T = c2 (a0^ ul^T + a1^ ur^T + ub^ a0^T + ut^ a1^T)
//                   with u^ = V^-1 u_side (q x q mat-vecs per pole);
//   * pole sum:     V is real, so sum_m Re(d_mk V W_m V^T) = V [sum_m Re(d_mk W_m)] V^T:
//                   the interior pole sums are accumulated in the spectral basis
//                   and transformed back once per step (k_spec_back).
//   UP:   h = N_I V W V^T (outward flux) from W through e_s = V^T d_s (four q-vectors).
//   DOWN: E^_k += Re(d_mk W_m), the interior solutions u_m are never formed.
// One CTA owns one (leaf, right-hand side) with both real parts and a
// contiguous group of half poles; thread t owns spectral mode (i', j') =
// (t & 15, t >> 4) of the zero-padded 16 x 16 grid (active when i', j' < q;
// compact mode index j' q + i' in G and E^).  Dinv is symmetric in (i', j'),
// so the thread reads it at t = j' 16 + i': consecutive threads, consecutive
// addresses (global and shared).
#pragma once

namespace rexp {
namespace dev {

constexpr int SP_T = 16;            // padded 1-D size of V, V^-1, Dinv rows
constexpr int SP_THREADS = 256;     // >= q^2 for q <= 16
constexpr int SP_PB = 4;            // half poles per batch (shared-memory staging)
constexpr int SP_LW = SP_T + 1;     // stride of W tiles (odd: conflict-free row and column walks)
constexpr int SP_NB = 4 * SP_T;     // max boundary nodes per leaf

struct SpecArgs {
    const double* V;        // 16 x 16 row-major, zero padded
    const double* Vinv;     // 16 x 16 row-major, zero padded
    const double* E01;      // e0 = V^T d_0, e1 = V^T d_{p-1} (d_r[k] = D[r][k+1]), 2 x 16
    const double* A01;      // a0^ = V^-1 D2[1..q][0], a1^ = V^-1 D2[1..q][p-1], 2 x 16
    const double2* Dinv;    // [nh][16*16] 1/(c2 (l_i + l_j) - sigma_m), (i', j') at i'*16 + j'
    const double2* cF;      // [nh][nF]
    const double2* dE;      // [nh][nE]
    const double* F;        // [R2][nF][NI] pole-independent RHS fields (k_pre)
    double* G;              // [nelem][R2][nF][q2] their spectral coefficients
    int q, p, nF, nE, nelem, R2, nh, ngroups, accumulate;
    double c1, c2;
    // UP
    double2* h;             // [nh][hps][R2]
    long long hps;
    // DOWN
    const double2* edge;    // [nh][NE][R2]
    long long NE;
    const int* gB;          // [nelem][4q]
    const int* own;         // [nelem][4q] 1 where this leaf owns the edge node's pole sum
    double* Ehat;           // [ngroups][nE][R2][nelem * q2] spectral pole-sum partials
    const double* Pi;       // [nE][nF][16*16] sum_m Re(d_mk c_mf Dinv_m), (i', j') at i'*16 + j'
    double* Eedge;          // [ngroups][nE][R2][NE] edge pole-sum partials
    // BACK
    double* E;              // [nE][R2][N]
    long long N;
    // fused RHS fields (k_spec_pre_fused)
    const double* u;        // state [nrhs][3][N] complex interleaved
    const int* elem_g;      // [nelem][p*p] (-1 at corners)
    const double* Dm;       // p x p differentiation matrix
};

__device__ __forceinline__ void sp_group_range(const SpecArgs& a, int grp, int& m0, int& m1) {
    const int base = a.nh / a.ngroups, rem = a.nh % a.ngroups;
    m0 = grp * base + min(grp, rem);
    m1 = m0 + base + (grp < rem ? 1 : 0);
}

// --------------------------------------------------------------------------
// k_spec_pre_fused: RSW RHS fields at the leaf's interior nodes (§2.1,
// eta0, div v0, curl v0 from the element's nodal values, R8) straight into
// their spectral coefficients G_f = V^-1 F_f V^-T (grid: nelem * R2 CTAs)
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(SP_THREADS) k_spec_pre_fused(SpecArgs a) {
    constexpr int PM = SP_T + 2;                       // p <= 18
    __shared__ double us[3][PM * PM];                  // v1, v2, eta at the element's p x p nodes
    __shared__ double ds[PM * PM];
    __shared__ double fs[3][SP_T * SP_T];
    __shared__ double ts[3][SP_T * SP_T];
    __shared__ double vis[SP_T * (SP_T + 1)];
    const int q = a.q, p = a.p, q2 = q * q, t = threadIdx.x;
    const int leaf = blockIdx.x / a.R2, r2 = blockIdx.x % a.R2;
    const int k = r2 >> 1, part = r2 & 1;
    for (int e = t; e < SP_T * SP_T; e += blockDim.x) vis[(e / SP_T) * (SP_T + 1) + e % SP_T] = a.Vinv[e];
    for (int e = t; e < p * p; e += blockDim.x) ds[e] = a.Dm[e];
    for (int e = t; e < 3 * p * p; e += blockDim.x) {
        const int fld = e / (p * p), node = e % (p * p);
        const int g = a.elem_g[(size_t)leaf * p * p + node];
        us[fld][node] = g >= 0 ? a.u[(((size_t)k * 3 + fld) * a.N + g) * 2 + part] : 0.0;
    }
    __syncthreads();
    for (int e = t; e < q2; e += blockDim.x) {
        const int i = e % q + 1, j = e / q + 1;        // interior node (i, j), node index j*p + i
        double dx0 = 0.0, dx1 = 0.0, dy0 = 0.0, dy1 = 0.0;
        for (int kk = 0; kk < p; ++kk) {
            const double dxw = ds[i * p + kk], dyw = ds[j * p + kk];
            dx0 = fma(dxw, us[0][j * p + kk], dx0);
            dx1 = fma(dxw, us[1][j * p + kk], dx1);
            dy0 = fma(dyw, us[0][kk * p + i], dy0);
            dy1 = fma(dyw, us[1][kk * p + i], dy1);
        }
        fs[0][e] = us[2][j * p + i];
        fs[1][e] = a.c1 * (dx0 + dy1);
        fs[2][e] = a.c1 * (dx1 - dy0);
    }
    __syncthreads();
    for (int e = t; e < 3 * q2; e += blockDim.x) {
        const int f = e / q2, node = e % q2, ip = node % q, j = node / q;
        double sum = 0.0;
        for (int i = 0; i < q; ++i) sum = fma(vis[ip * (SP_T + 1) + i], fs[f][j * q + i], sum);
        ts[f][j * q + ip] = sum;
    }
    __syncthreads();
    for (int e = t; e < 3 * q2; e += blockDim.x) {
        const int f = e / q2, mode = e % q2, ip = mode % q, jp = mode / q;
        double sum = 0.0;
        for (int j = 0; j < q; ++j) sum = fma(ts[f][j * q + ip], vis[jp * (SP_T + 1) + j], sum);
        a.G[((size_t)(f * q + ip) * q + jp) * ((size_t)a.nelem * a.R2) + (size_t)leaf * a.R2 + r2] = sum;
    }
}

// --------------------------------------------------------------------------
// k_spec_back: interior E_k = V (sum_groups E^_k + sum_f Pi_kf .* G_f) V^T and the
// owned edge nodes' sums over groups   (grid: nelem * R2 CTAs)
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(SP_THREADS) k_spec_back(SpecArgs a) {
    __shared__ double es[3][SP_T * SP_T];
    __shared__ double ts[3][SP_T * SP_T];
    __shared__ double vs[SP_T * (SP_T + 1)];
    __shared__ double eb[3][SP_NB];
    const int q = a.q, q2 = q * q, nbnd = 4 * q, t = threadIdx.x;
    const int leaf = blockIdx.x / a.R2, r2 = blockIdx.x % a.R2;
    const size_t ncol = (size_t)a.nelem * a.R2, col = blockIdx.x;   // column = leaf * R2 + r2
    for (int e = t; e < SP_T * SP_T; e += blockDim.x) vs[(e / SP_T) * (SP_T + 1) + e % SP_T] = a.V[e];
    __syncthreads();
    for (int e = t; e < a.nE * q2; e += blockDim.x) {
        const int kk = e / q2, mode = e % q2, ip = mode % q, jp = mode / q;
        const double* src = a.Ehat + ((size_t)(kk * q + ip) * q + jp) * ncol + col;
        double s = 0.0;
        for (int gi = 0; gi < 2 * a.ngroups; ++gi) s += src[(size_t)gi * a.nE * q2 * ncol];
        // pole-independent RHS part: sum_f Pi_kf G_f
        const double* G = a.G + ((size_t)ip * q + jp) * ncol + col;
        for (int f = 0; f < a.nF; ++f) s += a.Pi[((size_t)kk * a.nF + f) * SP_T * SP_T + ip * SP_T + jp] * G[(size_t)f * q2 * ncol];
        es[kk][mode] = s;   // E^[i'][j'] at j'*q + i'
    }
    // owned edge segments: sum over groups (into shared memory), then back from
    // the edge basis, E = V E' per segment (after the barrier below)
    for (int e = t; e < a.nE * nbnd; e += blockDim.x) {
        const int kk = e / nbnd, b = e % nbnd;
        double s = 0.0;
        if (a.own[(size_t)leaf * nbnd + b]) {
            const double* src = a.Eedge + ((size_t)kk * a.NE + a.gB[(size_t)leaf * nbnd + b]) * a.R2 + r2;
            for (int gi = 0; gi < a.ngroups; ++gi) s += src[(size_t)gi * a.nE * a.NE * a.R2];
        }
        eb[kk][b] = s;
    }
    __syncthreads();
    for (int e = t; e < a.nE * nbnd; e += blockDim.x) {
        const int kk = e / nbnd, b = e % nbnd;
        if (!a.own[(size_t)leaf * nbnd + b]) continue;
        const int side = b / q, s1 = b % q;
        double s = 0.0;
        for (int kq = 0; kq < q; ++kq) s = fma(vs[s1 * (SP_T + 1) + kq], eb[kk][side * q + kq], s);
        a.E[((size_t)kk * a.R2 + r2) * a.N + (a.N - a.NE) + a.gB[(size_t)leaf * nbnd + b]] = s;
    }
    // T1[(j', i)] = sum_i' V[i][i'] E^[i'][j']
    for (int e = t; e < a.nE * q2; e += blockDim.x) {
        const int kk = e / q2, node = e % q2, i = node % q, jp = node / q;
        double s = 0.0;
        for (int ipp = 0; ipp < q; ++ipp) s = fma(vs[i * (SP_T + 1) + ipp], es[kk][jp * q + ipp], s);
        ts[kk][jp * q + i] = s;
    }
    __syncthreads();
    // E[i][j] = sum_j' T1[(j', i)] V[j][j']
    for (int e = t; e < a.nE * q2; e += blockDim.x) {
        const int kk = e / q2, node = e % q2, i = node % q, j = node / q;
        double s = 0.0;
        for (int jpp = 0; jpp < q; ++jpp) s = fma(ts[kk][jpp * q + i], vs[j * (SP_T + 1) + jpp], s);
        a.E[((size_t)kk * a.R2 + r2) * a.N + (size_t)leaf * q2 + node] = s;
    }
}

// --------------------------------------------------------------------------
// Batched forms of the two once-per-step transforms (round 2): one CTA owns a
// leaf and RB consecutive real right-hand sides (thread = (slot, r), r fastest),
// so the state is read as whole complex values (16 B, node-fastest), G / E^ /
// Eedge are accessed in RB x 8-byte runs and E is written node-fastest - the
// one-(leaf, RHS) kernels above touch one 8-byte word per 32-byte sector
// (k_spec_pre_fused 0.41 TB/s, k_spec_back 0.55 TB/s on config 3,
// profiles/r02b_launches_c3.csv).  Dynamic shared memory: sp_pre_smem / sp_back_smem.
// --------------------------------------------------------------------------
template <int RB>
__host__ __device__ constexpr size_t sp_pre_smem(int p, int q) {
    return (size_t)(3 * p * p * RB + 3 * q * q * RB + SP_T * (SP_T + 1) + p * p) * sizeof(double);
}
template <int RB>
__global__ void __launch_bounds__(SP_THREADS) k_spec_pre_fused_b(SpecArgs a) {
    extern __shared__ double spsm[];
    const int q = a.q, p = a.p, q2 = q * q, pp = p * p, t = threadIdx.x;
    double* us = spsm;                       // [3][pp][RB]; reused as ts [3][q2][RB]
    double* fs = us + 3 * pp * RB;           // [3][q2][RB]
    double* vis = fs + 3 * q2 * RB;          // [16][17]
    double* ds = vis + SP_T * (SP_T + 1);    // [pp]
    const int nrb = a.R2 / RB;
    const int leaf = blockIdx.x / nrb, r20 = (blockIdx.x % nrb) * RB;
    constexpr int NS = SP_THREADS / RB;      // slots
    const int r = t % RB, slot = t / RB;
    for (int e = t; e < SP_T * SP_T; e += SP_THREADS) vis[(e / SP_T) * (SP_T + 1) + e % SP_T] = a.Vinv[e];
    for (int e = t; e < pp; e += SP_THREADS) ds[e] = a.Dm[e];
    // whole complex values: (c, fld, node), node fastest
    for (int e = t; e < (RB / 2) * 3 * pp; e += SP_THREADS) {
        const int node = e % pp, fld = (e / pp) % 3, c = e / (3 * pp);
        const int g = a.elem_g[(size_t)leaf * pp + node];
        double2 v = make_double2(0.0, 0.0);
        if (g >= 0) v = reinterpret_cast<const double2*>(a.u)[((size_t)(r20 / 2 + c) * 3 + fld) * a.N + g];
        us[(fld * pp + node) * RB + 2 * c] = v.x;
        us[(fld * pp + node) * RB + 2 * c + 1] = v.y;
    }
    __syncthreads();
    for (int e = slot; e < q2; e += NS) {
        const int i = e % q + 1, j = e / q + 1;
        double dx0 = 0.0, dx1 = 0.0, dy0 = 0.0, dy1 = 0.0;
        for (int kk = 0; kk < p; ++kk) {
            const double dxw = ds[i * p + kk], dyw = ds[j * p + kk];
            dx0 = fma(dxw, us[(0 * pp + j * p + kk) * RB + r], dx0);
            dx1 = fma(dxw, us[(1 * pp + j * p + kk) * RB + r], dx1);
            dy0 = fma(dyw, us[(0 * pp + kk * p + i) * RB + r], dy0);
            dy1 = fma(dyw, us[(1 * pp + kk * p + i) * RB + r], dy1);
        }
        fs[(0 * q2 + e) * RB + r] = us[(2 * pp + j * p + i) * RB + r];
        fs[(1 * q2 + e) * RB + r] = a.c1 * (dx0 + dy1);
        fs[(2 * q2 + e) * RB + r] = a.c1 * (dx1 - dy0);
    }
    __syncthreads();
    double* ts = us;
    for (int e = slot; e < 3 * q2; e += NS) {
        const int f = e / q2, node = e % q2, ip = node % q, j = node / q;
        double sum = 0.0;
        for (int i = 0; i < q; ++i) sum = fma(vis[ip * (SP_T + 1) + i], fs[(f * q2 + j * q + i) * RB + r], sum);
        ts[(f * q2 + j * q + ip) * RB + r] = sum;
    }
    __syncthreads();
    for (int e = slot; e < 3 * q2; e += NS) {
        const int f = e / q2, mode = e % q2, ip = mode % q, jp = mode / q;
        double sum = 0.0;
        for (int j = 0; j < q; ++j) sum = fma(ts[(f * q2 + j * q + ip) * RB + r], vis[jp * (SP_T + 1) + j], sum);
        a.G[((size_t)(f * q + ip) * q + jp) * ((size_t)a.nelem * a.R2) + (size_t)leaf * a.R2 + r20 + r] = sum;
    }
}

template <int RB>
__host__ __device__ constexpr size_t sp_back_smem(int q) {
    return (size_t)(2 * 3 * q * q * RB + SP_T * (SP_T + 1) + 3 * SP_NB * RB) * sizeof(double);
}
template <int RB>
__global__ void __launch_bounds__(SP_THREADS) k_spec_back_b(SpecArgs a) {
    extern __shared__ double spsm[];
    const int q = a.q, q2 = q * q, nbnd = 4 * q, t = threadIdx.x;
    double* es = spsm;                       // [3][q2][RB]; reused as the output tile [3][RB][q2]
    double* ts = es + 3 * q2 * RB;           // [3][q2][RB]
    double* vs = ts + 3 * q2 * RB;           // [16][17]
    double* eb = vs + SP_T * (SP_T + 1);     // [3][SP_NB][RB]
    const int nrb = a.R2 / RB;
    const int leaf = blockIdx.x / nrb, r20 = (blockIdx.x % nrb) * RB;
    constexpr int NS = SP_THREADS / RB;
    const int r = t % RB, slot = t / RB;
    const size_t ncol = (size_t)a.nelem * a.R2, col = (size_t)leaf * a.R2 + r20 + r;
    for (int e = t; e < SP_T * SP_T; e += SP_THREADS) vs[(e / SP_T) * (SP_T + 1) + e % SP_T] = a.V[e];
    for (int e = slot; e < a.nE * q2; e += NS) {
        const int kk = e / q2, mode = e % q2, ip = mode % q, jp = mode / q;
        const double* src = a.Ehat + ((size_t)(kk * q + ip) * q + jp) * ncol + col;
        double s = 0.0;
        for (int gi = 0; gi < 2 * a.ngroups; ++gi) s += src[(size_t)gi * a.nE * q2 * ncol];
        const double* G = a.G + ((size_t)ip * q + jp) * ncol + col;
        for (int f = 0; f < a.nF; ++f)
            s += a.Pi[((size_t)kk * a.nF + f) * SP_T * SP_T + ip * SP_T + jp] * G[(size_t)f * q2 * ncol];
        es[(kk * q2 + mode) * RB + r] = s;
    }
    for (int e = slot; e < a.nE * nbnd; e += NS) {
        const int kk = e / nbnd, b = e % nbnd;
        double s = 0.0;
        if (a.own[(size_t)leaf * nbnd + b]) {
            const double* src = a.Eedge + ((size_t)kk * a.NE + a.gB[(size_t)leaf * nbnd + b]) * a.R2 + r20 + r;
            for (int gi = 0; gi < a.ngroups; ++gi) s += src[(size_t)gi * a.nE * a.NE * a.R2];
        }
        eb[(kk * SP_NB + b) * RB + r] = s;
    }
    __syncthreads();
    for (int e = slot; e < a.nE * nbnd; e += NS) {
        const int kk = e / nbnd, b = e % nbnd;
        if (!a.own[(size_t)leaf * nbnd + b]) continue;
        const int side = b / q, s1 = b % q;
        double s = 0.0;
        for (int kq = 0; kq < q; ++kq) s = fma(vs[s1 * (SP_T + 1) + kq], eb[(kk * SP_NB + side * q + kq) * RB + r], s);
        a.E[((size_t)kk * a.R2 + r20 + r) * a.N + (a.N - a.NE) + a.gB[(size_t)leaf * nbnd + b]] = s;
    }
    for (int e = slot; e < a.nE * q2; e += NS) {
        const int kk = e / q2, node = e % q2, i = node % q, jp = node / q;
        double s = 0.0;
        for (int ipp = 0; ipp < q; ++ipp) s = fma(vs[i * (SP_T + 1) + ipp], es[(kk * q2 + jp * q + ipp) * RB + r], s);
        ts[(kk * q2 + jp * q + i) * RB + r] = s;
    }
    __syncthreads();
    double* out = es;                        // [3][RB][q2]
    for (int e = slot; e < a.nE * q2; e += NS) {
        const int kk = e / q2, node = e % q2, i = node % q, j = node / q;
        double s = 0.0;
        for (int jpp = 0; jpp < q; ++jpp) s = fma(ts[(kk * q2 + jpp * q + i) * RB + r], vs[j * (SP_T + 1) + jpp], s);
        out[(kk * RB + r) * q2 + node] = s;
    }
    __syncthreads();
    for (int e = t; e < a.nE * RB * q2; e += SP_THREADS) {
        const int node = e % q2, rr = (e / q2) % RB, kk = e / (q2 * RB);
        a.E[((size_t)kk * a.R2 + r20 + rr) * a.N + (size_t)leaf * q2 + node] = out[e];
    }
}

}  // namespace dev
}  // namespace rexp

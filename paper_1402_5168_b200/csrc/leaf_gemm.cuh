// Spectral leaf solves of the shared store as FP64 DMMA GEMMs over (pole x column).
//
// The spectral leaf algebra (leaf_spec.cuh header): per half pole
// m, leaf and real right-hand side, W_m = Dinv_m .* sum_f c_mf G_f in the
// eigenbasis of K = D2[1..q][1..q].  Both leaf passes are linear in the
// pole-independent data with pole-dependent coefficients, so for one edge
// index r of one orientation o they are dense products whose other dimension
// is every (leaf, RHS) column of the level at once:
//
// UP (flux of the particular solution, edge basis):
//   o = 0 (rows, r = i'):  h[m][bottom|top, r] = -/+ c1 sum_{f,j'} c_mf Dinv_m[r][j'] e_{0|1}[j'] G_f[r][j']
//   o = 1 (cols, r = j'):  h[m][left|right, r] = -/+ c1 sum_{f,i'} c_mf Dinv_m[i'][r] e_{0|1}[i'] G_f[i'][r]
//   C[(m, side, re|im) x col] = A_up[(m, side, re|im) x (f, t)] * B[(f, t) x col],  K = nF q,
//   B = the pole-independent spectral RHS fields G (k_spec_pre_fused), real.
// DOWN (pole sums of the boundary-driven interior solutions):
//   E^_k[mode] += sum_m Re(w_mk[mode] b_m[mode]),  w_mk = -c2 d_mk Dinv_m,
//   b_m = a0^[i'] ul[j'] + a1^[i'] ur[j'] + ub[i'] a0^[j'] + ut[i'] a1^[j'],
//   so for the two sides of orientation o at edge index r (o = 0: left/right,
//   r = j', free t = i'; o = 1: bottom/top, r = i', free t = j')
//   E^_k[t] = sum_{m, s, re|im} A_dn[(k, t) x (m, s, re|im)] u_m[side(o, s), r](re|im),
//   plus 2 nE rows with A = d_mk on side s only: the owned edge segments' pole
//   sums sum_m Re(d_mk u_m).  K = 4 x half poles: the pole sum IS the contraction.
//
// A_up and A_dn are formed on the host at setup (device.cu).  Real DMMA
// (mma.sync.m8n8k4.f64): the complex coefficients enter as separate re / im
// rows (UP) or columns (DOWN).  Operands are staged in shared memory by
// cp.async (16-byte copies); row strides are 4 (mod 16) doubles so the
// fragment reads of a half-warp hit 16 distinct banks.
#pragma once

#include "cgemm.cuh"

namespace rexp {
namespace dev {

struct LeafGemmArgs {
    int q, nelem, R2, ncol;   // ncol = nelem * R2 (column = leaf * R2 + r2)
    int nF, nE;
    const int* gB;            // [nelem][4q] edge node of each leaf boundary slot
    const int* own;           // [nelem][4q] 1 where the leaf owns that edge node's pole sum
    // UP
    const double* Aup;        // [2q][4 nh][KP] (row 4 m + 2 s + c) for this chunk: row 4 m0 of each (o, r) block
    long long aup_os;         // doubles between (o, r) blocks
    int Mrows;                // 4 * pc valid rows
    const double* G;          // [nF][q][q][ncol]
    double2* h;               // [pc][hps][R2]
    long long hps;
    double c1;
    // UP, parity-split form (k_leaf_gemm_up_eo): A rows 2 m + c, K = [even modes | odd modes]
    const double* Aup2;       // [2q][2 nh][LG_KP2]
    long long aup2_os;
    const int* kmap;          // [LG_KP2] k -> f q + t (-1: padding)
    // DOWN, parity-split form (k_leaf_gemm_down_eo): rows [even modes + edge-e | odd modes + edge-o],
    // K = (m, re|im); operand u_0 + u_1 for the first row group, u_0 - u_1 for the second
    const double* Adn2;       // [2q][16 MTH][lda2]
    long long adn2_os;
    int lda2;                 // 2 * nh
    const int* rmap;          // [16 MTH] row -> k q + t (interior), -1 - k (edge sums), INT_MIN (padding)
    // DOWN
    const double* Adn;        // [2q][8 MT][lda] for this chunk: column 4 m0
    long long adn_os;         // doubles between (o, r) blocks
    int lda;                  // 4 * nh (leading dimension)
    int Kdn;                  // 4 * pc
    int ksplit;               // K slices (grid.z = 2q * ksplit), one partial slot each
    const double2* edge;      // [pc][NE][R2]
    long long NE;
    double* Ehat;             // [slots][2][nE][q][q][ncol]  (this lane's first slot; per orientation)
    double* Eedge;            // [slots][nE][NE][R2]
    long long ehat_ss, eedge_ss;   // slot strides
    int accumulate;
};

// --------------------------------------------------------------------------
// UP: C tile BM x BN, whole K (KP) in one stage; warps WM x WN, warp tile
// (BM / WM) x (BN / WN).  grid (m-tiles, column tiles, 2q): consecutive CTAs
// share the B tile (L2), every CTA of an (o, r) shares its A block.
// Row order of A_up (chunk-local m): row 4 m + 2 s + c, c = 0 re, 1 im.
// --------------------------------------------------------------------------
constexpr int LG_LDK = 52;    // row stride of A tiles (doubles), = 4 mod 16

template <int KP, int BM, int BN>
constexpr size_t lg_up_smem() {
    return ((size_t)BM * LG_LDK + (size_t)KP * (BN + 4)) * sizeof(double);
}

template <int KP, int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN) k_leaf_gemm_up(LeafGemmArgs a) {
    constexpr int NT = 32 * WM * WN;
    constexpr int TM = BM / WM, TN = BN / WN, MT = TM / 8, NTL = TN / 8;
    constexpr int LDB = BN + 4;
    static_assert(KP % 4 == 0 && KP + 4 <= LG_LDK, "K padding");
    static_assert(MT % 2 == 0 || MT == 1, "m-tiles");
    extern __shared__ double lsm[];
    double* As = lsm;                   // [BM][LG_LDK]  A[row][k]
    double* Bs = lsm + BM * LG_LDK;     // [KP][LDB]     B[k][col]
    const int q = a.q;
    const int mt0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
    const int o = blockIdx.z / q, r = blockIdx.z % q;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int wm = wid / WN, wn = wid % WN;
    const int g = lane >> 2, t4 = lane & 3;
    const double* A = a.Aup + (size_t)blockIdx.z * a.aup_os;
    // A rows [mt0, mt0 + BM): KP contiguous doubles each
    for (int e = tid; e < BM * (KP / 2); e += NT) {
        const int row = e / (KP / 2), c2 = e % (KP / 2);
        double* d = As + row * LG_LDK + 2 * c2;
        if (mt0 + row < a.Mrows) cp_async16(d, A + (size_t)(mt0 + row) * KP + 2 * c2);
        else { d[0] = 0.0; d[1] = 0.0; }
    }
    // B rows k = (f, t): G_f[(o ? t : r)][(o ? r : t)][col0 .. col0 + BN)
    const int Kv = a.nF * q;
    for (int e = tid; e < KP * (BN / 2); e += NT) {
        const int kk = e / (BN / 2), c2 = e % (BN / 2);
        double* d = Bs + kk * LDB + 2 * c2;
        const int col = col0 + 2 * c2;
        if (kk < Kv && col < a.ncol) {
            const int f = kk / q, t = kk % q;
            const int ip = o ? t : r, jp = o ? r : t;
            cp_async16(d, a.G + ((size_t)(f * q + ip) * q + jp) * a.ncol + col);
        } else {
            d[0] = 0.0; d[1] = 0.0;
        }
    }
    cp_async_commit();
    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NTL; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KP / 4; ++ks) {
        const int kk = ks * 4 + t4;
        double av[MT], bv[NTL];
#pragma unroll
        for (int i = 0; i < MT; ++i) av[i] = As[(wm * TM + i * 8 + g) * LG_LDK + kk];
#pragma unroll
        for (int n = 0; n < NTL; ++n) bv[n] = Bs[kk * LDB + wn * TN + n * 8 + g];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int n = 0; n < NTL; ++n) dmma884(acc[i][n][0], acc[i][n][1], av[i], bv[n]);
    }
    // epilogue: row 2 P + c holds part c (re, im) of pair P = 2 m + s, i.e. threads
    // g (even) and g + 1 of a quad column share an output; they swap one value
    // (lane ^ 4) and each stores one complex: even g column j = 0, odd g j = 1
    const bool ev = (g & 1) == 0;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = mt0 + wm * TM + i * 8 + g;
        const int P = row >> 1, m = P >> 1, s = P & 1;
        const int side = o ? (s ? 1 : 3) : (s ? 2 : 0);
        double2* dst = a.h + ((size_t)m * a.hps + side * q + r) * a.R2;
#pragma unroll
        for (int n = 0; n < NTL; ++n) {
            const double x = ev ? acc[i][n][1] : acc[i][n][0];
            const double y = __shfl_xor_sync(0xffffffffu, x, 4);
            if (4 * m >= a.Mrows) continue;
            const int col = col0 + wn * TN + n * 8 + 2 * t4 + (ev ? 0 : 1);
            if (col >= a.ncol) continue;
            const int leaf = col / a.R2, r2 = col - leaf * a.R2;
            dst[(size_t)leaf * 4 * q * a.R2 + r2] = ev ? make_double2(acc[i][n][0], y) : make_double2(y, acc[i][n][1]);
        }
    }
}

// --------------------------------------------------------------------------
// UP, parity-split (round 2).  The eigenvectors of K are even or odd under the
// node reversal, and the end rows of the differentiation matrix are mirror
// images with opposite sign, so e_1 = -Pi e_0 (Pi = diag(mode parity)) and the
// coefficients of the two sides of an orientation differ only by the parity of
// the summed mode: A(side 1; t) = pi_t A(side 0; t).  With
//   E = sum_{t even} A(side 0; f, t) G_f[t],   O = sum_{t odd} A(side 0; f, t) G_f[t]
// the two sides are h_0 = E + O, h_1 = E - O: rows (m, re|im) only, K split into
// [even | odd] halves of LG_KH columns accumulated separately - 0.55 of the
// DMMAs of the (m, side, re|im) x (f, t) form.
// --------------------------------------------------------------------------
constexpr int LG_KH = 24, LG_KP2 = 2 * LG_KH;   // nF * ceil(q / 2) <= 24 for q <= 16

template <int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN) k_leaf_gemm_up_eo(LeafGemmArgs a) {
    constexpr int NT = 32 * WM * WN, KP = LG_KP2;
    constexpr int TM = BM / WM, TN = BN / WN, MT = TM / 8, NTL = TN / 8;
    constexpr int LDB = BN + 4;
    static_assert(KP + 4 <= LG_LDK, "K padding");
    extern __shared__ double lsm[];
    double* As = lsm;                   // [BM][LG_LDK]
    double* Bs = lsm + BM * LG_LDK;     // [KP][LDB]
    const int q = a.q;
    const int mt0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
    const int o = blockIdx.z / q, r = blockIdx.z % q;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int wm = wid / WN, wn = wid % WN;
    const int g = lane >> 2, t4 = lane & 3;
    const int Mrows = a.Mrows / 2;      // 2 rows per half pole
    const double* A = a.Aup2 + (size_t)blockIdx.z * a.aup2_os;
    for (int e = tid; e < BM * (KP / 2); e += NT) {
        const int row = e / (KP / 2), c2 = e % (KP / 2);
        double* d = As + row * LG_LDK + 2 * c2;
        if (mt0 + row < Mrows) cp_async16(d, A + (size_t)(mt0 + row) * KP + 2 * c2);
        else { d[0] = 0.0; d[1] = 0.0; }
    }
    for (int e = tid; e < KP * (BN / 2); e += NT) {
        const int kk = e / (BN / 2), c2 = e % (BN / 2);
        double* d = Bs + kk * LDB + 2 * c2;
        const int col = col0 + 2 * c2;
        const int ft = a.kmap[kk];
        if (ft >= 0 && col < a.ncol) {
            const int f = ft / q, t = ft % q;
            const int ip = o ? t : r, jp = o ? r : t;
            cp_async16(d, a.G + ((size_t)(f * q + ip) * q + jp) * a.ncol + col);
        } else {
            d[0] = 0.0; d[1] = 0.0;
        }
    }
    cp_async_commit();
    double acc[2][MT][NTL][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int n = 0; n < NTL; ++n) acc[h][i][n][0] = acc[h][i][n][1] = 0.0;
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int ks = 0; ks < LG_KH / 4; ++ks) {
            const int kk = h * LG_KH + ks * 4 + t4;
            double av[MT], bv[NTL];
#pragma unroll
            for (int i = 0; i < MT; ++i) av[i] = As[(wm * TM + i * 8 + g) * LG_LDK + kk];
#pragma unroll
            for (int n = 0; n < NTL; ++n) bv[n] = Bs[kk * LDB + wn * TN + n * 8 + g];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int n = 0; n < NTL; ++n) dmma884(acc[h][i][n][0], acc[h][i][n][1], av[i], bv[n]);
        }
    // epilogue: rows 2 m + c; threads g (even: re) and g + 1 (odd: im) of a quad column
    // swap one value (lane ^ 4) and each stores one complex per side
    const bool ev = (g & 1) == 0;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = mt0 + wm * TM + i * 8 + g;
        const int m = row >> 1;
#pragma unroll
        for (int n = 0; n < NTL; ++n) {
            // side 0 = E + O, side 1 = E - O for this thread's two columns
            const double s0a = acc[0][i][n][0] + acc[1][i][n][0], s0b = acc[0][i][n][1] + acc[1][i][n][1];
            const double s1a = acc[0][i][n][0] - acc[1][i][n][0], s1b = acc[0][i][n][1] - acc[1][i][n][1];
            const double y0 = __shfl_xor_sync(0xffffffffu, ev ? s0b : s0a, 4);
            const double y1 = __shfl_xor_sync(0xffffffffu, ev ? s1b : s1a, 4);
            if (2 * m >= Mrows) continue;
            const int col = col0 + wn * TN + n * 8 + 2 * t4 + (ev ? 0 : 1);
            if (col >= a.ncol) continue;
            const int leaf = col / a.R2, r2 = col - leaf * a.R2;
            const int sd0 = o ? 3 : 0, sd1 = o ? 1 : 2;
            double2* d0 = a.h + ((size_t)m * a.hps + sd0 * q + r) * a.R2 + (size_t)leaf * 4 * q * a.R2 + r2;
            double2* d1 = a.h + ((size_t)m * a.hps + sd1 * q + r) * a.R2 + (size_t)leaf * 4 * q * a.R2 + r2;
            *d0 = ev ? make_double2(s0a, y0) : make_double2(y0, s0b);
            *d1 = ev ? make_double2(s1a, y1) : make_double2(y1, s1b);
        }
    }
}
inline size_t lg_up_eo_smem(int BM, int BN) {
    return ((size_t)BM * LG_LDK + (size_t)LG_KP2 * (BN + 4)) * sizeof(double);
}

// --------------------------------------------------------------------------
// DOWN: C tile (8 MT) x BN, K = 4 pc in chunks of 16 (4 half poles) through an
// NST-stage cp.async ring; BN / 32 warps side by side in n, each MT x 4 tiles.
// Thread c < BN stages column c of every B chunk (its leaf's edge nodes are fixed).
// grid (column tiles, 2q * ksplit).
// --------------------------------------------------------------------------
constexpr int LGD_BK = 16, LGD_LDA = LGD_BK + 4;
constexpr int LGD_NST = 3;    // cp.async ring depth of the DOWN GEMM

template <int MT, int BN, int NST>
constexpr size_t lg_dn_smem() {
    return (size_t)NST * ((size_t)8 * MT * LGD_LDA + (size_t)(LGD_BK / 2) * (2 * BN + 8)) * sizeof(double);
}

template <int MT, int BN, int NST>
__global__ void __launch_bounds__(BN) k_leaf_gemm_down(LeafGemmArgs a) {
    constexpr int BM = 8 * MT, NT = BN, NTL = 4, LDP = 2 * BN + 8, BP = LGD_BK / 2;
    constexpr int ASZ = BM * LGD_LDA, BSZ = BP * LDP;
    extern __shared__ double lsm[];
    const int q = a.q;
    const int col0 = blockIdx.x * BN;
    const int orr = blockIdx.y / a.ksplit, ks = blockIdx.y % a.ksplit;
    const int o = orr / q, r = orr % q;
    const int tid = threadIdx.x, lane = tid & 31, wn = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    // this slice's K range (whole half poles: 4 k per pole)
    const int npole = a.Kdn / 4;
    const int pb = npole / a.ksplit, pr = npole % a.ksplit;
    const int p0 = ks * pb + min(ks, pr), p1 = p0 + pb + (ks < pr ? 1 : 0);
    const double* A = a.Adn + (size_t)orr * a.adn_os;
    // B column of this thread
    const int bcol = col0 + tid;
    const bool bok = bcol < a.ncol;
    const int bleaf = bok ? bcol / a.R2 : 0, br2 = bok ? bcol - bleaf * a.R2 : 0;
    const int sd0 = o ? 0 : 3, sd1 = o ? 2 : 1;          // side of s = 0, 1
    const long long ge0 = a.gB[(size_t)bleaf * 4 * q + sd0 * q + r];
    const long long ge1 = a.gB[(size_t)bleaf * 4 * q + sd1 * q + r];
    auto issue = [&](int st, int pp0) {
        double* As = lsm + st * (ASZ + BSZ);
        double* Bs = As + ASZ;
        // A: BM rows x 16 k (columns 4 pp0 ..), 8 16-byte pieces per row
        for (int e = tid; e < BM * (LGD_BK / 2); e += NT) {
            const int row = e / (LGD_BK / 2), c2 = e % (LGD_BK / 2);
            const int k = 4 * pp0 + 2 * c2;
            double* d = As + row * LGD_LDA + 2 * c2;
            if (k < 4 * p1) cp_async16(d, A + (size_t)row * a.lda + k);
            else { d[0] = 0.0; d[1] = 0.0; }
        }
        // B: pairs (m, s), m = pp0 .. pp0 + 3
#pragma unroll
        for (int pp = 0; pp < BP; ++pp) {
            const int m = pp0 + (pp >> 1);
            double* d = Bs + pp * LDP + 2 * tid;
            if (bok && m < p1)
                cp_async16(d, a.edge + ((size_t)m * a.NE + ((pp & 1) ? ge1 : ge0)) * a.R2 + br2);
            else { d[0] = 0.0; d[1] = 0.0; }
        }
        cp_async_commit();
    };
    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NTL; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    const int nch = (p1 - p0 + 3) / 4;
#pragma unroll
    for (int st = 0; st < NST - 1; ++st) {
        if (st < nch) issue(st, p0 + 4 * st);
        else cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait_group<NST - 2>();
        __syncthreads();
        const int nx = ch + NST - 1;
        if (nx < nch) issue(nx % NST, p0 + 4 * nx);
        else cp_async_commit();
        const double* As = lsm + (ch % NST) * (ASZ + BSZ);
        const double* Bs = As + ASZ;
#pragma unroll
        for (int kb = 0; kb < LGD_BK / 4; ++kb) {
            const int kk = kb * 4 + t4;
            double av[MT], bv[NTL];
#pragma unroll
            for (int i = 0; i < MT; ++i) av[i] = As[(i * 8 + g) * LGD_LDA + kk];
            // B[k][n]: pair 2 kb + (t4 >> 1), component t4 & 1
#pragma unroll
            for (int n = 0; n < NTL; ++n) bv[n] = Bs[(2 * kb + (t4 >> 1)) * LDP + 2 * (wn * 32 + n * 8 + g) + (t4 & 1)];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int n = 0; n < NTL; ++n) dmma884(acc[i][n][0], acc[i][n][1], av[i], bv[n]);
        }
    }
    // epilogue: rows (k, t) < nE q -> E^ ; rows nE q + (k, s) -> owned edge pole sums
    // both orientations contribute to every interior mode (left/right and
    // bottom/top sides): separate E^ slots per orientation, summed in k_spec_back;
    // the edge rows of (o, r) are distinct edge nodes
    double* Eh = a.Ehat + (size_t)(2 * ks + o) * a.ehat_ss;
    double* Ee = a.Eedge + (size_t)ks * a.eedge_ss;
    const int nint = a.nE * q;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = i * 8 + g;
        if (row >= nint + 2 * a.nE) continue;
#pragma unroll
        for (int n = 0; n < NTL; ++n)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int col = col0 + wn * 32 + n * 8 + 2 * t4 + j;
                if (col >= a.ncol) continue;
                double v = acc[i][n][j];
                if (row < nint) {
                    const int k = row / q, t = row % q;
                    const int ip = o ? r : t, jp = o ? t : r;
                    double* d = Eh + ((size_t)(k * q + ip) * q + jp) * a.ncol + col;
                    if (a.accumulate) v += *d;
                    *d = v;
                } else {
                    const int e = row - nint, k = e >> 1, s = e & 1;
                    const int leaf = col / a.R2, r2 = col - leaf * a.R2;
                    const int b = (s ? sd1 : sd0) * q + r;
                    if (!a.own[(size_t)leaf * 4 * q + b]) continue;
                    double* d = Ee + ((size_t)k * a.NE + a.gB[(size_t)leaf * 4 * q + b]) * a.R2 + r2;
                    if (a.accumulate) v += *d;
                    *d = v;
                }
            }
    }
}

// --------------------------------------------------------------------------
// DOWN, parity-split (round 2).  a1^ = Pi a0^ (D2's end columns are mirror
// images), so the coefficients of the two sides of an orientation differ by the
// parity of the output mode t: A((k, t); m, side 1) = pi_t A((k, t); m, side 0).
// Rows of even modes therefore contract with u_0 + u_1, rows of odd modes with
// u_0 - u_1, both over K = (m, re|im) only: half the DMMAs.  The owned edge sums
// sum_m Re(d_mk u_m[side]) ride along as a half-weight row in each group,
// side 0 = e + o, side 1 = e - o (same thread: the groups have equal sizes).
// Row groups of MTH m-tiles each; chunks of PB half poles (2 PB k).
// --------------------------------------------------------------------------
template <int MTH, int BN, int NST, int PB>
constexpr size_t lg_dn_eo_smem() {
    return (size_t)NST * ((size_t)16 * MTH * (2 * PB + 4) + (size_t)(2 * PB) * (2 * BN + 8)) * sizeof(double);
}

template <int MTH, int BN, int NST, int PB>
__global__ void __launch_bounds__(BN) k_leaf_gemm_down_eo(LeafGemmArgs a) {
    constexpr int MT = 2 * MTH, BM = 8 * MT, NT = BN, NTL = 4, LDP = 2 * BN + 8, BP = 2 * PB;
    constexpr int BK = 2 * PB, LDA = BK + 4;
    constexpr int ASZ = BM * LDA, BSZ = BP * LDP;
    static_assert(BK % 4 == 0, "k-steps of 4");
    extern __shared__ double lsm[];
    const int q = a.q;
    const int col0 = blockIdx.x * BN;
    const int orr = blockIdx.y / a.ksplit, ks = blockIdx.y % a.ksplit;
    const int o = orr / q, r = orr % q;
    const int tid = threadIdx.x, lane = tid & 31, wn = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int npole = a.Kdn / 4;
    const int pb = npole / a.ksplit, pr = npole % a.ksplit;
    const int p0 = ks * pb + min(ks, pr), p1 = p0 + pb + (ks < pr ? 1 : 0);
    const double* A = a.Adn2 + (size_t)orr * a.adn2_os;
    const int bcol = col0 + tid;
    const bool bok = bcol < a.ncol;
    const int bleaf = bok ? bcol / a.R2 : 0, br2 = bok ? bcol - bleaf * a.R2 : 0;
    const int sd0 = o ? 0 : 3, sd1 = o ? 2 : 1;
    const long long ge0 = a.gB[(size_t)bleaf * 4 * q + sd0 * q + r];
    const long long ge1 = a.gB[(size_t)bleaf * 4 * q + sd1 * q + r];
    auto issue = [&](int st, int pp0) {
        double* As = lsm + st * (ASZ + BSZ);
        double* Bs = As + ASZ;
        for (int e = tid; e < BM * (BK / 2); e += NT) {
            const int row = e / (BK / 2), c2 = e % (BK / 2);
            const int k = 2 * pp0 + 2 * c2;
            double* d = As + row * LDA + 2 * c2;
            if (k < 2 * p1) cp_async16(d, A + (size_t)row * a.lda2 + k);
            else { d[0] = 0.0; d[1] = 0.0; }
        }
#pragma unroll
        for (int pp = 0; pp < BP; ++pp) {
            const int m = pp0 + (pp >> 1);
            double* d = Bs + pp * LDP + 2 * tid;
            if (bok && m < p1)
                cp_async16(d, a.edge + ((size_t)m * a.NE + ((pp & 1) ? ge1 : ge0)) * a.R2 + br2);
            else { d[0] = 0.0; d[1] = 0.0; }
        }
        cp_async_commit();
    };
    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NTL; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    const int nch = (p1 - p0 + PB - 1) / PB;
#pragma unroll
    for (int st = 0; st < NST - 1; ++st) {
        if (st < nch) issue(st, p0 + PB * st);
        else cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait_group<NST - 2>();
        __syncthreads();
        const int nx = ch + NST - 1;
        if (nx < nch) issue(nx % NST, p0 + PB * nx);
        else cp_async_commit();
        const double* As = lsm + (ch % NST) * (ASZ + BSZ);
        const double* Bs = As + ASZ;
#pragma unroll
        for (int kb = 0; kb < BK / 4; ++kb) {
            const int kk = kb * 4 + t4;
            double av[MT], be[NTL], bo[NTL];
#pragma unroll
            for (int i = 0; i < MT; ++i) av[i] = As[(i * 8 + g) * LDA + kk];
            // k = (pole 2 kb + (t4 >> 1), component t4 & 1): u_0 +- u_1 of that pole
#pragma unroll
            for (int n = 0; n < NTL; ++n) {
                const int cidx = 2 * (wn * 32 + n * 8 + g) + (t4 & 1);
                const double u0 = Bs[(2 * (2 * kb + (t4 >> 1))) * LDP + cidx];
                const double u1 = Bs[(2 * (2 * kb + (t4 >> 1)) + 1) * LDP + cidx];
                be[n] = u0 + u1;
                bo[n] = u0 - u1;
            }
#pragma unroll
            for (int i = 0; i < MTH; ++i)
#pragma unroll
                for (int n = 0; n < NTL; ++n) {
                    dmma884(acc[i][n][0], acc[i][n][1], av[i], be[n]);
                    dmma884(acc[MTH + i][n][0], acc[MTH + i][n][1], av[MTH + i], bo[n]);
                }
        }
    }
    double* Eh = a.Ehat + (size_t)(2 * ks + o) * a.ehat_ss;
    double* Ee = a.Eedge + (size_t)ks * a.eedge_ss;
#pragma unroll
    for (int i = 0; i < MTH; ++i) {
        const int row = i * 8 + g;
        const int re = a.rmap[row], ro = a.rmap[8 * MTH + row];
#pragma unroll
        for (int n = 0; n < NTL; ++n)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int col = col0 + wn * 32 + n * 8 + 2 * t4 + j;
                if (col >= a.ncol) continue;
                const double ve = acc[i][n][j], vo = acc[MTH + i][n][j];
                if (re >= 0) {   // interior modes (the two groups' rows are different modes)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int kt = h ? ro : re;
                        if (kt < 0) continue;
                        const int k = kt / q, t = kt % q;
                        const int ip = o ? r : t, jp = o ? t : r;
                        double* d = Eh + ((size_t)(k * q + ip) * q + jp) * a.ncol + col;
                        double v = h ? vo : ve;
                        if (a.accumulate) v += *d;
                        *d = v;
                    }
                } else if (re > -1000000) {   // edge sums of k = -1 - re: side 0 = e + o, side 1 = e - o
                    const int k = -1 - re;
                    const int leaf = col / a.R2, r2 = col - leaf * a.R2;
#pragma unroll
                    for (int sdx = 0; sdx < 2; ++sdx) {
                        const int b = (sdx ? sd1 : sd0) * q + r;
                        if (!a.own[(size_t)leaf * 4 * q + b]) continue;
                        double* d = Ee + ((size_t)k * a.NE + a.gB[(size_t)leaf * 4 * q + b]) * a.R2 + r2;
                        double v = sdx ? ve - vo : ve + vo;
                        if (a.accumulate) v += *d;
                        *d = v;
                    }
                }
            }
    }
}

// variant ids (REXP_LGU / REXP_LGD): UP 0 = 64x128 (2x4 warps), 1 = 64x64 (2x2),
// 2 = 128x64 (4x2), 3 = 32x128 (1x4); DOWN 0 = BN 128 / 3 stages, 1 = 128 / 4,
// 2 = 64 / 3, 3 = 64 / 4
template <int KP>
inline void lg_up_launch(int var, dim3 g3, cudaStream_t s, const LeafGemmArgs& a) {
    switch (var) {
        case 1: k_leaf_gemm_up<KP, 64, 64, 2, 2><<<g3, 128, lg_up_smem<KP, 64, 64>(), s>>>(a); break;
        case 2: k_leaf_gemm_up<KP, 128, 64, 4, 2><<<g3, 256, lg_up_smem<KP, 128, 64>(), s>>>(a); break;
        case 3: k_leaf_gemm_up<KP, 32, 128, 1, 4><<<g3, 128, lg_up_smem<KP, 32, 128>(), s>>>(a); break;
        default: k_leaf_gemm_up<KP, 64, 128, 2, 4><<<g3, 256, lg_up_smem<KP, 64, 128>(), s>>>(a); break;
    }
}
inline void lg_up_tile(int var, int& BM, int& BN) {
    BM = var == 2 ? 128 : var == 3 ? 32 : 64;
    BN = (var == 1 || var == 2) ? 64 : 128;
}
template <int MT>
inline void lg_dn_launch(int var, dim3 g2, cudaStream_t s, const LeafGemmArgs& a) {
    switch (var) {
        case 1: k_leaf_gemm_down<MT, 128, 4><<<g2, 128, lg_dn_smem<MT, 128, 4>(), s>>>(a); break;
        case 2: k_leaf_gemm_down<MT, 64, 3><<<g2, 64, lg_dn_smem<MT, 64, 3>(), s>>>(a); break;
        case 3: k_leaf_gemm_down<MT, 64, 4><<<g2, 64, lg_dn_smem<MT, 64, 4>(), s>>>(a); break;
        default: k_leaf_gemm_down<MT, 128, 3><<<g2, 128, lg_dn_smem<MT, 128, 3>(), s>>>(a); break;
    }
}
inline int lg_dn_bn(int var) { return var >= 2 ? 64 : 128; }
inline void lg_allow() {
#define LG_ALLOW(...) cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
    LG_ALLOW(k_leaf_gemm_up<44, 64, 128, 2, 4>); LG_ALLOW(k_leaf_gemm_up<44, 64, 64, 2, 2>);
    LG_ALLOW(k_leaf_gemm_up<44, 128, 64, 4, 2>); LG_ALLOW(k_leaf_gemm_up<44, 32, 128, 1, 4>);
    LG_ALLOW(k_leaf_gemm_up<48, 64, 128, 2, 4>); LG_ALLOW(k_leaf_gemm_up<48, 64, 64, 2, 2>);
    LG_ALLOW(k_leaf_gemm_up<48, 128, 64, 4, 2>); LG_ALLOW(k_leaf_gemm_up<48, 32, 128, 1, 4>);
    LG_ALLOW(k_leaf_gemm_up_eo<32, 64, 2, 2>); LG_ALLOW(k_leaf_gemm_up_eo<32, 128, 2, 4>);
    LG_ALLOW(k_leaf_gemm_down_eo<2, 128, 3, 4>); LG_ALLOW(k_leaf_gemm_down_eo<3, 128, 3, 4>);
    LG_ALLOW(k_leaf_gemm_down_eo<4, 128, 3, 4>); LG_ALLOW(k_leaf_gemm_down_eo<2, 128, 2, 8>);
    LG_ALLOW(k_leaf_gemm_down_eo<3, 128, 2, 8>); LG_ALLOW(k_leaf_gemm_down_eo<4, 128, 2, 8>);
    LG_ALLOW(k_leaf_gemm_down<6, 128, 3>); LG_ALLOW(k_leaf_gemm_down<6, 128, 4>);
    LG_ALLOW(k_leaf_gemm_down<6, 64, 3>); LG_ALLOW(k_leaf_gemm_down<6, 64, 4>);
    LG_ALLOW(k_leaf_gemm_down<7, 128, 3>); LG_ALLOW(k_leaf_gemm_down<7, 128, 4>);
    LG_ALLOW(k_leaf_gemm_down<7, 64, 3>); LG_ALLOW(k_leaf_gemm_down<7, 64, 4>);
#undef LG_ALLOW
}

}  // namespace dev
}  // namespace rexp

// Tensor-product leaf solve for the constant-coefficient (shared) store.
//
// On a leaf the interior collocation operator is a Kronecker sum
//     A_II = c2 (I (x) K + K (x) I) - sigma,   K = D2[1..q][1..q],  c2 = (2/H)^2
// (§2.2 collocation; interior index (i, j), i fastest), so with
// K = V diag(l) V^-1 (real, kappa(V) ~ 1.6 for q <= 16):
//     A_II^{-1} F = V [ (V^-1 F V^-T) ./ (c2 (l_i + l_j) - sigma) ] V^T        (F: q x q)
// which is exactly the leaf inverse of the HPS solver, applied with four
// 16 x 16 (zero-padded) real x complex products on the FP64 tensor pipe
// (DMMA m8n8k4) instead of one dense q^2 x q^2 complex mat-vec: 7x fewer flops.
//
// One warp owns one (half pole, leaf, real RHS part) problem; tiles live in
// shared memory; only __syncwarp is needed.
//   UP:   u = A_II^{-1} f;  h = N_I u (outward normal flux at the 4q boundary nodes)
//   DOWN: u = A_II^{-1} (f - A_IB u_B) = interior solution (written for the pole sum)
#pragma once

namespace rexp {
namespace dev {

constexpr int FDM_T = 16;          // padded tile edge
constexpr int FDM_LDT = 16;        // tile stride (complex elements), XOR-swizzled columns:
constexpr int FDM_LDD = FDM_LDT;
// element (r, c) of a 16x16 complex tile lives at tix(r, c); the swizzle makes
// both the DMMA C-fragment stores (row g, cols 2t4+{0,1}) and the transposed
// B-fragment loads (row n = g, col k = t4) hit 8 distinct 16-byte slots per
// quarter warp (searched exhaustively)
__device__ __forceinline__ int tix(int r, int c) { return r * FDM_T + (c ^ ((5 * r) & 15)); }
constexpr int FDM_WARPS = 8;
constexpr int FDM_TILE_ELEMS = 2 * FDM_T * FDM_LDT + 4 * 16;     // tiles X, Y + boundary values

struct FdmArgs {
    const double* E01;      // 2 x 16: e0 = V^T d_0, e1 = V^T d_{p-1} (d_r[k] = D[r][k+1]), zero padded
    const double* V;        // 16 x 16 row-major, zero padded
    const double* Vinv;     // 16 x 16 row-major, zero padded
    const double2* Dinv;    // [nh][16*16] 1/(c2 (l_i + l_j) - sigma_m), zero padded
    const double* D;        // p x p
    const double* D2;       // p x p
    const double* F;        // [NI][nF][R2]
    const double2* cF;      // [nh][nF]
    int q, p, nF, nelem, R2, nh;
    double c1, c2;
    // UP
    double2* h;             // [nh][hps][R2]
    long long hps;
    // DOWN
    const double2* edge;    // [nh][NE][R2]
    long long NE;
    const int* gB;          // [nelem][4q]
    double2* w;             // [nh][nelem][q2][R2]
};

__device__ __forceinline__ void dmma884r(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// C (16x16 complex, in fragments) = A (16x16 real, fragments af) * B, where
// B[k][n] = TRANS ? X[n*LD + k] : X[k*LD + n]  (complex tile in shared memory).
constexpr int FDM_LDV = 20;        // stride of V, V^-1 in shared memory (conflict-free per half warp)

template <bool TRANS, int LD>
__device__ __forceinline__ void fdm_stage(const double* As, const double2* X, int g, int t4,
                                          double (&cr)[2][2][2], double (&ci)[2][2][2]) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) cr[mt][nt][0] = cr[mt][nt][1] = ci[mt][nt][0] = ci[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t4;
        double af[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) af[mt] = As[(mt * 8 + g) * FDM_LDV + k];   // A[m][k]
        double2 b[2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int n = nt * 8 + g;
            b[nt] = TRANS ? X[tix(n, k)] : X[tix(k, n)];
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma884r(cr[mt][nt][0], cr[mt][nt][1], af[mt], b[nt].x);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma884r(ci[mt][nt][0], ci[mt][nt][1], af[mt], b[nt].y);
    }
}

// Stage 1 with B = T held in registers in fragment layout: bf[ks][nt] = T[ks*4+t4][nt*8+g].
__device__ __forceinline__ void fdm_stage_reg(const double* As, const double2 (&bf)[4][2], int g, int t4,
                                              double (&cr)[2][2][2], double (&ci)[2][2][2]) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) cr[mt][nt][0] = cr[mt][nt][1] = ci[mt][nt][0] = ci[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        double af[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) af[mt] = As[(mt * 8 + g) * FDM_LDV + ks * 4 + t4];   // A[m][k]
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma884r(cr[mt][nt][0], cr[mt][nt][1], af[mt], bf[ks][nt].x);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma884r(ci[mt][nt][0], ci[mt][nt][1], af[mt], bf[ks][nt].y);
    }
}

// Right-hand side tile T (UP: f; DOWN: f - A_IB u_B) for pole m, then the
// four stages; returns U[i][j] in fragments (cr, ci) at (j = mt*8+g, i = nt*8+2t4+c).
template <bool DOWN, bool HALF = false>
__device__ __forceinline__ void fdm_solve(const FdmArgs& a, int m, int leaf, int r2, int lane, double2* P, double2* Q,
                                          double2* UB, const double* vf, const double* vif,
                                          double (&cr)[2][2][2], double (&ci)[2][2][2]) {
    const int g = lane >> 2, t4 = lane & 3;
    const int q = a.q, p = a.p, q2 = q * q, nb = 4 * q;
    const double2* cf = a.cF + (size_t)m * a.nF;
    const double2 c0 = cf[0];
    const double2 c1v = a.nF > 1 ? cf[1] : make_double2(0, 0);
    const double2 c2v = a.nF > 2 ? cf[2] : make_double2(0, 0);
    // boundary values of this leaf (DOWN) into the warp's UB area
    if (DOWN) {
        for (int b = lane; b < nb; b += 32)
            UB[b] = a.edge[((size_t)m * a.NE + a.gB[(size_t)leaf * nb + b]) * a.R2 + r2];
        __syncwarp();
    }
    // T directly in B-fragment layout: this lane's 8 elements T[i = ks*4+t4][j = nt*8+g]
    double fv[4][2][3];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int i = ks * 4 + t4, j = nt * 8 + g;
            fv[ks][nt][0] = fv[ks][nt][1] = fv[ks][nt][2] = 0.0;
            if (i < q && j < q) {
                const double* f = a.F + ((size_t)((size_t)leaf * q2 + j * q + i) * a.nF) * a.R2 + r2;
                fv[ks][nt][0] = f[0];
                if (a.nF > 1) fv[ks][nt][1] = f[a.R2];
                if (a.nF > 2) fv[ks][nt][2] = f[2 * a.R2];
            }
        }
    // D^-1 entries of this lane's stage-2 fragments, fetched while stages 1-2 run
    const double2* dv = a.Dinv + (size_t)m * FDM_T * FDM_T;
    double2 dinv[2][2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) dinv[mt][nt][c] = __ldg(dv + (nt * 8 + 2 * t4 + c) * FDM_T + mt * 8 + g);
    double2 bf[4][2];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int i = ks * 4 + t4, j = nt * 8 + g;
            double2 v = make_double2(0.0, 0.0);
            if (i < q && j < q) {
                v.x = c0.x * fv[ks][nt][0] + c1v.x * fv[ks][nt][1] + c2v.x * fv[ks][nt][2];
                v.y = c0.y * fv[ks][nt][0] + c1v.y * fv[ks][nt][1] + c2v.y * fv[ks][nt][2];
                if (DOWN) {
                    // A_IB u_B at interior (i+1, j+1): row i+1 meets left/right, column j+1 meets bottom/top
                    const double dl = a.D2[(i + 1) * p + 0], dr = a.D2[(i + 1) * p + (p - 1)];
                    const double db = a.D2[(j + 1) * p + 0], dt = a.D2[(j + 1) * p + (p - 1)];
                    const double2 ul = UB[3 * q + j], ur = UB[q + j], ub = UB[i], ut = UB[2 * q + i];
                    v.x -= a.c2 * (dl * ul.x + dr * ur.x + db * ub.x + dt * ut.x);
                    v.y -= a.c2 * (dl * ul.y + dr * ur.y + db * ub.y + dt * ut.y);
                }
            }
            bf[ks][nt] = v;
        }
    // stage 1: S1 = Vinv T            (contract i)        -> Q[i'][j]
    fdm_stage_reg(vif, bf, g, t4, cr, ci);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                Q[tix(mt * 8 + g, nt * 8 + 2 * t4 + c)] = make_double2(cr[mt][nt][c], ci[mt][nt][c]);
    __syncwarp();
    // stage 2: S2^T = Vinv S1^T       (contract j) -> C[j'][i'], scaled by Dinv (symmetric) -> P[j'][i']
    fdm_stage<true, FDM_LDT>(vif, Q, g, t4, cr, ci);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int jp = mt * 8 + g, ip = nt * 8 + 2 * t4 + c;
                const double2 d = dinv[mt][nt][c];
                const double xr = cr[mt][nt][c], xi = ci[mt][nt][c];
                P[tix(jp, ip)] = make_double2(xr * d.x - xi * d.y, xr * d.y + xi * d.x);
            }
    __syncwarp();
    if (HALF) return;   // spectral coefficients W^T left in P (P[tix(j', i')] = W[i'][j'])
    // stage 3: S3 = V W               (contract i'), W[i'][j'] = P[j'][i']  -> Q[i][j']
    fdm_stage<true, FDM_LDT>(vf, P, g, t4, cr, ci);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                Q[tix(mt * 8 + g, nt * 8 + 2 * t4 + c)] = make_double2(cr[mt][nt][c], ci[mt][nt][c]);
    __syncwarp();
    // stage 4: U^T = V S3^T           (contract j') -> C[j][i] = U[i][j]
    fdm_stage<true, FDM_LDT>(vf, Q, g, t4, cr, ci);
    __syncwarp();   // P, Q reusable by the caller after this point
}

// MODE 0 = UP (h = N_I A^-1 f, from the spectral coefficients), 1 = DOWN
// (interior solution u_m written for the pole sum).
template <int MODE>
__global__ void __launch_bounds__(32 * FDM_WARPS, 2) k_leaf_fdm(FdmArgs a) {
    extern __shared__ double2 fsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int q = a.q, p = a.p, q2 = q * q, nb = 4 * q;
    // V, V^-1 once per CTA (padded stride), then per-warp tiles
    double* vf = reinterpret_cast<double*>(fsm);
    double* vif = vf + FDM_T * FDM_LDV;
    for (int e = threadIdx.x; e < FDM_T * FDM_T; e += blockDim.x) {
        const int r = e / FDM_T, c = e % FDM_T;
        vf[r * FDM_LDV + c] = a.V[e];
        vif[r * FDM_LDV + c] = a.Vinv[e];
    }
    __syncthreads();
    double2* P = fsm + FDM_T * FDM_LDV + (size_t)warp * FDM_TILE_ELEMS;   // V, V^-1: 2 x 16 x FDM_LDV doubles
    double2* Q = P + FDM_T * FDM_LDT;
    double2* UB = Q + FDM_T * FDM_LDT;
    double cr[2][2][2], ci[2][2][2];
    const long long prob = (long long)blockIdx.x * FDM_WARPS + warp;

    const long long nprob = (long long)a.nh * a.nelem * a.R2;
    if (prob >= nprob) return;
    const int r2 = (int)(prob % a.R2);
    const int leaf = (int)((prob / a.R2) % a.nelem);
    const int m = (int)(prob / ((long long)a.R2 * a.nelem));
    if (MODE == 0) {
        // UP needs only the boundary flux h = N_I A^-1 f.  With A^-1 f = V W V^T:
        //   bottom/top  (d = D[0|p-1][1..q], row sums over j):  h = -/+ c1 V (W e),
        //   left/right  (column sums over i):                    h = -/+ c1 V (W^T e),
        // e = V^T d precomputed - four 16-vectors instead of stages 3-4.
        fdm_solve<false, true>(a, m, leaf, r2, lane, P, Q, UB, vf, vif, cr, ci);
        // y_s[r] = sum_c W[r][c] e_s[c]  (lanes 0-15),  z_s[r] = sum_c W[c][r] e_s[c]  (lanes 16-31);
        // P holds W^T: P[tix(j', i')] = W[i'][j']
        {
            const int r = lane & 15;
            const bool colsum = lane >= 16;
            double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
#pragma unroll 4
            for (int c = 0; c < FDM_T; ++c) {
                const double2 wv = colsum ? P[tix(r, c)] : P[tix(c, r)];   // W[c][r] : W[r][c]
                const double e0 = __ldg(a.E01 + c), e1 = __ldg(a.E01 + FDM_T + c);
                acc0.x = fma(wv.x, e0, acc0.x); acc0.y = fma(wv.y, e0, acc0.y);
                acc1.x = fma(wv.x, e1, acc1.x); acc1.y = fma(wv.y, e1, acc1.y);
            }
            // UB[0..15] = y0, [16..31] = y1, [32..47] = z0, [48..63] = z1
            UB[(colsum ? 32 : 0) + r] = acc0;
            UB[(colsum ? 48 : 16) + r] = acc1;
        }
        __syncwarp();
        for (int b = lane; b < nb; b += 32) {
            const int side = b / q, s1 = b % q;
            // bottom: -V y0, right: +V z1, top: +V y1, left: -V z0  (index s1 = i or j)
            const int src = side == 0 ? 0 : side == 1 ? 48 : side == 2 ? 16 : 32;
            const double sgn = (side == 0 || side == 3) ? -a.c1 : a.c1;
            double sx = 0.0, sy = 0.0;
#pragma unroll 4
            for (int k = 0; k < FDM_T; ++k) {
                const double v = vf[s1 * FDM_LDV + k];
                const double2 y = UB[src + k];
                sx = fma(v, y.x, sx);
                sy = fma(v, y.y, sy);
            }
            a.h[((size_t)m * a.hps + (size_t)leaf * nb + b) * a.R2 + r2] = make_double2(sgn * sx, sgn * sy);
        }
        return;
    }
    fdm_solve<true>(a, m, leaf, r2, lane, P, Q, UB, vf, vif, cr, ci);
    {
        double2* wl = a.w + (((size_t)m * a.nelem + leaf) * q2) * a.R2 + r2;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int j = mt * 8 + g, i = nt * 8 + 2 * t4 + c;
                    if (i < q && j < q) wl[(size_t)(j * q + i) * a.R2] = make_double2(cr[mt][nt][c], ci[mt][nt][c]);
                }
    }
}

}  // namespace dev
}  // namespace rexp

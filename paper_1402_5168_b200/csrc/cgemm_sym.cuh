// Symmetric-pair DMMA GEMM for the merge levels of the spectral shared store.
//
// A level whose reflection along the interface maps each child onto itself
// acts on the edge data as a signed involution without fixed points (pairs
// A <-> B with sign s, device.cu: DeviceStore::sym_pairs).  Every operator of
// the level commutes with it, so the store keeps only the half pair
// M+- = A_AA +- A_AB S ([M+ | M-], each hr x hk column-major) and the product
// over all nodes' columns is two half-size GEMMs:
//     B+- [k][col] = x_{A_k}(col) +- s_k x_{B_k}(col)
//     P = M+ B+,  D = M- B-,   y_{A_r} = (P + D)/2,  y_{B_r} = s_r (P - D)/2.
// Same tiling and DMMA scheme as k_cgemm (cgemm.cuh); A tiles of both halves by
// cp.async, B formed from the mode's gathers through registers, double-buffered.
#pragma once

#include "cgemm.cuh"

namespace rexp {
namespace dev {

struct CgemmSymArgs {
    CgemmArgs g;              // A = [M+ | M-] per pole, rows = hr, K = hk, the mode's gathers
    const int *iA, *iB;       // input pairs (k)
    const double* is;
    const int *oA, *oB;       // output pairs (rows)
    const double* os;
    int n3, next;             // full interface / boundary sizes of the level
    // second reflection (device.cu: sym_pairs2): partners of the boundary pairs and their signs;
    // UP-Y writes them too, DOWN adds them to the gathered operand (-1: the pair has no partner)
    int sym2;
    const int *xA2, *xB2;
    const double *xsA2, *xsB2;
};

struct BRawSym { double v[8]; };

// x at full input position pos for column col: UPX s3 = h^a_3 + h^b_3 (two gathers),
// UPY w3, DOWN u_ext
template <int R2T, int MODE>
__device__ __forceinline__ void cgs_fetch1(const CgemmSymArgs& s, int m, int pos, int node, int r2, double* out,
                                           int pos2 = -1, double sg2 = 0.0) {
    const CgemmArgs& a = s.g;
    const int R2 = R2T ? R2T : a.R2;
    if (MODE == CG_UPX) {
        const double2* src = a.src + (size_t)m * a.src_ps * R2;
        const int base = cg_child_base(a, node);
        const double2 v0 = src[(size_t)(base + a.bi0[pos]) * R2 + r2];
        const double2 v1 = src[(size_t)(base + a.bi1[pos]) * R2 + r2];
        out[0] = v0.x; out[1] = v0.y; out[2] = v1.x; out[3] = v1.y;
    } else if (MODE == CG_UPY) {
        const double2 v = a.src[(size_t)m * a.src_ps * R2 + ((size_t)node * s.n3 + pos) * R2 + r2];
        out[0] = v.x; out[1] = v.y; out[2] = 0.0; out[3] = 0.0;
    } else {   // DOWN (+ the reflection-2 partner, summed like UP-X's second child)
        const double2 v = a.src[((size_t)m * a.src_ps + a.bi0[(size_t)node * s.next + pos]) * R2 + r2];
        out[0] = v.x; out[1] = v.y; out[2] = 0.0; out[3] = 0.0;
        if (pos2 >= 0) {
            const double2 w = a.src[((size_t)m * a.src_ps + a.bi0[(size_t)node * s.next + pos2]) * R2 + r2];
            out[2] = sg2 * w.x; out[3] = sg2 * w.y;
        }
    }
}

// additive epilogue terms of the thread's outputs (UP-Y: child h[ext], DOWN: w3),
// fetched before the K loop so their latency overlaps the operand loads (PF)
template <int R2T, int MODE, int MT>
__device__ __forceinline__ void cgs_prefetch_add(const CgemmSymArgs& s, int m, int row0, int col0, int mrow0,
                                                 int warp, int g, int t4, double2 (&pre)[MT][2][2]) {
    const CgemmArgs& a = s.g;
    const int R2 = R2T ? R2T : a.R2;
    const int hr = a.rows, ncols = a.nodes * R2;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pre[i][j][0] = pre[i][j][1] = make_double2(0.0, 0.0);
            const int rr = row0 + mrow0 + i * 8 + g;
            const int col = col0 + warp * 8 + 2 * t4 + j;
            if (rr >= hr || col >= ncols) continue;
            const int node = col / R2, r2 = col % R2;
            const int ra = s.oA[rr], rbw = s.oB[rr];
            if (MODE == CG_UPY) {
                const int base = cg_child_base(a, node);
                pre[i][j][0] = a.add[((size_t)m * a.add_ps + base + a.ai0[ra]) * R2 + r2];
                pre[i][j][1] = a.add[((size_t)m * a.add_ps + base + a.ai0[rbw]) * R2 + r2];
            } else if (MODE == CG_DOWN) {
                const double2* w3 = a.add + (size_t)m * a.add_ps * R2;
                pre[i][j][0] = w3[((size_t)node * s.n3 + ra) * R2 + r2];
                pre[i][j][1] = w3[((size_t)node * s.n3 + rbw) * R2 + r2];
            }
        }
}

// epilogue: half row rr -> rows oA[rr] (y_A) and oB[rr] (y_B); PF: the additive
// terms were prefetched into pre
template <int R2T, int MODE, int MT, bool PF = false>
__device__ __forceinline__ void cgs_epilogue(const CgemmSymArgs& s, int m, int row0, int col0, int mrow0, int warp,
                                             int g, int t4, const double (&acc)[2][MT][4],
                                             const double2 (*pre)[2][2] = nullptr) {
    const CgemmArgs& a = s.g;
    const int R2 = R2T ? R2T : a.R2;
    const int hr = a.rows, ncols = a.nodes * R2;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int rr = row0 + mrow0 + i * 8 + g;
        if (rr >= hr) continue;
        const int ra = s.oA[rr], rbw = s.oB[rr];
        const double so = 0.5 * s.os[rr];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int col = col0 + warp * 8 + 2 * t4 + j;
            if (col >= ncols) continue;
            const int node = col / R2, r2 = col % R2;
            const double pr = acc[0][i][j], pi = acc[0][i][2 + j], dr = acc[1][i][j], di = acc[1][i][2 + j];
            double2 yA = make_double2(0.5 * (pr + dr), 0.5 * (pi + di));
            double2 yB = make_double2(so * (pr - dr), so * (pi - di));
            if (MODE == CG_UPX) {
                double2* dst = a.dst + (size_t)m * a.dst_ps * R2;
                dst[((size_t)node * s.n3 + ra) * R2 + r2] = yA;
                dst[((size_t)node * s.n3 + rbw) * R2 + r2] = yB;
            } else if (MODE == CG_UPY) {
                const int base = cg_child_base(a, node);
                const double2 ea = PF ? pre[i][j][0] : a.add[((size_t)m * a.add_ps + base + a.ai0[ra]) * R2 + r2];
                const double2 eb = PF ? pre[i][j][1] : a.add[((size_t)m * a.add_ps + base + a.ai0[rbw]) * R2 + r2];
                double2* dst = a.dst + (size_t)m * a.dst_ps * R2;
                dst[((size_t)node * s.next + ra) * R2 + r2] = make_double2(yA.x + ea.x, yA.y + ea.y);
                dst[((size_t)node * s.next + rbw) * R2 + r2] = make_double2(yB.x + eb.x, yB.y + eb.y);
                if (s.sym2) {   // the reflection-2 partners carry the same values up to the edge-basis sign
                    const int pa = s.xA2[rr], pb = s.xB2[rr];
                    if (pa >= 0) {
                        const double ga = s.xsA2[rr], gb = s.xsB2[rr];
                        const double2 fa = a.add[((size_t)m * a.add_ps + base + a.ai0[pa]) * R2 + r2];
                        const double2 fb = a.add[((size_t)m * a.add_ps + base + a.ai0[pb]) * R2 + r2];
                        dst[((size_t)node * s.next + pa) * R2 + r2] = make_double2(fma(ga, yA.x, fa.x), fma(ga, yA.y, fa.y));
                        dst[((size_t)node * s.next + pb) * R2 + r2] = make_double2(fma(gb, yB.x, fb.x), fma(gb, yB.y, fb.y));
                    }
                }
            } else {   // DOWN: u3 = y + w3, scattered to the edge array
                const double2* w3 = a.add + (size_t)m * a.add_ps * R2;
                const double2 wa = PF ? pre[i][j][0] : w3[((size_t)node * s.n3 + ra) * R2 + r2];
                const double2 wb = PF ? pre[i][j][1] : w3[((size_t)node * s.n3 + rbw) * R2 + r2];
                a.dst[((size_t)m * a.dst_ps + a.so0[(size_t)node * s.n3 + ra]) * R2 + r2] =
                    make_double2(yA.x + wa.x, yA.y + wa.y);
                a.dst[((size_t)m * a.dst_ps + a.so0[(size_t)node * s.n3 + rbw]) * R2 + r2] =
                    make_double2(yB.x + wb.x, yB.y + wb.y);
            }
        }
    }
}

// NST: 2 = B+- formed through registers (double-buffered); 3 = cp.async ring of
// 3 stages; 12 / 11 = cp.async ring of 2 / 1 stage(s) (smaller footprint: more
// CTAs per SM for the short-K, latency-bound low levels)
template <int NST>
__host__ __device__ constexpr int cgs_ring() { return NST >= 10 ? NST - 10 : NST; }
template <int MT, int WN, int BK, int WM = 1, int NST = 2, int MODE = CG_UPY>
__host__ __device__ constexpr size_t cgemm_sym_smem_bytes() {
    // the UP-X ring stages both children's raw gathers of x_A and x_B (4 tiles per stage)
    constexpr int XT = (MODE == CG_UPX && NST >= 10) ? 2 : 1;
    return (size_t)cgs_ring<NST>() * 2 * BK * ((8 * MT * WM + 2) + XT * (8 * WN + 2)) * sizeof(double2);
}

// gathered source address of x at full input position pos (UP-Y, DOWN: one 16-byte value)
template <int R2T, int MODE>
__device__ __forceinline__ const double2* cgs_src(const CgemmSymArgs& s, int m, int pos, int node, int r2) {
    const CgemmArgs& a = s.g;
    const int R2 = R2T ? R2T : a.R2;
    if (MODE == CG_UPY) return a.src + (size_t)m * a.src_ps * R2 + ((size_t)node * s.n3 + pos) * R2 + r2;
    return a.src + ((size_t)m * a.src_ps + a.bi0[(size_t)node * s.next + pos]) * R2 + r2;   // DOWN
}

// NST = 2: B+- formed through registers.  NST = 3 (UP-Y / DOWN): both halves of A
// and the raw x_A, x_B tiles by cp.async into a 3-stage ring; B+- formed in the
// compute loop (b+- = x_A +- s x_B).
template <int MT, int WN, int BK, int R2T, int MODE, int WM = 1, int NST = 2, bool PF = false>
__global__ void __launch_bounds__(32 * WN * WM) k_cgemm_sym(CgemmSymArgs s) {
    const CgemmArgs& a = s.g;
    constexpr int BM = 8 * MT * WM, BN = 8 * WN, NT = 32 * WN * WM;
    const int R2 = R2T ? R2T : a.R2;
    constexpr int LDA = BM + 2, LDB = BN + 2;
    constexpr int BPT = (BK * BN + NT - 1) / NT;
    extern __shared__ double2 sm[];

    const int m = blockIdx.y;
    const int rb = blockIdx.x % a.nrowblk;
    const int cb = blockIdx.x / a.nrowblk;
    const int row0 = rb * BM, col0 = cb * BN;
    const int ncols = a.nodes * R2;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int warp = wid % WN, wm = wid / WN;
    const int g = lane >> 2, t4 = lane & 3;
    const int mrow0 = wm * MT * 8;
    const int hr = a.rows, hk = a.K;
    const double2* Ap = a.A + (size_t)m * 2 * hr * hk;   // M+
    const double2* Am = Ap + (size_t)hr * hk;            // M-

    constexpr bool kRingX = MODE == CG_UPX && NST >= 10;   // UP-X: h^a_3 and h^b_3 copied raw, summed in the loop
    if constexpr (NST >= 3 && (MODE == CG_UPY || MODE == CG_DOWN || kRingX)) {
        // ring of RS stages: [stage][half] A tiles, then [stage][A|B] raw x tiles
        constexpr int RS = cgs_ring<NST>();
        auto AsN = [&](int st, int hf) { return sm + (st * 2 + hf) * BK * LDA; };
        auto XsN = [&](int st, int ab) { return sm + RS * 2 * BK * LDA + (st * 2 + ab) * BK * LDB; };
        auto XsN2 = [&](int st, int ab) { return sm + RS * 2 * BK * (LDA + LDB) + (st * 2 + ab) * BK * LDB; };
        auto issue = [&](int st, int k0) {
            for (int e = tid; e < 2 * BK * BM; e += NT) {
                const int hf = e / (BK * BM), ee = e % (BK * BM);
                const int kk = ee / BM, r = ee % BM;
                const int row = row0 + r, k = k0 + kk;
                double2* base = AsN(st, hf);
                const double2* M = hf ? Am : Ap;
                if (row < hr && k < hk) cp_async16(base + kk * LDA + r, M + (size_t)k * hr + row);
                else base[kk * LDA + r] = make_double2(0.0, 0.0);
            }
            for (int e = tid; e < 2 * BK * BN; e += NT) {
                const int ab = e / (BK * BN), ee = e % (BK * BN);
                const int kk = ee / BN, c = ee % BN;
                const int k = k0 + kk, col = col0 + c;
                double2* base = XsN(st, ab);
                if constexpr (kRingX) {
                    double2* base2 = XsN2(st, ab);
                    if (k < hk && col < ncols) {
                        const int pos = ab ? s.iB[k] : s.iA[k], node = col / R2, r2 = col % R2;
                        const double2* srcm = a.src + (size_t)m * a.src_ps * R2;
                        const int cbase = cg_child_base(a, node);
                        cp_async16(base + kk * LDB + c, srcm + (size_t)(cbase + a.bi0[pos]) * R2 + r2);
                        cp_async16(base2 + kk * LDB + c, srcm + (size_t)(cbase + a.bi1[pos]) * R2 + r2);
                    } else {
                        base[kk * LDB + c] = make_double2(0.0, 0.0);
                        base2[kk * LDB + c] = make_double2(0.0, 0.0);
                    }
                } else {
                    if (k < hk && col < ncols)
                        cp_async16(base + kk * LDB + c,
                                   cgs_src<R2T, MODE>(s, m, ab ? s.iB[k] : s.iA[k], col / R2, col % R2));
                    else base[kk * LDB + c] = make_double2(0.0, 0.0);
                    if (MODE == CG_DOWN && s.sym2) {   // reflection-2 partner of the gathered value
                        double2* base2 = XsN2(st, ab);
                        const int pos2 = (k < hk && col < ncols) ? (ab ? s.xB2[k] : s.xA2[k]) : -1;
                        if (pos2 >= 0) cp_async16(base2 + kk * LDB + c, cgs_src<R2T, MODE>(s, m, pos2, col / R2, col % R2));
                        else base2[kk * LDB + c] = make_double2(0.0, 0.0);
                    }
                }
            }
            cp_async_commit();
        };
        double acc3[2][MT][4], q3[2][MT][2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                acc3[hf][i][0] = acc3[hf][i][1] = acc3[hf][i][2] = acc3[hf][i][3] = 0.0;
                q3[hf][i][0] = q3[hf][i][1] = 0.0;
            }
        const int nch = (hk + BK - 1) / BK;
#pragma unroll
        for (int st = 0; st < RS - 1; ++st) {
            if (st < nch) issue(st, st * BK);
            else cp_async_commit();
        }
        double2 pre3[PF ? MT : 1][2][2];
        if constexpr (PF) cgs_prefetch_add<R2T, MODE, MT>(s, m, row0, col0, mrow0, warp, g, t4, pre3);
        for (int ch = 0; ch < nch; ++ch) {
            if constexpr (RS == 1) {
                if (ch > 0) __syncthreads();    // everyone is done with the single stage
                issue(0, ch * BK);
                cp_async_wait_all();
                __syncthreads();
            } else {
                cp_async_wait_group<(RS >= 2 ? RS - 2 : 0)>();
                __syncthreads();
                const int nx = ch + RS - 1;
                if (nx < nch) issue(nx % RS, nx * BK);
                else cp_async_commit();
            }
            const int st = RS == 1 ? 0 : ch % RS;
            const double2* XA = XsN(st, 0);
            const double2* XB = XsN(st, 1);
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                const int kk = ks * 4 + t4;
                const int k = ch * BK + kk;
                const double sg = k < hk ? __ldg(s.is + k) : 0.0;
                double2 xa = XA[kk * LDB + warp * 8 + g], xb = XB[kk * LDB + warp * 8 + g];
                if constexpr (kRingX) {
                    const double2 xa2 = XsN2(st, 0)[kk * LDB + warp * 8 + g], xb2 = XsN2(st, 1)[kk * LDB + warp * 8 + g];
                    xa.x += xa2.x; xa.y += xa2.y;
                    xb.x += xb2.x; xb.y += xb2.y;
                }
                if (MODE == CG_DOWN && s.sym2) {
                    const double2 xa2 = XsN2(st, 0)[kk * LDB + warp * 8 + g], xb2 = XsN2(st, 1)[kk * LDB + warp * 8 + g];
                    const double ga = k < hk ? __ldg(s.xsA2 + k) : 0.0, gb = k < hk ? __ldg(s.xsB2 + k) : 0.0;
                    xa.x = fma(ga, xa2.x, xa.x); xa.y = fma(ga, xa2.y, xa.y);
                    xb.x = fma(gb, xb2.x, xb.x); xb.y = fma(gb, xb2.y, xb.y);
                }
                const double2 bp = make_double2(xa.x + sg * xb.x, xa.y + sg * xb.y);
                const double2 bm = make_double2(xa.x - sg * xb.x, xa.y - sg * xb.y);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const double2* Ab = AsN(st, hf);
                    const double2 b = hf ? bm : bp;
                    double2 av[MT];
#pragma unroll
                    for (int i = 0; i < MT; ++i) av[i] = Ab[kk * LDA + mrow0 + i * 8 + g];
#if REXP_CMUL3
                    const double bs = b.x + b.y;
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][0], acc3[hf][i][1], av[i].x, b.x);
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][2], acc3[hf][i][3], av[i].x + av[i].y, bs);
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(q3[hf][i][0], q3[hf][i][1], av[i].y, b.y);
#else
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][0], acc3[hf][i][1], av[i].x, b.x);
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][2], acc3[hf][i][3], av[i].x, b.y);
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][0], acc3[hf][i][1], av[i].y, -b.y);
#pragma unroll
                    for (int i = 0; i < MT; ++i) dmma884(acc3[hf][i][2], acc3[hf][i][3], av[i].y, b.x);
#endif
                }
            }
        }
#if REXP_CMUL3
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int i = 0; i < MT; ++i) cmul3_finish(acc3[hf][i], q3[hf][i]);
#endif
        cgs_epilogue<R2T, MODE, MT, PF>(s, m, row0, col0, mrow0, warp, g, t4, acc3, pre3);
        return;
    }
    // buffers: [buf][half] A tiles, then [buf][half] B tiles
    auto As = [&](int buf, int hf) { return sm + (buf * 2 + hf) * BK * LDA; };
    auto Bs = [&](int buf, int hf) { return sm + 4 * BK * LDA + (buf * 2 + hf) * BK * LDB; };

    auto issue_A = [&](int buf, int k0) {
        for (int e = tid; e < 2 * BK * BM; e += NT) {
            const int hf = e / (BK * BM), ee = e % (BK * BM);
            const int kk = ee / BM, r = ee % BM;
            const int row = row0 + r, k = k0 + kk;
            double2* base = As(buf, hf);
            const double2* M = hf ? Am : Ap;
            if (row < hr && k < hk) cp_async16(base + kk * LDA + r, M + (size_t)k * hr + row);
            else base[kk * LDA + r] = make_double2(0.0, 0.0);
        }
        cp_async_commit();
    };
    BRawSym braw[BPT];
    auto fetch_B = [&](int k0) {
#pragma unroll
        for (int u = 0; u < BPT; ++u) {
            const int e = tid + u * NT;
            const int kk = e / BN, c = e % BN;
            const int k = k0 + kk, col = col0 + c;
#pragma unroll
            for (int j = 0; j < 8; ++j) braw[u].v[j] = 0.0;
            if (e < BK * BN && k < hk && col < ncols) {
                const int node = col / R2, r2 = col % R2;
                if (MODE == CG_DOWN && s.sym2) {
                    cgs_fetch1<R2T, MODE>(s, m, s.iA[k], node, r2, braw[u].v, s.xA2[k], s.xsA2[k]);
                    cgs_fetch1<R2T, MODE>(s, m, s.iB[k], node, r2, braw[u].v + 4, s.xB2[k], s.xsB2[k]);
                } else {
                    cgs_fetch1<R2T, MODE>(s, m, s.iA[k], node, r2, braw[u].v);
                    cgs_fetch1<R2T, MODE>(s, m, s.iB[k], node, r2, braw[u].v + 4);
                }
            }
        }
    };
    auto store_B = [&](int buf, int k0) {
#pragma unroll
        for (int u = 0; u < BPT; ++u) {
            const int e = tid + u * NT;
            if (e < BK * BN) {
                const int kk = e / BN, c = e % BN;
                const int k = k0 + kk;
                const double sg = k < hk ? s.is[k] : 0.0;
                const double* v = braw[u].v;
                const double xar = v[0] + v[2], xai = v[1] + v[3];   // UPX: two-child sum (others: v[2], v[3] = 0)
                const double xbr = v[4] + v[6], xbi = v[5] + v[7];
                Bs(buf, 0)[kk * LDB + c] = make_double2(xar + sg * xbr, xai + sg * xbi);
                Bs(buf, 1)[kk * LDB + c] = make_double2(xar - sg * xbr, xai - sg * xbi);
            }
        }
    };

    double acc[2][MT][4], q2[2][MT][2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            acc[hf][i][0] = acc[hf][i][1] = acc[hf][i][2] = acc[hf][i][3] = 0.0;
            q2[hf][i][0] = q2[hf][i][1] = 0.0;
        }

    const int nchunks = (hk + BK - 1) / BK;
    issue_A(0, 0);
    fetch_B(0);
    double2 pre2[PF ? MT : 1][2][2];
    if constexpr (PF) cgs_prefetch_add<R2T, MODE, MT>(s, m, row0, col0, mrow0, warp, g, t4, pre2);
    store_B(0, 0);
    cp_async_wait_all();
    __syncthreads();
    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        const bool more = ch + 1 < nchunks;
        if (more) {
            issue_A(buf ^ 1, (ch + 1) * BK);
            fetch_B((ch + 1) * BK);
        }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const double2* Ab = As(buf, hf);
            const double2* Bb = Bs(buf, hf);
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                const int kk = ks * 4 + t4;
                const double2 b = Bb[kk * LDB + warp * 8 + g];
                double2 av[MT];
#pragma unroll
                for (int i = 0; i < MT; ++i) av[i] = Ab[kk * LDA + mrow0 + i * 8 + g];
#if REXP_CMUL3
                const double bs = b.x + b.y;
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][0], acc[hf][i][1], av[i].x, b.x);
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][2], acc[hf][i][3], av[i].x + av[i].y, bs);
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(q2[hf][i][0], q2[hf][i][1], av[i].y, b.y);
#else
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][0], acc[hf][i][1], av[i].x, b.x);
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][2], acc[hf][i][3], av[i].x, b.y);
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][0], acc[hf][i][1], av[i].y, -b.y);
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[hf][i][2], acc[hf][i][3], av[i].y, b.x);
#endif
            }
        }
        if (more) {
            store_B(buf ^ 1, (ch + 1) * BK);
            cp_async_wait_all();
        }
        __syncthreads();
    }
#if REXP_CMUL3
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int i = 0; i < MT; ++i) cmul3_finish(acc[hf][i], q2[hf][i]);
#endif
    cgs_epilogue<R2T, MODE, MT, PF>(s, m, row0, col0, mrow0, warp, g, t4, acc, pre2);
}

}  // namespace dev
}  // namespace rexp

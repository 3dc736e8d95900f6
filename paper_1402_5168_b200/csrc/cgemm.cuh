// Batched complex128 GEMM on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64)
// for the SHARED operator store: per half pole m (grid.y) one operator A_m
// (rows x K, column-major complex) multiplies the gathered right-hand sides of
// every node of a tree level at once,
//     C[rows x (nodes*R2)] = A_m[rows x K] * B[K x (nodes*R2)],
// so the leaf solves and the low merge levels become dense GEMMs.
// Complex product as four real DMMAs per k-step:
//     Cr += Ar Br + Ai (-Bi),   Ci += Ar Bi + Ai Br.
// CTA = WN warps; warp w owns n-tile w (8 columns) and MT m-tiles (8 rows each):
// BM = 8 MT, BN = 8 WN.  K is staged through shared memory in BK = 16 chunks
// (A via cp.async 16-byte copies, B through a mode-specific gather/formation),
// double-buffered.  Row strides padded by 2 complex so the 8 threads of a
// quarter-warp hit 8 distinct 16-byte slots (conflict-free LDS.128).
#pragma once

namespace rexp {
namespace dev {

enum CgemmMode { CG_LEAF_UP = 0, CG_LEAF_DOWN = 1, CG_UPX = 2, CG_UPY = 3, CG_DOWN = 4, CG_ROOT = 5 };

struct CgemmArgs {
    const double2* A;       // [nh][rows*K] column-major (shared store)
    int rows, K, nodes;
    int R2;                 // real right-hand sides per node (used when the template R2 is 0)
    int nrowblk;
    // LEAF_UP
    const double* F;        // [R2][nF][NI]
    const double2* cF;      // [nh][nF]
    int nF, q2;
    // generic gathers
    const double2* src;     // pole-strided source of B (edge, h, w3)
    long long src_ps;       // per-pole stride in R2-vectors
    const int* bi0;         // [nodes][K] gather indices (or leaf_gB)
    const int* bi1;         // second gather (UPX)
    // epilogue
    double2* dst;           // pole-strided destination
    long long dst_ps;
    const double2* add;     // additive term source (UPY: child h via ai0, DOWN: w3 contiguous)
    long long add_ps;
    const int* ai0;         // UPY: [nodes][rows] ext index into add
    const int* so0;         // DOWN: [nodes][rows] scatter index
    // UPX / UPY gathers are affine in the node (mesh.cpp): index(node, k) =
    // ca(node) * nchild + index(0, k), ca(node) = 2 node (x-merge) or
    // node + (node / nbx) nbx (y-merge); only node 0's rows (bi0, bi1, ai0) are read
    int nbx, xdir, nchild;
};

__device__ __forceinline__ int cg_child_base(const CgemmArgs& a, int node) {
    return (a.xdir ? 2 * node : node + (node / a.nbx) * a.nbx) * a.nchild;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Complex products on the real DMMA: REXP_CMUL3 = 1 (default) uses the
// three-multiply form per 8x8 tile,
//   P1 += Ar Br (acc[0..1]),  P3 += (Ar + Ai)(Br + Bi) (acc[2..3]),  P2 += Ai Bi (q[0..1]),
// finished after the K loop as Cr = P1 - P2, Ci = P3 - P1 - P2 (cmul3_finish):
// 3 DMMAs per complex k-step instead of 4 (the merge GEMMs are DMMA-issue bound,
// profiles/r01_merge_ncu_details.txt: math_pipe_throttle).  0 = four real products.
#ifndef REXP_CMUL3
#define REXP_CMUL3 1
#endif
__device__ __forceinline__ void cmul3_finish(double* acc, const double* q) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const double p1 = acc[j], p2 = q[j], p3 = acc[2 + j];
        acc[j] = p1 - p2;
        acc[2 + j] = p3 - p1 - p2;
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// B gather in two phases so the global loads of chunk c+1 are in flight while
// chunk c is multiplied: cg_fetch issues the loads into registers, cg_form
// turns them into the B element (after the math).
struct BRaw { double v[4]; };

template <int R2T, int MODE>
__device__ __forceinline__ void cg_fetch(const CgemmArgs& a, int m, int k, int col, BRaw& r) {
    const int R2 = R2T ? R2T : a.R2;
    const int node = col / R2, r2 = col % R2;
    if (MODE == CG_LEAF_UP) {
        const size_t NI = (size_t)a.nodes * a.q2;
        const double* f = a.F + (size_t)r2 * a.nF * NI + (size_t)node * a.q2 + k;
        r.v[0] = f[0];
        r.v[1] = a.nF > 1 ? f[NI] : 0.0;
        r.v[2] = a.nF > 2 ? f[2 * NI] : 0.0;
    } else if (MODE == CG_UPX || MODE == CG_ROOT) {
        // ROOT: one node, node-independent seam positions pos1/pos2 (P^T h)
        const double2* s = a.src + (size_t)m * a.src_ps * R2;
        const int base = MODE == CG_ROOT ? 0 : cg_child_base(a, node);
        const double2 v0 = s[(size_t)(base + a.bi0[k]) * R2 + r2];
        const double2 v1 = s[(size_t)(base + a.bi1[k]) * R2 + r2];
        r.v[0] = v0.x; r.v[1] = v0.y; r.v[2] = v1.x; r.v[3] = v1.y;
    } else if (MODE == CG_UPY) {
        const double2 v = a.src[(size_t)m * a.src_ps * R2 + ((size_t)node * a.K + k) * R2 + r2];
        r.v[0] = v.x; r.v[1] = v.y;
    } else {  // LEAF_DOWN, DOWN: gather from the pole's edge array
        const double2 v = a.src[((size_t)m * a.src_ps + a.bi0[(size_t)node * a.K + k]) * R2 + r2];
        r.v[0] = v.x; r.v[1] = v.y;
    }
}

// modes whose B element is one gathered 16-byte value (copyable by cp.async)
template <int MODE>
__host__ __device__ constexpr bool cg_plain_b() { return MODE == CG_UPY || MODE == CG_DOWN || MODE == CG_LEAF_DOWN; }

template <int R2T, int MODE>
__device__ __forceinline__ const double2* cg_src_ptr(const CgemmArgs& a, int m, int k, int col) {
    const int R2 = R2T ? R2T : a.R2;
    const int node = col / R2, r2 = col % R2;
    if (MODE == CG_UPY) return a.src + (size_t)m * a.src_ps * R2 + ((size_t)node * a.K + k) * R2 + r2;
    return a.src + ((size_t)m * a.src_ps + a.bi0[(size_t)node * a.K + k]) * R2 + r2;   // DOWN, LEAF_DOWN
}

template <int MODE>
__device__ __forceinline__ double2 cg_form(const BRaw& r, const double2* cf) {
    if (MODE == CG_LEAF_UP) {
        double2 v;
        v.x = fma(cf[0].x, r.v[0], fma(cf[1].x, r.v[1], cf[2].x * r.v[2]));
        v.y = fma(cf[0].y, r.v[0], fma(cf[1].y, r.v[1], cf[2].y * r.v[2]));
        return v;
    } else if (MODE == CG_UPX || MODE == CG_ROOT) {
        return make_double2(r.v[0] + r.v[2], r.v[1] + r.v[3]);
    } else {
        return make_double2(r.v[0], r.v[1]);
    }
}

template <int R2T, int MODE>
__device__ __forceinline__ void cg_store(const CgemmArgs& a, int m, int row, int col, double2 v) {
    const int R2 = R2T ? R2T : a.R2;
    const int node = col / R2, r2 = col % R2;
    if (MODE == CG_LEAF_UP) {
        a.dst[(((size_t)m * a.nodes + node) * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_LEAF_DOWN) {   // additive w folded in by the caller
        a.dst[(((size_t)m * a.nodes + node) * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_UPX) {
        a.dst[(size_t)m * a.dst_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_UPY) {   // additive child h[ext] folded in by the caller
        a.dst[(size_t)m * a.dst_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_ROOT) {   // seam values into the pole's edge array
        a.dst[((size_t)m * a.dst_ps + a.so0[row]) * R2 + r2] = v;
    } else {  // DOWN (additive w3 folded in by the caller)
        a.dst[((size_t)m * a.dst_ps + a.so0[(size_t)node * a.rows + row]) * R2 + r2] = v;
    }
}

// NST: 2 = B through registers (double-buffered), 3 = cp.async ring of 3 stages,
// 11 = cp.async, one stage (short-K levels: small footprint, more CTAs per SM)
template <int NST>
__host__ __device__ constexpr int cg_ring() { return NST >= 10 ? NST - 10 : NST; }
template <int MT, int WN, int BK, int NTW = 1, int WM = 1, int NST = 2>
__host__ __device__ constexpr size_t cgemm_smem_bytes() {
    return (size_t)(cg_ring<NST>() < 2 ? 2 : cg_ring<NST>()) * BK * ((8 * MT * WM + 2) + (8 * WN * NTW + 2)) *
           sizeof(double2);
}
// UP-Y (compile-time R2): the additive child term of the tile is staged too
template <int MT, int WN, int BK, int NTW = 1, int WM = 1, int NST = 2, int MODE = 0>
__host__ __device__ constexpr size_t cgemm_smem_total() {
    return cgemm_smem_bytes<MT, WN, BK, NTW, WM, NST>() +
           (MODE == CG_UPY ? (size_t)(8 * MT * WM) * (8 * WN * NTW) * sizeof(double2) : 0);
}

// MT m-tiles and NTW n-tiles per warp; WN warps side by side in n, WM in m.
// NST = 2: A by cp.async and B through registers, one chunk ahead.  NST >= 3
// (plain-gather B modes): A and B both by cp.async into an NST-stage ring,
// NST - 1 chunks in flight, one barrier per chunk.
template <int MT, int WN, int BK, int R2T, int MODE, int NTW = 1, int MINB = 1, int WM = 1, int NST = 2>
__global__ void __launch_bounds__(32 * WN * WM, MINB) k_cgemm(CgemmArgs a) {
    constexpr int BM = 8 * MT * WM, BN = 8 * WN * NTW, NT = 32 * WN * WM;
    const int R2 = R2T ? R2T : a.R2;
    static_assert(BK % 4 == 0, "BK must be a multiple of the DMMA k (4)");
    constexpr int LDA = BM + 2, LDB = BN + 2;
    constexpr int BPT = (BK * BN + NT - 1) / NT;     // B elements per thread per chunk
    extern __shared__ double2 sm[];

    const int m = blockIdx.y;
    const int rb = blockIdx.x % a.nrowblk;
    const int cb = blockIdx.x / a.nrowblk;
    const int row0 = rb * BM, col0 = cb * BN;
    const int ncols = a.nodes * R2;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int warp = wid % WN, wm = wid / WN;          // n position, m position of this warp
    const int g = lane >> 2, t4 = lane & 3;
    const int mrow0 = wm * MT * 8;                     // first row of this warp inside the CTA tile
    const double2* Am = a.A + (size_t)m * a.rows * a.K;
    double2 cf[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
    if (MODE == CG_LEAF_UP) {
        const double2* c = a.cF + (size_t)m * a.nF;
        cf[0] = c[0];
        if (a.nF > 1) cf[1] = c[1];
        if (a.nF > 2) cf[2] = c[2];
    }

    auto As = [&](int buf) { return sm + buf * BK * LDA; };
    auto Bs = [&](int buf) { return sm + 2 * BK * LDA + buf * BK * LDB; };

    auto issue_A = [&](int buf, int k0) {
        double2* base = As(buf);
        for (int e = tid; e < BK * BM; e += NT) {
            const int kk = e / BM, r = e % BM;
            const int row = row0 + r, k = k0 + kk;
            if (row < a.rows && k < a.K) cp_async16(base + kk * LDA + r, Am + (size_t)k * a.rows + row);
            else base[kk * LDA + r] = make_double2(0.0, 0.0);
        }
        cp_async_commit();
    };
    BRaw braw[BPT];
    // B element of thread slot e: (kk, c).  With compile-time R2 the merge modes map
    // consecutive e to (real part, k, node) so consecutive threads read consecutive
    // addresses of the node-major gathered vectors
    constexpr bool kBmap = R2T != 0 && MODE != CG_LEAF_UP && MODE != CG_LEAF_DOWN && (BN % (R2T ? R2T : 1)) == 0;
    auto bslot = [&](int e, int& kk, int& c) {
        if (kBmap) {
            constexpr int R = R2T ? R2T : 1;
            const int r2 = e % R, t2 = e / R;
            kk = t2 % BK;
            c = (t2 / BK) * R + r2;
        } else {
            kk = e / BN;
            c = e % BN;
        }
    };
    auto fetch_B = [&](int k0) {
#pragma unroll
        for (int u = 0; u < BPT; ++u) {
            const int e = tid + u * NT;
            int kk, c;
            bslot(e, kk, c);
            const int k = k0 + kk, col = col0 + c;
            braw[u].v[0] = braw[u].v[1] = braw[u].v[2] = braw[u].v[3] = 0.0;
            if (e < BK * BN && k < a.K && col < ncols) cg_fetch<R2T, MODE>(a, m, k, col, braw[u]);
        }
    };
    auto store_B = [&](int buf) {
        double2* base = Bs(buf);
#pragma unroll
        for (int u = 0; u < BPT; ++u) {
            const int e = tid + u * NT;
            if (e < BK * BN) {
                int kk, c;
                bslot(e, kk, c);
                base[kk * LDB + c] = cg_form<MODE>(braw[u], cf);
            }
        }
    };

    double acc[MT][NTW][4];
    double accq[MT][NTW][2];   // REXP_CMUL3: P2 = sum Ai Bi
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NTW; ++n) {
            acc[i][n][0] = acc[i][n][1] = acc[i][n][2] = acc[i][n][3] = 0.0;
            accq[i][n][0] = accq[i][n][1] = 0.0;
        }

    // additive epilogue terms (LEAF_DOWN: w, DOWN: w3, UPY: child h[ext]) fetched
    // before the K loop so their latency overlaps the products
    // UP-Y with compile-time R2 uses the staged, coalesced epilogue below instead
    constexpr bool kStagedUPY = (MODE == CG_UPY && R2T != 0 && (BN % (R2T ? R2T : 1) == 0 || (R2T ? R2T : 1) % BN == 0));
    constexpr bool kAdd = (MODE == CG_LEAF_DOWN || MODE == CG_DOWN || (MODE == CG_UPY && !kStagedUPY));
    double2 addv[kAdd ? MT : 1][kAdd ? NTW : 1][2];
    if (kAdd) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int row = row0 + mrow0 + i * 8 + g;
                    const int col = col0 + (warp * NTW + n) * 8 + 2 * t4 + j;
                    addv[i][n][j] = make_double2(0.0, 0.0);
                    if (row < a.rows && col < ncols) {
                        const int node = col / R2, r2 = col % R2;
                        if (MODE == CG_LEAF_DOWN)
                            addv[i][n][j] = a.dst[(((size_t)m * a.nodes + node) * a.rows + row) * R2 + r2];
                        else if (MODE == CG_UPY)
                            addv[i][n][j] = a.add[((size_t)m * a.add_ps + cg_child_base(a, node) + a.ai0[row]) * R2 + r2];
                        else
                            addv[i][n][j] = a.add[(size_t)m * a.add_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2];
                    }
                }
    }

    // UP-Y staged epilogue: the tile's additive child term h[ext] -> shared memory by
    // cp.async now (it lands with the first operand chunk), [run][row][RUN] order: a run
    // is one node's R2 columns (R2 <= BN) or the tile's BN columns of one node (R2 > BN)
    double2* Adds = sm + cgemm_smem_bytes<MT, WN, BK, NTW, WM, NST>() / sizeof(double2);
    constexpr int RUN = R2T == 0 ? 1 : R2T < BN ? R2T : BN;
    if constexpr (kStagedUPY) {
        constexpr int R = R2T ? R2T : 1;
        for (int e = tid; e < (BN / RUN) * BM * RUN; e += NT) {
            const int j = e % RUN, rl = (e / RUN) % BM, nl = e / (RUN * BM);
            const int row = row0 + rl, col = col0 + nl * RUN + j;
            if (row < a.rows && col < ncols)
                cp_async16(Adds + e,
                           a.add + ((size_t)m * a.add_ps + cg_child_base(a, col / R) + a.ai0[row]) * R + col % R);
        }
        cp_async_commit();
    }
    const int nchunks = (a.K + BK - 1) / BK;
    auto compute = [&](const double2* Ab, const double2* Bb) {
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            const int kk = ks * 4 + t4;
            double2 b[NTW];
#pragma unroll
            for (int n = 0; n < NTW; ++n) b[n] = Bb[kk * LDB + (warp * NTW + n) * 8 + g];   // B[k = t4][n = g]
            double2 av[MT];
#pragma unroll
            for (int i = 0; i < MT; ++i) av[i] = Ab[kk * LDA + mrow0 + i * 8 + g];   // A[m = g][k = t4]
#if REXP_CMUL3
            double bs[NTW], as[MT];
#pragma unroll
            for (int n = 0; n < NTW; ++n) bs[n] = b[n].x + b[n].y;
#pragma unroll
            for (int i = 0; i < MT; ++i) as[i] = av[i].x + av[i].y;
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][0], acc[i][n][1], av[i].x, b[n].x);   // P1
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][2], acc[i][n][3], as[i], bs[n]);       // P3
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(accq[i][n][0], accq[i][n][1], av[i].y, b[n].y);  // P2
#else
            // four passes so each accumulator is revisited only every 2*MT*NTW DMMAs
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][0], acc[i][n][1], av[i].x, b[n].x);    // Cr += Ar Br
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][2], acc[i][n][3], av[i].x, b[n].y);    // Ci += Ar Bi
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][0], acc[i][n][1], av[i].y, -b[n].y);   // Cr += Ai (-Bi)
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma884(acc[i][n][2], acc[i][n][3], av[i].y, b[n].x);    // Ci += Ai Br
#endif
        }
    };
    if constexpr (NST >= 3 && cg_plain_b<MODE>()) {
        constexpr int RS = cg_ring<NST>();
        auto AsN = [&](int buf) { return sm + buf * BK * LDA; };
        auto BsN = [&](int buf) { return sm + (RS < 2 ? 2 : RS) * BK * LDA + buf * BK * LDB; };
        auto issue = [&](int buf, int k0) {
            double2* ab = AsN(buf);
            for (int e = tid; e < BK * BM; e += NT) {
                const int kk = e / BM, r = e % BM;
                const int row = row0 + r, k = k0 + kk;
                if (row < a.rows && k < a.K) cp_async16(ab + kk * LDA + r, Am + (size_t)k * a.rows + row);
                else ab[kk * LDA + r] = make_double2(0.0, 0.0);
            }
            double2* bb = BsN(buf);
            for (int e = tid; e < BK * BN; e += NT) {
                const int kk = e / BN, cc = e % BN;
                const int k = k0 + kk, col = col0 + cc;
                if (k < a.K && col < ncols) cp_async16(bb + kk * LDB + cc, cg_src_ptr<R2T, MODE>(a, m, k, col));
                else bb[kk * LDB + cc] = make_double2(0.0, 0.0);
            }
            cp_async_commit();
        };
#pragma unroll
        for (int st = 0; st < RS - 1; ++st) {
            if (st < nchunks) issue(st, st * BK);
            else cp_async_commit();
        }
        for (int ch = 0; ch < nchunks; ++ch) {
            if constexpr (RS == 1) {
                if (ch > 0) __syncthreads();  // everyone is done with the single stage
                issue(0, ch * BK);
                cp_async_wait_all();
                __syncthreads();
                compute(AsN(0), BsN(0));
            } else {
                cp_async_wait_group<(RS >= 2 ? RS - 2 : 0)>();   // chunk ch has landed (this thread's copies)
                __syncthreads();                  // everyone's copies; the buffer refilled below is free
                const int nx = ch + RS - 1;
                if (nx < nchunks) issue(nx % RS, nx * BK);
                else cp_async_commit();
                compute(AsN(ch % RS), BsN(ch % RS));
            }
        }
    } else {
        issue_A(0, 0);
        fetch_B(0);
        store_B(0);
        cp_async_wait_all();
        __syncthreads();
        for (int ch = 0; ch < nchunks; ++ch) {
            const int buf = ch & 1;
            const bool more = ch + 1 < nchunks;
            if (more) {
                issue_A(buf ^ 1, (ch + 1) * BK);
                fetch_B((ch + 1) * BK);
            }
            compute(As(buf), Bs(buf));
            if (more) {
                store_B(buf ^ 1);
                cp_async_wait_all();
            }
            __syncthreads();
        }
    }
#if REXP_CMUL3
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NTW; ++n) cmul3_finish(acc[i][n], accq[i][n]);
#endif
    if constexpr (kStagedUPY) {
        // staged epilogue: C tile -> shared memory [local col][row], then each node's
        // rows x R2 run (contiguous in h) written and its child term h[ext] read
        // with consecutive threads on consecutive addresses
        constexpr int LDC = BM + 1;
        static_assert((size_t)BN * LDC * sizeof(double2) <= cgemm_smem_bytes<MT, WN, BK, NTW, WM, NST>(),
                      "the C tile must fit in the A/B buffers (Adds follows them)");
        double2* Cs = sm;   // BN x LDC, reuses the A/B buffers
        cp_async_wait_all();
        __syncthreads();    // every warp is done reading them (the 3-stage loop ends without a barrier)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int n = 0; n < NTW; ++n)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    Cs[((warp * NTW + n) * 8 + 2 * t4 + j) * LDC + mrow0 + i * 8 + g] =
                        make_double2(acc[i][n][j], acc[i][n][2 + j]);
        __syncthreads();
        constexpr int NPT = BN / RUN;                  // runs per tile
        double2* dst = a.dst + (size_t)m * a.dst_ps * R2T;
        for (int e = tid; e < NPT * BM * RUN; e += NT) {
            const int j = e % RUN, rl = (e / RUN) % BM, nl = e / (RUN * BM);
            const int row = row0 + rl, col = col0 + nl * RUN + j;
            if (row >= a.rows || col >= ncols) continue;
            const int node = col / R2T, r2 = col % R2T;
            const double2 ad = Adds[e];
            const double2 v = Cs[(nl * RUN + j) * LDC + rl];
            dst[((size_t)node * a.rows + row) * R2T + r2] = make_double2(v.x + ad.x, v.y + ad.y);
        }
        return;
    }
    // epilogue: C[g][2 t4 + j] of each tile
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = row0 + mrow0 + i * 8 + g;
        if (row >= a.rows) continue;
#pragma unroll
        for (int n = 0; n < NTW; ++n)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int col = col0 + (warp * NTW + n) * 8 + 2 * t4 + j;
                if (col >= ncols) continue;
                double2 v = make_double2(acc[i][n][j], acc[i][n][2 + j]);
                if (kAdd) {
                    v.x += addv[i][n][j].x;
                    v.y += addv[i][n][j].y;
                }
                cg_store<R2T, MODE>(a, m, row, col, v);
            }
    }
}

}  // namespace dev
}  // namespace rexp

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

enum CgemmMode { CG_LEAF_UP = 0, CG_LEAF_DOWN = 1, CG_UPX = 2, CG_UPY = 3, CG_DOWN = 4 };

struct CgemmArgs {
    const double2* A;       // [nh][rows*K] column-major (shared store)
    int rows, K, nodes;
    int nrowblk;
    // LEAF_UP
    const double* F;        // [NI][nF][R2]
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
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int R2, int MODE>
__device__ __forceinline__ double2 cg_load_b(const CgemmArgs& a, int m, int k, int col) {
    const int node = col / R2, r2 = col % R2;
    if (MODE == CG_LEAF_UP) {
        const double* f = a.F + ((size_t)(node * a.q2 + k) * a.nF) * R2 + r2;
        const double2* c = a.cF + (size_t)m * a.nF;
        double2 v = make_double2(0.0, 0.0);
        for (int t = 0; t < a.nF; ++t) {
            const double x = f[(size_t)t * R2];
            const double2 ct = c[t];
            v.x = fma(ct.x, x, v.x);
            v.y = fma(ct.y, x, v.y);
        }
        return v;
    } else if (MODE == CG_UPX) {
        const double2* s = a.src + (size_t)m * a.src_ps * R2;
        const double2 v0 = s[(size_t)a.bi0[(size_t)node * a.K + k] * R2 + r2];
        const double2 v1 = s[(size_t)a.bi1[(size_t)node * a.K + k] * R2 + r2];
        return make_double2(v0.x + v1.x, v0.y + v1.y);
    } else if (MODE == CG_UPY) {
        return a.src[(size_t)m * a.src_ps * R2 + ((size_t)node * a.K + k) * R2 + r2];
    } else {  // LEAF_DOWN, DOWN: gather from the pole's edge array
        return a.src[((size_t)m * a.src_ps + a.bi0[(size_t)node * a.K + k]) * R2 + r2];
    }
}

template <int R2, int MODE>
__device__ __forceinline__ void cg_store(const CgemmArgs& a, int m, int row, int col, double2 v) {
    const int node = col / R2, r2 = col % R2;
    if (MODE == CG_LEAF_UP) {
        a.dst[(((size_t)m * a.nodes + node) * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_LEAF_DOWN) {
        double2* p = a.dst + (((size_t)m * a.nodes + node) * a.rows + row) * R2 + r2;
        const double2 w = *p;
        *p = make_double2(w.x + v.x, w.y + v.y);
    } else if (MODE == CG_UPX) {
        a.dst[(size_t)m * a.dst_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2] = v;
    } else if (MODE == CG_UPY) {
        const double2 ad = a.add[((size_t)m * a.add_ps + a.ai0[(size_t)node * a.rows + row]) * R2 + r2];
        a.dst[(size_t)m * a.dst_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2] =
            make_double2(ad.x + v.x, ad.y + v.y);
    } else {  // DOWN
        const double2 ad = a.add[(size_t)m * a.add_ps * R2 + ((size_t)node * a.rows + row) * R2 + r2];
        a.dst[((size_t)m * a.dst_ps + a.so0[(size_t)node * a.rows + row]) * R2 + r2] =
            make_double2(ad.x + v.x, ad.y + v.y);
    }
}

constexpr int CG_BK = 16;

template <int MT, int WN>
constexpr size_t cgemm_smem_bytes() {
    return 2 * (size_t)CG_BK * ((8 * MT + 2) + (8 * WN + 2)) * sizeof(double2);
}

template <int MT, int WN, int R2, int MODE>
__global__ void __launch_bounds__(32 * WN) k_cgemm(CgemmArgs a) {
    constexpr int BM = 8 * MT, BN = 8 * WN, BK = CG_BK;
    constexpr int LDA = BM + 2, LDB = BN + 2;
    extern __shared__ double2 sm[];
    double2* As[2] = {sm, sm + BK * LDA};
    double2* Bs[2] = {sm + 2 * BK * LDA, sm + 2 * BK * LDA + BK * LDB};

    const int m = blockIdx.y;
    const int rb = blockIdx.x % a.nrowblk;
    const int cb = blockIdx.x / a.nrowblk;
    const int row0 = rb * BM, col0 = cb * BN;
    const int ncols = a.nodes * R2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const double2* Am = a.A + (size_t)m * a.rows * a.K;

    auto load_chunk = [&](int buf, int k0) {
        // A: BK columns x BM rows (column-major in global, contiguous rows)
        for (int e = tid; e < BK * BM; e += 32 * WN) {
            const int kk = e / BM, r = e % BM;
            double2* dst = As[buf] + kk * LDA + r;
            const int row = row0 + r, k = k0 + kk;
            if (row < a.rows && k < a.K) cp_async16(dst, Am + (size_t)k * a.rows + row);
            else *dst = make_double2(0.0, 0.0);
        }
        // B: BK x BN, formed / gathered per mode
        for (int e = tid; e < BK * BN; e += 32 * WN) {
            const int kk = e / BN, c = e % BN;
            const int k = k0 + kk, col = col0 + c;
            double2 v = make_double2(0.0, 0.0);
            if (k < a.K && col < ncols) v = cg_load_b<R2, MODE>(a, m, k, col);
            Bs[buf][kk * LDB + c] = v;
        }
        cp_async_commit();
    };

    double acc[MT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;

    const int nchunks = (a.K + BK - 1) / BK;
    load_chunk(0, 0);
    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        cp_async_wait_all();
        __syncthreads();
        if (ch + 1 < nchunks) load_chunk(buf ^ 1, (ch + 1) * BK);
        const double2* Ab = As[buf];
        const double2* Bb = Bs[buf];
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            const int kk = ks * 4 + t4;
            const double2 b = Bb[kk * LDB + warp * 8 + g];   // B[k = t4][n = g]
            const double nbi = -b.y;
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const double2 av = Ab[kk * LDA + i * 8 + g];  // A[m = g][k = t4]
                dmma884(acc[i][0], acc[i][1], av.x, b.x);    // Cr += Ar Br
                dmma884(acc[i][0], acc[i][1], av.y, nbi);    // Cr += Ai (-Bi)
                dmma884(acc[i][2], acc[i][3], av.x, b.y);    // Ci += Ar Bi
                dmma884(acc[i][2], acc[i][3], av.y, b.x);    // Ci += Ai Br
            }
        }
    }
    // epilogue: C[g][2 t4 + j] of each tile
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = row0 + i * 8 + g;
        if (row >= a.rows) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int col = col0 + warp * 8 + 2 * t4 + j;
            if (col < ncols) cg_store<R2, MODE>(a, m, row, col, make_double2(acc[i][j], acc[i][2 + j]));
        }
    }
}

}  // namespace dev
}  // namespace rexp

// Fused multi-level merge sweeps for the shared operator store (see fused_tree.hpp).
//
// One CTA = one half pole x CS sibling subtrees x RC real right-hand-side columns
// (CS * RC = 8 = one DMMA n-tile per node), carried through nlev merge levels
// (§2.3: the upward pass w3 = -X (h^a_3 + h^b_3), h = h_child[ext] + Y w3
// and the downward pass u3 = S u_ext + w3) with every level's boundary data in
// shared memory.  Warp roles: CW consumer warps run the FP64 DMMAs
// (mma.sync.m8n8k4.f64, three-multiply complex product as in cgemm.cuh); one
// producer warp streams the operators of all the group's stages, in order,
// through a ring of shared-memory slots with 1-D bulk copies (cp.async.bulk,
// one per operator column, padded leading dimension) completing on mbarriers,
// so the next stage's operator is in flight while the current one is multiplied.
#include "fused_tree.hpp"

#include <algorithm>
#include <cstdio>

#include "cgemm.cuh"

namespace rexp {
namespace dev {

namespace {

constexpr int FT_CW = 12;                   // consumer warps
constexpr int FT_NT = 32 * (FT_CW + 1);     // + the producer warp
constexpr int FT_IT = 2;                    // (m-tile, n-tile) items per consumer warp
constexpr int FT_HDR = 1024;                // mbarriers (128 B) + node id table
#ifndef FT_MINB
#define FT_MINB 2                           // resident CTAs per SM the register budget allows
#endif

__host__ __device__ inline int ceil4(int v) { return (v + 3) & ~3; }

// ---- mbarrier / bulk-copy primitives (sm_90+) --------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned ok = 0;
    for (unsigned spin = 0; !ok; ++spin) {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (spin > (1u << 22)) __trap();   // a lost arrival must fail loudly, not hang the GPU
    }
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * FT_CW) : "memory"); }

// ---- one operator stage ------------------------------------------------------
struct Ring {
    int slot = 0;
    unsigned phase = 0;
    __device__ __forceinline__ void advance(int nslots) {
        if (++slot == nslots) { slot = 0; phase ^= 1u; }
    }
};

// producer side of one stage: one bulk copy per K chunk (the packed image already
// has the padded shared-memory layout) into the next ring slot
__device__ __forceinline__ void ft_produce(const FtStageDesc& st, const double2* img, Ring& rg, const FtArgs& a,
                                           unsigned ring, unsigned full, unsigned empty, int lane) {
    const unsigned bytes = static_cast<unsigned>(st.nh * st.bk * st.lda) * 16u;
    const double2* src = img + st.img_off;
    for (int c = 0; c < st.nchunks; ++c) {
        mbar_wait(empty + 8 * rg.slot, rg.phase ^ 1u);
        if (lane == 0) {
            mbar_expect_tx(full + 8 * rg.slot, bytes);
            bulk_g2s(ring + rg.slot * a.slot_bytes, src + static_cast<size_t>(c) * (bytes / 16), bytes,
                     full + 8 * rg.slot);
        }
        __syncwarp();
        rg.advance(a.nslots);
    }
}

// consumer side: C = M B over the stage's K chunks; items (m-tile, n-tile[, k
// slice]) are dealt to the warps round-robin.  KS > 1 (DOWN: few rows, long K)
// splits the k-steps of every chunk over KS warps per tile; the partial sums are
// combined through `scratch` in a fixed order.  epi(row, col, P[4], D[4]) gets
// the tile's values {re(col), re(col+1), im(col), im(col+1)} of both halves.
template <class Epi>
__device__ __forceinline__ void ft_gemm(const FtStageDesc& st, const double2* Bp, const double2* Bm, int ldb,
                                        int ncols, int KS, double* scratch, Ring& rg, const FtArgs& a,
                                        const char* ringp, unsigned full, unsigned empty, int warp, int lane,
                                        Epi epi) {
    const int g = lane >> 2, t4 = lane & 3;
    const int ntl = ncols >> 3, ntiles = ((st.hr + 7) >> 3) * ntl, nitems = ntiles * KS;
    const int ksteps = st.bk >> 2;
    double acc[FT_IT][2][6];
#pragma unroll
    for (int u = 0; u < FT_IT; ++u)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int e = 0; e < 6; ++e) acc[u][hf][e] = 0.0;
    for (int c = 0; c < st.nchunks; ++c) {
        const int k0 = c * st.bk;
        mbar_wait(full + 8 * rg.slot, rg.phase);
        const double2* As = reinterpret_cast<const double2*>(ringp + static_cast<size_t>(rg.slot) * a.slot_bytes);
#pragma unroll
        for (int u = 0; u < FT_IT; ++u) {
            const int it = warp + FT_CW * u;
            if (it < nitems) {
                const int tile = it % ntiles, sl = it / ntiles;
                const int mi = tile / ntl, ni = tile - mi * ntl;
                const double2* Ab = As + mi * 8 + g;
                const double2* Bb0 = Bp + k0 * ldb + ni * 8 + g;
                const double2* Bb1 = Bm + k0 * ldb + ni * 8 + g;
                for (int ks = sl; ks < ksteps; ks += KS) {
                    const int kk = ks * 4 + t4;
                    {
                        const double2 av = Ab[kk * st.lda];
                        const double2 bv = Bb0[kk * ldb];
                        dmma884(acc[u][0][0], acc[u][0][1], av.x, bv.x);
                        dmma884(acc[u][0][2], acc[u][0][3], av.x + av.y, bv.x + bv.y);
                        dmma884(acc[u][0][4], acc[u][0][5], av.y, bv.y);
                    }
                    if (st.nh == 2) {
                        const double2 av = Ab[(st.bk + kk) * st.lda];
                        const double2 bv = Bb1[kk * ldb];
                        dmma884(acc[u][1][0], acc[u][1][1], av.x, bv.x);
                        dmma884(acc[u][1][2], acc[u][1][3], av.x + av.y, bv.x + bv.y);
                        dmma884(acc[u][1][4], acc[u][1][5], av.y, bv.y);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * rg.slot);
        rg.advance(a.nslots);
    }
    // three-multiply form -> {re, re, im, im}
#pragma unroll
    for (int u = 0; u < FT_IT; ++u)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double p1 = acc[u][hf][j], p3 = acc[u][hf][2 + j], p2 = acc[u][hf][4 + j];
                acc[u][hf][j] = p1 - p2;
                acc[u][hf][2 + j] = p3 - p1 - p2;
            }
    if (KS > 1) {
        // partial sums of slices >= 1 -> scratch [slice - 1][tile][hf][e][lane]
        consumer_sync();   // every warp is done reading B (scratch aliases it)
#pragma unroll
        for (int u = 0; u < FT_IT; ++u) {
            const int it = warp + FT_CW * u;
            if (it < nitems && it >= ntiles) {
                const int tile = it % ntiles, sl = it / ntiles;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        scratch[((((sl - 1) * ntiles + tile) * 2 + hf) * 4 + e) * 32 + lane] = acc[u][hf][e];
            }
        }
        consumer_sync();
#pragma unroll
        for (int u = 0; u < FT_IT; ++u) {
            const int it = warp + FT_CW * u;
            if (it < ntiles) {
                for (int sl = 1; sl < KS; ++sl)
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            acc[u][hf][e] += scratch[((((sl - 1) * ntiles + it) * 2 + hf) * 4 + e) * 32 + lane];
            }
        }
    }
#pragma unroll
    for (int u = 0; u < FT_IT; ++u) {
        const int it = warp + FT_CW * u;
        if (it < ntiles) {
            const int mi = it / ntl, ni = it - mi * ntl;
            const int row = mi * 8 + g;
            if (row < st.hr) epi(row, ni * 8 + 2 * t4, acc[u][0], acc[u][1]);
        }
    }
}

// global node ids of the group's levels, top-down: ids[(l + 1) * stride + i], l = -1 .. nlev - 1
__device__ __forceinline__ void ft_node_ids(const FtArgs& a, int* ids, int stride, int top0, int tid) {
    if (tid == 0) {
        for (int s = 0; s < a.CS; ++s) ids[a.nlev * stride + s] = top0 + s;
        int cnt = a.CS;
        for (int l = a.nlev - 1; l >= 0; --l) {
            const FtLevel& L = a.lv[l];
            for (int i = 0; i < cnt; ++i) {
                const int node = ids[(l + 1) * stride + i];
                const int ca = L.xdir ? 2 * node : node + (node / L.nbx) * L.nbx;
                ids[l * stride + 2 * i] = ca;
                ids[l * stride + 2 * i + 1] = ca + (L.xdir ? 1 : L.nbx);
            }
            cnt *= 2;
        }
    }
}

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

// common prologue: barriers, node ids, the group's index tables -> shared memory
__device__ __forceinline__ void ft_prologue(const FtArgs& a, char* smem, int* ids, int stride, int top0, int tid) {
    const unsigned full = smem_u32(smem), empty = full + 64;
    if (tid == 0) {
        for (int s = 0; s < a.nslots; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, FT_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    ft_node_ids(a, ids, stride, top0, tid);
    int* it = reinterpret_cast<int*>(smem + a.off_tab);
    for (int e = tid; e < a.n_itab; e += FT_NT) it[e] = a.itab[e];
    double* dt = reinterpret_cast<double*>(it + ((a.n_itab + 1) & ~1));
    for (int e = tid; e < a.n_dtab; e += FT_NT) dt[e] = a.dtab[e];
    __syncthreads();
}

// ------------------------------------------------------------------------------
// UP: levels lv[0 .. nlev-1]; reads the child h of lv[0], writes every level's w3
// and the top level's h.  Per level: B_X = gathered h^a_3 + h^b_3 (pair form),
// GEMM X whose accumulators P, D are directly the pair-form operand of GEMM Y
// (B+ = y_A + s y_B = P, B- = D), GEMM Y + the children's exterior rows.
// ------------------------------------------------------------------------------
__global__ void __launch_bounds__(FT_NT, FT_MINB) k_ft_up(const __grid_constant__ FtArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = blockIdx.y;
    const int cb = blockIdx.x % a.ncb, top0 = (blockIdx.x / a.ncb) * a.CS;
    const int c0 = cb * a.RC, RC = a.RC, R2 = a.R2, lgRC = a.lgRC;
    const unsigned full = smem_u32(smem), empty = full + 64, ring = smem_u32(smem + a.off_ring);
    int* ids = reinterpret_cast<int*>(smem + 128);
    const int stride = a.CS << a.nlev;
    ft_prologue(a, smem, ids, stride, top0, tid);

    if (warp == FT_CW) {
        Ring rg;
        const double2* img = a.img + m * a.img_ps;
        for (int l = 0; l < a.nlev; ++l) {
            const FtLevel& L = a.lv[l];
            if (!L.xdiag) ft_produce(L.st[0], img, rg, a, ring, full, empty, lane);
            ft_produce(L.st[1], img, rg, a, ring, full, empty, lane);
        }
        return;
    }

    // ---- consumers ----
    const int* itab = reinterpret_cast<const int*>(smem + a.off_tab);
    const double* dtab = reinterpret_cast<const double*>(itab + ((a.n_itab + 1) & ~1));
    double2* cur = reinterpret_cast<double2*>(smem + a.off_a);
    double2* nxt = reinterpret_cast<double2*>(smem + a.off_b);
    double2* Bxp = reinterpret_cast<double2*>(smem + a.off_bx);
    double2* Bxm = reinterpret_cast<double2*>(smem + a.off_bx + a.bhalf);
    double2* Byp = reinterpret_cast<double2*>(smem + a.off_by);
    double2* Bym = reinterpret_cast<double2*>(smem + a.off_by + a.bhalf);
    const char* ringp = smem + a.off_ring;
    constexpr int CT = 32 * FT_CW;
    {
        const int nin = a.CS << a.nlev, nc = a.lv[0].nchild;
        const double2* hm = a.hin + static_cast<size_t>(m) * a.hps * R2 + c0;
        for (int i = 0; i < nin; ++i) {
            const double2* src = hm + static_cast<size_t>(ids[i]) * nc * R2;
            double2* dst = cur + i * nc * RC;
            for (int e = tid; e < nc * RC; e += CT) cp_async16(dst + e, src + static_cast<size_t>(e >> lgRC) * R2 + (e & (RC - 1)));
        }
        cp_async_commit();
        cp_async_wait_all();
    }
    consumer_sync();
    Ring rg;
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * RC, ldb = ncols + 2, lgc = ilog2(ncols);
        const int n3 = L.n3, next = L.next, nc = L.nchild;
        const int* lid = ids + (l + 1) * stride;
        const bool top = l == a.nlev - 1;
        const double2* curc = cur;
        const int4* xg = reinterpret_cast<const int4*>(itab + L.t_xg);
        const double* xs = dtab + L.d_xs;
        double2* wg = L.w3 + static_cast<size_t>(m) * L.nodes * n3 * R2 + c0;
        const int Ky = L.st[1].hk, KPy = L.st[1].bk * L.st[1].nchunks;
        if (L.xdiag) {
            // w3 = -X (h^a_3 + h^b_3) with a diagonal X (the store holds -X): directly GEMM Y's operand
            const double2* Xm = L.X + m * L.ppX;
            for (int e = tid; e < KPy * ncols; e += CT) {
                const int k = e >> lgc, col = e & (ncols - 1);
                double2 w = make_double2(0.0, 0.0);
                if (k < n3) {
                    const int i = col >> lgRC, j = col & (RC - 1);
                    const int4 o = xg[k];
                    const double2 u = curc[((2 * i) * nc + o.x) * RC + j], v = curc[((2 * i) * nc + o.y) * RC + j];
                    const double2 x = __ldg(Xm + static_cast<size_t>(k) * (n3 + 1));
                    const double sx = u.x + v.x, sy = u.y + v.y;
                    w = make_double2(x.x * sx - x.y * sy, x.x * sy + x.y * sx);
                    wg[(static_cast<size_t>(lid[i]) * n3 + k) * R2 + j] = w;
                }
                Byp[k * ldb + col] = w;
            }
        } else {
            const FtStageDesc& st = L.st[0];
            const int KPx = st.bk * st.nchunks;
            for (int e = tid; e < KPx * ncols; e += CT) {
                const int k = e >> lgc, col = e & (ncols - 1);
                double2 vp = make_double2(0.0, 0.0), vm = vp;
                if (k < st.hk) {
                    const int i = col >> lgRC, j = col & (RC - 1);
                    const int4 o = xg[k];
                    const double2* cb2 = curc + (2 * i) * nc * RC + j;
                    const double2 a0 = cb2[o.x * RC], a1 = cb2[o.y * RC];
                    vp = make_double2(a0.x + a1.x, a0.y + a1.y);
                    if (L.sym) {
                        const double2 b0 = cb2[o.z * RC], b1 = cb2[o.w * RC];
                        const double s = xs[k];
                        const double xbr = s * (b0.x + b1.x), xbi = s * (b0.y + b1.y);
                        vm = make_double2(vp.x - xbr, vp.y - xbi);
                        vp = make_double2(vp.x + xbr, vp.y + xbi);
                    }
                }
                Bxp[k * ldb + col] = vp;
                if (L.sym) Bxm[k * ldb + col] = vm;
            }
            // zero the K padding of GEMM Y's operand (rows written by no epilogue)
            for (int e = tid; e < (KPy - Ky) * ncols; e += CT) {
                const int k = Ky + (e >> lgc), col = e & (ncols - 1);
                Byp[k * ldb + col] = make_double2(0.0, 0.0);
                if (L.sym) Bym[k * ldb + col] = make_double2(0.0, 0.0);
            }
            consumer_sync();
            const int2* xrow = reinterpret_cast<const int2*>(itab + L.t_xrow);
            const double* xso = dtab + L.d_xso;
            ft_gemm(st, Bxp, Bxm, ldb, ncols, 1, nullptr, rg, a, ringp, full, empty, warp, lane,
                    [&](int row, int col, const double* P, const double* D) {
                        const int i = col >> lgRC, j = col & (RC - 1);
                        double2* wn = wg + static_cast<size_t>(lid[i]) * n3 * R2 + j;
                        if (L.sym) {
                            const int2 r = xrow[row];
                            const double so = xso[row];
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj) {
                                Byp[row * ldb + col + jj] = make_double2(P[jj], P[2 + jj]);
                                Bym[row * ldb + col + jj] = make_double2(D[jj], D[2 + jj]);
                                wn[static_cast<size_t>(r.x) * R2 + jj] =
                                    make_double2(0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                                wn[static_cast<size_t>(r.y) * R2 + jj] =
                                    make_double2(so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                            }
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj) {
                                const double2 v = make_double2(P[jj], P[2 + jj]);
                                Byp[row * ldb + col + jj] = v;
                                wn[static_cast<size_t>(row) * R2 + jj] = v;
                            }
                        }
                    });
        }
        consumer_sync();
        // ---- h = h_child[ext] + Y w3 ----
        {
            const int4* yrow = reinterpret_cast<const int4*>(itab + L.t_yrow);
            const double* yso = dtab + L.d_yso;
            double2* hg = a.hout + static_cast<size_t>(m) * a.hps * R2 + c0;
            double2* nx = nxt;
            ft_gemm(L.st[1], Byp, Bym, ldb, ncols, 1, nullptr, rg, a, ringp, full, empty, warp, lane,
                    [&](int row, int col, const double* P, const double* D) {
                        const int i = col >> lgRC, j = col & (RC - 1);
                        const int4 r = yrow[row];
                        const double2* cc = curc + (2 * i) * nc * RC + j;
                        double2* og = hg + static_cast<size_t>(lid[i]) * next * R2 + j;
                        double2* os = nx + i * next * RC + j;
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            double2 vA, vB;
                            if (L.sym) {
                                const double so = yso[row];
                                vA = make_double2(0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                                vB = make_double2(so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                                const double2 cB = cc[r.w * RC + jj];
                                vB.x += cB.x; vB.y += cB.y;
                            } else {
                                vA = make_double2(P[jj], P[2 + jj]);
                            }
                            const double2 cA = cc[r.z * RC + jj];
                            vA.x += cA.x; vA.y += cA.y;
                            if (top) {
                                og[static_cast<size_t>(r.x) * R2 + jj] = vA;
                                if (L.sym) og[static_cast<size_t>(r.y) * R2 + jj] = vB;
                            } else {
                                os[r.x * RC + jj] = vA;
                                if (L.sym) os[r.y * RC + jj] = vB;
                            }
                        }
                    });
        }
        consumer_sync();
        double2* t = cur; cur = nxt; nxt = t;
    }
}

// ------------------------------------------------------------------------------
// DOWN: levels lv[nlev-1 .. 0]; gathers the top boxes' boundary values from the
// edge array, scatters every level's interface values u3 = S u_ext + w3.
// ------------------------------------------------------------------------------
__global__ void __launch_bounds__(FT_NT, FT_MINB) k_ft_down(const __grid_constant__ FtArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = blockIdx.y;
    const int cb = blockIdx.x % a.ncb, top0 = (blockIdx.x / a.ncb) * a.CS;
    const int c0 = cb * a.RC, RC = a.RC, R2 = a.R2, lgRC = a.lgRC;
    const unsigned full = smem_u32(smem), empty = full + 64, ring = smem_u32(smem + a.off_ring);
    int* ids = reinterpret_cast<int*>(smem + 128);
    const int stride = a.CS << a.nlev;
    ft_prologue(a, smem, ids, stride, top0, tid);

    if (warp == FT_CW) {
        Ring rg;
        const double2* img = a.img + m * a.img_ps;
        for (int l = a.nlev - 1; l >= 0; --l) ft_produce(a.lv[l].st[2], img, rg, a, ring, full, empty, lane);
        return;
    }

    const int* itab = reinterpret_cast<const int*>(smem + a.off_tab);
    const double* dtab = reinterpret_cast<const double*>(itab + ((a.n_itab + 1) & ~1));
    double2* cur = reinterpret_cast<double2*>(smem + a.off_a);
    double2* nxt = reinterpret_cast<double2*>(smem + a.off_b);
    double2* W = reinterpret_cast<double2*>(smem + a.off_w);    // every level's w3, top level first
    double2* U3 = reinterpret_cast<double2*>(smem + a.off_u);
    double2* Bp = reinterpret_cast<double2*>(smem + a.off_bx);
    double2* Bm = reinterpret_cast<double2*>(smem + a.off_bx + a.bhalf);
    const char* ringp = smem + a.off_ring;
    constexpr int CT = 32 * FT_CW;
    double2* em = a.edge + static_cast<size_t>(m) * a.NE * R2 + c0;
    {
        // the top boxes' boundary values and all w3 terms of the group
        const FtLevel& T = a.lv[a.nlev - 1];
        const int* tids = ids + a.nlev * stride;
        for (int i = 0; i < a.CS; ++i) {
            const int* ge = T.gext + static_cast<size_t>(tids[i]) * T.next;
            double2* dst = cur + i * T.next * RC;
            for (int e = tid; e < T.next * RC; e += CT)
                cp_async16(dst + e, em + static_cast<size_t>(__ldg(ge + (e >> lgRC))) * R2 + (e & (RC - 1)));
        }
        int woff = 0;
        for (int l = a.nlev - 1; l >= 0; --l) {
            const FtLevel& L = a.lv[l];
            const int nl = a.CS << (a.nlev - 1 - l);
            const int* lid = ids + (l + 1) * stride;
            const double2* wgl = L.w3 + static_cast<size_t>(m) * L.nodes * L.n3 * R2 + c0;
            for (int i = 0; i < nl; ++i) {
                const double2* src = wgl + static_cast<size_t>(lid[i]) * L.n3 * R2;
                double2* dst = W + woff + i * L.n3 * RC;
                for (int e = tid; e < L.n3 * RC; e += CT)
                    cp_async16(dst + e, src + static_cast<size_t>(e >> lgRC) * R2 + (e & (RC - 1)));
            }
            woff += nl * L.n3 * RC;
        }
        cp_async_commit();
        cp_async_wait_all();
    }
    consumer_sync();
    Ring rg;
    int woff = 0;
    for (int l = a.nlev - 1; l >= 0; --l) {
        const FtLevel& L = a.lv[l];
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * RC, ldb = ncols + 2, lgc = ilog2(ncols);
        const int n3 = L.n3, next = L.next, nc = L.nchild;
        const int* lid = ids + (l + 1) * stride;
        const FtStageDesc& st = L.st[2];
        const double2* curc = cur;
        {
            const int2* dg = reinterpret_cast<const int2*>(itab + L.t_dg);
            const double* ds = dtab + L.d_ds;
            const int KP = st.bk * st.nchunks;
            for (int e = tid; e < KP * ncols; e += CT) {
                const int k = e >> lgc, col = e & (ncols - 1);
                double2 vp = make_double2(0.0, 0.0), vm = vp;
                if (k < st.hk) {
                    const int i = col >> lgRC, j = col & (RC - 1);
                    const int2 o = dg[k];
                    const double2* cb2 = curc + i * next * RC + j;
                    vp = cb2[o.x * RC];
                    if (L.sym) {
                        const double2 b = cb2[o.y * RC];
                        const double s = ds[k];
                        vm = make_double2(vp.x - s * b.x, vp.y - s * b.y);
                        vp = make_double2(vp.x + s * b.x, vp.y + s * b.y);
                    }
                }
                Bp[k * ldb + col] = vp;
                if (L.sym) Bm[k * ldb + col] = vm;
            }
        }
        consumer_sync();
        // k slices: as many as the warps allow (few output rows, long K)
        const int ntiles = ((st.hr + 7) >> 3) * (ncols >> 3);
        int KS = (FT_CW * FT_IT) / ntiles;
        KS = KS < 1 ? 1 : KS > 6 ? 6 : KS;
        const double2* Wl = W + woff;
        const int2* drow = reinterpret_cast<const int2*>(itab + L.t_drow);
        const double* dso = dtab + L.d_dso;
        ft_gemm(st, Bp, Bm, ldb, ncols, KS, reinterpret_cast<double*>(Bp), rg, a, ringp, full, empty, warp, lane,
                [&](int row, int col, const double* P, const double* D) {
                    const int i = col >> lgRC, j = col & (RC - 1);
                    const int2 r = drow[row];
                    const int* g3 = L.g3 + static_cast<size_t>(lid[i]) * n3;
                    const double2* wl = Wl + i * n3 * RC + j;
                    double2* us = U3 + i * n3 * RC + j;
                    double2* eA = em + static_cast<size_t>(__ldg(g3 + r.x)) * R2 + j;
                    double2* eB = L.sym ? em + static_cast<size_t>(__ldg(g3 + r.y)) * R2 + j : eA;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        double2 vA;
                        if (L.sym) {
                            const double so = dso[row];
                            vA = make_double2(0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                            double2 vB = make_double2(so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                            const double2 wB = wl[r.y * RC + jj];
                            vB.x += wB.x; vB.y += wB.y;
                            us[r.y * RC + jj] = vB;
                            eB[jj] = vB;
                        } else {
                            vA = make_double2(P[jj], P[2 + jj]);
                        }
                        const double2 wA = wl[r.x * RC + jj];
                        vA.x += wA.x; vA.y += wA.y;
                        us[r.x * RC + jj] = vA;
                        eA[jj] = vA;
                    }
                });
        consumer_sync();
        woff += nl * n3 * RC;
        if (l > 0) {
            // the children's boundary values: parent boundary rows and the new interface values
            const int* dch = itab + L.t_dch;
            const int2* dch3 = reinterpret_cast<const int2*>(dch + next);
            for (int i = 0; i < nl; ++i) {
                double2* cdst = nxt + (2 * i) * nc * RC;
                const double2* usrc = curc + i * next * RC;
                for (int e = tid; e < next * RC; e += CT) cdst[dch[e >> lgRC] * RC + (e & (RC - 1))] = usrc[e];
                const double2* u3 = U3 + i * n3 * RC;
                for (int e = tid; e < n3 * RC; e += CT) {
                    const int2 o = dch3[e >> lgRC];
                    const double2 v = u3[e];
                    cdst[o.x * RC + (e & (RC - 1))] = v;
                    cdst[o.y * RC + (e & (RC - 1))] = v;
                }
            }
            consumer_sync();
            double2* t = cur; cur = nxt; nxt = t;
        }
    }
}

// operator -> chunked, padded image: [chunk][hf][kk < bk][r < lda]
struct PackArgs {
    const double2* M;
    long long pp;          // per-pole stride of M
    double2* img;          // pole 0's image + the stage's offset
    long long img_ps;
    int hr, hk, nh, lda, bk, nchunks;
};
__global__ void k_ft_pack(PackArgs p) {
    const long long tot = static_cast<long long>(p.nchunks) * p.nh * p.bk * p.lda;
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= tot) return;
    const long long m = blockIdx.y;
    const int r = static_cast<int>(e % p.lda);
    const int kk = static_cast<int>((e / p.lda) % p.bk);
    const int hf = static_cast<int>((e / (static_cast<long long>(p.lda) * p.bk)) % p.nh);
    const int c = static_cast<int>(e / (static_cast<long long>(p.lda) * p.bk * p.nh));
    const int k = c * p.bk + kk;
    double2 v = make_double2(0.0, 0.0);
    if (r < p.hr && k < p.hk)
        v = p.M[m * p.pp + static_cast<long long>(hf) * p.hr * p.hk + static_cast<long long>(k) * p.hr + r];
    p.img[m * p.img_ps + e] = v;
}

inline int align_up(int v, int a) { return (v + a - 1) / a * a; }

}  // namespace

bool ft_plan(FtArgs& a, const FtHostLevel* hl, bool down, std::vector<int>& itab, std::vector<double>& dtab) {
    itab.clear();
    dtab.clear();
    if (a.nlev < 1 || a.nlev > FT_MAXLEV) return false;
    if (a.R2 >= 8) {
        if (a.R2 % 8) return false;
        a.RC = 8;
    } else {
        if (a.R2 < 1 || 8 % a.R2) return false;
        a.RC = a.R2;
    }
    a.CS = 8 / a.RC;
    a.lgRC = a.RC == 8 ? 3 : a.RC == 4 ? 2 : a.RC == 2 ? 1 : 0;
    a.ncb = a.R2 / a.RC;
    if (a.lv[a.nlev - 1].nodes % a.CS) return false;
    if ((a.nlev + 1) * (a.CS << a.nlev) * 4 + 128 > FT_HDR) return false;
    a.nslots = 3;
    a.slot_bytes = 12 * 1024;
    // stage descriptors
    long long img = 0;
    size_t bmax = 0;
    for (int l = 0; l < a.nlev; ++l) {
        FtLevel& L = a.lv[l];
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * a.RC, ldb = ncols + 2;
        const int h3 = L.sym ? L.n3 / 2 : L.n3, hx = L.sym ? L.next / 2 : L.next;
        for (int which = 0; which < 3; ++which) {
            FtStageDesc& st = L.st[which];
            st = FtStageDesc{};
            if (down != (which == 2)) continue;
            if (which == 0 && L.xdiag) continue;
            st.nh = L.sym ? 2 : 1;
            st.hr = which == 1 ? hx : h3;
            st.hk = which == 2 ? hx : h3;
            st.lda = (st.hr + 7) / 8 * 8 + 2;
            int bk = (a.slot_bytes / (st.nh * st.lda * 16)) & ~3;
            if (bk < 4) return false;
            bk = std::min(bk, ceil4(st.hk));
            st.nchunks = (st.hk + bk - 1) / bk;
            bk = ceil4((st.hk + st.nchunks - 1) / st.nchunks);   // even chunks
            st.nchunks = (st.hk + bk - 1) / bk;
            st.bk = bk;
            st.img_off = img;
            img += static_cast<long long>(st.nchunks) * st.nh * st.bk * st.lda;
            bmax = std::max(bmax, static_cast<size_t>(st.bk) * st.nchunks * ldb * 16);
            const int ntiles = (st.hr + 7) / 8 * (ncols / 8);
            if (ntiles > FT_CW * FT_IT) return false;
            if (down) {
                const int KS = std::min(6, std::max(1, FT_CW * FT_IT / ntiles));
                // the k-slice partial sums alias both B halves
                bmax = std::max(bmax, (static_cast<size_t>(KS - 1) * ntiles * 2 * 4 * 32 * 8 + 1) / 2);
            }
        }
        if (!down && L.xdiag) bmax = std::max(bmax, static_cast<size_t>(L.st[1].bk) * L.st[1].nchunks * ldb * 16);
    }
    a.img_ps = img;
    // index tables
    auto pad_i = [&](int mult) { while (itab.size() % mult) itab.push_back(0); };
    for (int l = 0; l < a.nlev; ++l) {
        FtLevel& L = a.lv[l];
        const FtHostLevel& H = hl[l];
        const int nc = L.nchild, h3 = L.sym ? L.n3 / 2 : L.n3, hx = L.sym ? L.next / 2 : L.next;
        auto cpos = [&](int r) { return H.extc[r] * nc + H.extp[r]; };
        if (!down) {
            pad_i(4);
            L.t_xg = static_cast<int>(itab.size());
            L.d_xs = static_cast<int>(dtab.size());
            for (int k = 0; k < h3; ++k) {
                const int pA = L.sym ? H.iA[k] : k, pB = L.sym ? H.iB[k] : k;
                itab.insert(itab.end(), {H.ia3p[pA], nc + H.ib3p[pA], H.ia3p[pB], nc + H.ib3p[pB]});
                dtab.push_back(L.sym ? H.is[k] : 0.0);
            }
            pad_i(2);
            L.t_xrow = static_cast<int>(itab.size());
            L.d_xso = static_cast<int>(dtab.size());
            for (int r = 0; r < h3; ++r) {
                itab.insert(itab.end(), {L.sym ? H.iA[r] : r, L.sym ? H.iB[r] : r});
                dtab.push_back(L.sym ? 0.5 * H.is[r] : 0.0);
            }
            pad_i(4);
            L.t_yrow = static_cast<int>(itab.size());
            L.d_yso = static_cast<int>(dtab.size());
            for (int r = 0; r < hx; ++r) {
                const int ra = L.sym ? H.eA[r] : r, rb = L.sym ? H.eB[r] : r;
                itab.insert(itab.end(), {ra, rb, cpos(ra), cpos(rb)});
                dtab.push_back(L.sym ? 0.5 * H.es[r] : 0.0);
            }
        } else {
            pad_i(2);
            L.t_dg = static_cast<int>(itab.size());
            L.d_ds = static_cast<int>(dtab.size());
            for (int k = 0; k < hx; ++k) {
                itab.insert(itab.end(), {L.sym ? H.eA[k] : k, L.sym ? H.eB[k] : k});
                dtab.push_back(L.sym ? H.es[k] : 0.0);
            }
            L.t_drow = static_cast<int>(itab.size());
            L.d_dso = static_cast<int>(dtab.size());
            for (int r = 0; r < h3; ++r) {
                itab.insert(itab.end(), {L.sym ? H.iA[r] : r, L.sym ? H.iB[r] : r});
                dtab.push_back(L.sym ? 0.5 * H.is[r] : 0.0);
            }
            L.t_dch = static_cast<int>(itab.size());
            for (int r = 0; r < L.next; ++r) itab.push_back(cpos(r));
            if ((L.t_dch + L.next) % 2) return false;   // the int2 part must stay 8-byte aligned (next is even)
            for (int k = 0; k < L.n3; ++k) itab.insert(itab.end(), {H.ia3p[k], nc + H.ib3p[k]});
        }
    }
    a.n_itab = static_cast<int>(itab.size());
    a.n_dtab = static_cast<int>(dtab.size());
    // state buffers: levels alternate between A and B (UP: the child h of lv[0] in A;
    // DOWN: the top boxes' boundary values in A)
    size_t sa = 0, sb = 0, sw = 0, su = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        const size_t nl = static_cast<size_t>(a.CS) << (a.nlev - 1 - l);
        sw += nl * L.n3 * a.RC * 16;
        su = std::max(su, nl * L.n3 * a.RC * 16);
        if (!down) {
            const size_t in = 2 * nl * L.nchild * a.RC * 16;
            (l % 2 == 0 ? sa : sb) = std::max(l % 2 == 0 ? sa : sb, in);
            if (l < a.nlev - 1) {
                const size_t out = nl * L.next * a.RC * 16;
                (l % 2 == 0 ? sb : sa) = std::max(l % 2 == 0 ? sb : sa, out);
            }
        } else {
            const int d = a.nlev - 1 - l;   // depth from the top
            const size_t in = nl * L.next * a.RC * 16;
            (d % 2 == 0 ? sa : sb) = std::max(d % 2 == 0 ? sa : sb, in);
        }
    }
    a.off_tab = FT_HDR;
    a.off_ring = align_up(a.off_tab + ((a.n_itab + 1) & ~1) * 4 + a.n_dtab * 8, 128);
    a.off_a = a.off_ring + a.nslots * a.slot_bytes;
    a.off_b = a.off_a + align_up(static_cast<int>(sa), 128);
    a.off_w = a.off_b + align_up(static_cast<int>(sb), 128);
    a.off_u = a.off_w + (down ? align_up(static_cast<int>(sw), 128) : 0);
    a.off_bx = a.off_u + (down ? align_up(static_cast<int>(su), 128) : 0);
    a.bhalf = align_up(static_cast<int>(bmax), 128);
    a.off_by = a.off_bx + 2 * a.bhalf;
    a.smem_bytes = a.off_by + (down ? 0 : 2 * a.bhalf);
    return a.smem_bytes <= 220 * 1024;
}

void ft_allow() {
    cudaFuncSetAttribute(k_ft_up, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_ft_down, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

void ft_pack(const FtArgs& a, bool down, double2* img, int npoles, cudaStream_t s) {
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        for (int which = 0; which < 3; ++which) {
            const FtStageDesc& st = L.st[which];
            if (st.nchunks == 0) continue;
            if (down != (which == 2)) continue;
            PackArgs p;
            p.M = which == 0 ? L.X : which == 1 ? L.Y : L.S;
            p.pp = which == 0 ? L.ppX : which == 1 ? L.ppY : L.ppS;
            p.img = img + st.img_off;
            p.img_ps = a.img_ps;
            p.hr = st.hr; p.hk = st.hk; p.nh = st.nh; p.lda = st.lda; p.bk = st.bk; p.nchunks = st.nchunks;
            const long long tot = static_cast<long long>(st.nchunks) * st.nh * st.bk * st.lda;
            k_ft_pack<<<dim3(static_cast<unsigned>((tot + 255) / 256), static_cast<unsigned>(npoles)), 256, 0, s>>>(p);
        }
    }
}

void ft_launch_up(const FtArgs& a, int top_nodes, int pc, cudaStream_t s) {
    k_ft_up<<<dim3(static_cast<unsigned>(top_nodes / a.CS * a.ncb), static_cast<unsigned>(pc)), FT_NT, a.smem_bytes, s>>>(a);
}

void ft_launch_down(const FtArgs& a, int top_nodes, int pc, cudaStream_t s) {
    k_ft_down<<<dim3(static_cast<unsigned>(top_nodes / a.CS * a.ncb), static_cast<unsigned>(pc)), FT_NT, a.smem_bytes,
                s>>>(a);
}

}  // namespace dev
}  // namespace rexp

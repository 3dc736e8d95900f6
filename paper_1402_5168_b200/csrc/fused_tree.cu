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
struct FtStage {
    const double2* M;   // this pole's operator ([M+ | M-] when nh == 2), column-major hr x hk
    int hr, hk, nh, lda, bk;
};

// which: 0 = X, 1 = Y, 2 = S
__host__ __device__ inline FtStage ft_stage(const FtLevel& L, int which, long long m, int slot_bytes) {
    FtStage s;
    const int n3 = L.sym ? L.n3 / 2 : L.n3, nx = L.sym ? L.next / 2 : L.next;
    s.nh = L.sym ? 2 : 1;
    s.hr = which == 1 ? nx : n3;
    s.hk = which == 2 ? nx : n3;
    const double2* base = which == 0 ? L.X : which == 1 ? L.Y : L.S;
    const long long pp = which == 0 ? L.ppX : which == 1 ? L.ppY : L.ppS;
    s.M = base + m * pp;
    s.lda = ((s.hr + 7) / 8) * 8 + 2;
    int bk = (slot_bytes / (s.nh * s.lda * 16)) & ~3;
    if (bk > ceil4(s.hk)) bk = ceil4(s.hk);
    s.bk = bk;
    return s;
}

struct Ring {
    int slot = 0;
    unsigned phase = 0;
    __device__ __forceinline__ void advance(int nslots) {
        if (++slot == nslots) { slot = 0; phase ^= 1u; }
    }
};

// producer side of one stage: every K chunk -> the next ring slot
__device__ __forceinline__ void ft_produce(const FtStage& st, Ring& rg, const FtArgs& a, unsigned ring, unsigned full,
                                           unsigned empty, int lane) {
    for (int k0 = 0; k0 < st.hk; k0 += st.bk) {
        const int kc = min(st.bk, st.hk - k0);
        mbar_wait(empty + 8 * rg.slot, rg.phase ^ 1u);
        if (lane == 0) mbar_expect_tx(full + 8 * rg.slot, static_cast<unsigned>(st.nh * kc * st.hr * 16));
        __syncwarp();
        const unsigned dst0 = ring + rg.slot * a.slot_bytes;
        for (int idx = lane; idx < st.nh * kc; idx += 32) {
            const int hf = idx / kc, c = idx % kc;
            bulk_g2s(dst0 + static_cast<unsigned>((hf * st.bk + c) * st.lda) * 16u,
                     st.M + static_cast<size_t>(hf) * st.hr * st.hk + static_cast<size_t>(k0 + c) * st.hr,
                     static_cast<unsigned>(st.hr * 16), full + 8 * rg.slot);
        }
        rg.advance(a.nslots);
    }
}

// consumer side: C = M B over the stage's K chunks; items (m-tile, n-tile[, k
// slice]) are dealt to the warps round-robin.  KS > 1 (DOWN: few rows, long K)
// splits the k-steps of every chunk over KS warps per tile; the partial sums are
// combined through `scratch` in a fixed order.  epi(row, col, P[4], D[4]) gets
// the tile's values {re(col), re(col+1), im(col), im(col+1)} of both halves.
template <class Epi>
__device__ __forceinline__ void ft_gemm(const FtStage& st, const double2* Bp, const double2* Bm, int ldb, int ncols,
                                        int KS, double* scratch, Ring& rg, const FtArgs& a, const char* ringp,
                                        unsigned full, unsigned empty, int warp, int lane, Epi epi) {
    const int g = lane >> 2, t4 = lane & 3;
    const int ntl = ncols >> 3, ntiles = ((st.hr + 7) >> 3) * ntl, nitems = ntiles * KS;
    double acc[FT_IT][2][6];
#pragma unroll
    for (int u = 0; u < FT_IT; ++u)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int e = 0; e < 6; ++e) acc[u][hf][e] = 0.0;
    for (int k0 = 0; k0 < st.hk; k0 += st.bk) {
        const int kc = min(st.bk, st.hk - k0);
        const int ksteps = (kc + 3) >> 2;
        mbar_wait(full + 8 * rg.slot, rg.phase);
        const double2* As = reinterpret_cast<const double2*>(ringp + static_cast<size_t>(rg.slot) * a.slot_bytes);
#pragma unroll
        for (int u = 0; u < FT_IT; ++u) {
            const int it = warp + FT_CW * u;
            if (it < nitems) {
                const int tile = it % ntiles, sl = it / ntiles;
                const int mi = tile / ntl, ni = tile % ntl;
                for (int ks = sl; ks < ksteps; ks += KS) {
                    const int kk = ks * 4 + t4;
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        if (hf < st.nh) {
                            const double2 av = As[(hf * st.bk + kk) * st.lda + mi * 8 + g];
                            const double2 bv = (hf ? Bm : Bp)[(k0 + kk) * ldb + ni * 8 + g];
                            dmma884(acc[u][hf][0], acc[u][hf][1], av.x, bv.x);
                            dmma884(acc[u][hf][2], acc[u][hf][3], av.x + av.y, bv.x + bv.y);
                            dmma884(acc[u][hf][4], acc[u][hf][5], av.y, bv.y);
                        }
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
            const int mi = it / ntl, ni = it % ntl;
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

// B (or B+-) of a stage from a gathered vector x(node i, position, column j)
template <class XF>
__device__ __forceinline__ void ft_form_b(double2* Bp, double2* Bm, int ldb, int ncols, int hk, bool sym,
                                          const int* pA, const int* pB, const double* ps, int RC, int tid, XF x) {
    const int KP = ceil4(hk);
    for (int e = tid; e < KP * ncols; e += 32 * FT_CW) {
        const int k = e / ncols, col = e % ncols;
        double2 vp = make_double2(0.0, 0.0), vm = vp;
        if (k < hk) {
            const int i = col / RC, j = col % RC;
            if (sym) {
                const double2 xa = x(i, pA[k], j), xb = x(i, pB[k], j);
                const double s = ps[k];
                vp = make_double2(xa.x + s * xb.x, xa.y + s * xb.y);
                vm = make_double2(xa.x - s * xb.x, xa.y - s * xb.y);
            } else {
                vp = x(i, k, j);
            }
        }
        Bp[k * ldb + col] = vp;
        if (sym) Bm[k * ldb + col] = vm;
    }
}

// ------------------------------------------------------------------------------
// UP: levels lv[0 .. nlev-1]; reads the child h of lv[0], writes every level's w3
// and the top level's h.
// ------------------------------------------------------------------------------
__global__ void __launch_bounds__(FT_NT, 1) k_ft_up(const __grid_constant__ FtArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = blockIdx.y;
    const int cb = blockIdx.x % a.ncb, top0 = (blockIdx.x / a.ncb) * a.CS;
    const int c0 = cb * a.RC, RC = a.RC, R2 = a.R2;
    const unsigned full = smem_u32(smem), empty = full + 64, ring = smem_u32(smem + a.off_ring);
    int* ids = reinterpret_cast<int*>(smem + 128);
    const int stride = a.CS << a.nlev;

    // zero the ring once: padded rows / columns of a slot are multiplied (by zero
    // rows of B or into unused C rows) and must stay finite
    for (int e = tid; e < a.nslots * a.slot_bytes / 16; e += FT_NT)
        reinterpret_cast<double2*>(smem + a.off_ring)[e] = make_double2(0.0, 0.0);
    if (tid == 0) {
        for (int s = 0; s < a.nslots; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, FT_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    ft_node_ids(a, ids, stride, top0, tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    if (warp == FT_CW) {
        Ring rg;
        for (int l = 0; l < a.nlev; ++l) {
            const FtLevel& L = a.lv[l];
            if (!L.xdiag) ft_produce(ft_stage(L, 0, m, a.slot_bytes), rg, a, ring, full, empty, lane);
            ft_produce(ft_stage(L, 1, m, a.slot_bytes), rg, a, ring, full, empty, lane);
        }
        return;
    }

    // ---- consumers ----
    double2* cur = reinterpret_cast<double2*>(smem + a.off_a);
    double2* nxt = reinterpret_cast<double2*>(smem + a.off_b);
    double2* W = reinterpret_cast<double2*>(smem + a.off_w);
    double2* Bp = reinterpret_cast<double2*>(smem + a.off_bp);
    double2* Bm = reinterpret_cast<double2*>(smem + a.off_bm);
    const char* ringp = smem + a.off_ring;
    constexpr int CT = 32 * FT_CW;
    {
        const int nin = a.CS << a.nlev, nc = a.lv[0].nchild;
        const double2* hm = a.hin + static_cast<size_t>(m) * a.hps * R2;
        for (int e = tid; e < nin * nc * RC; e += CT) {
            const int j = e % RC, r = (e / RC) % nc, i = e / (RC * nc);
            cp_async16(cur + e, hm + (static_cast<size_t>(ids[i]) * nc + r) * R2 + c0 + j);
        }
        cp_async_commit();
        cp_async_wait_all();
    }
    consumer_sync();
    Ring rg;
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * RC, ldb = ncols + 2;
        const int n3 = L.n3, next = L.next, nc = L.nchild;
        const int* lid = ids + (l + 1) * stride;
        const bool top = l == a.nlev - 1;
        const double2* curc = cur;
        auto xsum = [&](int i, int pos, int j) {   // h^a_3 + h^b_3 of node i
            const double2 u = curc[((2 * i) * nc + L.ia3p[pos]) * RC + j];
            const double2 v = curc[((2 * i + 1) * nc + L.ib3p[pos]) * RC + j];
            return make_double2(u.x + v.x, u.y + v.y);
        };
        // ---- w3 = -X (h^a_3 + h^b_3) (the store holds -X) ----
        if (L.xdiag) {
            const double2* Xm = L.X + m * L.ppX;
            for (int e = tid; e < nl * n3 * RC; e += CT) {
                const int j = e % RC, k = (e / RC) % n3, i = e / (RC * n3);
                const double2 s3 = xsum(i, k, j);
                const double2 x = __ldg(Xm + static_cast<size_t>(k) * (n3 + 1));
                W[e] = make_double2(x.x * s3.x - x.y * s3.y, x.x * s3.y + x.y * s3.x);
            }
        } else {
            const FtStage st = ft_stage(L, 0, m, a.slot_bytes);
            ft_form_b(Bp, Bm, ldb, ncols, st.hk, L.sym != 0, L.siA, L.siB, L.sis, RC, tid, xsum);
            consumer_sync();
            ft_gemm(st, Bp, Bm, ldb, ncols, 1, nullptr, rg, a, ringp, full, empty, warp, lane,
                    [&](int row, int col, const double* P, const double* D) {
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int i = (col + jj) / RC, j = (col + jj) % RC;
                            if (L.sym) {
                                const double so = 0.5 * L.sis[row];
                                W[(i * n3 + L.siA[row]) * RC + j] =
                                    make_double2(0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                                W[(i * n3 + L.siB[row]) * RC + j] =
                                    make_double2(so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                            } else {
                                W[(i * n3 + row) * RC + j] = make_double2(P[jj], P[2 + jj]);
                            }
                        }
                    });
        }
        consumer_sync();
        // w3 -> global (the downward pass adds it)
        {
            double2* wg = L.w3 + static_cast<size_t>(m) * L.nodes * n3 * R2;
            for (int e = tid; e < nl * n3 * RC; e += CT) {
                const int j = e % RC, k = (e / RC) % n3, i = e / (RC * n3);
                wg[(static_cast<size_t>(lid[i]) * n3 + k) * R2 + c0 + j] = W[e];
            }
        }
        // ---- h = h_child[ext] + Y w3 ----
        {
            const FtStage st = ft_stage(L, 1, m, a.slot_bytes);
            const double2* Wc = W;
            ft_form_b(Bp, Bm, ldb, ncols, st.hk, L.sym != 0, L.siA, L.siB, L.sis, RC, tid,
                      [&](int i, int pos, int j) { return Wc[(i * n3 + pos) * RC + j]; });
            consumer_sync();
            double2* hg = a.hout + static_cast<size_t>(m) * a.hps * R2;
            double2* nx = nxt;
            auto put = [&](int i, int r, int j, double re, double im) {
                const double2 c = curc[((2 * i + L.extc[r]) * nc + L.extp[r]) * RC + j];
                const double2 v = make_double2(re + c.x, im + c.y);
                if (top) hg[(static_cast<size_t>(lid[i]) * next + r) * R2 + c0 + j] = v;
                else nx[(i * next + r) * RC + j] = v;
            };
            ft_gemm(st, Bp, Bm, ldb, ncols, 1, nullptr, rg, a, ringp, full, empty, warp, lane,
                    [&](int row, int col, const double* P, const double* D) {
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int i = (col + jj) / RC, j = (col + jj) % RC;
                            if (L.sym) {
                                const double so = 0.5 * L.ses[row];
                                put(i, L.seA[row], j, 0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                                put(i, L.seB[row], j, so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                            } else {
                                put(i, row, j, P[jj], P[2 + jj]);
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
__global__ void __launch_bounds__(FT_NT, 1) k_ft_down(const __grid_constant__ FtArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = blockIdx.y;
    const int cb = blockIdx.x % a.ncb, top0 = (blockIdx.x / a.ncb) * a.CS;
    const int c0 = cb * a.RC, RC = a.RC, R2 = a.R2;
    const unsigned full = smem_u32(smem), empty = full + 64, ring = smem_u32(smem + a.off_ring);
    int* ids = reinterpret_cast<int*>(smem + 128);
    const int stride = a.CS << a.nlev;

    for (int e = tid; e < a.nslots * a.slot_bytes / 16; e += FT_NT)
        reinterpret_cast<double2*>(smem + a.off_ring)[e] = make_double2(0.0, 0.0);
    if (tid == 0) {
        for (int s = 0; s < a.nslots; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, FT_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    ft_node_ids(a, ids, stride, top0, tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    if (warp == FT_CW) {
        Ring rg;
        for (int l = a.nlev - 1; l >= 0; --l)
            ft_produce(ft_stage(a.lv[l], 2, m, a.slot_bytes), rg, a, ring, full, empty, lane);
        return;
    }

    double2* cur = reinterpret_cast<double2*>(smem + a.off_a);
    double2* nxt = reinterpret_cast<double2*>(smem + a.off_b);
    double2* W = reinterpret_cast<double2*>(smem + a.off_w);    // every level's w3, top level first
    double2* U3 = reinterpret_cast<double2*>(smem + a.off_u);
    double2* Bp = reinterpret_cast<double2*>(smem + a.off_bp);
    double2* Bm = reinterpret_cast<double2*>(smem + a.off_bm);
    const char* ringp = smem + a.off_ring;
    constexpr int CT = 32 * FT_CW;
    double2* em = a.edge + static_cast<size_t>(m) * a.NE * R2;
    {
        // the top boxes' boundary values and all w3 terms of the group
        const FtLevel& T = a.lv[a.nlev - 1];
        const int* tid_ = ids + a.nlev * stride;
        for (int e = tid; e < a.CS * T.next * RC; e += CT) {
            const int j = e % RC, r = (e / RC) % T.next, i = e / (RC * T.next);
            cp_async16(cur + e, em + static_cast<size_t>(T.gext[static_cast<size_t>(tid_[i]) * T.next + r]) * R2 + c0 + j);
        }
        int woff = 0;
        for (int l = a.nlev - 1; l >= 0; --l) {
            const FtLevel& L = a.lv[l];
            const int nl = a.CS << (a.nlev - 1 - l);
            const int* lid = ids + (l + 1) * stride;
            const double2* wg = L.w3 + static_cast<size_t>(m) * L.nodes * L.n3 * R2;
            for (int e = tid; e < nl * L.n3 * RC; e += CT) {
                const int j = e % RC, k = (e / RC) % L.n3, i = e / (RC * L.n3);
                cp_async16(W + woff + e, wg + (static_cast<size_t>(lid[i]) * L.n3 + k) * R2 + c0 + j);
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
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * RC, ldb = ncols + 2;
        const int n3 = L.n3, next = L.next, nc = L.nchild;
        const int* lid = ids + (l + 1) * stride;
        const FtStage st = ft_stage(L, 2, m, a.slot_bytes);
        const double2* curc = cur;
        ft_form_b(Bp, Bm, ldb, ncols, st.hk, L.sym != 0, L.seA, L.seB, L.ses, RC, tid,
                  [&](int i, int pos, int j) { return curc[(i * next + pos) * RC + j]; });
        consumer_sync();
        // k slices: as many as the warps allow (few output rows, long K)
        const int ntiles = ((st.hr + 7) >> 3) * (ncols >> 3);
        int KS = (FT_CW * FT_IT) / ntiles;
        KS = KS < 1 ? 1 : KS > 6 ? 6 : KS;
        const double2* Wl = W + woff;
        auto put = [&](int i, int k, int j, double re, double im) {
            const double2 w = Wl[(i * n3 + k) * RC + j];
            const double2 v = make_double2(re + w.x, im + w.y);
            U3[(i * n3 + k) * RC + j] = v;
            em[static_cast<size_t>(L.g3[static_cast<size_t>(lid[i]) * n3 + k]) * R2 + c0 + j] = v;
        };
        ft_gemm(st, Bp, Bm, ldb, ncols, KS, reinterpret_cast<double*>(Bp), rg, a, ringp, full, empty, warp, lane,
                [&](int row, int col, const double* P, const double* D) {
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int i = (col + jj) / RC, j = (col + jj) % RC;
                        if (L.sym) {
                            const double so = 0.5 * L.sis[row];
                            put(i, L.siA[row], j, 0.5 * (P[jj] + D[jj]), 0.5 * (P[2 + jj] + D[2 + jj]));
                            put(i, L.siB[row], j, so * (P[jj] - D[jj]), so * (P[2 + jj] - D[2 + jj]));
                        } else {
                            put(i, row, j, P[jj], P[2 + jj]);
                        }
                    }
                });
        consumer_sync();
        woff += nl * n3 * RC;
        if (l > 0) {
            // the children's boundary values: parent boundary rows and the new interface values
            for (int e = tid; e < nl * (next + n3) * RC; e += CT) {
                const int j = e % RC, r = (e / RC) % (next + n3), i = e / (RC * (next + n3));
                if (r < next) {
                    nxt[((2 * i + L.extc[r]) * nc + L.extp[r]) * RC + j] = curc[(i * next + r) * RC + j];
                } else {
                    const int k = r - next;
                    const double2 v = U3[(i * n3 + k) * RC + j];
                    nxt[((2 * i) * nc + L.ia3p[k]) * RC + j] = v;
                    nxt[((2 * i + 1) * nc + L.ib3p[k]) * RC + j] = v;
                }
            }
            consumer_sync();
            double2* t = cur; cur = nxt; nxt = t;
        }
    }
}

inline int align_up(int v, int a) { return (v + a - 1) / a * a; }

}  // namespace

bool ft_plan(FtArgs& a, bool down) {
    if (a.nlev < 1 || a.nlev > FT_MAXLEV) return false;
    if (a.R2 >= 8) {
        if (a.R2 % 8) return false;
        a.RC = 8;
    } else {
        if (8 % a.R2) return false;
        a.RC = a.R2;
    }
    a.CS = 8 / a.RC;
    a.ncb = a.R2 / a.RC;
    if (a.lv[a.nlev - 1].nodes % a.CS) return false;
    if ((a.nlev + 1) * (a.CS << a.nlev) * 4 + 128 > FT_HDR) return false;
    // state buffers: levels alternate between A and B (UP: the child h of lv[0] in A;
    // DOWN: the top boxes' boundary values in A)
    size_t sa = 0, sb = 0, sw = 0, su = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        const size_t nl = static_cast<size_t>(a.CS) << (a.nlev - 1 - l);
        sw += nl * L.n3 * a.RC * 16;
        su = std::max(su, nl * L.n3 * a.RC * 16);
        if (!down) {
            // lv[l] reads its children (buffer l % 2 == 0 ? A : B) and writes the other (unless top)
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
    // B staging and the ring: the largest padded column decides the smallest slot
    size_t sbp = 0, sbm = 0;
    int colmax = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const FtLevel& L = a.lv[l];
        const int nl = a.CS << (a.nlev - 1 - l), ncols = nl * a.RC, ldb = ncols + 2;
        for (int which = down ? 2 : 0; which <= (down ? 2 : 1); ++which) {
            if (which == 0 && L.xdiag) continue;
            const FtStage st = ft_stage(L, which, 0, 1 << 30);
            const size_t b = static_cast<size_t>(ceil4(st.hk)) * ldb * 16;
            sbp = std::max(sbp, b);
            if (L.sym) sbm = std::max(sbm, b);
            colmax = std::max(colmax, st.nh * st.lda * 16);
            const int ntiles = ((st.hr + 7) / 8) * (ncols / 8);
            if (ntiles > FT_CW * FT_IT) return false;
            if (down) {
                int KS = std::min(6, std::max(1, FT_CW * FT_IT / ntiles));
                sbp = std::max(sbp, static_cast<size_t>(KS - 1) * ntiles * 2 * 4 * 32 * 8);
            }
        }
    }
    a.nslots = 3;
    a.slot_bytes = align_up(std::max(4 * colmax, 12 * 1024), 128);
    a.off_ring = FT_HDR;
    a.off_a = a.off_ring + a.nslots * a.slot_bytes;
    a.off_b = a.off_a + align_up(static_cast<int>(sa), 128);
    a.off_w = a.off_b + align_up(static_cast<int>(sb), 128);
    a.off_u = a.off_w + align_up(static_cast<int>(sw), 128);
    a.off_bp = a.off_u + (down ? align_up(static_cast<int>(su), 128) : 0);
    a.off_bm = a.off_bp + align_up(static_cast<int>(sbp), 128);
    a.smem_bytes = a.off_bm + align_up(static_cast<int>(sbm), 128);
    return a.smem_bytes <= 220 * 1024;
}

void ft_allow() {
    cudaFuncSetAttribute(k_ft_up, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_ft_down, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
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

// Tile instantiations of the symmetric-pair DMMA GEMM (cgemm_sym.cuh).
#include "cgemm_launch.hpp"
#include "cgemm_sym.cuh"

namespace rexp {
namespace dev {
namespace {

template <int MT, int WN, int BK, int R2T, int MODE, int NST, bool PF>
void cgs_launch(dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    constexpr int WM = WN == 2 ? 4 : WN == 4 ? 2 : 1;
    size_t smem = cgemm_sym_smem_bytes<MT, WN, BK, WM, NST, MODE>();
    // DOWN rings with the second reflection stage the partners' raw tiles too
    if (MODE == CG_DOWN && NST >= 3 && a.sym2) smem += (size_t)cgs_ring<NST>() * 2 * BK * (8 * WN + 2) * sizeof(double2);
    if constexpr (NST != 2) {
        // a ring that does not fit (3 stages of a wide tile plus the partner tiles): register-staged form
        if (smem > 200 * 1024) {
            cgs_launch<MT, WN, BK, R2T, MODE, 2, false>(grid, s, a);
            return;
        }
    }
    k_cgemm_sym<MT, WN, BK, R2T, MODE, WM, NST, PF><<<grid, 32 * WN * WM, smem, s>>>(a);
}
template <int MT, int WN, int BK, int R2T, int MODE, int NST, bool PF>
void cgs_allow1() {
    constexpr int WM = WN == 2 ? 4 : WN == 4 ? 2 : 1;
    cudaFuncSetAttribute(k_cgemm_sym<MT, WN, BK, R2T, MODE, WM, NST, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
}
template <int BK, int R2T, int MODE, int NST, bool PF>
void cgs_tiles_n(int MT, int WN, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    if (MT == 2) {
        if (WN == 2) cgs_launch<2, 2, BK, R2T, MODE, NST, PF>(grid, s, a);
        else if (WN == 4) cgs_launch<2, 4, BK, R2T, MODE, NST, PF>(grid, s, a);
        else cgs_launch<2, 8, BK, R2T, MODE, NST, PF>(grid, s, a);
    } else {
        if (WN == 2) cgs_launch<4, 2, BK, R2T, MODE, NST, PF>(grid, s, a);
        else if (WN == 4) cgs_launch<4, 4, BK, R2T, MODE, NST, PF>(grid, s, a);
        else cgs_launch<4, 8, BK, R2T, MODE, NST, PF>(grid, s, a);
    }
}
// PF variants (additive epilogue terms prefetched before the K loop): UP-Y / DOWN
// with compile-time R2 = 128 (many right-hand sides: latency-bound low levels)
template <int R2T, int MODE>
constexpr bool cgs_has_pf() { return R2T == 128 && (MODE == CG_UPY || MODE == CG_DOWN); }
// nst = 3: 3-stage cp.async ring (UP-Y / DOWN only)
// nst: 2 = register-staged B, 3 = cp.async ring of 3, 12 / 11 = cp.async ring of
// 2 / 1 (the ring variants: UP-Y / DOWN only; 12 / 11 compiled for R2 = 128)
template <int BK, int R2T, int MODE>
void cgs_tiles(int MT, int WN, int nst, bool pf, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    if constexpr (cgs_has_pf<R2T, MODE>()) {
        if (nst == 12) { pf ? cgs_tiles_n<BK, R2T, MODE, 12, true>(MT, WN, grid, s, a)
                            : cgs_tiles_n<BK, R2T, MODE, 12, false>(MT, WN, grid, s, a); return; }
        if (nst == 11) { pf ? cgs_tiles_n<BK, R2T, MODE, 11, true>(MT, WN, grid, s, a)
                            : cgs_tiles_n<BK, R2T, MODE, 11, false>(MT, WN, grid, s, a); return; }
        if (pf) {
            if (nst >= 3) cgs_tiles_n<BK, R2T, MODE, 3, true>(MT, WN, grid, s, a);
            else cgs_tiles_n<BK, R2T, MODE, 2, true>(MT, WN, grid, s, a);
            return;
        }
    }
    if constexpr (MODE == CG_UPY || MODE == CG_DOWN) {
        if (nst >= 3) {
            cgs_tiles_n<BK, R2T, MODE, 3, false>(MT, WN, grid, s, a);
            return;
        }
    }
    // UP-X single-stage cp.async ring (both children's gathers copied raw), R2 = 128
    if constexpr (MODE == CG_UPX && R2T == 128) {
        if (nst == 11) {
            cgs_tiles_n<BK, R2T, MODE, 11, false>(MT, WN, grid, s, a);
            return;
        }
    }
    cgs_tiles_n<BK, R2T, MODE, 2, false>(MT, WN, grid, s, a);
}
template <int BK, int R2T, int MODE, int NST, bool PF>
void cgs_allow_n() {
    cgs_allow1<2, 2, BK, R2T, MODE, NST, PF>(); cgs_allow1<2, 4, BK, R2T, MODE, NST, PF>();
    cgs_allow1<2, 8, BK, R2T, MODE, NST, PF>(); cgs_allow1<4, 2, BK, R2T, MODE, NST, PF>();
    cgs_allow1<4, 4, BK, R2T, MODE, NST, PF>(); cgs_allow1<4, 8, BK, R2T, MODE, NST, PF>();
}
template <int BK, int R2T, int MODE>
void cgs_allow_tiles() {
    cgs_allow_n<BK, R2T, MODE, 2, false>();
    if constexpr (MODE == CG_UPY || MODE == CG_DOWN) cgs_allow_n<BK, R2T, MODE, 3, false>();
    if constexpr (MODE == CG_UPX && R2T == 128) cgs_allow_n<BK, R2T, MODE, 11, false>();
    if constexpr (cgs_has_pf<R2T, MODE>()) {
        cgs_allow_n<BK, R2T, MODE, 2, true>();
        cgs_allow_n<BK, R2T, MODE, 3, true>();
        cgs_allow_n<BK, R2T, MODE, 12, true>();
        cgs_allow_n<BK, R2T, MODE, 12, false>();
        cgs_allow_n<BK, R2T, MODE, 11, true>();
        cgs_allow_n<BK, R2T, MODE, 11, false>();
    }
}
// BK = 16 always: the pair kernel stages A and B for both halves, so the
// smaller chunk keeps two or more CTAs per SM (BK = 28 with 64-row tiles needs
// ~180 KB of shared memory)
template <int MODE>
void cgs_run_mode(int R2, int MT, int WN, int nst, bool pf, int K, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    (void)K;
    if (R2 == 2) cgs_tiles<16, 2, MODE>(MT, WN, nst, pf, grid, s, a);
    else if (R2 == 4) cgs_tiles<16, 4, MODE>(MT, WN, nst, pf, grid, s, a);
    else if (R2 == 128) cgs_tiles<16, 128, MODE>(MT, WN, nst, pf, grid, s, a);   // 64 RHS (c3): shifts, not divisions
    else cgs_tiles<16, 0, MODE>(MT, WN, nst, pf, grid, s, a);
}
template <int MODE>
void cgs_allow_mode() {
    cgs_allow_tiles<16, 2, MODE>();
    cgs_allow_tiles<16, 4, MODE>();
    cgs_allow_tiles<16, 128, MODE>();
    cgs_allow_tiles<16, 0, MODE>();
}

}  // namespace

void cgs_run(int mode, int R2, int MT, int WN, int nst, bool pf, int K, dim3 grid, cudaStream_t s,
             const CgemmSymArgs& a) {
    if (mode == CG_UPX) cgs_run_mode<CG_UPX>(R2, MT, WN, nst, pf, K, grid, s, a);
    else if (mode == CG_UPY) cgs_run_mode<CG_UPY>(R2, MT, WN, nst, pf, K, grid, s, a);
    else cgs_run_mode<CG_DOWN>(R2, MT, WN, nst, pf, K, grid, s, a);
}
void cgs_allow() {
    cgs_allow_mode<CG_UPX>();
    cgs_allow_mode<CG_UPY>();
    cgs_allow_mode<CG_DOWN>();
}

}  // namespace dev
}  // namespace rexp

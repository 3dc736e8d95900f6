// Tile instantiations of the symmetric-pair DMMA GEMM (cgemm_sym.cuh).
#include "cgemm_launch.hpp"
#include "cgemm_sym.cuh"

namespace rexp {
namespace dev {
namespace {

template <int MT, int WN, int BK, int R2T, int MODE>
void cgs_launch(dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    constexpr int WM = WN == 2 ? 4 : WN == 4 ? 2 : 1;
    k_cgemm_sym<MT, WN, BK, R2T, MODE, WM><<<grid, 32 * WN * WM, cgemm_sym_smem_bytes<MT, WN, BK, WM>(), s>>>(a);
}
template <int MT, int WN, int BK, int R2T, int MODE>
void cgs_allow1() {
    constexpr int WM = WN == 2 ? 4 : WN == 4 ? 2 : 1;
    cudaFuncSetAttribute(k_cgemm_sym<MT, WN, BK, R2T, MODE, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
}
template <int BK, int R2T, int MODE>
void cgs_tiles(int MT, int WN, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    if (MT == 2) {
        if (WN == 2) cgs_launch<2, 2, BK, R2T, MODE>(grid, s, a);
        else if (WN == 4) cgs_launch<2, 4, BK, R2T, MODE>(grid, s, a);
        else cgs_launch<2, 8, BK, R2T, MODE>(grid, s, a);
    } else {
        if (WN == 2) cgs_launch<4, 2, BK, R2T, MODE>(grid, s, a);
        else if (WN == 4) cgs_launch<4, 4, BK, R2T, MODE>(grid, s, a);
        else cgs_launch<4, 8, BK, R2T, MODE>(grid, s, a);
    }
}
template <int BK, int R2T, int MODE>
void cgs_allow_tiles() {
    cgs_allow1<2, 2, BK, R2T, MODE>(); cgs_allow1<2, 4, BK, R2T, MODE>(); cgs_allow1<2, 8, BK, R2T, MODE>();
    cgs_allow1<4, 2, BK, R2T, MODE>(); cgs_allow1<4, 4, BK, R2T, MODE>(); cgs_allow1<4, 8, BK, R2T, MODE>();
}
template <int MODE>
void cgs_run_mode(int R2, int MT, int WN, int K, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    const bool b28 = (K % 28) == 0;
    if (R2 == 2) {
        if (b28) cgs_tiles<28, 2, MODE>(MT, WN, grid, s, a);
        else cgs_tiles<16, 2, MODE>(MT, WN, grid, s, a);
    } else if (R2 == 4) {
        if (b28) cgs_tiles<28, 4, MODE>(MT, WN, grid, s, a);
        else cgs_tiles<16, 4, MODE>(MT, WN, grid, s, a);
    } else {
        if (b28) cgs_tiles<28, 0, MODE>(MT, WN, grid, s, a);
        else cgs_tiles<16, 0, MODE>(MT, WN, grid, s, a);
    }
}
template <int MODE>
void cgs_allow_mode() {
    cgs_allow_tiles<16, 2, MODE>(); cgs_allow_tiles<28, 2, MODE>();
    cgs_allow_tiles<16, 4, MODE>(); cgs_allow_tiles<28, 4, MODE>();
    cgs_allow_tiles<16, 0, MODE>(); cgs_allow_tiles<28, 0, MODE>();
}

}  // namespace

void cgs_run(int mode, int R2, int MT, int WN, int K, dim3 grid, cudaStream_t s, const CgemmSymArgs& a) {
    if (mode == CG_UPX) cgs_run_mode<CG_UPX>(R2, MT, WN, K, grid, s, a);
    else if (mode == CG_UPY) cgs_run_mode<CG_UPY>(R2, MT, WN, K, grid, s, a);
    else cgs_run_mode<CG_DOWN>(R2, MT, WN, K, grid, s, a);
}
void cgs_allow() {
    cgs_allow_mode<CG_UPX>();
    cgs_allow_mode<CG_UPY>();
    cgs_allow_mode<CG_DOWN>();
}

}  // namespace dev
}  // namespace rexp

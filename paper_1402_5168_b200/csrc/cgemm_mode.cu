// Tile instantiations of k_cgemm for one mode (compiled once per CG_MODE value).
#include "cgemm_launch.hpp"

#ifndef CG_MODE
#error "compile with -DCG_MODE=<0..5>"
#endif

namespace rexp {
namespace dev {
namespace {

template <int MT, int WN, int BK, int R2T, int MODE, int WM = 1, int MINB = 1, int NST = 2>
void cg_launch(dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    k_cgemm<MT, WN, BK, R2T, MODE, 1, MINB, WM, NST>
        <<<grid, 32 * WN * WM, cgemm_smem_total<MT, WN, BK, 1, WM, NST, (R2T != 0 ? MODE : 0)>(), s>>>(a);
}
// leaf tiles: MT in {4, 5}, WN = 8; merge tiles: MT in {2, 4} with
//   WN = 8, WM = 1 | WN = 4, WM = 2 | WN = 2, WM = 4
template <int BK, int R2T, int MODE, int MINB>
void cg_tiles_b(int MT, int WN, dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    if (MT == 2) {
        if (WN == 2) cg_launch<2, 2, BK, R2T, MODE, 4, MINB>(grid, s, a);
        else if (WN == 4) cg_launch<2, 4, BK, R2T, MODE, 2, MINB>(grid, s, a);
        else cg_launch<2, 8, BK, R2T, MODE, 1, MINB>(grid, s, a);
    } else {
        if (WN == 2) cg_launch<4, 2, BK, R2T, MODE, 4, MINB>(grid, s, a);
        else if (WN == 4) cg_launch<4, 4, BK, R2T, MODE, 2, MINB>(grid, s, a);
        else cg_launch<4, 8, BK, R2T, MODE, 1, MINB>(grid, s, a);
    }
}
// 3-stage cp.async ring (plain-gather B modes), MINB = 1
template <int BK, int R2T, int MODE>
void cg_tiles_s3(int MT, int WN, dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    if constexpr (MODE == CG_UPY || MODE == CG_DOWN) {
        if (MT == 2) {
            if (WN == 2) cg_launch<2, 2, BK, R2T, MODE, 4, 1, 3>(grid, s, a);
            else if (WN == 4) cg_launch<2, 4, BK, R2T, MODE, 2, 1, 3>(grid, s, a);
            else cg_launch<2, 8, BK, R2T, MODE, 1, 1, 3>(grid, s, a);
        } else {
            if (WN == 2) cg_launch<4, 2, BK, R2T, MODE, 4, 1, 3>(grid, s, a);
            else if (WN == 4) cg_launch<4, 4, BK, R2T, MODE, 2, 1, 3>(grid, s, a);
            else cg_launch<4, 8, BK, R2T, MODE, 1, 1, 3>(grid, s, a);
        }
    } else {
        cg_tiles_b<BK, R2T, MODE, 1>(MT, WN, grid, s, a);
    }
}
// single-stage cp.async (plain-gather B modes, R2 = 128): short-K levels
template <int BK, int R2T, int MODE>
void cg_tiles_s1(int MT, int WN, dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    if constexpr ((MODE == CG_UPY || MODE == CG_DOWN) && R2T == 128) {
        if (MT == 2) {
            if (WN == 2) cg_launch<2, 2, BK, R2T, MODE, 4, 1, 11>(grid, s, a);
            else if (WN == 4) cg_launch<2, 4, BK, R2T, MODE, 2, 1, 11>(grid, s, a);
            else cg_launch<2, 8, BK, R2T, MODE, 1, 1, 11>(grid, s, a);
        } else {
            if (WN == 2) cg_launch<4, 2, BK, R2T, MODE, 4, 1, 11>(grid, s, a);
            else if (WN == 4) cg_launch<4, 4, BK, R2T, MODE, 2, 1, 11>(grid, s, a);
            else cg_launch<4, 8, BK, R2T, MODE, 1, 1, 11>(grid, s, a);
        }
    } else {
        cg_tiles_s3<BK, R2T, MODE>(MT, WN, grid, s, a);
    }
}
// MINB = 4: register budget for 4 resident 256-thread CTAs per SM (<= 64 registers);
// MINB = 3 selects the 3-stage cp.async pipeline instead (StageCfg::minb), 6 the
// single-stage one
template <int BK, int R2T, int MODE>
void cg_tiles(int MT, int WN, int MINB, dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    if (MODE == CG_LEAF_UP || MODE == CG_LEAF_DOWN) {
        if (MT == 4) cg_launch<4, 8, BK, R2T, MODE>(grid, s, a);
        else cg_launch<5, 8, BK, R2T, MODE>(grid, s, a);
        return;
    }
    if (MINB == 6) cg_tiles_s1<BK, R2T, MODE>(MT, WN, grid, s, a);
    else if (MINB >= 4) cg_tiles_b<BK, R2T, MODE, 4>(MT, WN, grid, s, a);
    else if (MINB == 3) cg_tiles_s3<BK, R2T, MODE>(MT, WN, grid, s, a);
    else cg_tiles_b<BK, R2T, MODE, 1>(MT, WN, grid, s, a);
}
template <int MT, int WN, int BK, int R2T, int MODE, int WM = 1, int MINB = 1, int NST = 2>
void cg_allow1() {
    cudaFuncSetAttribute(k_cgemm<MT, WN, BK, R2T, MODE, 1, MINB, WM, NST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}
template <int BK, int R2T, int MODE>
void cg_allow_tiles() {
    if (MODE == CG_LEAF_UP || MODE == CG_LEAF_DOWN) {
        cg_allow1<4, 8, BK, R2T, MODE>(); cg_allow1<5, 8, BK, R2T, MODE>();
        return;
    }
    cg_allow1<2, 2, BK, R2T, MODE, 4>(); cg_allow1<2, 4, BK, R2T, MODE, 2>(); cg_allow1<2, 8, BK, R2T, MODE>();
    cg_allow1<4, 2, BK, R2T, MODE, 4>(); cg_allow1<4, 4, BK, R2T, MODE, 2>(); cg_allow1<4, 8, BK, R2T, MODE>();
    cg_allow1<2, 2, BK, R2T, MODE, 4, 4>(); cg_allow1<2, 4, BK, R2T, MODE, 2, 4>(); cg_allow1<2, 8, BK, R2T, MODE, 1, 4>();
    cg_allow1<4, 2, BK, R2T, MODE, 4, 4>(); cg_allow1<4, 4, BK, R2T, MODE, 2, 4>(); cg_allow1<4, 8, BK, R2T, MODE, 1, 4>();
    if constexpr (MODE == CG_UPY || MODE == CG_DOWN) {
        cg_allow1<2, 2, BK, R2T, MODE, 4, 1, 3>(); cg_allow1<2, 4, BK, R2T, MODE, 2, 1, 3>();
        cg_allow1<2, 8, BK, R2T, MODE, 1, 1, 3>(); cg_allow1<4, 2, BK, R2T, MODE, 4, 1, 3>();
        cg_allow1<4, 4, BK, R2T, MODE, 2, 1, 3>(); cg_allow1<4, 8, BK, R2T, MODE, 1, 1, 3>();
    }
    if constexpr ((MODE == CG_UPY || MODE == CG_DOWN) && R2T == 128) {
        cg_allow1<2, 2, BK, R2T, MODE, 4, 1, 11>(); cg_allow1<2, 4, BK, R2T, MODE, 2, 1, 11>();
        cg_allow1<2, 8, BK, R2T, MODE, 1, 1, 11>(); cg_allow1<4, 2, BK, R2T, MODE, 4, 1, 11>();
        cg_allow1<4, 4, BK, R2T, MODE, 2, 1, 11>(); cg_allow1<4, 8, BK, R2T, MODE, 1, 1, 11>();
    }
}

// BK = 28 when K is a multiple of 28 (q = 14: every K of the tree), else 16;
// R2 = 2, 4 (and 128 for up-Y / down) compiled in, anything else at run time
// MINB bit 16: use BK = 16 even when K is a multiple of 28 (smaller shared-memory
// footprint, more resident CTAs; an autotuner candidate)
// R2 = 128 (64 RHS, config 3) compiled in for the first-level up-Y / down GEMMs
// (staged up-Y epilogue, shifts instead of divisions); the levels above run the pair GEMM
constexpr bool kR2x128 = CG_MODE == CG_UPY || CG_MODE == CG_DOWN;
void run(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a) {
    constexpr int M = CG_MODE;
    const bool b28 = (K % 28) == 0 && !(MINB & 16);
    MINB &= 15;
    if (R2 == 2) {
        if (b28) cg_tiles<28, 2, M>(MT, WN, MINB, grid, s, a);
        else cg_tiles<16, 2, M>(MT, WN, MINB, grid, s, a);
    } else if (R2 == 4) {
        if (b28) cg_tiles<28, 4, M>(MT, WN, MINB, grid, s, a);
        else cg_tiles<16, 4, M>(MT, WN, MINB, grid, s, a);
    } else if (kR2x128 && R2 == 128) {
        if constexpr (kR2x128) {
            if (b28) cg_tiles<28, 128, M>(MT, WN, MINB, grid, s, a);
            else cg_tiles<16, 128, M>(MT, WN, MINB, grid, s, a);
        }
    } else {
        if (b28) cg_tiles<28, 0, M>(MT, WN, MINB, grid, s, a);
        else cg_tiles<16, 0, M>(MT, WN, MINB, grid, s, a);
    }
}
void allow() {
    constexpr int M = CG_MODE;
    cg_allow_tiles<16, 2, M>(); cg_allow_tiles<28, 2, M>();
    cg_allow_tiles<16, 4, M>(); cg_allow_tiles<28, 4, M>();
    cg_allow_tiles<16, 0, M>(); cg_allow_tiles<28, 0, M>();
    if constexpr (kR2x128) { cg_allow_tiles<16, 128, M>(); cg_allow_tiles<28, 128, M>(); }
}

}  // namespace

#if CG_MODE == 0
void cg_run_leaf_up(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_leaf_up() { allow(); }
#elif CG_MODE == 1
void cg_run_leaf_down(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_leaf_down() { allow(); }
#elif CG_MODE == 2
void cg_run_upx(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_upx() { allow(); }
#elif CG_MODE == 3
void cg_run_upy(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_upy() { allow(); }
#elif CG_MODE == 4
void cg_run_down(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_down() { allow(); }
#else
void cg_run_root(int R2, int MT, int WN, int MINB, int K, dim3 g, cudaStream_t s, const CgemmArgs& a) { run(R2, MT, WN, MINB, K, g, s, a); }
void cg_allow_root() { allow(); }
#endif

}  // namespace dev
}  // namespace rexp

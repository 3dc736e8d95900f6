// Host-side launchers of the DMMA complex GEMM (k_cgemm) - one translation
// unit per mode (cgemm_mode.cu compiled with -DCG_MODE=...) so the tile
// instantiations build in parallel.
#pragma once

#include <cuda_runtime.h>

#include "cgemm.cuh"

namespace rexp {
namespace dev {

// WM (warps along m) implied by WN for merge tiles: 8 -> 1, 4 -> 2, 2 -> 4
inline int cg_wm(int WN) { return WN == 2 ? 4 : WN == 4 ? 2 : 1; }

void cg_run_leaf_up(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_run_leaf_down(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_run_upx(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_run_upy(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_run_down(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_run_root(int R2, int MT, int WN, int MINB, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a);
void cg_allow_leaf_up();
void cg_allow_leaf_down();
void cg_allow_upx();
void cg_allow_upy();
void cg_allow_down();
void cg_allow_root();

inline void cg_run_mode(int mode, int R2, int MT, int WN, int K, dim3 grid, cudaStream_t s, const CgemmArgs& a,
                        int MINB = 1) {
    switch (mode) {
        case CG_LEAF_UP: cg_run_leaf_up(R2, MT, WN, MINB, K, grid, s, a); break;
        case CG_LEAF_DOWN: cg_run_leaf_down(R2, MT, WN, MINB, K, grid, s, a); break;
        case CG_UPX: cg_run_upx(R2, MT, WN, MINB, K, grid, s, a); break;
        case CG_UPY: cg_run_upy(R2, MT, WN, MINB, K, grid, s, a); break;
        case CG_DOWN: cg_run_down(R2, MT, WN, MINB, K, grid, s, a); break;
        default: cg_run_root(R2, MT, WN, MINB, K, grid, s, a); break;
    }
}
inline void cg_allow_all() {
    cg_allow_leaf_up(); cg_allow_leaf_down(); cg_allow_upx(); cg_allow_upy(); cg_allow_down(); cg_allow_root();
}

}  // namespace dev
}  // namespace rexp

// Standalone tuning harness for k_cgemm (LEAF_UP / LEAF_DOWN shapes of config 1).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1402_5168_b200/csrc/cgemm.cuh"
using namespace rexp::dev;

template <int MT, int WN, int BK, int MODE, int NTW, int MINB>
float run(CgemmArgs a, int nh, int reps) {
    const int R2 = 2;
    int ncols = a.nodes * R2;
    a.nrowblk = (a.rows + 8 * MT - 1) / (8 * MT);
    int ncb = (ncols + 8 * WN * NTW - 1) / (8 * WN * NTW);
    size_t smem = cgemm_smem_bytes<MT, WN, BK, NTW>();
    auto k = k_cgemm<MT, WN, BK, R2, MODE, NTW, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    dim3 grid(a.nrowblk * ncb, nh);
    k<<<grid, 32 * WN, smem>>>(a);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k<<<grid, 32 * WN, smem>>>(a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaFuncAttributes at; cudaFuncGetAttributes(&at, k);
    int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * WN, smem);
    double fl = 8.0 * a.rows * a.K * (double)ncols * nh;
    printf("MODE %d MT %d WN %d BK %d NTW %d MINB %d: %.3f ms  %.2f TF  regs %d spill %zu occ %d  err=%s\n", MODE, MT, WN, BK, NTW, MINB,
           ms / reps, fl / (ms / reps * 1e-3) / 1e12, at.numRegs, at.localSizeBytes, occ, cudaGetErrorString(cudaGetLastError()));
    return ms / reps;
}

int main() {
    const int nh = 282, nelem = 256, q2 = 196, nb = 56, R2 = 2, nF = 3;
    double2 *A, *S, *w, *edge, *cF; double* F; int* gB;
    cudaMalloc(&A, (size_t)nh * q2 * q2 * 16); cudaMalloc(&S, (size_t)nh * q2 * nb * 16);
    cudaMalloc(&w, (size_t)nh * nelem * q2 * R2 * 16); cudaMalloc(&edge, (size_t)nh * 7168 * R2 * 16);
    cudaMalloc(&F, (size_t)nelem * q2 * nF * R2 * 8); cudaMalloc(&cF, nh * nF * 16); cudaMalloc(&gB, nelem * nb * 4);
    cudaMemset(A, 0, (size_t)nh * q2 * q2 * 16); cudaMemset(S, 0, (size_t)nh * q2 * nb * 16);
    cudaMemset(F, 0, (size_t)nelem * q2 * nF * R2 * 8); cudaMemset(cF, 0, nh * nF * 16);
    cudaMemset(edge, 0, (size_t)nh * 7168 * R2 * 16); cudaMemset(w, 0, (size_t)nh * nelem * q2 * R2 * 16);
    std::vector<int> h(nelem * nb); for (int i = 0; i < nelem * nb; ++i) h[i] = (i * 7) % 7168;
    cudaMemcpy(gB, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CgemmArgs up{}; up.A = A; up.rows = q2; up.K = q2; up.nodes = nelem; up.F = F; up.cF = cF; up.nF = nF; up.q2 = q2; up.dst = w;
    CgemmArgs dn{}; dn.A = S; dn.rows = q2; dn.K = nb; dn.nodes = nelem; dn.src = edge; dn.src_ps = 7168; dn.bi0 = gB; dn.dst = w;
    int reps = 10;
    run<5, 8, 28, CG_LEAF_UP, 1, 1>(up, nh, reps);
    run<5, 8, 28, CG_LEAF_UP, 1, 2>(up, nh, reps);
    run<5, 8, 28, CG_LEAF_UP, 2, 1>(up, nh, reps);
    run<5, 4, 28, CG_LEAF_UP, 2, 1>(up, nh, reps);
    run<5, 4, 28, CG_LEAF_UP, 4, 1>(up, nh, reps);
    run<5, 8, 16, CG_LEAF_UP, 2, 1>(up, nh, reps);
    run<4, 8, 28, CG_LEAF_UP, 2, 1>(up, nh, reps);
    run<5, 8, 28, CG_LEAF_UP, 1, 3>(up, nh, reps);
    run<5, 8, 28, CG_LEAF_DOWN, 1, 1>(dn, nh, reps);
    run<5, 8, 16, CG_LEAF_DOWN, 1, 1>(dn, nh, reps);
    run<5, 8, 28, CG_LEAF_DOWN, 2, 1>(dn, nh, reps);
    run<5, 4, 28, CG_LEAF_DOWN, 2, 1>(dn, nh, reps);
    run<5, 8, 28, CG_LEAF_DOWN, 1, 2>(dn, nh, reps);
    run<2, 8, 28, CG_LEAF_DOWN, 2, 1>(dn, nh, reps);
    return 0;
}

// Fused multi-level merge sweeps of the shared (constant-coefficient) store
// (fused_tree.cu): one CTA carries a subtree of 2^nlev child boxes for one half
// pole and 8 right-hand-side columns through nlev consecutive merge levels with
// the boundary data h / u resident in shared memory, so a fused group reads its
// children's h (or its top box's boundary values) once and writes only the top
// level's h (and every level's w3 / interface values).  DESIGN.md §2 "Fused
// subtree sweeps".
#pragma once

#include <cuda_runtime.h>

namespace rexp {
namespace dev {

constexpr int FT_MAXLEV = 3;

struct FtLevel {
    const double2 *X, *Y, *S;        // operators of the launch's first half pole ([M+ | M-] when sym)
    long long ppX, ppY, ppS;         // per-pole strides (complex elements)
    int n3, next, nchild, nbx, xdir, sym, xdiag, nodes;
    const int *ia3p, *ib3p;          // [n3] interface positions in child a / child b
    const int *extc, *extp;          // [next] parent boundary row -> (child 0/1, position)
    const int *siA, *siB, *seA, *seB;   // symmetric pairs of the interface / boundary (sym)
    const double *sis, *ses;
    double2* w3;                     // [pc][nodes * n3][R2]
    const int *gext, *g3;            // [nodes][next], [nodes][n3] global edge ids (DOWN)
};

struct FtArgs {
    FtLevel lv[FT_MAXLEV];           // bottom-up
    int nlev, R2, RC, CS;            // RC columns per node and CS subtrees per CTA: RC * CS = 8
    int ncb;                         // column blocks per node (R2 / RC)
    const double2* hin;              // UP: child h of the lowest level [pc][hps][R2]
    double2* hout;                   // UP: h of the top level
    long long hps;
    double2* edge;                   // DOWN: [pc][NE][R2]
    long long NE;
    // shared-memory plan (bytes from the dynamic base), ft_plan
    int nslots, slot_bytes, off_ring, off_a, off_b, off_w, off_bp, off_bm, off_u, smem_bytes;
};

// fills the shared-memory plan for an UP (down = false) or DOWN group; returns
// false if the group does not fit (items per warp, shared memory)
bool ft_plan(FtArgs& a, bool down);
void ft_allow();
void ft_launch_up(const FtArgs& a, int top_nodes, int pc, cudaStream_t s);
void ft_launch_down(const FtArgs& a, int top_nodes, int pc, cudaStream_t s);

}  // namespace dev
}  // namespace rexp

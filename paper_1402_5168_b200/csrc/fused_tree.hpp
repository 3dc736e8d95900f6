// Fused multi-level merge sweeps of the shared (constant-coefficient) store
// (fused_tree.cu): one CTA carries a subtree of 2^nlev child boxes for one half
// pole and 8 right-hand-side columns through nlev consecutive merge levels with
// the boundary data h / u resident in shared memory, so a fused group reads its
// children's h (or its top box's boundary values) once and writes only the top
// level's h (and every level's w3 / interface values).  DESIGN.md §2 "Fused
// subtree sweeps".
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace rexp {
namespace dev {

constexpr int FT_MAXLEV = 3;

// host copies of a level's node-independent index tables (plan input)
struct FtHostLevel {
    std::vector<int> ia3p, ib3p, extc, extp;   // [n3], [n3], [next], [next]
    std::vector<int> iA, iB, eA, eB;           // symmetric pairs (sym levels)
    std::vector<double> is, es;
};

// one operator stage: its chunked, padded image (per pole: nchunks x [nh][bk][lda]
// complex, zero padding) is what the producer warp copies, one bulk copy per chunk
struct FtStageDesc {
    long long img_off;    // offset (complex elements) inside a pole's image
    int hr, hk, nh, lda, bk, nchunks;
};

struct FtLevel {
    const double2 *X, *Y, *S;        // operators of the launch's first half pole ([M+ | M-] when sym)
    long long ppX, ppY, ppS;         // per-pole strides (complex elements)
    int n3, next, nchild, nbx, xdir, sym, xdiag, nodes;
    double2* w3;                     // [pc][nodes * n3][R2]
    const int *gext, *g3;            // [nodes][next], [nodes][n3] global edge ids (DOWN)
    FtStageDesc st[3];               // X, Y, S
    // offsets into the group's int / double tables (see ft_plan)
    int t_xg, t_xrow, t_yrow, t_dg, t_drow, t_dch;
    int d_xs, d_xso, d_yso, d_ds, d_dso;
};

struct FtArgs {
    FtLevel lv[FT_MAXLEV];           // bottom-up
    int nlev, R2, RC, CS;            // RC columns per node and CS subtrees per CTA: RC * CS = 8
    int lgRC, ncb;                   // column blocks per node (R2 / RC)
    const double2* hin;              // UP: child h of the lowest level [pc][hps][R2]
    double2* hout;                   // UP: h of the top level
    long long hps;
    double2* edge;                   // DOWN: [pc][NE][R2]
    long long NE;
    const double2* img;              // packed operator images of the launch's first half pole
    long long img_ps;                // per-pole image size (complex elements)
    const int* itab;
    const double* dtab;
    int n_itab, n_dtab;
    // shared-memory plan (bytes from the dynamic base), ft_plan
    int nslots, slot_bytes, off_tab, off_ring, off_a, off_b, off_w, off_u, off_bx, off_by, bhalf, smem_bytes;
};

// fills the stage descriptors, index tables and shared-memory plan for an UP
// (down = false) or DOWN group; returns false if the group does not fit
bool ft_plan(FtArgs& a, const FtHostLevel* hl, bool down, std::vector<int>& itab, std::vector<double>& dtab);
void ft_allow();
// packs the operators of `npoles` half poles (a.lv[].X/Y/S, per-pole strides) into `img`
void ft_pack(const FtArgs& a, bool down, double2* img, int npoles, cudaStream_t s);
void ft_launch_up(const FtArgs& a, int top_nodes, int pc, cudaStream_t s);
void ft_launch_down(const FtArgs& a, int top_nodes, int pc, cudaStream_t s);

}  // namespace dev
}  // namespace rexp

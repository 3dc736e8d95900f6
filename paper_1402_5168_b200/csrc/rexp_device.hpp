// Device operator store and hot-path launcher (see device.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "fused_tree.hpp"
#include "rexp_internal.hpp"

namespace rexp {
namespace dev {

struct StageCfg {
    int kind = 0;   // 0: DMMA GEMM (k_cgemm), 1: GEMV (k_gemv), 2: symmetric-pair GEMV (k_gemv_sym)
    int MT = 4, WN = 8;
    int minb = 1;   // 4: register-capped variant (4 resident CTAs per SM)
    int rb = 64;    // GEMV row block (CS = 256 / rb column groups)
    int nb = 0;     // symmetric-pair GEMV: nodes per CTA (0 = as many as fit)
};

struct Level {
    int nodes = 0, n3 = 0, next = 0, nchild = 0, child_nodes = 0, nbx = 1, dir = 0;
    bool sym = false;   // stored as the symmetric half pair [M+ | M-] (k_gemv_sym, see sym_pairs)
    bool xdiag = false; // X diagonal in the edge basis: up-X as k_upx_diag
    int *siA = nullptr, *siB = nullptr, *seA = nullptr, *seB = nullptr;   // interface / boundary pairs
    double *sis = nullptr, *ses = nullptr;                                 // their signs
    std::vector<int> h_iA, h_iB, h_eA, h_eB;
    std::vector<double> h_is, h_es;
    // second reflection (across the interface: it swaps the two children and leaves the
    // interface fixed), R2 >= 16: only one boundary pair (A, B) of each reflection-2 orbit
    // is computed (Y rows) / multiplied (S columns); e2* are compact over those hx2 pairs
    bool sym2 = false;
    int hx2 = 0;
    int *e2A = nullptr, *e2B = nullptr, *e2pA = nullptr, *e2pB = nullptr;   // positions, partners (-1: none)
    double *e2s = nullptr, *e2sA = nullptr, *e2sB = nullptr;                 // reflection-1 sign, partner signs
    std::vector<int> h_e2A, h_e2B;
    std::vector<double> h_e2s;
    double2 *X = nullptr, *Y = nullptr, *S = nullptr;   // [nh][nodes_stored][...] col-major
    int *ia3 = nullptr, *ib3 = nullptr, *ext = nullptr, *gext = nullptr, *g3 = nullptr;
    int *ia3p = nullptr, *ib3p = nullptr, *extc = nullptr, *extp = nullptr;   // node-independent forms (fused sweeps)
    double2* w3 = nullptr;                              // [chunk][nodes][n3][R2]
    size_t ppX = 0, ppY = 0, ppS = 0;                   // per-pole operator sizes (complex)
};

struct SpecArgs;

class DeviceStore {
  public:
    ~DeviceStore();
    int init(const Problem& P, const Tree& T, const PoleTables& pt, int h0, int h1, bool shared, int nrhs);
    int upload_ops(const std::vector<HostLevelOps>& ops, int m0);
    void release();
    // one full step on a device state [nrhs][3][N] complex128 (CUDA graph replay
    // unless timing or REXP_GRAPH=0; step_eager launches the kernels directly)
    int step(double* d_state, cudaStream_t s);
    int step_eager(double* d_state, cudaStream_t s);
    bool use_graph = true;
    // all half poles of the handle, chunk by chunk: leaf solves, merge sweeps and
    // the weighted pole sums E (written to d_E_out)
    int solve_sum(const double* d_state, double* d_E_out, cudaStream_t s);
    int recover(const double* d_E_in, double* d_state, cudaStream_t s);
    int launches_per_step() const;

    // per-kernel-class CUDA-event timing on the launching stream
    enum { T_PRE = 0, T_LEAF_UP, T_LEAF_FLUX, T_MERGE_UP, T_ROOT, T_MERGE_DOWN, T_LEAF_DOWN, T_POLE_SUM, T_RECOVER, T_NCLASS };
    int timing_begin();
    int timing_end(double* ms, int32_t* launches);

    int model = 0, n = 0, p = 0, q = 0, q2 = 0, nb = 0, nelem = 0;
    long long N = 0, NI = 0, NV = 0, NE = 0;
    int h0 = 0, h1 = 0, nh = 0, nrhs = 1, R2 = 2, nF = 0, nE = 0, ns = 0;
    bool shared = true;
    bool fdm = false;          // tensor-product leaf inverse (constant coefficients)
    double c1 = 0.0;
    std::vector<double> scal;
    int64_t store_bytes = 0, work_bytes = 0;
    double* d_u = nullptr;     // device state buffer for host-pointer applies
    double* d_E = nullptr;     // pole sums [nE][R2][N]

  private:
    template <typename T>
    int alloc(T** p, size_t count);
    template <typename T>
    int put(T** p, const std::vector<T>& v);
    int check(const char* what);
    void configure_kernels();

    void tbeg(cudaStream_t s);
    void tend(int cls, cudaStream_t s);
    bool timing = false;
    struct TEntry { int cls; cudaEvent_t a, b; };
    std::vector<TEntry> tlog;
    std::vector<cudaEvent_t> tpool;
    size_t tpool_used = 0;
    cudaEvent_t tcur = nullptr;
    cudaEvent_t next_event();

    std::vector<void*> allocs;
    // pole lanes: per-lane work buffers, pole range and stream (see init)
    struct LaneBufs {
        double2* edge = nullptr;
        double2* h[2] = {nullptr, nullptr};
        std::vector<double2*> w3;
        int m0 = 0, m1 = 0;
        cudaStream_t stream = nullptr;
        cudaEvent_t done = nullptr;
    };
    std::vector<LaneBufs> lane_bufs;
    int nlanes = 1, cur_lane = 0;
    cudaEvent_t ev_fork = nullptr;
    void use_lane(int ln);
    int sym_pairs(const Tree& T, const MergeLevel& L, Level& D);
    int sym_pairs2(const Tree& T, const MergeLevel& L, Level& D);
    std::vector<double> mode_parity;   // +-1: parity of eigenvector k of K under i -> q-1-i
    cudaGraphExec_t graph_exec = nullptr;
    const double* graph_state = nullptr;
    cudaStream_t cap_stream = nullptr;
    void drop_graph();
    double *d_D = nullptr, *d_Dw = nullptr, *d_kappa = nullptr, *d_NI = nullptr, *d_F = nullptr;
    int *d_elem_g = nullptr, *d_leaf_gB = nullptr, *d_rpos1 = nullptr, *d_rpos2 = nullptr, *d_rgs = nullptr;
    double2 *d_cF = nullptr, *d_dE = nullptr, *d_Dinv = nullptr;
    double *d_V = nullptr, *d_Vinv = nullptr, *d_D2 = nullptr, *d_E01 = nullptr, *d_A01 = nullptr;
    double *d_G = nullptr, *d_Ehat = nullptr, *d_Eedge = nullptr, *d_Pi = nullptr;   // spectral RHS fields, pole-sum partials
    int* d_leaf_own = nullptr;                  // [nelem][4q] edge-node ownership for the pole sums
    double *d_Aup = nullptr, *d_Adn = nullptr;  // leaf GEMM coefficients (leaf_gemm.cuh), [2q][..]
    double* d_Aup2 = nullptr;                   // parity-split UP coefficients (k_leaf_gemm_up_eo)
    int* d_kmap = nullptr;
    bool lg_eo = false;
    double* d_Adn2 = nullptr;                   // parity-split DOWN coefficients (k_leaf_gemm_down_eo)
    int* d_rmap = nullptr;
    bool lg_dn_eo = false;
    int lg_dn_mth = 3, lg_dn_eo_pb = 4;
    int lg_KP = 44, lg_MT = 6;                  // their K padding (UP) / row tiles (DOWN)
    int lg_up_var = 0, lg_dn_var = 0;           // tile variants (leaf_gemm.cuh)
    int ngroups = 1;                            // K slices of the leaf DOWN GEMM = pole-sum partial slots per lane
    int chunk = 1;             // half poles per work-buffer chunk
    int num_sms = 148;
    size_t pp_Ainv = 0, pp_Sleaf = 0, pp_Xroot = 0;
    int tree_chunk(int m0, int pc, cudaStream_t s);
    int launch_stage(int kind, size_t li, const StageCfg& cfg, int m0, int pc, cudaStream_t s);
    public:
    int tune_stages(bool measure);   // heuristic defaults; measure = time the candidates (after upload)
    std::string stage_report() const;
    bool tuned = false;
    private:
    std::vector<StageCfg> t_upx, t_upy, t_down;
    // fused subtree sweeps (fused_tree.cu): groups of consecutive levels run by one kernel
    struct FtGroup { int l0 = 0, nlev = 0; FtArgs args; double2* img = nullptr; };
    std::vector<FtGroup> ft_up, ft_down;   // by lowest level, ascending
    std::string ft_times;                  // autotuner: fused vs single-level times
    int h_sel = -1;                        // h buffer holding the current children (-1: by level parity)
    int plan_fused(const Tree& T);
    int pack_fused();
    bool ft_packed = false;
    bool spec_batch = true;                // batched k_spec_pre_fused_b / k_spec_back_b (REXP_SPEC_BATCH=0: one (leaf, RHS) per CTA)
    const FtGroup* ft_group(const std::vector<FtGroup>& v, int l0) const;
    int launch_fused(const FtGroup& g, bool down, int m0, int pc, cudaStream_t s);
    StageCfg t_root;
    SpecArgs spec_args(int m0, int pc) const;
    int pole_sum_chunk(int m0, int pc, bool accumulate, double* d_E_out, cudaStream_t s);
    double2 *d_Ainv = nullptr, *d_Sleaf = nullptr, *d_Xroot = nullptr;
    double2 *d_w = nullptr, *d_edge = nullptr;
    double2* d_h[2] = {nullptr, nullptr};
    long long hstride = 0;
    std::vector<Level> levels;
};

}  // namespace dev
}  // namespace rexp

/*
 * rexp.h - C ABI of the B200 rational-exponential time stepper.
 *
 * Implements the apply phase of Haut, Babb, Martinsson, Wingate,
 * "A high-order scheme for solving wave propagation problems via the direct
 * construction of an approximate time-evolution operator":
 *
 *     u_{n+1} = exp(tau L) u_n  ~=  sum_m b_m (tau L - alpha_m)^{-1} u_n
 *
 * (Eq. "error in exp(t*L)"), with every
 * shifted resolvent applied through a precomputed hierarchical (nested
 * dissection / HPS) solver of the spectral-element collocation system
 * (§2.2-2.3) after the elliptic reformulations of
 * PAPER.md §2.1 (lines 266-396).
 *
 * Everything is plain C: host or device pointers and sizes; no torch types.
 * All functions return 0 on success and a negative REXP_E* code on failure;
 * rexp_last_error() then returns a thread-local human-readable message.
 * Nothing here falls back to a CPU implementation of the apply: if CUDA is
 * unavailable, rexp_setup() with device >= 0 fails with REXP_ENODEV.
 *
 * ----------------------------------------------------------------------------
 * Discretization and node ordering (§2.2, Fig. 1)
 * ----------------------------------------------------------------------------
 * Periodic unit square split into n x n equal elements (n a power of two,
 * n >= 2); each element carries a p x p Chebyshev-Lobatto grid
 * t_k = -cos(pi k/(p-1)), k = 0..p-1.  Let q = p - 2 and H = 1/n.  Element
 * (ex, ey), e = ey*n + ex, spans [ex H,(ex+1)H] x [ey H,(ey+1)H]; local node
 * (i, j) sits at (ex H + (t_i+1)H/2, ey H + (t_j+1)H/2).  Corner nodes are
 * not unknowns (no collocation or flux row references them).  The N global
 * nodes, N = n^2 (q^2 + 2q), are ordered
 *     interior   g = e*q^2 + (j-1)*q + (i-1)             i, j in 1..q
 *     vertical   g = NI + e*q + (j-1)        left edge x = ex*H of element e
 *     horizontal g = NI + NV + e*q + (i-1)   bottom edge y = ey*H of element e
 * with NI = n^2 q^2, NV = NH = n^2 q.
 *
 * State vectors are complex128 stored as interleaved (re, im) doubles, laid
 * out [nrhs][3][N]:
 *     model REXP_MODEL_RSW : fields (v1, v2, eta) of the linear rotating
 *         shallow-water system  v_t = -f J v + grad eta,  eta_t = div v
 *         (g = H = 1, J = [[0,1],[-1,0]]);
 *     model REXP_MODEL_WAVE: fields (w, z, v) = (u_x, u_y, u_t) of
 *         u_tt = kappa Lap u in first-order form.
 *
 * ----------------------------------------------------------------------------
 * Rational approximation (§3)
 * ----------------------------------------------------------------------------
 * rexp_setup builds R(iy) = sum_m b_m/(iy - alpha_m) with
 * |R(iy) - e^{iy}| <= delta on |y| <= tau*Lambda and |R(iy)| <= 1 + delta on
 * the real line (Eqs. "RM_prop1", "RM_prop2"), as the product S*R_gauss of
 * the §3.1/§3.2 Gaussian-sum + Table-1 approximant and the §3.3 filter
 * (readings R1-R6).  It fails with REXP_EACCURACY if dense sampling
 * finds either bound violated.  The pole set is conjugate-closed and, because
 * the operators are real, each conjugate pair is applied once to the real and
 * imaginary parts of the state; the "half poles" are the
 * poles with Im(alpha) >= 0.
 */
#ifndef REXP_H
#define REXP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REXP_MODEL_RSW 0
#define REXP_MODEL_WAVE 1

#define REXP_STORE_AUTO 0     /* shared for RSW (constant coefficients), per-node otherwise */
#define REXP_STORE_SHARED 1   /* one operator set per tree level (translation invariant)     */
#define REXP_STORE_PERNODE 2  /* one operator set per tree node                              */

#define REXP_OK 0
#define REXP_EINVAL -1        /* invalid argument                                  */
#define REXP_EACCURACY -2     /* rational approximation failed its delta checks    */
#define REXP_ENODEV -3        /* no CUDA device / CUDA error                       */
#define REXP_ENOMEM -4        /* allocation failed (host or device)                */
#define REXP_ESINGULAR -5     /* a factorization met a zero pivot                  */
#define REXP_ESTATE -6        /* handle not in a state that allows this call       */

typedef struct rexp_problem {
    int32_t model;        /* REXP_MODEL_RSW or REXP_MODEL_WAVE                         */
    int32_t n;            /* elements per direction: power of two, 2..1024             */
    int32_t p;            /* Chebyshev nodes per direction per element: 4..32          */
    double f;             /* Coriolis parameter f (RSW); ignored for WAVE              */
    const double* kappa;  /* WAVE: kappa > 0 at the N global nodes (HOST pointer, read
                             during rexp_setup only, not retained); NULL for RSW       */
} rexp_problem;

typedef struct rexp_options {
    int32_t nrhs;         /* independent complex states applied together: 1..64
                             (per-node store: 1..4)                                      */
    int32_t store;        /* REXP_STORE_*                                               */
    int32_t device;       /* CUDA ordinal for the operator store; -1 = host-only build
                             (operators kept on the host for rexp_export_*; rexp_apply
                             then returns REXP_ESTATE)                                  */
    int32_t half_begin;   /* half-pole range [half_begin, half_end) owned by this handle */
    int32_t half_end;     /* (pole-sharded multi-GPU); -1, -1 = all                      */
    int32_t nthreads;     /* host threads used by the factorization; 0 = all cores      */
} rexp_options;

typedef struct rexp_handle rexp_handle;

/* Fill *opt with defaults: nrhs 1, store AUTO, device 0, all half poles, all cores. */
void rexp_default_options(rexp_options* opt);

/*
 * setup(L, tau, delta, Lambda)  (§1.3 "build stage", lines 167-179).
 * Computes the poles/weights (alpha_m, b_m) for the interval |y| <= tau*Lambda,
 * factors every (tau L - alpha_m) (its elliptic reformulation, §2.1) into the
 * merge-tree solution operators on the host, and uploads them to the device
 * store.  Nothing here is part of the timed apply.  On success *out owns all
 * memory; release it with rexp_free.
 */
int rexp_setup(const rexp_problem* prob, double tau, double delta, double Lambda,
               const rexp_options* opt, rexp_handle** out);

/*
 * apply(u, nsteps): u <- (sum_m b_m (tau L - alpha_m)^{-1})^nsteps u, in place.
 * u: complex128 [nrhs][3][N] interleaved.  If u_on_device != 0, u is a device
 * pointer on the handle's device and the call is asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  Otherwise u is a host
 * pointer; the call copies it to the device, steps, copies back and
 * synchronizes `stream` before returning.  Requires a handle that owns all
 * half poles (single-GPU).  Each step is replayed from a CUDA graph captured
 * on first use for this state pointer (recaptured when the pointer changes;
 * the capture uses a private stream, replay runs on `stream`); the pole lanes
 * of the spectral path fork from and join back to `stream` inside the step.
 * Environment REXP_GRAPH=0 launches the kernels directly.
 */
int rexp_apply(rexp_handle* h, double* u, int32_t nsteps, int32_t u_on_device, void* stream);

/* Release everything owned by the handle (safe on NULL). */
void rexp_free(rexp_handle* h);

/* Message describing the last error on this thread ("" if none). */
const char* rexp_last_error(void);

/* ---- pole-sharded step (multi-GPU: partial pole sums + all-reduce + finish) ----
 * rexp_step_partial writes this handle's share of the pole sums E into e_dev
 * (doubles, length rexp_partial_len); the caller sums e_dev over ranks (e.g.
 * NCCL all-reduce) and calls rexp_step_finish, which recovers the new state
 * from the summed E and the old state.  Both asynchronous on `stream`;
 * u_dev is a device pointer [nrhs][3][N] complex128. */
int64_t rexp_partial_len(const rexp_handle* h);
int rexp_step_partial(rexp_handle* h, const double* u_dev, double* e_dev, void* stream);
int rexp_step_finish(rexp_handle* h, const double* e_dev, double* u_dev, void* stream);

/* ---- queries ---- */
int64_t rexp_num_nodes(const rexp_handle* h);          /* N                              */
int32_t rexp_num_poles(const rexp_handle* h);          /* all poles (2M+1 in the paper)  */
int32_t rexp_num_half_poles(const rexp_handle* h);     /* poles with Im(alpha) >= 0      */
/* alpha, b: complex128 interleaved, length rexp_num_poles (host pointers). */
int rexp_get_poles(const rexp_handle* h, double* alpha, double* b);
/* measured sup |R(iy) - e^{iy}| on |y| <= tau*Lambda and sup |R(iy)| on the sample set */
int rexp_get_accuracy(const rexp_handle* h, double* err, double* maxmod);
/* node coordinates x[N], y[N] (host pointers) in the ordering above */
int rexp_node_coords(const rexp_handle* h, double* x, double* y);
/* the same without a handle (e.g. to sample kappa before rexp_setup) */
int64_t rexp_mesh_num_nodes(int32_t n, int32_t p);
int rexp_mesh_coords(int32_t n, int32_t p, double* x, double* y);
/* bytes of the device operator store / of the per-step work buffers */
int64_t rexp_store_bytes(const rexp_handle* h);
int64_t rexp_work_bytes(const rexp_handle* h);
/* number of kernel launches one step issues (for the bench's gpu_launches) */
int32_t rexp_launches_per_step(const rexp_handle* h);
/* leaf solver of the device store: 0 = dense q^2 x q^2 leaf operators,
 * 1 = spectral (tensor-product) leaf path of the constant-coefficient store:
 * leaf solves and interior pole sums in the eigenbasis of D2[1..q][1..q],
 * edge data in the spectral edge basis, symmetric-pair merge levels and the
 * Fourier root; -1 = no device store */
int32_t rexp_leaf_solver(const rexp_handle* h);
/* kernel chosen for every merge stage (X, Y, down per level) and the closure
 * by the setup-time autotuner, as text (for reports): gemmMxN (DMMA GEMM; r =
 * register-capped, s3 = 3-stage cp.async, k16 = BK 16), gemvRB, symRB[nNB] /
 * symgemmMxN (symmetric-pair forms), diag (diagonal first-level up-X),
 * root[fourier] */
int rexp_stage_report(const rexp_handle* h, char* buf, int32_t len);

/* ---- per-kernel timing (bench) ----
 * Between rexp_timing_begin and rexp_timing_end every kernel launch of the
 * handle is bracketed by CUDA events on its launching stream; timing_end
 * synchronizes on the last event and returns, per kernel class
 *   0 pre, 1 leaf_up, 2 leaf_flux, 3 merge_up, 4 root, 5 merge_down,
 *   6 leaf_down, 7 pole_sum, 8 recover,
 * the summed device milliseconds ms[9] and launch counts launches[9]. */
int rexp_timing_begin(rexp_handle* h);
int rexp_timing_end(rexp_handle* h, double* ms, int32_t* launches);

/* ---- test hooks (setup verification on the host; not part of the apply) ----
 * Describe / export the operator store of a HOST-ONLY handle (device = -1):
 * levels 0 = leaves, 1..L = merge levels (bottom-up), L+1 = periodic root.
 * info = {nodes, nodes_stored, n3|q^2|ns, next|4q|4nq, nchild, dir, half_begin, half_end}.
 * which (leaves) 0 = A_II^{-1}, 1 = S_leaf; (merges) 0 = -X, 1 = Y, 2 = S;
 * (root) 0 = -(P^T T P)^{-1}.  Matrices are column-major complex128.
 * Index lists: (leaves) 3 = leaf boundary edge indices, 4 = element-local map;
 * (merges) 0 = ia3, 1 = ib3, 2 = ext, 3 = gext, 4 = g3; (root) 0 = pos1, 1 = pos2, 2 = seam edges. */
int32_t rexp_export_num_levels(const rexp_handle* h);
int rexp_export_level_info(const rexp_handle* h, int32_t lev, int64_t info[8]);
int rexp_export_matrix(const rexp_handle* h, int32_t half_index, int32_t lev, int32_t node,
                       int32_t which, double* out);
int rexp_export_index(const rexp_handle* h, int32_t lev, int32_t which, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* REXP_H */

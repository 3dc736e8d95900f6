// C ABI of include/rexp.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "rexp_device.hpp"
#include "rexp_internal.hpp"

namespace rexp {
namespace {
// one message per calling thread (include/rexp.h: "thread-local")
thread_local std::string t_err;
}  // namespace
void set_error(const std::string& msg) { t_err = msg; }
}  // namespace rexp

struct rexp_handle {
    rexp::Problem P;
    rexp::Tree T;
    rexp::RationalApprox ra;
    rexp::PoleTables pt;
    int h0 = 0, h1 = 0;
    bool shared = true;
    int nrhs = 1;
    int device = -1;
    std::vector<rexp::HostLevelOps> host_ops;   // kept only for host-only handles
    std::unique_ptr<rexp::dev::DeviceStore> dev;
};

using namespace rexp;

extern "C" {

const char* rexp_last_error(void) { return t_err.c_str(); }

void rexp_default_options(rexp_options* opt) {
    if (!opt) return;
    opt->nrhs = 1;
    opt->store = REXP_STORE_AUTO;
    opt->device = 0;
    opt->half_begin = -1;
    opt->half_end = -1;
    opt->nthreads = 0;
}

int rexp_setup(const rexp_problem* prob, double tau, double delta, double Lambda, const rexp_options* opt_in,
               rexp_handle** out) {
    if (!prob || !out) {
        set_error("rexp_setup: null argument");
        return REXP_EINVAL;
    }
    *out = nullptr;
    rexp_options opt;
    rexp_default_options(&opt);
    if (opt_in) opt = *opt_in;
    if (prob->model != REXP_MODEL_RSW && prob->model != REXP_MODEL_WAVE) {
        set_error("rexp_setup: unknown model");
        return REXP_EINVAL;
    }
    if (!(tau > 0.0) || !(Lambda > 0.0) || !(delta > 0.0)) {
        set_error("rexp_setup: tau, Lambda, delta must be positive");
        return REXP_EINVAL;
    }
    if (opt.nrhs < 1 || opt.nrhs > 64) {
        set_error("rexp_setup: nrhs must be in 1..64");
        return REXP_EINVAL;
    }
    if (prob->p > 18) {
        set_error("rexp_setup: this build supports p <= 18 ((p-2)^2 <= 256 rows per leaf CTA)");
        return REXP_EINVAL;
    }
    std::unique_ptr<rexp_handle> h(new rexp_handle());
    h->P.model = prob->model;
    h->P.n = prob->n;
    h->P.p = prob->p;
    h->P.f = prob->f;
    h->P.tau = tau;
    h->P.delta = delta;
    h->P.Lambda = Lambda;
    int rc = build_tree(prob->n, prob->p, h->T);
    if (rc) return rc;
    if (prob->model == REXP_MODEL_WAVE) {
        if (!prob->kappa) {
            set_error("rexp_setup: WAVE needs kappa");
            return REXP_EINVAL;
        }
        h->P.kappa.assign(prob->kappa, prob->kappa + h->T.N);
        for (double k : h->P.kappa)
            if (!(k > 0.0)) {
                set_error("rexp_setup: kappa must be positive");
                return REXP_EINVAL;
            }
    }
    if ((rc = build_exp_approx(tau * Lambda, delta, h->ra))) return rc;
    build_pole_tables(h->P, h->ra, h->pt);
    const int nh = static_cast<int>(h->pt.alpha.size());
    h->h0 = opt.half_begin < 0 ? 0 : opt.half_begin;
    h->h1 = opt.half_end < 0 ? nh : opt.half_end;
    if (h->h0 < 0 || h->h1 > nh || h->h0 >= h->h1) {
        set_error("rexp_setup: invalid half-pole range");
        return REXP_EINVAL;
    }
    int store = opt.store;
    if (store == REXP_STORE_AUTO) store = prob->model == REXP_MODEL_RSW ? REXP_STORE_SHARED : REXP_STORE_PERNODE;
    if (store == REXP_STORE_SHARED && prob->model == REXP_MODEL_WAVE) {
        set_error("rexp_setup: the shared store needs constant coefficients (RSW)");
        return REXP_EINVAL;
    }
    h->shared = store == REXP_STORE_SHARED;
    h->nrhs = opt.nrhs;
    h->device = opt.device;
    if (!h->shared && opt.nrhs != 1 && opt.nrhs != 2 && opt.nrhs != 4) {
        set_error("rexp_setup: the per-node store supports nrhs = 1, 2 or 4");
        return REXP_EINVAL;
    }
    if (opt.device < 0) {
        std::vector<HostLevelOps> ops;
        if ((rc = factor_host(h->P, h->T, h->pt, h->h0, h->h1, h->shared, opt.nthreads, ops))) return rc;
        h->host_ops = std::move(ops);
    } else {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= opt.device) {
            cudaGetLastError();
            set_error("rexp_setup: no CUDA device " + std::to_string(opt.device));
            return REXP_ENODEV;
        }
        if (cudaSetDevice(opt.device) != cudaSuccess) {
            set_error("rexp_setup: cudaSetDevice failed");
            return REXP_ENODEV;
        }
        h->dev.reset(new dev::DeviceStore());
        if ((rc = h->dev->init(h->P, h->T, h->pt, h->h0, h->h1, h->shared, h->nrhs))) return rc;
        // factor on the host and upload in pole chunks of <= ~8 GB of operators
        const int64_t nhl = h->h1 - h->h0;
        const int64_t per_pole = std::max<int64_t>(1, h->dev->store_bytes / std::max<int64_t>(1, nhl));
        const int64_t cmax = std::max<int64_t>(1, (int64_t(8) << 30) / per_pole);
        for (int c0 = h->h0; c0 < h->h1; c0 += static_cast<int>(cmax)) {
            const int c1 = static_cast<int>(std::min<int64_t>(h->h1, c0 + cmax));
            std::vector<HostLevelOps> ops;
            if ((rc = factor_host(h->P, h->T, h->pt, c0, c1, h->shared, opt.nthreads, ops, h->shared,
                                  h->dev->fdm)))
                return rc;
            if ((rc = h->dev->upload_ops(ops, c0 - h->h0))) return rc;
        }
        if ((rc = h->dev->tune_stages(true))) return rc;
    }
    *out = h.release();
    return REXP_OK;
}

void rexp_free(rexp_handle* h) {
    if (!h) return;
    if (h->dev) {
        cudaSetDevice(h->device);
        h->dev.reset();
    }
    delete h;
}

static int need_device(rexp_handle* h, bool all_poles) {
    if (!h || !h->dev) {
        set_error("handle has no device store (host-only setup?)");
        return REXP_ESTATE;
    }
    if (all_poles && (h->h0 != 0 || h->h1 != static_cast<int>(h->pt.alpha.size()))) {
        set_error("rexp_apply needs a handle that owns all half poles; use step_partial/finish");
        return REXP_ESTATE;
    }
    if (cudaSetDevice(h->device) != cudaSuccess) {
        set_error("cudaSetDevice failed");
        return REXP_ENODEV;
    }
    return REXP_OK;
}

int rexp_apply(rexp_handle* h, double* u, int32_t nsteps, int32_t u_on_device, void* stream) {
    int rc = need_device(h, true);
    if (rc) return rc;
    if (!u || nsteps < 0) {
        set_error("rexp_apply: bad arguments");
        return REXP_EINVAL;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = static_cast<size_t>(h->nrhs) * 3 * h->T.N * 2 * sizeof(double);
    double* du = u;
    if (!u_on_device) {
        du = h->dev->d_u;
        if (cudaMemcpyAsync(du, u, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            set_error("rexp_apply: H2D copy failed");
            return REXP_ENODEV;
        }
    }
    for (int k = 0; k < nsteps; ++k)
        if ((rc = h->dev->step(du, s))) return rc;
    if (!u_on_device) {
        if (cudaMemcpyAsync(u, du, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            set_error("rexp_apply: D2H copy failed");
            return REXP_ENODEV;
        }
    }
    return REXP_OK;
}

int64_t rexp_partial_len(const rexp_handle* h) {
    if (!h) return -1;
    return static_cast<int64_t>(h->pt.nE) * 2 * h->nrhs * h->T.N;
}

int rexp_step_partial(rexp_handle* h, const double* u_dev, double* e_dev, void* stream) {
    int rc = need_device(h, false);
    if (rc) return rc;
    if (!u_dev || !e_dev) {
        set_error("rexp_step_partial: null state or pole-sum pointer");
        return REXP_EINVAL;
    }
    return h->dev->solve_sum(u_dev, e_dev, static_cast<cudaStream_t>(stream));
}

int rexp_step_finish(rexp_handle* h, const double* e_dev, double* u_dev, void* stream) {
    int rc = need_device(h, false);
    if (rc) return rc;
    if (!u_dev || !e_dev) {
        set_error("rexp_step_finish: null state or pole-sum pointer");
        return REXP_EINVAL;
    }
    return h->dev->recover(e_dev, u_dev, static_cast<cudaStream_t>(stream));
}

int64_t rexp_num_nodes(const rexp_handle* h) { return h ? h->T.N : -1; }

int64_t rexp_mesh_num_nodes(int32_t n, int32_t p) {
    if (n < 2 || p < 4) return -1;
    const int64_t q = p - 2;
    return static_cast<int64_t>(n) * n * (q * q + 2 * q);
}

int rexp_mesh_coords(int32_t n, int32_t p, double* x, double* y) {
    if (!x || !y) return REXP_EINVAL;
    Tree T;
    const int rc = build_tree(n, p, T);
    if (rc) return rc;
    std::memcpy(x, T.x.data(), T.x.size() * sizeof(double));
    std::memcpy(y, T.y.data(), T.y.size() * sizeof(double));
    return REXP_OK;
}
int32_t rexp_num_poles(const rexp_handle* h) { return h ? static_cast<int32_t>(h->ra.poles.size()) : -1; }
int32_t rexp_num_half_poles(const rexp_handle* h) { return h ? static_cast<int32_t>(h->pt.alpha.size()) : -1; }

int rexp_get_poles(const rexp_handle* h, double* alpha, double* b) {
    if (!h || !alpha || !b) return REXP_EINVAL;
    for (size_t k = 0; k < h->ra.poles.size(); ++k) {
        alpha[2 * k] = h->ra.poles[k].real();
        alpha[2 * k + 1] = h->ra.poles[k].imag();
        b[2 * k] = h->ra.res[k].real();
        b[2 * k + 1] = h->ra.res[k].imag();
    }
    return REXP_OK;
}

int rexp_get_accuracy(const rexp_handle* h, double* err, double* maxmod) {
    if (!h) return REXP_EINVAL;
    if (err) *err = h->ra.err;
    if (maxmod) *maxmod = h->ra.maxmod;
    return REXP_OK;
}

int rexp_node_coords(const rexp_handle* h, double* x, double* y) {
    if (!h || !x || !y) return REXP_EINVAL;
    std::memcpy(x, h->T.x.data(), h->T.x.size() * sizeof(double));
    std::memcpy(y, h->T.y.data(), h->T.y.size() * sizeof(double));
    return REXP_OK;
}

int64_t rexp_store_bytes(const rexp_handle* h) {
    if (!h) return -1;
    if (h->dev) return h->dev->store_bytes;
    int64_t b = 0;
    for (auto& L : h->host_ops)
        for (int k = 0; k < 3; ++k) b += static_cast<int64_t>(L.m[k].size()) * 16;
    return b;
}
int64_t rexp_work_bytes(const rexp_handle* h) { return (h && h->dev) ? h->dev->work_bytes : 0; }
int32_t rexp_launches_per_step(const rexp_handle* h) {
    if (!h) return -1;
    if (h->dev) return h->dev->launches_per_step();
    return 6 + 3 * static_cast<int32_t>(h->T.levels.size());
}


int rexp_stage_report(const rexp_handle* h, char* buf, int32_t len) {
    if (!h || !h->dev || !buf || len <= 0) return REXP_EINVAL;
    const std::string s = h->dev->stage_report();
    std::strncpy(buf, s.c_str(), static_cast<size_t>(len) - 1);
    buf[len - 1] = 0;
    return REXP_OK;
}

int32_t rexp_leaf_solver(const rexp_handle* h) {
    if (!h || !h->dev) return -1;
    return h->dev->fdm ? 1 : 0;
}

int rexp_timing_begin(rexp_handle* h) {
    int rc = need_device(h, false);
    if (rc) return rc;
    return h->dev->timing_begin();
}

int rexp_timing_end(rexp_handle* h, double* ms, int32_t* launches) {
    int rc = need_device(h, false);
    if (rc) return rc;
    return h->dev->timing_end(ms, launches);
}

int32_t rexp_export_num_levels(const rexp_handle* h) {
    return h ? static_cast<int32_t>(h->T.levels.size()) + 2 : -1;
}

int rexp_export_level_info(const rexp_handle* h, int32_t lev, int64_t info[8]) {
    if (!h || !info) return REXP_EINVAL;
    const int L = static_cast<int>(h->T.levels.size());
    if (lev < 0 || lev > L + 1) return REXP_EINVAL;
    for (int k = 0; k < 8; ++k) info[k] = 0;
    const int q = h->T.q;
    if (lev == 0) {
        info[0] = h->T.nelem;
        info[1] = h->shared ? 1 : h->T.nelem;
        info[2] = q * q;
        info[3] = 4 * q;
    } else if (lev <= L) {
        const MergeLevel& M = h->T.levels[lev - 1];
        info[0] = M.nodes;
        info[1] = h->shared ? 1 : M.nodes;
        info[2] = M.n3;
        info[3] = M.next;
        info[4] = M.nchild;
        info[5] = M.dir;
    } else {
        info[0] = 1;
        info[1] = 1;
        info[2] = h->T.ns;
        info[3] = 4 * h->T.n * q;
    }
    info[6] = h->h0;
    info[7] = h->h1;
    return REXP_OK;
}

int rexp_export_matrix(const rexp_handle* h, int32_t half_index, int32_t lev, int32_t node, int32_t which,
                       double* out) {
    if (!h || !out || h->host_ops.empty()) {
        set_error("rexp_export_matrix needs a host-only handle");
        return REXP_ESTATE;
    }
    if (lev < 0 || lev >= static_cast<int>(h->host_ops.size())) return REXP_EINVAL;
    const HostLevelOps& L = h->host_ops[lev];
    if (which < 0 || which >= L.nmat || node < 0 || node >= L.nodes_stored) return REXP_EINVAL;
    const int slot = half_index - h->h0;
    if (slot < 0 || slot >= h->h1 - h->h0) return REXP_EINVAL;
    const size_t sz = static_cast<size_t>(L.rows[which]) * L.cols[which];
    const cd* src = L.m[which].data() + (static_cast<size_t>(slot) * L.nodes_stored + node) * sz;
    std::memcpy(out, src, sz * sizeof(cd));
    return REXP_OK;
}

int rexp_export_index(const rexp_handle* h, int32_t lev, int32_t which, int32_t* out) {
    if (!h || !out) return REXP_EINVAL;
    const int L = static_cast<int>(h->T.levels.size());
    const std::vector<int32_t>* v = nullptr;
    if (lev == 0) {
        if (which == 3) v = &h->T.leaf_gB;
        else if (which == 4) v = &h->T.elem_g;
    } else if (lev >= 1 && lev <= L) {
        const MergeLevel& M = h->T.levels[lev - 1];
        const std::vector<int32_t>* opts[5] = {&M.ia3, &M.ib3, &M.ext, &M.gext, &M.g3};
        if (which >= 0 && which < 5) v = opts[which];
    } else if (lev == L + 1) {
        const std::vector<int32_t>* opts[3] = {&h->T.root_pos1, &h->T.root_pos2, &h->T.root_gs};
        if (which >= 0 && which < 3) v = opts[which];
    }
    if (!v) return REXP_EINVAL;
    std::memcpy(out, v->data(), v->size() * sizeof(int32_t));
    return REXP_OK;
}

}  // extern "C"

"""Which side limits the full-step parity at config-1 size?  (GPU + oracle)

For a few large-weight half poles of config 1: the GPU path's single-pole pole sums
E_1 = w Re(b eta) (rexp_step_partial on a one-pole handle) against the oracle's eta
as it stands (one sparse-LU solve) and against the same solve after one step of
iterative refinement with a long-double residual.  tools/g_pole_err.sh runs it.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.models import RSW  # noqa: E402
from oracle.rational import build_exp_approx  # noqa: E402
from oracle.specelem import Mesh  # noqa: E402
from paper_1402_5168_b200 import api  # noqa: E402
from workloads import CONFIGS, rsw_initial_state  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1_rsw_16x16_p16"]
tau, f = cfg["tau"], cfg["f"]
Lam = cfg["Lambda_tau"] / tau
m = Mesh(cfg["n"], cfg["p"])
model = RSW(m, f)
ap = build_exp_approx(cfg["Lambda_tau"], cfg["delta"], verify=False)
halfs = [(a, b) for a, b in zip(ap["poles"], ap["res"]) if a.imag >= 0]
mags = np.array([abs(b) for _, b in halfs])
order = np.argsort(-mags)
u0 = rsw_initial_state(m.x, m.y, cfg["seed"])
ur = u0.real.astype(complex)
ld = np.longdouble


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for k in [int(order[0]), int(order[7]), int(order[40])]:
    alpha, b = halfs[k]
    w = 2.0 if alpha.imag > 0 else 1.0
    beta = alpha / tau
    k2 = beta * beta + f * f
    lu = model.factor(beta)
    r = model.resolvent(alpha, tau, ur, lu=lu)
    eta = r[2] * tau                                  # the elliptic solve's output (reading R9)
    B = m.collocation_matrix(np.full(m.NI, k2, dtype=complex)).tocsr()
    # the right-hand side RSW.resolvent solved for, rebuilt from its own formulas
    v01, v02, eta0 = ur
    a1 = (beta * v01 - f * v02) / k2
    a2 = (beta * v02 + f * v01) / k2
    F = np.zeros(m.N, dtype=complex)
    F[: m.NI] = ((k2 / beta) * (eta0 + model.Gx @ a1 + model.Gy @ a2))[: m.NI]
    x = lu.solve(F)
    dr, di = B.data.real.astype(ld), B.data.imag.astype(ld)
    for it in range(2):
        xr, xi = x.real.astype(ld)[B.indices], x.imag.astype(ld)[B.indices]
        pr = np.add.reduceat(dr * xr - di * xi, B.indptr[:-1])
        pi = np.add.reduceat(dr * xi + di * xr, B.indptr[:-1])
        res = (F.real.astype(ld) - pr).astype(float) + 1j * (F.imag.astype(ld) - pi).astype(float)
        x = x + lu.solve(res)
    hk = api.setup("rsw", cfg["n"], cfg["p"], tau, cfg["delta"], Lam, f=f, half_range=(k, k + 1))
    u = torch.from_numpy(u0.copy()).reshape(1, 3, -1).cuda()
    e = torch.zeros(hk.partial_len, dtype=torch.float64, device="cuda")
    api.step_partial(hk, u, e)
    torch.cuda.synchronize()
    E = e.cpu().numpy().reshape(3, 2, -1)
    hk.close()
    bt = b / tau
    ref_plain = w * (bt * eta).real
    ref_refined = w * (bt * x).real
    print(f"half pole {k} alpha {alpha:.3f} |b| {abs(b):.2e}: oracle eta vs rebuilt solve {rel(lu.solve(F), eta):.1e}; "
          f"GPU vs oracle {rel(E[0][0], ref_plain):.2e}; GPU vs refined oracle {rel(E[0][0], ref_refined):.2e}; "
          f"oracle vs refined {rel(ref_plain, ref_refined):.2e}", flush=True)

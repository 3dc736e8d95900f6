"""How accurate is the oracle's own sparse-LU solve at config-1 size?  (oracle/ only, CPU)

For sampled poles of config 1: x = lu.solve(F) (what oracle.models.RSW.resolvent uses),
one step of iterative refinement with the residual r = F - B x accumulated in long
double, and the size of the correction relative to x.  The weighted corrections
b_m dx_m of the sampled poles, relative to the step's output norm, say how much of
the 1e-10 parity budget the oracle's own rounding can use up.
    python tools/oracle_refine_check.py [npoles]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.evolve import EvolutionOperator  # noqa: E402
from oracle.models import RSW  # noqa: E402
from oracle.specelem import Mesh  # noqa: E402
from workloads import CONFIGS, initial_state  # noqa: E402

cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c1_rsw_16x16_p16"]
npick = int(sys.argv[1]) if len(sys.argv) > 1 else 12
m = Mesh(cfg["n"], cfg["p"])
model = RSW(m, cfg["f"])
op = EvolutionOperator(model, cfg["tau"], cfg["Lambda_tau"] / cfg["tau"], cfg["delta"])
u0 = initial_state("rsw", m.x, m.y, cfg["seed"])
order = np.argsort(-np.abs(op.res))
picks = sorted(set(list(order[: npick // 2]) + list(order[:: max(1, len(order) // (npick // 2))][: npick // 2])))
print(f"{len(op.poles)} poles, sum|b| = {np.abs(op.res).sum():.3e}, max|b| = {np.abs(op.res).max():.3e}")
tot_dx = 0.0
for k in picks:
    alpha = op.poles[k]
    beta = alpha / cfg["tau"]
    k2 = beta * beta + cfg["f"] ** 2
    B = m.collocation_matrix(np.full(m.NI, k2, dtype=complex)).tocsr()
    lu = model.factor(beta)
    x_full = model.resolvent(alpha, cfg["tau"], u0, lu=lu)
    # the elliptic right-hand side as RSW.resolvent forms it: recover F from B and the solution
    eta = x_full[2] * cfg["tau"]
    F = B @ eta
    x = lu.solve(F)
    # residual in long double: CSR products and row sums done by hand (scipy has no long double kernels)
    ld = np.longdouble
    dr, di = B.data.real.astype(ld), B.data.imag.astype(ld)
    xr, xi = x.real.astype(ld)[B.indices], x.imag.astype(ld)[B.indices]
    pr = np.add.reduceat(dr * xr - di * xi, B.indptr[:-1])
    pi = np.add.reduceat(dr * xi + di * xr, B.indptr[:-1])
    r = (F.real.astype(ld) - pr).astype(float) + 1j * (F.imag.astype(ld) - pi).astype(float)
    dx = lu.solve(r)
    rel = np.linalg.norm(dx) / np.linalg.norm(x)
    w = abs(op.res[k]) * np.linalg.norm(dx) / cfg["tau"]
    tot_dx += w
    print(f"pole {k:4d} alpha {alpha:.3f} |b| {abs(op.res[k]):.2e}  |dx|/|x| {rel:.2e}  |b dx|/|u0| "
          f"{w / np.linalg.norm(u0[2]):.2e}", flush=True)
print(f"sum over {len(picks)} sampled poles of |b dx| / |u0| = {tot_dx / np.linalg.norm(u0[2]):.2e}")

"""Brute-force matrix exponential on tiny grids (BASELINE.json north_star pin).

On a 2 x 2 element mesh with p = 6 (96 nodes per field, 288 unknowns) every
resolvent the oracle applies is formed as a dense matrix (the oracle applied
to unit vectors).  The discrete resolvents R_a = (tau L_h - a)^{-1} of the
elliptic reformulation (§2.1) are projected: edge-node values of the
elliptic right-hand side never enter the interior collocation system
(PAPER.md:416-445), so R_a has a null space and L_h is only defined on its
range.  There R_a is diagonalised, R_a = V diag(mu) V^-1, and the eigenvalues
of tau L_h are lambda = a + 1/mu (mu != 0).  The brute-force evolution is
V diag(e^lambda) V^-1 (range only) and the oracle's step
sum_m b_m R_m u must reproduce it to within the rational
approximation error delta times the eigenvector
conditioning, for tau Lambda covering the whole discrete spectrum.

* Wave: the resolvents of all poles are resolvents of ONE
  operator (resolvent identity R_a - R_b = (a - b) R_a R_b to rounding), and
  the step equals the brute-force exponential to ~1e-9.
* RSW: the reformulation uses div(A grad eta) = beta Lap eta
  / (beta^2 + f^2), exact in the continuum; discretely the collocation
  Laplacian is not div_h grad_h, so the resolvents agree with one operator
  approximately (the identity's defect is ~1e-3 on these grids, carried by
  the unresolved top of the discrete spectrum - reading R14).  The step is checked against
  the brute-force exponential of L_h recovered from one pole to that level.
"""
import numpy as np
import pytest

from oracle.evolve import EvolutionOperator
from oracle.models import RSW, Wave
from oracle.specelem import Mesh
from workloads import rsw_initial_state, wave_initial_state, wave_speed_field

TAU = 0.05


def _resolvent_matrix(model, alpha, tau):
    n3 = 3 * model.mesh.N
    lu = model.factor(alpha / tau)
    R = np.zeros((n3, n3), complex)
    for j in range(n3):
        e = np.zeros(n3, complex)
        e[j] = 1.0
        R[:, j] = model.resolvent(alpha, tau, e.reshape(3, -1), lu=lu).reshape(-1)
    return R


def _setup(name, p):
    m = Mesh(2, p)
    if name == "rsw":
        return m, RSW(m, 1.0), rsw_initial_state(m.x, m.y, 3)
    return m, Wave(m, wave_speed_field(m.x, m.y, 3)), wave_initial_state(m.x, m.y, 3)


@pytest.mark.parametrize("name,p,ident_tol,step_tol", [("wave", 6, 1e-12, 1e-8), ("rsw", 6, 5e-3, 2e-3),
                                                       ("rsw", 8, 1e-2, 2e-3)])
def test_step_equals_bruteforce_expm(name, p, ident_tol, step_tol):
    m, model, u0 = _setup(name, p)
    a1, a2 = 1.3 + 0.7j, -0.4 + 2.1j
    R1 = _resolvent_matrix(model, a1, TAU)
    R2 = _resolvent_matrix(model, a2, TAU)
    lhs = R1 - R2
    defect = np.abs(lhs - (a1 - a2) * R1 @ R2).max() / np.abs(lhs).max()
    assert defect <= ident_tol, defect
    mu, V = np.linalg.eig(R1)
    nz = np.abs(mu) > 1e-9 * np.abs(mu).max()
    lam = a1 + 1.0 / mu[nz]
    # skew-Hermitian up to discretization: a purely imaginary spectrum
    assert np.abs(lam.real).max() <= 1e-2 * np.abs(lam.imag).max()
    Lam = 1.02 * np.abs(lam.imag).max() / TAU
    op = EvolutionOperator(model, TAU, Lam, 1e-10)
    got = op.step(u0).reshape(-1)
    c = np.linalg.solve(V, u0.reshape(-1))
    ref = V[:, nz] @ (np.exp(lam) * c[nz])
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(f"{name} p={p}: resolvent-identity defect {defect:.1e}, step vs brute-force expm {err:.1e}")
    assert err <= step_tol


def test_bruteforce_catches_a_wrong_weight():
    """The pin is sharp: one pole weight off by 1e-6 (relative) breaks it."""
    m, model, u0 = _setup("wave", 6)
    a1 = 1.3 + 0.7j
    R1 = _resolvent_matrix(model, a1, TAU)
    mu, V = np.linalg.eig(R1)
    nz = np.abs(mu) > 1e-9 * np.abs(mu).max()
    lam = a1 + 1.0 / mu[nz]
    Lam = 1.02 * np.abs(lam.imag).max() / TAU
    op = EvolutionOperator(model, TAU, Lam, 1e-10)
    k = int(np.argmax(np.abs(op.res)))
    op.res = op.res.copy()
    op.res[k] *= 1 + 1e-6
    c = np.linalg.solve(V, u0.reshape(-1))
    ref = V[:, nz] @ (np.exp(lam) * c[nz])
    err = np.linalg.norm(op.step(u0).reshape(-1) - ref) / np.linalg.norm(ref)
    assert err > 1e-8

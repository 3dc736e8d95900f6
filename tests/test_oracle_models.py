"""Pins for oracle/models.py and oracle/evolve.py.

Closed forms: for constant coefficients on the periodic square a Fourier mode
e^{2 pi i k.x} r is an exact eigen-direction of L, so the
resolvent and exp(tau L) act on it through the 3x3 symbol matrix.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.evolve import EvolutionOperator
from oracle.models import RSW, Wave
from oracle.rational import build_exp_approx
from oracle.specelem import Mesh


def _mode(m, k1, k2, vec):
    ph = np.exp(2j * math.pi * (k1 * m.x + k2 * m.y))
    return np.asarray(vec, dtype=complex)[:, None] * ph[None, :], ph


@pytest.fixture(scope="module")
def rsw16():
    return RSW(Mesh(4, 16), f=1.0)


@pytest.mark.parametrize("alpha", [-4.6 + 3.0j, 4.6 - 20.0j, -9.2 + 0.0j, 4.6 + 60.0j])
@pytest.mark.parametrize("k", [(1, 2), (-3, 1)])
def test_rsw_resolvent_fourier_mode_closed_form(rsw16, alpha, k):
    tau = 0.5
    m = rsw16.mesh
    vec = [0.3, -0.2 + 0.1j, 1.0]
    u, ph = _mode(m, *k, vec)
    got = rsw16.resolvent(alpha, tau, u)
    S = rsw16.symbol(*k)
    ref = np.linalg.solve(tau * S - alpha * np.eye(3), vec)
    assert np.abs(got - ref[:, None] * ph[None, :]).max() < 1e-9 * np.abs(ref).max() * 1e2


def test_rsw_printed_A_sign_fails_closed_form(rsw16):
    """Reading R10: with the paper's printed A_alpha = (alpha I + f J)/(alpha^2+f^2)
    the reformulation does NOT invert (L - beta); with beta I - f J it does."""
    m = rsw16.mesh
    f, beta = 1.0, 1.3 + 0.7j
    k = (1, 1)
    vec = np.array([0.3, -0.2, 1.0], dtype=complex)
    S = rsw16.symbol(*k)
    ref = np.linalg.solve(S - beta * np.eye(3), vec)
    kk = 2j * math.pi * np.array(k)
    J = np.array([[0, 1], [-1, 0]])
    for sgn, ok in [(-1.0, True), (+1.0, False)]:
        A = (beta * np.eye(2) + sgn * f * J) / (beta ** 2 + f ** 2)
        k2 = beta ** 2 + f ** 2
        rhs = (k2 / beta) * (vec[2] + kk @ (A @ vec[:2]))
        eta = rhs / ((kk @ kk) - k2)          # Laplacian symbol is kk.kk = -(2 pi |k|)^2
        v = A @ (kk * eta - vec[:2])
        got = np.array([v[0], v[1], eta])
        assert (np.abs(got - ref).max() < 1e-12) == ok


def test_rsw_conjugation_identity(rsw16):
    """conj((tau L - alpha)^{-1} u0) = (tau L - conj(alpha))^{-1} u0 for real u0."""
    m = rsw16.mesh
    rng = np.random.default_rng(0)
    u = np.stack([np.sin(2 * math.pi * m.x) * rng.uniform(), np.cos(4 * math.pi * m.y), np.sin(2 * math.pi * (m.x - m.y))])
    a = -4.6 + 7.0j
    r1 = rsw16.resolvent(a, 0.5, u)
    r2 = rsw16.resolvent(np.conj(a), 0.5, u)
    assert np.abs(np.conj(r1) - r2).max() < 1e-11 * np.abs(r1).max()


def test_rsw_resolvent_defect_identity(rsw16):
    """(tau L - alpha) R u = u up to discretization error, for smooth u."""
    m = rsw16.mesh
    u = np.stack([np.cos(2 * math.pi * m.x) * np.sin(2 * math.pi * m.y),
                  np.sin(4 * math.pi * m.x), np.exp(np.sin(2 * math.pi * m.x) * np.cos(2 * math.pi * m.y))]).astype(complex)
    for a in [-4.6 + 2.0j, 4.6 - 30.0j]:
        r = rsw16.resolvent(a, 0.5, u)
        d = 0.5 * rsw16.forward(r) - a * r - u
        assert np.abs(d).max() < 1e-7 * np.abs(u).max()


def test_wave_constant_kappa_matches_symbol():
    m = Mesh(4, 16)
    wv = Wave(m, np.ones(m.N))
    k1, k2 = 2, -1
    vec = [0.2, 0.5j, 1.0]
    u, ph = _mode(m, k1, k2, vec)
    a1, a2 = 2j * math.pi * k1, 2j * math.pi * k2
    S = np.array([[0, 0, a1], [0, 0, a2], [a1, a2, 0]], dtype=complex)
    for alpha in [-4.6 + 5.0j, 4.6 + 40.0j]:
        got = wv.resolvent(alpha, 0.5, u)
        ref = np.linalg.solve(0.5 * S - alpha * np.eye(3), vec)
        assert np.abs(got - ref[:, None] * ph[None, :]).max() < 1e-9 * np.abs(ref).max() * 1e2


def test_wave_variable_kappa_defect_and_conjugation():
    m = Mesh(4, 16)
    kappa = (0.75 + 0.25 * np.sin(2 * math.pi * m.x)) * (1.0 + 0.3 * np.cos(2 * math.pi * m.y))
    wv = Wave(m, kappa)
    u0 = np.sin(2 * math.pi * m.x) * np.sin(2 * math.pi * m.y)
    u = np.stack([2 * math.pi * np.cos(2 * math.pi * m.x) * np.sin(2 * math.pi * m.y),
                  2 * math.pi * np.sin(2 * math.pi * m.x) * np.cos(2 * math.pi * m.y), 0.3 * u0]).astype(complex)
    a = -4.6 + 9.0j
    r = wv.resolvent(a, 0.5, u)
    d = 0.5 * wv.forward(r) - a * r - u
    assert np.abs(d).max() < 1e-7 * np.abs(u).max()
    r2 = wv.resolvent(np.conj(a), 0.5, u)
    assert np.abs(np.conj(r) - r2).max() < 1e-11 * np.abs(r).max()


# ---------------------------------------------------------------------------
# the evolution operator
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def op16():
    m = Mesh(4, 16)
    return EvolutionOperator(RSW(m, 1.0), tau=0.25, Lambda=80.0, delta=1e-10)


def test_step_fourier_mode_exact_evolution(op16):
    """exp(tau L) is diagonal in Fourier space; one and three
    big steps on a resolved mode match expm(tau * symbol)."""
    m = op16.model.mesh
    k = (1, -2)
    vec = np.array([0.1, 0.4 - 0.2j, 1.0])
    u, ph = _mode(m, *k, vec)
    S = op16.model.symbol(*k)
    assert np.abs(np.linalg.eigvals(op16.tau * S)).max() < op16.tau * op16.Lambda
    u3 = u
    for n in range(1, 4):
        u3 = op16.step(u3)
        ref = sla.expm(n * op16.tau * S) @ vec
        assert np.abs(u3 - ref[:, None] * ph[None, :]).max() < 1e-8
    # norm conservation of the skew-Hermitian flow on this mode
    assert abs(np.linalg.norm(u3[:, 0]) - np.linalg.norm(vec)) < 1e-8


def test_step_linearity_and_half_pole_identity(op16):
    m = op16.model.mesh
    rng = np.random.default_rng(5)
    a = np.stack([np.sin(2 * math.pi * (m.x + 2 * m.y)), np.cos(2 * math.pi * m.x), np.sin(4 * math.pi * m.y)])
    b = np.stack([np.cos(2 * math.pi * m.y), np.sin(2 * math.pi * (m.x - m.y)), np.cos(2 * math.pi * m.x) ** 2])
    c1, c2 = 0.7 - 0.2j, -1.3j
    lhs = op16.step(c1 * a + c2 * b)
    sa, sb = op16.step(a), op16.step(b)
    assert np.abs(lhs - (c1 * sa + c2 * sb)).max() < 1e-11 * np.abs(lhs).max()
    # real input -> real output (conjugate-closed poles/residues)
    assert np.abs(sa.imag).max() < 1e-11 * np.abs(sa).max()
    # the conjugate-pair identity the GPU path relies on:
    #   sum_all b_m R_m a = sum_{Im alpha >= 0} w_m Re(b_m R_m a),  w = 2 (Im>0), 1 (Im=0)
    p, r = op16.poles, op16.res
    acc = np.zeros_like(sa)
    for mm in range(len(p)):
        if p[mm].imag > 1e-12 * abs(p[mm]):
            acc += 2.0 * (r[mm] * op16.resolvent(mm, a)).real
        elif abs(p[mm].imag) <= 1e-12 * abs(p[mm]):
            acc += (r[mm] * op16.resolvent(mm, a)).real
    assert np.abs(acc - sa.real).max() < 1e-11 * np.abs(sa).max()


def test_poles_counts_match_policy():
    """Reading R5: hS = 2.5 h and the smallest filter margin >= 8 that passes the
    delta / 1 + delta checks (a smaller margin fails them)."""
    from oracle.rational import M0_MARGIN_MIN, _check, compose_rational, exp_approx_params, \
        gaussian_coeffs_chi, gaussian_coeffs_exp, product_rational
    for A, npoles, margin in [(20.0, 316, 8), (60.0, 528, 8), (100.0, 736, 8), (160.0, 1060, 9), (10.0, 276, 9)]:
        ap = build_exp_approx(A, 1e-10)
        assert len(ap["poles"]) == npoles and ap["params"]["margin"] == margin, A
        if margin > M0_MARGIN_MIN:
            prm = exp_approx_params(A, margin - 1)
            pR, rR = compose_rational(prm["h"], gaussian_coeffs_exp(prm["h"], prm["M"]))
            pS, rS = compose_rational(prm["hS"], gaussian_coeffs_chi(prm["M0"]))
            err, mm = _check(*product_rational(pS, rS, pR, rR), A, 32)
            assert err > 1e-10 or mm > 1 + 1e-10


def test_refined_lu_is_the_same_solve_with_a_smaller_residual():
    """RefinedLU (reading R15) solves the SAME collocation system as a plain
    sparse LU - the two solutions differ only at rounding level - and its
    residual, evaluated independently in long double with dense arithmetic, is
    smaller; on a tiny system it reproduces numpy's dense solve."""
    import scipy.sparse.linalg as spla
    from oracle.models import RefinedLU
    m = Mesh(4, 12)
    beta = (4.6 + 41.7j) / 0.2
    B = m.collocation_matrix(np.full(m.NI, beta * beta + 1.0, dtype=complex))
    rng = np.random.default_rng(3)
    F = np.zeros(m.N, dtype=complex)
    F[: m.NI] = rng.standard_normal(m.NI) + 1j * rng.standard_normal(m.NI)
    x_plain = spla.splu(B.tocsc()).solve(F)
    x_ref = RefinedLU(B).solve(F)
    assert np.linalg.norm(x_ref - x_plain) <= 1e-10 * np.linalg.norm(x_plain)   # same system, same answer

    def residual(x):   # independent of RefinedLU.residual: dense long-double products
        Bd = B.toarray()
        ld = np.longdouble
        Br, Bi = Bd.real.astype(ld), Bd.imag.astype(ld)
        xr, xi = x.real.astype(ld), x.imag.astype(ld)
        rr = F.real.astype(ld) - (Br @ xr - Bi @ xi)
        ri = F.imag.astype(ld) - (Br @ xi + Bi @ xr)
        return float(np.sqrt((rr * rr + ri * ri).sum()))

    r_plain, r_ref = residual(x_plain), residual(x_ref)
    print(f"residual plain {r_plain:.2e} refined {r_ref:.2e}")
    assert r_ref <= 0.5 * r_plain
    # tiny system against the dense definition
    m2 = Mesh(2, 6)
    B2 = m2.collocation_matrix(np.full(m2.NI, 2.0 + 1.0j, dtype=complex))
    F2 = rng.standard_normal(m2.N) + 1j * rng.standard_normal(m2.N)
    assert np.linalg.norm(RefinedLU(B2).solve(F2) - np.linalg.solve(B2.toarray(), F2)) <= 1e-12 * np.linalg.norm(F2)

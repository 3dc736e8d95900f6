"""Pins for oracle/rational.py against what PAPER.md and mathematics fix.

Each test would fail for a plausible mistake in the oracle: a mistyped Table-1
entry or the wrong rational form (test_table1_*), a wrong sign/index/scale in
the Gaussian coefficients (appendix bound), a wrong convolution limit or pole
map (compose vs direct), a broken filter/product (stability bound).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import rational as R
from oracle.evolve import rational_apply_dense

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_table1_transcription_spot_values():
    mu, a = R.table1()
    L = R.L_TABLE
    assert L == GOLD["table1_L"]["value"]
    assert mu == GOLD["table1_mu"]["value"]
    assert a[L] == GOLD["table1_a0"]["value"]
    assert a[L + 1] == complex(*GOLD["table1_a1"]["value"])
    assert a[0] == complex(*GOLD["table1_am11"]["value"])


def test_table1_gaussian_rational_sup_error_matches_paper():
    """sup_x |psi_1 - Re sum a_j/(ix+mu+ij)| ~ 7e-13 (Fig. 3)."""
    x = np.linspace(-50.0, 50.0, 100001)
    err = np.abs(R.gaussian_rational_psi1(x) - R.psi1(x)).max()
    paper = GOLD["gaussian_rational_sup_error"]["value"]
    assert err <= 1.5 * paper
    assert err >= 0.5 * paper          # same approximant, not an accidentally better one
    # far field: both sides decay; the rational tail stays below the same bound
    xf = np.logspace(1.7, 6, 2000)
    assert np.abs(R.gaussian_rational_psi1(xf) - R.psi1(xf)).max() <= 1.5 * paper


def test_table1_even_part_not_worse():
    """Reading R2: the even part of the approximant cannot be worse (triangle inequality)."""
    x = np.linspace(-50.0, 50.0, 100001)
    _, ae = R.table1_even()
    err_e = np.abs(R.gaussian_rational_psi1(x, a=ae) - R.psi1(x)).max()
    err_o = np.abs(R.gaussian_rational_psi1(x) - R.psi1(x)).max()
    assert err_e <= err_o * (1 + 1e-6)
    assert np.allclose(ae, np.conj(ae[::-1]), rtol=0, atol=0)


def test_psi_hat_closed_form_against_quadrature():
    h = 0.23
    x = np.linspace(-40 * h, 40 * h, 200001)
    dx = x[1] - x[0]
    for xi in [0.0, 0.7, 1.0, 2.3]:
        num = np.sum(R.psi_h(x, h) * np.exp(-2j * math.pi * x * xi)) * dx
        assert abs(num - R.psi_h_hat(xi, h)) < 1e-11


@pytest.mark.parametrize("h,M,t", [(0.2, 50, 0.5), (0.17, 40, 1.0), (0.25, 30, 1.0)])
def test_gaussian_sum_within_appendix_bound(h, M, t):
    """Appendix A: pointwise error <= Poisson bound."""
    X = (M - 2) * h
    x = np.linspace(-X * 1.1, X * 1.1, 4001)
    c = R.gaussian_coeffs_exp(h, M, t)
    err = np.abs(R.gaussian_sum(x, h, c) - np.exp(2j * math.pi * t * x))
    bound = R.appendix_error_bound(h, M, x, t)
    assert np.all(err <= bound * (1 + 1e-6) + 1e-14)
    # and the bound is tight enough to mean something inside the interval
    inner = np.abs(x) <= (M - 12) * h
    assert err[inner].max() < 5e-9
    # |c_m| constant
    assert np.allclose(np.abs(c), h / R.psi_h_hat(t, h))


@pytest.mark.parametrize("h,M", [(0.17, 20), (0.34, 9)])
def test_compose_partial_fractions_equal_direct_sum(h, M):
    """The pole/residue form equals sum_m c_m * [Table-1 rational of psi_1(x/h+m)]."""
    rng = np.random.default_rng(0)
    coeffs = rng.standard_normal(2 * M + 1) + 1j * rng.standard_normal(2 * M + 1)
    poles, res = R.compose_rational(h, coeffs)
    _, ae = R.table1_even()
    x = np.linspace(-(M + 15) * h, (M + 15) * h, 3001)
    direct = np.zeros(x.shape, dtype=complex)
    for m, cm in zip(range(-M, M + 1), coeffs):
        direct += cm * R.gaussian_rational_psi1(x / h + m, a=ae)
    pf = R.rational_eval(poles, res, 2j * math.pi * x)
    assert np.abs(pf - direct).max() < 1e-12 * np.abs(coeffs).sum()
    assert len(poles) == 2 * (2 * (M + R.L_TABLE) + 1)


def test_fig4_172_pairs_reach_1e10_on_28():
    """PAPER.md:755-758 (Fig. 4): 172 conjugate pairs give ~1e-10 on -28 <= x <= 28."""
    K = GOLD["fig4_pairs"]["value"]
    X = GOLD["fig4_half_interval_x"]["value"]
    M = K - R.L_TABLE
    h = X / (M - 10)
    poles, res = R.compose_rational(h, R.gaussian_coeffs_exp(h, M))
    assert len(poles) // 2 == 2 * K + 1
    x = np.linspace(-X, X, 56001)
    val = R.rational_eval(poles, res, 2j * math.pi * x)
    err_cos = np.abs(0.5 * (val + val[::-1]) - np.cos(2 * math.pi * x)).max()
    err_sin = np.abs(0.5 * (val - val[::-1]) / 1j - np.sin(2 * math.pi * x)).max()
    assert max(err_cos, err_sin) <= GOLD["fig4_sup_error"]["value"]


def test_unfiltered_approximant_overshoots():
    """§3.3: the bare Gaussian approximant exceeds 1 near |x| ~ Mh."""
    h, M = 0.17, 40
    poles, res = R.compose_rational(h, R.gaussian_coeffs_exp(h, M))
    y = 2 * math.pi * np.linspace(-(M + 10) * h, (M + 10) * h, 20001)
    assert np.abs(R.rational_eval(poles, res, 1j * y)).max() > 1.1


@pytest.mark.parametrize("A", [20.0, 60.0])
def test_build_exp_approx_accuracy_stability_symmetry(A):
    ap = R.build_exp_approx(A, 1e-10)
    p, b = ap["poles"], ap["res"]
    assert ap["err"] <= 1e-10
    assert ap["maxmod"] <= 1.0 + 1e-10
    # independent dense re-check on a different sample set, incl. far field
    y = np.concatenate([np.random.default_rng(1).uniform(-A, A, 5000)])
    assert np.abs(R.rational_eval(p, b, 1j * y) - np.exp(1j * y)).max() <= 1e-10
    yf = np.concatenate([np.linspace(A, 6 * A, 5000), -np.linspace(A, 6 * A, 5000), [1e8, -1e8]])
    assert np.abs(R.rational_eval(p, b, 1j * yf)).max() <= 1.0 + 1e-10
    # poles off the imaginary axis, distinct, conjugate-closed with conjugate residues
    assert np.all(np.abs(p.real) > 1.0)
    d = np.abs(p[:, None] - p[None, :]) + np.eye(len(p))
    assert d.min() > 1e-6
    for k in range(len(p)):
        j = np.argmin(np.abs(p - np.conj(p[k])))
        assert abs(p[j] - np.conj(p[k])) < 1e-12 * abs(p[k])
        assert abs(b[j] - np.conj(b[k])) < 1e-12 * max(1.0, abs(b[k]))


def test_product_rational_equals_pointwise_product():
    pS, rS = R.compose_rational(0.34, R.gaussian_coeffs_chi(8))
    pR, rR = R.compose_rational(0.17, R.gaussian_coeffs_exp(0.17, 16))
    p, b = R.product_rational(pS, rS, pR, rR)
    z = 1j * np.random.default_rng(2).uniform(-40, 40, 3000) + 0.3
    lhs = R.rational_eval(p, b, z)
    rhs = R.rational_eval(pS, rS, z) * R.rational_eval(pR, rR, z)
    assert np.abs(lhs - rhs).max() < 1e-11


def test_matrix_function_brute_force():
    """sum b_m (A - alpha_m)^{-1} u vs expm(A) u for a skew-symmetric A with
    spectrum inside [-0.9 tau Lambda, 0.9 tau Lambda]: error <= delta ||u||
    (spectral theorem + Eq. RM_prop1)."""
    A_int = 20.0
    ap = R.build_exp_approx(A_int, 1e-10)
    rng = np.random.default_rng(3)
    n = 14
    Q = rng.standard_normal((n, n))
    S = Q - Q.T
    S *= 0.9 * A_int / np.abs(np.linalg.eigvals(S)).max()
    u = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    got = rational_apply_dense(ap["poles"], ap["res"], S, u)
    ref = sla.expm(S) @ u
    assert np.linalg.norm(got - ref) <= 2e-10 * np.linalg.norm(u)

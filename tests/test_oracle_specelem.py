"""Pins for oracle/specelem.py (§2.2): exactness on polynomials,
closed-form Laplacian/gradient of Fourier modes, manufactured solutions,
spectral convergence, index bookkeeping."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.specelem import Mesh, cheb_points, lagrange_diff_matrix


@pytest.mark.parametrize("p", [4, 6, 10, 16])
def test_diff_matrix_exact_on_polynomials(p):
    t = cheb_points(p)
    D = lagrange_diff_matrix(t)
    for deg in range(p):
        assert np.abs(D @ t ** deg - (deg * t ** (deg - 1) if deg else 0 * t)).max() < 1e-10 * max(1, deg) ** 2
    assert np.abs(D @ np.ones(p)).max() < 1e-12


def test_edge_tangential_stencil_exact_on_polynomials():
    m = Mesh(2, 12)
    s = m.s_edge
    for deg in range(m.p):
        ref = deg * s[1:-1] ** (deg - 1) if deg else 0 * s[1:-1]
        assert np.abs(m.Dw @ s ** deg - ref).max() < 1e-9 * max(1, deg) ** 2


def test_node_counts_and_bijection():
    m = Mesh(2, 4)
    # hand count: 4 elements x (2x2 interior + 2 owned edges x 2 nodes) = 32
    assert m.N == 32
    for n, p in [(2, 4), (4, 6), (4, 10)]:
        m = Mesh(n, p)
        g = m.G[m.G >= 0]
        assert set(g.tolist()) == set(range(m.N))
        counts = np.bincount(g, minlength=m.N)
        assert np.all(counts[: m.NI] == 1)         # interior nodes belong to one element
        assert np.all(counts[m.NI:] == 2)          # edge nodes shared by exactly two elements
        assert np.sum(m.G < 0) == 4 * n * n        # corners excluded


def test_coordinates_periodic_and_on_grid():
    m = Mesh(4, 6)
    assert np.all((m.x >= 0) & (m.x < 1)) and np.all((m.y >= 0) & (m.y < 1))
    # vertical-edge nodes lie on x = ex * H
    V = slice(m.NI, m.NI + m.NV)
    assert np.allclose(np.round(m.x[V] * m.n) / m.n, m.x[V], atol=1e-15)


def _mode(m, k1, k2):
    return np.exp(2j * math.pi * (k1 * m.x + k2 * m.y))


@pytest.mark.parametrize("k1,k2", [(1, 0), (1, 2), (-2, 3)])
def test_collocation_rows_on_fourier_mode(k1, k2):
    m = Mesh(4, 16)
    sigma = 3.0 + 1.0j
    B = m.collocation_matrix(np.full(m.NI, sigma))
    ph = _mode(m, k1, k2)
    r = B @ ph
    lam = -(2 * math.pi) ** 2 * (k1 * k1 + k2 * k2) - sigma
    assert np.abs(r[: m.NI] - lam * ph[: m.NI]).max() < 1e-7 * abs(lam)
    assert np.abs(r[m.NI:]).max() < 1e-8 * 2 * math.pi * math.hypot(k1, k2) * m.n


@pytest.mark.parametrize("k1,k2", [(1, 2), (0, 3), (3, -1)])
def test_gradient_on_fourier_mode_all_node_classes(k1, k2):
    m = Mesh(4, 16)
    ph = _mode(m, k1, k2)
    gx, gy = m.grad(ph)
    assert np.abs(gx - 2j * math.pi * k1 * ph).max() < 1e-8
    assert np.abs(gy - 2j * math.pi * k2 * ph).max() < 1e-8
    Gx, Gy = m.grad_matrices()
    assert np.abs(Gx @ ph - gx).max() < 1e-12
    assert np.abs(Gy @ ph - gy).max() < 1e-12


def _manufactured_error(n, p, sigma):
    m = Mesh(n, p)
    u = np.sin(2 * math.pi * m.x) * np.cos(4 * math.pi * m.y) + 0.5 * np.cos(2 * math.pi * (m.x + m.y))
    lap = -(2 * math.pi) ** 2 * (1 + 4) * np.sin(2 * math.pi * m.x) * np.cos(4 * math.pi * m.y) \
        - (2 * math.pi) ** 2 * 2 * 0.5 * np.cos(2 * math.pi * (m.x + m.y))
    F = np.zeros(m.N, dtype=complex)
    F[: m.NI] = (lap - sigma * u)[: m.NI]
    B = m.collocation_matrix(np.full(m.NI, sigma, dtype=complex))
    sol = spla.splu(B).solve(F)
    return np.abs(sol - u).max()


def test_manufactured_solution_and_spectral_convergence():
    sigma = 5.0 - 40.0j
    e16 = _manufactured_error(4, 16, sigma)
    e8 = _manufactured_error(4, 8, sigma)
    assert e16 < 1e-9
    assert e8 / e16 > 1e3


def test_solution_is_c1_across_edges():
    """Flux rows: the two one-sided normal derivatives agree at edge nodes."""
    m = Mesh(4, 10)
    rng = np.random.default_rng(0)
    F = np.zeros(m.N, dtype=complex)
    F[: m.NI] = rng.standard_normal(m.NI)
    u = spla.splu(m.collocation_matrix(np.full(m.NI, 2.0 + 0j))).solve(F)
    B = m.collocation_matrix(np.full(m.NI, 2.0 + 0j))
    assert np.abs((B @ u)[m.NI:]).max() < 1e-9 * np.abs(u).max() * m.n * m.p ** 2

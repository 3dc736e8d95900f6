"""Seeded synthetic workloads shared by the oracle tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only the BASELINE.json configurations
(as plain parameters) and initial-condition / coefficient-field generators that
take node coordinates (computed by whichever side calls them) and a seed.

Recipe (DESIGN.md §4 "Inputs"), following BASELINE.json configs:
  * RSW initial condition: eta = periodised Gaussian bump (sigma = 0.1, centre
    drawn from the seed) + complex random Fourier perturbation of amplitude 1e-2
    on modes 0 < |k|_inf <= 4; zero velocity.  The perturbation has complex
    amplitudes, so the state is genuinely complex128.
  * Wave equation: u0 as the RSW eta above, state (w, z, v) = (u0_x, u0_y, 0)
    with the derivatives taken analytically; kappa = c(x)^2 with c a smooth
    random field (Fourier modes |k|_inf <= 6) scaled into [0.5, 1.5].
"""
from __future__ import annotations

import math

import numpy as np

# name -> parameters.  "tau" is our choice (BASELINE.json fixes only tau*Lambda).
CONFIGS = {
    "c0_rsw_4x4_p10": dict(model="rsw", n=4, p=10, f=1.0, Lambda_tau=20.0, tau=0.2, delta=1e-10,
                           nsteps=10, nrhs=1, seed=1234),
    "c1_rsw_16x16_p16": dict(model="rsw", n=16, p=16, f=1.0, Lambda_tau=60.0, tau=0.5, delta=1e-10,
                             nsteps=100, nrhs=1, seed=1234),
    "c2_wave_32x32_p16": dict(model="wave", n=32, p=16, Lambda_tau=100.0, tau=0.5, delta=1e-10,
                              nsteps=50, nrhs=1, seed=1234),
    "c3_rsw_32x32_p16_x64": dict(model="rsw", n=32, p=16, f=1.0, Lambda_tau=60.0, tau=0.25, delta=1e-10,
                                 nsteps=50, nrhs=64, seed=1234),
    # reduced-size stand-in for c2 that fits one B200 (per-node store ~10 GB):
    # the variable-coefficient (HBM-bound GEMV) path at a measurable scale
    "c2r_wave_8x8_p16": dict(model="wave", n=8, p=16, Lambda_tau=20.0, tau=0.2, delta=1e-10,
                             nsteps=10, nrhs=1, seed=1234),
    "c4_wave_64x64_p12": dict(model="wave", n=64, p=12, Lambda_tau=160.0, tau=0.5, delta=1e-10,
                              nsteps=200, nrhs=1, seed=1234),
}


def _periodic_gaussian(x, y, x0, y0, sigma):
    out = np.zeros_like(x)
    for sx in (-1.0, 0.0, 1.0):
        for sy in (-1.0, 0.0, 1.0):
            out += np.exp(-((x - x0 - sx) ** 2 + (y - y0 - sy) ** 2) / (2.0 * sigma * sigma))
    return out


def _modes(rng, kmax):
    ks = [(k1, k2) for k1 in range(-kmax, kmax + 1) for k2 in range(-kmax, kmax + 1) if (k1, k2) != (0, 0)]
    amp = rng.standard_normal(len(ks)) + 1j * rng.standard_normal(len(ks))
    return ks, amp


def scalar_bump(x, y, seed, sigma=0.1, amp=1e-2, kmax=4):
    """Gaussian bump + complex low-wavenumber perturbation, and its gradient."""
    rng = np.random.default_rng(seed)
    x0, y0 = rng.uniform(0.0, 1.0, size=2)
    g = _periodic_gaussian(x, y, x0, y0, sigma)
    gx = np.zeros_like(x)
    gy = np.zeros_like(x)
    for sx in (-1.0, 0.0, 1.0):
        for sy in (-1.0, 0.0, 1.0):
            e = np.exp(-((x - x0 - sx) ** 2 + (y - y0 - sy) ** 2) / (2.0 * sigma * sigma))
            gx += -(x - x0 - sx) / (sigma * sigma) * e
            gy += -(y - y0 - sy) / (sigma * sigma) * e
    ks, a = _modes(rng, kmax)
    scale = amp / math.sqrt(len(ks))
    u = g.astype(complex)
    ux = gx.astype(complex)
    uy = gy.astype(complex)
    for (k1, k2), ak in zip(ks, a):
        ph = np.exp(2j * math.pi * (k1 * x + k2 * y))
        u += scale * ak * ph
        ux += scale * ak * 2j * math.pi * k1 * ph
        uy += scale * ak * 2j * math.pi * k2 * ph
    return u, ux, uy


def rsw_initial_state(x, y, seed):
    """(v1, v2, eta) complex128, shape (3, N)."""
    eta, _, _ = scalar_bump(x, y, seed)
    z = np.zeros_like(eta)
    return np.stack([z, z.copy(), eta])


def wave_initial_state(x, y, seed):
    """(w, z, v) = (u0_x, u0_y, 0), complex128, shape (3, N)."""
    u, ux, uy = scalar_bump(x, y, seed)
    return np.stack([ux, uy, np.zeros_like(u)])


def wave_speed_field(x, y, seed, kmax=6):
    """kappa = c^2, c smooth random (|k|_inf <= 6) scaled into [0.5, 1.5]."""
    rng = np.random.default_rng(seed + 7919)
    c = np.zeros_like(x, dtype=float)
    for k1 in range(-kmax, kmax + 1):
        for k2 in range(0, kmax + 1):
            if k2 == 0 and k1 < 0:
                continue
            a, b = rng.standard_normal(2) / (1.0 + k1 * k1 + k2 * k2)
            ph = 2.0 * math.pi * (k1 * x + k2 * y)
            c += a * np.cos(ph) + b * np.sin(ph)
    # scale into [0.5, 1.5] using the field's exact extremes on a fine uniform grid
    s = np.linspace(0.0, 1.0, 257)[:-1]
    X, Y = np.meshgrid(s, s, indexing="ij")
    cf = np.zeros_like(X)
    rng = np.random.default_rng(seed + 7919)
    for k1 in range(-kmax, kmax + 1):
        for k2 in range(0, kmax + 1):
            if k2 == 0 and k1 < 0:
                continue
            a, b = rng.standard_normal(2) / (1.0 + k1 * k1 + k2 * k2)
            ph = 2.0 * math.pi * (k1 * X + k2 * Y)
            cf += a * np.cos(ph) + b * np.sin(ph)
    lo, hi = cf.min(), cf.max()
    pad = 0.02 * (hi - lo)
    c01 = (c - (lo - pad)) / ((hi + pad) - (lo - pad))
    c01 = np.clip(c01, 0.0, 1.0)
    cc = 0.5 + c01
    return cc * cc


def initial_state(model, x, y, seed):
    return rsw_initial_state(x, y, seed) if model == "rsw" else wave_initial_state(x, y, seed)

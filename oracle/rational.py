"""Oracle: rational approximation of exp(iy) (§1.2, §3).

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` may be imported by the
product path (``paper_1402_5168_b200``); only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg use it.  Plain, slow, fp64 numpy, written to be
checked against the paper by eye.

Notation follows PAPER.md:
  * psi_h(x) = (4 pi)^{-1/2} exp(-x^2 / (4 h^2))           (§3)
  * Gaussian sum  f(x) ~ sum_{m=-M}^{M} c_m psi_h(x + m h)  (§3 Eq. "intro,
    approx of f(x) via Gaussians", §3.1)
  * c_m = (h / psihat_h(1)) e^{-2 pi i m h} for f = e^{2 pi i x}
    (§3.1 Eq. "coeff. for exp, gauss")
  * psi_1(x) ~ Re sum_{j=-L}^{L} a_j / (i x + mu + i j), L = 11
    (§3.2 Eq. "approx of Gaussian via rationals", Table 1)
  * R_M(i y) = sum_m b_m / (i y - alpha_m) ~ e^{i y} on |y| <= tau Lambda
    (§1.2 Eq. "def_RM"/"RM_prop1")
  * filter: S(iy) ~ chi(x) = sum_{|m|<=M0} psi_{hS}(x + m hS), and the
    stable approximant is the proper rational function S(iy) R(iy)
    (§3.3, Eq. "partition of unity-1").

Readings of the paper taken here (all listed in DESIGN.md §3):
  R1  Table 1 is used in the form Re sum a_j/(ix + mu + ij) (the form of
      Eq. "approx of Gaussian via rationals"); pinned by the 7e-13 sup error
      the paper prints (§3.2).
  R2  a_j is replaced by its even part  a~_j = (a_j + conj(a_{-j}))/2 :
      psi_1 is real and even, the table pairs agree only to ~1e-6, and the
      even part of the approximant has sup error <= that of the original.
      Makes the rational function exactly conjugate-symmetric.
  R3  Convolution limits j in [max(-L, n-M), min(L, n+M)] (the paper's
      L_2 repeats L_1, PAPER.md:520 - a typo).
  R4  Scaled variable x = y / (2 pi): e^{iy} = e^{2 pi i x}, A = tau*Lambda
      maps to X = A / (2 pi) (§3.1 works with e^{2 pi i x}).
  R5  Parameter policy (paper gives no h):  h = 0.17, hS = 2.5 h,
      M0 = ceil(X / hS) + c, M = ceil(M0 hS / h), with c the smallest margin
      >= 8 for which the approximant passes the delta / 1 + delta checks of
      §1.2 (Eqs. "RM_prop1", "RM_prop2").  The filter lattice hS differs from
      h so the poles of S and R are distinct (§3.3).
  R6  Stability filter = §3.3's first construction, the product S(iy)R(iy)
      written as one proper rational function (union of pole sets, residue of
      each factor multiplied by the other factor evaluated at the pole).
      S = Q (no pole reduction; the reduction algorithm of [HAU-BEY] is out
      of scope).
"""
from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# Table 1, verbatim.
# ---------------------------------------------------------------------------
MU = -4.315321510875024
L_TABLE = 11
_A_TABLE = {
    -11: (-1.0845749544592896e-7, 2.77075431662228e-8),
    -10: (1.858753344202957e-8, -9.105375434750162e-7),
    -9: (3.6743713227243024e-6, 7.073284346322969e-7),
    -8: (-2.7990058083347696e-6, 0.0000112564827639346),
    -7: (0.000014918577548849352, -0.0000316278486761932),
    -6: (-0.0010751767283285608, -0.00047282220513073084),
    -5: (0.003816465653840016, 0.017839810396560574),
    -4: (0.12124105653274578, -0.12327042473830248),
    -3: (-0.9774980792734348, -0.1877130220537587),
    -2: (1.3432866123333178, 3.2034715228495942),
    -1: (4.072408546157305, -6.123755543580666),
    0: (-9.442699917778205, 0.0),
    1: (4.072408620272648, 6.123755841848161),
    2: (1.3432860877712938, -3.2034712658530275),
    3: (-0.9774985292598916, 0.18771238018072134),
    4: (0.1212417070363373, 0.12326987628935386),
    5: (0.0038169724770333343, -0.017839242222443888),
    6: (-0.0010756025812659208, 0.0004731874917343858),
    7: (0.000014713754789095218, 0.000031358475831136815),
    8: (-2.659323898804944e-6, -0.000011341571201752273),
    9: (3.6970377676364553e-6, -6.517457477594937e-7),
    10: (3.883933649142257e-9, 9.128496023863376e-7),
    11: (-1.0816457995911385e-7, -2.954309729192276e-8),
}


def table1():
    """(mu, a) with a[j + L] = a_j, j = -11..11, verbatim from Table 1."""
    a = np.array([complex(*_A_TABLE[j]) for j in range(-L_TABLE, L_TABLE + 1)])
    return MU, a


def table1_even():
    """Reading R2: even part a~_j = (a_j + conj(a_{-j})) / 2."""
    mu, a = table1()
    return mu, 0.5 * (a + np.conj(a[::-1]))


def psi1(x):
    """psi_1(x) = (4 pi)^{-1/2} e^{-x^2/4}  (§3, PAPER.md:495 with h = 1)."""
    x = np.asarray(x, dtype=float)
    return (4.0 * math.pi) ** -0.5 * np.exp(-x * x / 4.0)


def psi_h(x, h):
    """psi_h(x) = (4 pi)^{-1/2} e^{-x^2/(4 h^2)}  (§3)."""
    x = np.asarray(x, dtype=float)
    return (4.0 * math.pi) ** -0.5 * np.exp(-x * x / (4.0 * h * h))


def psi_h_hat(xi, h):
    """Fourier transform of psi_h, fhat(xi) = int f(x) e^{-2 pi i x xi} dx.

    Closed form of a Gaussian integral: h * exp(-4 pi^2 h^2 xi^2).
    """
    xi = np.asarray(xi, dtype=float)
    return h * np.exp(-4.0 * math.pi ** 2 * h * h * xi * xi)


def gaussian_rational_psi1(x, a=None, mu=MU):
    """Re sum_j a_j / (i x + mu + i j)  (Eq. "approx of Gaussian via rationals")."""
    if a is None:
        _, a = table1()
    j = np.arange(-L_TABLE, L_TABLE + 1)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    out = np.zeros(x.shape, dtype=float)
    for jj, aj in zip(j, a):
        out += (aj / (1j * x + mu + 1j * jj)).real
    return out


# ---------------------------------------------------------------------------
# §3.1 Gaussian sums
# ---------------------------------------------------------------------------
def gaussian_coeffs_exp(h, M, t=1.0):
    """c_m = (h / psihat_h(t)) e^{-2 pi i m t h}, m = -M..M.

    Approximates e^{2 pi i t x} by sum_m c_m psi_h(x + m h).
    """
    m = np.arange(-M, M + 1)
    return (h / psi_h_hat(t, h)) * np.exp(-2j * math.pi * m * t * h)


def gaussian_coeffs_chi(M0):
    """Unit coefficients of chi(x) = sum_{|m|<=M0} psi_h(x + m h) (Eq. "partition of unity-1").

    With psi_h(x) = psi_1(x/h) and int psi_1 = 1, sum over all m of
    psi_1(x/h + m) ~ 1 (Poisson), so the unit coefficients give a window ~1
    on |x| <= (M0 - m0) h.
    """
    return np.ones(2 * M0 + 1, dtype=complex)


def gaussian_sum(x, h, coeffs):
    """Direct evaluation sum_{m=-M}^{M} c_m psi_h(x + m h) (no rational step)."""
    M = (len(coeffs) - 1) // 2
    x = np.atleast_1d(np.asarray(x, dtype=float))
    out = np.zeros(x.shape, dtype=complex)
    for m, cm in zip(range(-M, M + 1), coeffs):
        out += cm * psi_h(x + m * h, h)
    return out


def appendix_error_bound(h, M, x, t=1.0, kmax=50, mtail=400):
    """Appendix A / Eq. "error bound for e^ix, partial-1".

    Poisson summation gives, for the sum with c_m = (h/psihat_h(t)) e^{-2 pi i m t h},
      |e^{2 pi i t x} - sum_{|m|<=M} c_m psi_h(x+mh)|
         <= (1/psihat_h(t)) ( sum_{k != 0} psihat_h(t + k/h)
                              + h sum_{|m|>M} psi_h(x + m h) ).
    (The printed bound drops the shift by t and the factor h in the second sum;
    this is the bound the Appendix derivation actually yields.)
    """
    k = np.concatenate([np.arange(-kmax, 0), np.arange(1, kmax + 1)])
    alias = np.sum(psi_h_hat(t + k / h, h))
    x = np.atleast_1d(np.asarray(x, dtype=float))
    m = np.concatenate([np.arange(-M - mtail, -M), np.arange(M + 1, M + mtail + 1)])
    tail = h * psi_h(x[:, None] + m[None, :] * h, h).sum(axis=1)
    return (alias + tail) / psi_h_hat(t, h)


# ---------------------------------------------------------------------------
# §3 composition: Gaussian sum + Table 1  ->  partial fractions in y = 2 pi x
# ---------------------------------------------------------------------------
def compose_rational(h, coeffs, even_table=True):
    """Poles/residues of sum_m c_m psi_h(x+mh) with psi_h -> Table-1 rational.

    Derivation (§3), with y = 2 pi x:
      psi_h(x + m h) = psi_1(x/h + m) ~ Re sum_j a_j / (i(x/h + m) + mu + i j)
                     = pi h sum_j [ a_j / (iy - alpha+_{j+m}) - conj(a_j) / (iy - alpha-_{j+m}) ]
      alpha+_n = -2 pi h (mu + i n),   alpha-_n = 2 pi h (mu - i n)
    so   sum_m c_m psi_h(x + m h) ~ sum_n [ b+_n/(iy - alpha+_n) + b-_n/(iy - alpha-_n) ]
      b+_n =  pi h C_n,  C_n = sum_{m+j=n} c_m a_j
      b-_n = -pi h D_n,  D_n = sum_{m+j=n} c_m conj(a_j)
    n = -(M+L)..(M+L), j in [max(-L, n-M), min(L, n+M)]  (reading R3).
    Returns (poles, residues) as complex arrays; the value at iy is
    sum b/(iy - alpha).
    """
    mu, a = table1_even() if even_table else table1()
    L = L_TABLE
    M = (len(coeffs) - 1) // 2
    K = M + L
    ns = np.arange(-K, K + 1)
    C = np.zeros(2 * K + 1, dtype=complex)
    D = np.zeros(2 * K + 1, dtype=complex)
    for idx, n in enumerate(ns):
        for j in range(max(-L, n - M), min(L, n + M) + 1):
            m = n - j
            C[idx] += coeffs[m + M] * a[j + L]
            D[idx] += coeffs[m + M] * np.conj(a[j + L])
    alpha_p = -2.0 * math.pi * h * (mu + 1j * ns)
    alpha_m = 2.0 * math.pi * h * (mu - 1j * ns)
    poles = np.concatenate([alpha_p, alpha_m])
    res = np.concatenate([math.pi * h * C, -math.pi * h * D])
    return poles, res


def rational_eval(poles, res, z):
    """sum_m b_m / (z - alpha_m) at complex points z (Eq. "def_RM" with z = iy)."""
    z = np.atleast_1d(np.asarray(z, dtype=complex))
    out = np.zeros(z.shape, dtype=complex)
    for i in range(0, z.size, 4096):
        zz = z[i:i + 4096]
        out[i:i + 4096] = (res[None, :] / (zz[:, None] - poles[None, :])).sum(axis=1)
    return out


def product_rational(pS, rS, pR, rR):
    """S*R as one proper rational function (§3.3).

    Both factors are proper with simple, disjoint poles, so
      S(z) R(z) = sum_k rS_k R(pS_k)/(z - pS_k) + sum_m rR_m S(pR_m)/(z - pR_m).
    """
    gap = np.abs(pS[:, None] - pR[None, :]).min()
    if gap < 1e-8:
        raise ValueError("pole collision between filter and approximant")
    res_S = rS * rational_eval(pR, rR, pS)
    res_R = rR * rational_eval(pS, rS, pR)
    return np.concatenate([pS, pR]), np.concatenate([res_S, res_R])


# ---------------------------------------------------------------------------
# build: the (alpha_m, b_m) of exp(tau L) ~ sum_m b_m (tau L - alpha_m)^{-1}
# ---------------------------------------------------------------------------
H_DEFAULT = 0.17
HS_RATIO = 2.5
M0_MARGIN_MIN = 8
M0_MARGIN_MAX = 16


def exp_approx_params(A, margin=M0_MARGIN_MIN):
    """Reading R5: parameter policy for the interval [-A, A] (A = tau*Lambda)."""
    X = A / (2.0 * math.pi)
    h = H_DEFAULT
    hS = HS_RATIO * h
    M0 = int(math.ceil(X / hS)) + margin
    M = int(math.ceil(M0 * hS / h - 1e-9))
    return dict(X=X, h=h, hS=hS, M=M, M0=M0, margin=margin)


def _check(poles, res, A, nsamp_per_unit):
    """Sup error against e^{iy} on |y| <= A and sup |R(iy)| on the real line
    (dense sampling, the paper's own verification style, Figs. 3-5)."""
    y = np.linspace(-A, A, int(2 * A * nsamp_per_unit) + 1)
    err = np.abs(rational_eval(poles, res, 1j * y) - np.exp(1j * y)).max()
    far = np.concatenate([np.linspace(-4 * A - 60, 4 * A + 60, int(8 * A * nsamp_per_unit) + 1),
                          np.logspace(0, 7, 400), -np.logspace(0, 7, 400)])
    maxmod = max(np.abs(rational_eval(poles, res, 1j * far)).max(),
                 np.abs(rational_eval(poles, res, 1j * y)).max())
    return float(err), float(maxmod)


def build_exp_approx(A, delta, verify=True, nsamp_per_unit=32):
    """Poles alpha_m and weights b_m with |e^{iy} - R(iy)| <= delta on |y| <= A
    and |R(iy)| <= 1 + delta on the real line (§1.2 Eqs. "RM_prop1", "RM_prop2").

    R = S * R_gauss  (reading R6); the filter margin c of reading R5 grows
    from 8 until both checks pass (they always run: they pick c).  With
    verify=True a failure at the largest margin raises.
    Returns dict(poles, res, params, err, maxmod).
    """
    for margin in range(M0_MARGIN_MIN, M0_MARGIN_MAX + 1):
        prm = exp_approx_params(A, margin)
        h, hS, M, M0 = prm["h"], prm["hS"], prm["M"], prm["M0"]
        pR, rR = compose_rational(h, gaussian_coeffs_exp(h, M))
        pS, rS = compose_rational(hS, gaussian_coeffs_chi(M0))
        poles, res = product_rational(pS, rS, pR, rR)
        err, maxmod = _check(poles, res, A, nsamp_per_unit)
        if err <= delta and maxmod <= 1.0 + delta:
            break
    out = dict(poles=poles, res=res, params=prm, err=err, maxmod=maxmod)
    if verify:
        if err > delta:
            raise ValueError(f"rational approximation error {err:.3e} exceeds delta={delta:.1e}")
        if maxmod > 1.0 + delta:
            raise ValueError(f"|R(iy)| reaches {maxmod:.12f} > 1 + delta")
    return out

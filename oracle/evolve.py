"""Oracle: the approximate time-evolution operator and its repeated application
(§1.1-1.2, Eq. "error in exp(t*L)").

TEST INFRASTRUCTURE ONLY (see oracle/rational.py header).

    u_{n+1} = sum_{m} b_m (tau L - alpha_m)^{-1} u_n

Every pole is solved explicitly (no conjugate-pair shortcut): this is the
plain definition, against which the GPU path's conjugate-pair/real-split
evaluation (Eq. "conjugate, matrix inverses") is checked.
"""
from __future__ import annotations

import numpy as np

from .rational import build_exp_approx


class EvolutionOperator:
    def __init__(self, model, tau, Lambda, delta, approx=None):
        self.model = model
        self.tau = float(tau)
        self.Lambda = float(Lambda)
        self.delta = float(delta)
        self.approx = approx if approx is not None else build_exp_approx(self.tau * self.Lambda, self.delta)
        self.poles = self.approx["poles"]
        self.res = self.approx["res"]
        self._lu = [None] * len(self.poles)

    def factor_all(self):
        for m, a in enumerate(self.poles):
            if self._lu[m] is None:
                self._lu[m] = self.model.factor(a / self.tau)

    def resolvent(self, m, u):
        if self._lu[m] is None:
            self._lu[m] = self.model.factor(self.poles[m] / self.tau)
        return self.model.resolvent(self.poles[m], self.tau, u, lu=self._lu[m])

    def step(self, u):
        """One big step: sum_m b_m (tau L - alpha_m)^{-1} u (ascending m)."""
        u = np.asarray(u, dtype=complex)
        out = np.zeros_like(u)
        for m in range(len(self.poles)):
            out += self.res[m] * self.resolvent(m, u)
        return out

    def evolve(self, u, nsteps):
        for _ in range(nsteps):
            u = self.step(u)
        return u


def rational_apply_dense(poles, res, Amat, u):
    """sum_m b_m (A - alpha_m)^{-1} u for a small dense matrix A (brute-force pins)."""
    n = Amat.shape[0]
    out = np.zeros(n, dtype=complex)
    for a, b in zip(poles, res):
        out += b * np.linalg.solve(Amat - a * np.eye(n), u)
    return out

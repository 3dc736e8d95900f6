"""Oracle: multidomain Chebyshev collocation on the periodic unit square
(§2.2 "Discretization", Fig. 1; §2.3).

TEST INFRASTRUCTURE ONLY (see oracle/rational.py header).  Plain numpy /
scipy.sparse, fp64 / complex128.

Discretization: the square is split into n x n equal
elements, each carrying a p x p tensor grid of Chebyshev(-Lobatto) nodes.
The global node set {x_j} consists of
  * element-interior nodes ("filled circles", Fig. 1): the PDE is collocated
    there with spectral differentiation on the local p x p grid;
  * interface nodes ("hollow squares"): nodes on element edges, shared by the
    two adjacent elements; continuity of the normal flux is enforced there.
Reading R7: corner nodes are not unknowns.  No interior
collocation row and no edge flux row references a corner value (row i / column
j of the local grid only ever touches the two edge nodes at its ends), so the
corners decouple; PAPER.md:445 defers them to the HPS tutorial, whose solver
drops them.

Global ordering (the C-ABI convention of include/rexp.h, restated here so the
oracle is readable on its own):
  interior block  : g = e*(p-2)^2 + (j-1)*(p-2) + (i-1),  e = ey*n + ex,  i,j in 1..p-2
  vertical edges  : g = NI + e*(p-2) + (j-1)   (the LEFT edge x = ex*H of element e)
  horizontal edges: g = NI + NV + e*(p-2) + (i-1)  (the BOTTOM edge y = ey*H of element e)
Element (ex, ey) spans [ex H, (ex+1) H] x [ey H, (ey+1) H], H = 1/n; local node
(i, j) sits at (ex H + (t_i + 1) H/2, ey H + (t_j + 1) H/2), t_k = -cos(pi k/(p-1)).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def cheb_points(p):
    """Chebyshev-Lobatto points t_k = -cos(pi k / (p-1)), k = 0..p-1 (ascending)."""
    k = np.arange(p)
    return -np.cos(math.pi * k / (p - 1))


def lagrange_diff_matrix(t):
    """D[i, k] = l_k'(t_i) for the Lagrange basis on nodes t (any distinct nodes).

    Barycentric form: w_k = 1 / prod_{l != k}(t_k - t_l);
    D[i,k] = (w_k / w_i) / (t_i - t_k) (i != k),  D[i,i] = -sum_{k != i} D[i,k].
    """
    t = np.asarray(t, dtype=float)
    n = t.size
    w = np.array([1.0 / np.prod([t[k] - t[l] for l in range(n) if l != k]) for k in range(n)])
    D = np.zeros((n, n))
    for i in range(n):
        for k in range(n):
            if i != k:
                D[i, k] = (w[k] / w[i]) / (t[i] - t[k])
        D[i, i] = -np.sum(D[i, :])
    return D


class Mesh:
    """Periodic n x n element mesh with p x p Chebyshev nodes per element."""

    def __init__(self, n, p):
        if n < 2 or p < 4:
            raise ValueError("need n >= 2 elements per direction and p >= 4")
        self.n, self.p = n, p
        self.q = p - 2
        self.H = 1.0 / n
        self.t = cheb_points(p)
        self.D = lagrange_diff_matrix(self.t)          # d/dt on [-1, 1]
        self.D2 = self.D @ self.D
        # edge-tangential differentiation (reading R8): the p-2 nodes of the edge
        # plus the nearest node of each collinear neighbour edge, i.e. nodes
        # s = (-1-eps, t_1, ..., t_{p-2}, 1+eps), eps = 1 + t_1; rows of the
        # p-2 edge nodes only.
        eps = 1.0 + self.t[1]
        self.s_edge = np.concatenate([[-1.0 - eps], self.t[1:-1], [1.0 + eps]])
        self.Dw = lagrange_diff_matrix(self.s_edge)[1:-1, :]
        q = self.q
        self.nelem = n * n
        self.NI = self.nelem * q * q
        self.NV = self.nelem * q
        self.NH = self.nelem * q
        self.N = self.NI + self.NV + self.NH
        self._build_index()

    # -- indexing -----------------------------------------------------------
    def elem(self, ex, ey):
        n = self.n
        return (ey % n) * n + (ex % n)

    def gidx(self, ex, ey, i, j):
        """Global index of local node (i, j) of element (ex, ey); -1 for corners."""
        p, q = self.p, self.q
        ci = i in (0, p - 1)
        cj = j in (0, p - 1)
        if ci and cj:
            return -1
        if not ci and not cj:
            return self.elem(ex, ey) * q * q + (j - 1) * q + (i - 1)
        if ci:  # vertical edge: left (i=0) of (ex,ey), right (i=p-1) = left of (ex+1,ey)
            e = self.elem(ex if i == 0 else ex + 1, ey)
            return self.NI + e * q + (j - 1)
        e = self.elem(ex, ey if j == 0 else ey + 1)
        return self.NI + self.NV + e * q + (i - 1)

    def _build_index(self):
        n, p = self.n, self.p
        G = np.full((self.nelem, p, p), -1, dtype=np.int64)   # [e, j, i]
        for ey in range(n):
            for ex in range(n):
                e = self.elem(ex, ey)
                for j in range(p):
                    for i in range(p):
                        G[e, j, i] = self.gidx(ex, ey, i, j)
        self.G = G
        xs = np.zeros(self.N)
        ys = np.zeros(self.N)
        H = self.H
        for ey in range(n):
            for ex in range(n):
                e = self.elem(ex, ey)
                for j in range(p):
                    for i in range(p):
                        g = G[e, j, i]
                        if g >= 0:
                            xs[g] = (ex * H + (self.t[i] + 1.0) * H / 2.0) % 1.0
                            ys[g] = (ey * H + (self.t[j] + 1.0) * H / 2.0) % 1.0
        self.x, self.y = xs, ys

    def is_interior(self):
        m = np.zeros(self.N, dtype=bool)
        m[: self.NI] = True
        return m

    # -- collocation matrix (§2.2) -----------------------------------------
    def collocation_matrix(self, sigma_int):
        """B = B0 - diag(sigma on interior rows); B0 = collocation_matrix_explicit(0)."""
        if getattr(self, "_B0", None) is None:
            self._B0 = self.collocation_matrix_explicit(np.zeros(self.NI))
        d = np.zeros(self.N, dtype=complex)
        d[: self.NI] = sigma_int
        return (self._B0 - sp.diags(d)).tocsc()

    def collocation_matrix_explicit(self, sigma_int):
        """B for (Laplacian - sigma(x)) u = f  with flux continuity on edges.

        Rows g < NI (interior node (e,i,j)):
            (2/H)^2 [sum_k D2[i,k] u(e;k,j) + sum_k D2[j,k] u(e;i,k)] - sigma_g u_g
        Rows on a vertical edge (left edge of element e, left neighbour eL):
            (2/H) [sum_k D[p-1,k] u(eL;k,j) - sum_k D[0,k] u(e;k,j)]     (= 0)
        Rows on a horizontal edge analogously with the bottom neighbour.
        sigma_int: length-NI array (sigma at interior nodes; complex allowed).
        """
        n, p, q, H = self.n, self.p, self.q, self.H
        D, D2, G = self.D, self.D2, self.G
        s = (2.0 / H) ** 2
        rows, cols, vals = [], [], []
        for ey in range(n):
            for ex in range(n):
                e = self.elem(ex, ey)
                for j in range(1, p - 1):
                    for i in range(1, p - 1):
                        g = G[e, j, i]
                        for k in range(p):
                            rows.append(g); cols.append(G[e, j, k]); vals.append(s * D2[i, k])
                            rows.append(g); cols.append(G[e, k, i]); vals.append(s * D2[j, k])
                        rows.append(g); cols.append(g); vals.append(-sigma_int[g])
                eL = self.elem(ex - 1, ey)
                eB = self.elem(ex, ey - 1)
                for j in range(1, p - 1):          # left edge of e
                    g = G[e, j, 0]
                    for k in range(p):
                        rows.append(g); cols.append(G[eL, j, k]); vals.append((2.0 / H) * D[p - 1, k])
                        rows.append(g); cols.append(G[e, j, k]); vals.append(-(2.0 / H) * D[0, k])
                for i in range(1, p - 1):          # bottom edge of e
                    g = G[e, 0, i]
                    for k in range(p):
                        rows.append(g); cols.append(G[eB, k, i]); vals.append((2.0 / H) * D[p - 1, k])
                        rows.append(g); cols.append(G[e, k, i]); vals.append(-(2.0 / H) * D[0, k])
        B = sp.coo_matrix((np.array(vals, dtype=complex), (rows, cols)), shape=(self.N, self.N))
        return B.tocsc()

    # -- derivatives of a nodal field --------------------------------------
    def grad(self, u):
        """(du/dx, du/dy) at every global node (reading R8).

        interior nodes: spectral differentiation along the element's row/column;
        edge nodes: normal derivative = mean of the two one-sided spectral
        derivatives; tangential derivative = differentiation of the degree-(p-1)
        interpolant through the p-2 edge nodes and the nearest node of each
        collinear neighbour edge (matrix Dw, nodes s_edge).
        """
        n, p, q, H = self.n, self.p, self.q, self.H
        D, Dw, G = self.D, self.Dw, self.G
        c = 2.0 / H
        u = np.asarray(u)
        ux = np.zeros(self.N, dtype=u.dtype)
        uy = np.zeros(self.N, dtype=u.dtype)
        for ey in range(n):
            for ex in range(n):
                e = self.elem(ex, ey)
                eL = self.elem(ex - 1, ey)
                eB = self.elem(ex, ey - 1)
                for j in range(1, p - 1):
                    for i in range(1, p - 1):
                        g = G[e, j, i]
                        ux[g] = c * sum(D[i, k] * u[G[e, j, k]] for k in range(p))
                        uy[g] = c * sum(D[j, k] * u[G[e, k, i]] for k in range(p))
                for j in range(1, p - 1):   # left edge
                    g = G[e, j, 0]
                    right_side = c * sum(D[0, k] * u[G[e, j, k]] for k in range(p))
                    left_side = c * sum(D[p - 1, k] * u[G[eL, j, k]] for k in range(p))
                    ux[g] = 0.5 * (right_side + left_side)
                    line = [u[G[eB, p - 2, 0]]] + [u[G[e, l, 0]] for l in range(1, p - 1)] \
                        + [u[G[self.elem(ex, ey + 1), 1, 0]]]
                    uy[g] = c * sum(Dw[j - 1, l] * line[l] for l in range(p))
                for i in range(1, p - 1):   # bottom edge
                    g = G[e, 0, i]
                    top_side = c * sum(D[0, k] * u[G[e, k, i]] for k in range(p))
                    bot_side = c * sum(D[p - 1, k] * u[G[eB, k, i]] for k in range(p))
                    uy[g] = 0.5 * (top_side + bot_side)
                    line = [u[G[eL, 0, p - 2]]] + [u[G[e, 0, l]] for l in range(1, p - 1)] \
                        + [u[G[self.elem(ex + 1, ey), 0, 1]]]
                    ux[g] = c * sum(Dw[i - 1, l] * line[l] for l in range(p))
        return ux, uy

    def grad_matrices(self):
        """Sparse matrices Gx, Gy with Gx @ u == grad(u)[0] (same definition, assembled)."""
        n, p, q, H = self.n, self.p, self.q, self.H
        D, Dw, G = self.D, self.Dw, self.G
        c = 2.0 / H
        rx, cx, vx, ry, cy, vy = [], [], [], [], [], []
        for ey in range(n):
            for ex in range(n):
                e = self.elem(ex, ey)
                eL = self.elem(ex - 1, ey)
                eB = self.elem(ex, ey - 1)
                for j in range(1, p - 1):
                    for i in range(1, p - 1):
                        g = G[e, j, i]
                        for k in range(p):
                            rx.append(g); cx.append(G[e, j, k]); vx.append(c * D[i, k])
                            ry.append(g); cy.append(G[e, k, i]); vy.append(c * D[j, k])
                for j in range(1, p - 1):
                    g = G[e, j, 0]
                    for k in range(p):
                        rx.append(g); cx.append(G[e, j, k]); vx.append(0.5 * c * D[0, k])
                        rx.append(g); cx.append(G[eL, j, k]); vx.append(0.5 * c * D[p - 1, k])
                    line = [G[eB, p - 2, 0]] + [G[e, l, 0] for l in range(1, p - 1)] + [G[self.elem(ex, ey + 1), 1, 0]]
                    for l in range(p):
                        ry.append(g); cy.append(line[l]); vy.append(c * Dw[j - 1, l])
                for i in range(1, p - 1):
                    g = G[e, 0, i]
                    for k in range(p):
                        ry.append(g); cy.append(G[e, k, i]); vy.append(0.5 * c * D[0, k])
                        ry.append(g); cy.append(G[eB, k, i]); vy.append(0.5 * c * D[p - 1, k])
                    line = [G[eL, 0, p - 2]] + [G[e, 0, l] for l in range(1, p - 1)] + [G[self.elem(ex + 1, ey), 0, 1]]
                    for l in range(p):
                        rx.append(g); cx.append(line[l]); vx.append(c * Dw[i - 1, l])
        Gx = sp.coo_matrix((vx, (rx, cx)), shape=(self.N, self.N)).tocsr()
        Gy = sp.coo_matrix((vy, (ry, cy)), shape=(self.N, self.N)).tocsr()
        return Gx, Gy

    def quadrature_weights(self):
        """Nodal weights for a discrete L2 norm (used only for diagnostics):
        tensor Clenshaw-Curtis-free trapezoid-like weights, H^2/(p-1)^2 per node."""
        return np.full(self.N, (self.H / (self.p - 1)) ** 2)

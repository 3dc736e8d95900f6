// Spectral-element mesh (§2.2, Fig. 1) and the nested-dissection /
// HPS merge tree (§2.3): index lists that the factorization and the
// device kernels share.  Restated from the paper; shares no code with oracle/.
#include <cmath>

#include "rexp_internal.hpp"

namespace rexp {

std::vector<double> lagrange_diff(const std::vector<double>& t) {
    const int n = static_cast<int>(t.size());
    std::vector<double> w(n), D(n * n, 0.0);
    for (int k = 0; k < n; ++k) {
        double prod = 1.0;
        for (int l = 0; l < n; ++l)
            if (l != k) prod *= (t[k] - t[l]);
        w[k] = 1.0 / prod;
    }
    for (int i = 0; i < n; ++i) {
        double diag = 0.0;
        for (int k = 0; k < n; ++k) {
            if (k == i) continue;
            const double v = (w[k] / w[i]) / (t[i] - t[k]);
            D[i * n + k] = v;
            diag -= v;
        }
        D[i * n + i] = diag;
    }
    return D;
}

Cheb make_cheb(int p) {
    constexpr double kPi = 3.14159265358979323846;
    Cheb c;
    c.p = p;
    c.t.resize(p);
    for (int k = 0; k < p; ++k) c.t[k] = -std::cos(kPi * k / (p - 1));
    c.D = lagrange_diff(c.t);
    c.D2.assign(p * p, 0.0);
    for (int i = 0; i < p; ++i)
        for (int k = 0; k < p; ++k) {
            double s = 0.0;
            for (int l = 0; l < p; ++l) s += c.D[i * p + l] * c.D[l * p + k];
            c.D2[i * p + k] = s;
        }
    // Reading R8: tangential derivative along an edge from the p-2 edge nodes and
    // the nearest node of each collinear neighbour edge: nodes (-1-eps, t_1..t_{p-2}, 1+eps).
    const double eps = 1.0 + c.t[1];
    std::vector<double> s(p);
    s[0] = -1.0 - eps;
    for (int k = 1; k <= p - 2; ++k) s[k] = c.t[k];
    s[p - 1] = 1.0 + eps;
    const std::vector<double> Ds = lagrange_diff(s);
    c.Dw.assign((p - 2) * p, 0.0);
    for (int r = 0; r < p - 2; ++r)
        for (int k = 0; k < p; ++k) c.Dw[r * p + k] = Ds[(r + 1) * p + k];
    return c;
}

namespace {

struct BoxGeom {
    int n, q;
    int64_t NV;
    int elem(int ex, int ey) const { return ((ey % n + n) % n) * n + ((ex % n + n) % n); }
    // global edge index (V block first, then H block) of the boundary of box at
    // element offset (x0, y0), size a x b, position pos in [bottom, right, top, left]
    int32_t gedge(int x0, int y0, int a, int b, int pos) const {
        const int seg_b = a * q, seg_r = b * q;
        if (pos < seg_b) {  // bottom
            const int s = pos / q, i = pos % q;
            return static_cast<int32_t>(NV + static_cast<int64_t>(elem(x0 + s, y0)) * q + i);
        }
        pos -= seg_b;
        if (pos < seg_r) {  // right
            const int s = pos / q, j = pos % q;
            return static_cast<int32_t>(static_cast<int64_t>(elem(x0 + a, y0 + s)) * q + j);
        }
        pos -= seg_r;
        if (pos < seg_b) {  // top
            const int s = pos / q, i = pos % q;
            return static_cast<int32_t>(NV + static_cast<int64_t>(elem(x0 + s, y0 + b)) * q + i);
        }
        pos -= seg_b;
        {  // left
            const int s = pos / q, j = pos % q;
            return static_cast<int32_t>(static_cast<int64_t>(elem(x0, y0 + s)) * q + j);
        }
    }
};

}  // namespace

int build_tree(int n, int p, Tree& T) {
    if (n < 2 || (n & (n - 1)) != 0 || n > 1024) {
        set_error("n must be a power of two in [2, 1024]");
        return REXP_EINVAL;
    }
    if (p < 4 || p > 32) {
        set_error("p must be in [4, 32]");
        return REXP_EINVAL;
    }
    const int q = p - 2;
    T.n = n;
    T.p = p;
    T.q = q;
    T.nelem = n * n;
    T.NI = static_cast<int64_t>(T.nelem) * q * q;
    T.NV = static_cast<int64_t>(T.nelem) * q;
    T.NH = T.NV;
    T.N = T.NI + T.NV + T.NH;
    T.NE = T.NV + T.NH;
    if (T.N >= (int64_t(1) << 31)) {
        set_error("mesh too large for 32-bit node indices");
        return REXP_EINVAL;
    }
    BoxGeom bg{n, q, T.NV};

    // element-local -> global map and coordinates
    const Cheb ch = make_cheb(p);
    const double H = 1.0 / n;
    T.elem_g.assign(static_cast<size_t>(T.nelem) * p * p, -1);
    T.x.assign(T.N, 0.0);
    T.y.assign(T.N, 0.0);
    for (int ey = 0; ey < n; ++ey)
        for (int ex = 0; ex < n; ++ex) {
            const int e = ey * n + ex;
            for (int j = 0; j < p; ++j)
                for (int i = 0; i < p; ++i) {
                    const bool ci = (i == 0 || i == p - 1), cj = (j == 0 || j == p - 1);
                    int64_t g = -1;
                    if (!ci && !cj) {
                        g = static_cast<int64_t>(e) * q * q + (j - 1) * q + (i - 1);
                    } else if (ci && !cj) {
                        const int ev = bg.elem(i == 0 ? ex : ex + 1, ey);
                        g = T.NI + static_cast<int64_t>(ev) * q + (j - 1);
                    } else if (!ci && cj) {
                        const int eh = bg.elem(ex, j == 0 ? ey : ey + 1);
                        g = T.NI + T.NV + static_cast<int64_t>(eh) * q + (i - 1);
                    }
                    T.elem_g[static_cast<size_t>(e) * p * p + j * p + i] = static_cast<int32_t>(g);
                    if (g >= 0) {
                        T.x[g] = std::fmod(ex * H + (ch.t[i] + 1.0) * H / 2.0, 1.0);
                        T.y[g] = std::fmod(ey * H + (ch.t[j] + 1.0) * H / 2.0, 1.0);
                    }
                }
        }

    // leaf boundary: [bottom, right, top, left], same convention as boxes
    T.leaf_gB.resize(static_cast<size_t>(T.nelem) * 4 * q);
    for (int ey = 0; ey < n; ++ey)
        for (int ex = 0; ex < n; ++ex) {
            const int e = ey * n + ex;
            for (int pos = 0; pos < 4 * q; ++pos)
                T.leaf_gB[static_cast<size_t>(e) * 4 * q + pos] = bg.gedge(ex, ey, 1, 1, pos);
        }

    // merge levels.  Boxes alternate x- and y-merges; the x-merge that reaches the
    // full width n closes the periodic x seam at the same time (both vertical
    // interfaces, a.right|b.left and a.left|b.right), leaving a cylinder whose
    // boundary is [bottom, top] only; the root then merges the two cylinders
    // across both horizontal interfaces (DESIGN.md §6 "periodic closure").
    T.levels.clear();
    int ac = 1, bc = 1;
    int lev = 0;
    bool cylinder = false;
    while (!cylinder) {
        MergeLevel L;
        L.dir = (lev % 2 == 0) ? 0 : 1;
        L.a = L.dir == 0 ? 2 * ac : ac;
        L.b = L.dir == 0 ? bc : 2 * bc;
        cylinder = L.dir == 0 && L.a == n;
        L.nbx = n / L.a;
        L.nby = n / L.b;
        L.nodes = L.nbx * L.nby;
        L.nchild = 2 * (ac + bc) * q;
        L.child_nodes = (n / ac) * (n / bc);
        L.next = cylinder ? 2 * L.a * q : 2 * (L.a + L.b) * q;
        const int cbx = n / ac;  // child boxes per row
        // child boundary offsets
        const int c_bot = 0, c_right = ac * q, c_top = (ac + bc) * q, c_left = (2 * ac + bc) * q;
        std::vector<std::pair<int, int>> order;  // parent position -> (child 0/1, child pos)
        if (cylinder) {
            L.n3 = 2 * bc * q;
            for (int t = 0; t < bc * q; ++t) {      // middle seam
                L.ia3_pos.push_back(c_right + t);
                L.ib3_pos.push_back(c_left + t);
            }
            for (int t = 0; t < bc * q; ++t) {      // periodic x seam
                L.ia3_pos.push_back(c_left + t);
                L.ib3_pos.push_back(c_right + t);
            }
            for (int t = 0; t < ac * q; ++t) order.push_back({0, c_bot + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({1, c_bot + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({0, c_top + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({1, c_top + t});
        } else if (L.dir == 0) {
            L.n3 = bc * q;
            for (int t = 0; t < L.n3; ++t) {
                L.ia3_pos.push_back(c_right + t);
                L.ib3_pos.push_back(c_left + t);
            }
            for (int t = 0; t < ac * q; ++t) order.push_back({0, c_bot + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({1, c_bot + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({1, c_right + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({0, c_top + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({1, c_top + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({0, c_left + t});
        } else {
            L.n3 = ac * q;
            for (int t = 0; t < L.n3; ++t) {
                L.ia3_pos.push_back(c_top + t);
                L.ib3_pos.push_back(c_bot + t);
            }
            for (int t = 0; t < ac * q; ++t) order.push_back({0, c_bot + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({0, c_right + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({1, c_right + t});
            for (int t = 0; t < ac * q; ++t) order.push_back({1, c_top + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({0, c_left + t});
            for (int t = 0; t < bc * q; ++t) order.push_back({1, c_left + t});
        }
        if (static_cast<int>(order.size()) != L.next) {
            set_error("internal: merge ordering size mismatch");
            return REXP_EINVAL;
        }
        L.ia3.resize(static_cast<size_t>(L.nodes) * L.n3);
        L.ib3.resize(static_cast<size_t>(L.nodes) * L.n3);
        L.g3.resize(static_cast<size_t>(L.nodes) * L.n3);
        L.ext.resize(static_cast<size_t>(L.nodes) * L.next);
        L.ext_is_b.resize(static_cast<size_t>(L.nodes) * L.next);
        L.ext_pos.resize(static_cast<size_t>(L.nodes) * L.next);
        L.gext.resize(static_cast<size_t>(L.nodes) * L.next);
        for (int by = 0; by < L.nby; ++by)
            for (int bx = 0; bx < L.nbx; ++bx) {
                const int node = by * L.nbx + bx;
                int ca_x, ca_y, cb_x, cb_y;
                if (L.dir == 0) {
                    ca_x = 2 * bx; ca_y = by; cb_x = 2 * bx + 1; cb_y = by;
                } else {
                    ca_x = bx; ca_y = 2 * by; cb_x = bx; cb_y = 2 * by + 1;
                }
                const int ca = ca_y * cbx + ca_x, cb = cb_y * cbx + cb_x;
                const int x0 = bx * L.a, y0 = by * L.b;
                const int ax0 = ca_x * ac, ay0 = ca_y * bc;
                for (int t = 0; t < L.n3; ++t) {
                    L.ia3[static_cast<size_t>(node) * L.n3 + t] = ca * L.nchild + L.ia3_pos[t];
                    L.ib3[static_cast<size_t>(node) * L.n3 + t] = cb * L.nchild + L.ib3_pos[t];
                    const int32_t g = bg.gedge(ax0, ay0, ac, bc, L.ia3_pos[t]);
                    L.g3[static_cast<size_t>(node) * L.n3 + t] = g;
                    const int bx0 = cb_x * ac, by0 = cb_y * bc;
                    if (bg.gedge(bx0, by0, ac, bc, L.ib3_pos[t]) != g) {
                        set_error("internal: interface node mismatch");
                        return REXP_EINVAL;
                    }
                }
                for (int r = 0; r < L.next; ++r) {
                    const int c = order[r].first, cpos = order[r].second;
                    const size_t o = static_cast<size_t>(node) * L.next + r;
                    L.ext[o] = (c == 0 ? ca : cb) * L.nchild + cpos;
                    L.ext_is_b[o] = c;
                    L.ext_pos[o] = cpos;
                    // cylinder boundary [bottom, top]: skip the box's right side
                    const int bpos = (cylinder && r >= L.a * q) ? r + L.b * q : r;
                    L.gext[o] = bg.gedge(x0, y0, L.a, L.b, bpos);
                    const int cx0 = (c == 0 ? ca_x : cb_x) * ac, cy0 = (c == 0 ? ca_y : cb_y) * bc;
                    if (bg.gedge(cx0, cy0, ac, bc, cpos) != L.gext[o]) {
                        set_error("internal: parent/child boundary mismatch");
                        return REXP_EINVAL;
                    }
                }
            }
        T.levels.push_back(std::move(L));
        ac = T.levels.back().a;
        bc = T.levels.back().b;
        ++lev;
    }
    // root: cylinder 0 (y0 = 0) and cylinder 1 (y0 = n/2) meet on the middle seam
    // (0.top | 1.bottom) and the periodic y seam (0.bottom | 1.top); positions are
    // flat indices into the cylinder level's boundary array, pos1 in cylinder 0
    // and pos2 in cylinder 1
    const MergeLevel& C = T.levels.back();
    if (C.nodes != 2 || C.next != 2 * n * q) {
        set_error("internal: cylinder level shape");
        return REXP_EINVAL;
    }
    const int nq = n * q;
    T.ns = 2 * nq;
    T.root_pos1.resize(T.ns);
    T.root_pos2.resize(T.ns);
    T.root_gs.resize(T.ns);
    for (int t = 0; t < nq; ++t) {
        T.root_pos1[t] = nq + t;                // cylinder 0 top
        T.root_pos2[t] = C.next + t;            // cylinder 1 bottom
        T.root_pos1[nq + t] = t;                // cylinder 0 bottom
        T.root_pos2[nq + t] = C.next + nq + t;  // cylinder 1 top
    }
    for (int s = 0; s < T.ns; ++s) {
        T.root_gs[s] = C.gext[T.root_pos1[s]];
        if (C.gext[T.root_pos2[s]] != T.root_gs[s]) {
            set_error("internal: periodic seam mismatch");
            return REXP_EINVAL;
        }
    }
    return REXP_OK;
}

}  // namespace rexp

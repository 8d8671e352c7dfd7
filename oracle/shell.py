"""Discrete-shell oracle for BASELINE config 4 (test infrastructure only).

Energies (vectorized over elements, written once and evaluated on hyper-dual numbers, so
gradients and second derivatives -- d2E/dx2 and the rest-shape block d2E/dx dX -- are exact):

* StVK membrane triangle (plane stress): E_m = t A [alpha/2 tr(G)^2 + beta tr(G^2)] with the
  Green strain G = 1/2 (Abar^{-1} a - I) from the deformed / rest first fundamental forms,
  alpha = E nu / (1 - nu^2), beta = E / (2 (1 + nu)); plus self-weight rho g t A/3 sum z
  (lumped by rest area, gravity along -z).
* Dihedral hinge (Discrete Shells): E_b = k_b (theta - theta_bar)^2 3 |e_bar|^2 /
  (A1_bar + A2_bar), k_b = E t^3 / (24 (1 - nu^2)), theta = atan2(((n1 x n2) . e)/|e|, n1 . n2)
  for the hinge (x0, x1 | x2, x3): triangles (x0, x1, x2) and (x1, x0, x3).

The reference package has no shell element; these are validated by finite
differences (tests/test_oracle.py) and independently re-implemented in CUDA.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .sgn_cpu import Csc, csc_structural, solve_static


class HD:
    """Hyper-dual numbers a + b e1 + c e2 + d e1 e2 (e1^2 = e2^2 = 0), elementwise arrays."""

    __slots__ = ("a", "b", "c", "d")

    def __init__(self, a, b=0.0, c=0.0, d=0.0):
        self.a, self.b, self.c, self.d = a, b, c, d

    @staticmethod
    def lift(v):
        return v if isinstance(v, HD) else HD(v)

    def __add__(self, o):
        o = HD.lift(o)
        return HD(self.a + o.a, self.b + o.b, self.c + o.c, self.d + o.d)

    __radd__ = __add__

    def __neg__(self):
        return HD(-self.a, -self.b, -self.c, -self.d)

    def __sub__(self, o):
        return self + (-HD.lift(o))

    def __rsub__(self, o):
        return HD.lift(o) - self

    def __mul__(self, o):
        o = HD.lift(o)
        return HD(self.a * o.a, self.a * o.b + self.b * o.a, self.a * o.c + self.c * o.a,
                  self.a * o.d + self.b * o.c + self.c * o.b + self.d * o.a)

    __rmul__ = __mul__

    def _f(self, f0, f1, f2):
        """Chain rule for a scalar function with value f0, f' = f1, f'' = f2."""
        return HD(f0, f1 * self.b, f1 * self.c, f1 * self.d + f2 * self.b * self.c)

    def recip(self):
        return self._f(1.0 / self.a, -1.0 / self.a ** 2, 2.0 / self.a ** 3)

    def __truediv__(self, o):
        return self * HD.lift(o).recip()

    def __rtruediv__(self, o):
        return HD.lift(o) * self.recip()

    def sqrt(self):
        s = np.sqrt(self.a)
        return self._f(s, 0.5 / s, -0.25 / (s * self.a))


def hd_atan2(y: HD, x: HD) -> HD:
    r2 = x.a * x.a + y.a * y.a
    fy, fx = x.a / r2, -y.a / r2
    fyy, fxx, fxy = -2.0 * x.a * y.a / r2 ** 2, 2.0 * x.a * y.a / r2 ** 2, (y.a ** 2 - x.a ** 2) / r2 ** 2
    return HD(np.arctan2(y.a, x.a), fy * y.b + fx * x.b, fy * y.c + fx * x.c,
              fy * y.d + fx * x.d + fyy * y.b * y.c + fxy * (y.b * x.c + y.c * x.b) + fxx * x.b * x.c)


def _dot(u, v):
    return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]


def _cross(u, v):
    return [u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]]


def _sub(u, v):
    return [u[0] - v[0], u[1] - v[1], u[2] - v[2]]


def membrane_energy(x, X, t, alpha, beta, rho_g):
    """x, X: [vertex][axis] lists of arrays/HD (3 vertices)."""
    e1, e2 = _sub(x[1], x[0]), _sub(x[2], x[0])
    E1, E2 = _sub(X[1], X[0]), _sub(X[2], X[0])
    a00, a01, a11 = _dot(e1, e1), _dot(e1, e2), _dot(e2, e2)
    b00, b01, b11 = _dot(E1, E1), _dot(E1, E2), _dot(E2, E2)
    det = b00 * b11 - b01 * b01
    area = 0.5 * (det.sqrt() if isinstance(det, HD) else np.sqrt(det))
    # M = Abar^{-1} a
    m00 = (b11 * a00 - b01 * a01) / det
    m01 = (b11 * a01 - b01 * a11) / det
    m10 = (b00 * a01 - b01 * a00) / det
    m11 = (b00 * a11 - b01 * a01) / det
    trG = 0.5 * (m00 + m11 - 2.0)
    trG2 = 0.25 * ((m00 - 1.0) * (m00 - 1.0) + 2.0 * m01 * m10 + (m11 - 1.0) * (m11 - 1.0))
    psi = 0.5 * alpha * trG * trG + beta * trG2
    zsum = x[0][2] + x[1][2] + x[2][2]
    return t * area * psi + (rho_g * t / 3.0) * area * zsum


def _theta(x0, x1, x2, x3):
    e = _sub(x1, x0)
    n1 = _cross(e, _sub(x2, x0))
    n2 = _cross(_sub(x3, x0), e)
    le = _dot(e, e)
    le = le.sqrt() if isinstance(le, HD) else np.sqrt(le)
    s = _dot(_cross(n1, n2), e) / le
    c = _dot(n1, n2)
    if isinstance(s, HD) or isinstance(c, HD):
        return hd_atan2(HD.lift(s), HD.lift(c)), n1, n2, e
    return np.arctan2(s, c), n1, n2, e


def hinge_energy(x, X, kb):
    th, _, _, _ = _theta(*x)
    thb, n1b, n2b, eb = _theta(*X)
    l2 = _dot(eb, eb)
    a1 = _dot(n1b, n1b)
    a2 = _dot(n2b, n2b)
    a1 = 0.5 * (a1.sqrt() if isinstance(a1, HD) else np.sqrt(a1))
    a2 = 0.5 * (a2.sqrt() if isinstance(a2, HD) else np.sqrt(a2))
    d = th - thb
    return kb * d * d * (3.0 * l2 / (a1 + a2))


def _as_lists(P):
    """(ne, nv, 3) -> [vertex][axis] arrays."""
    return [[P[:, v, i] for i in range(3)] for v in range(P.shape[1])]


def element_derivs(energy, xe, Xe, *args):
    """(grad[ne, nd], hess[ne, nd, nd], mixed[ne, nd, nd]) by hyper-dual evaluation."""
    ne, nv, _ = xe.shape
    nd = nv * 3
    grad = np.empty((ne, nd))
    hess = np.empty((ne, nd, nd))
    mixed = np.empty((ne, nd, nd))
    base_x, base_X = _as_lists(xe), _as_lists(Xe)

    for i in range(nd):
        for j in range(i, nd):
            xs = [[HD(base_x[v][a]) for a in range(3)] for v in range(nv)]
            vi, ai = divmod(i, 3)
            vj, aj = divmod(j, 3)
            xs[vi][ai] = HD(base_x[vi][ai], np.ones(ne), 0.0, 0.0)
            cur = xs[vj][aj]
            xs[vj][aj] = HD(cur.a, cur.b, np.ones(ne), 0.0)
            E = energy(xs, [[HD(base_X[v][a]) for a in range(3)] for v in range(nv)], *args)
            hess[:, i, j] = hess[:, j, i] = E.d
            if j == i:
                grad[:, i] = E.b
        for j in range(nd):
            xs = [[HD(base_x[v][a]) for a in range(3)] for v in range(nv)]
            Xs = [[HD(base_X[v][a]) for a in range(3)] for v in range(nv)]
            vi, ai = divmod(i, 3)
            vj, aj = divmod(j, 3)
            xs[vi][ai] = HD(base_x[vi][ai], np.ones(ne), 0.0, 0.0)
            Xs[vj][aj] = HD(base_X[vj][aj], 0.0, np.ones(ne), 0.0)
            mixed[:, i, j] = energy(xs, Xs, *args).d
    return grad, hess, mixed


def element_energy(energy, xe, Xe, *args):
    return energy(_as_lists(xe), _as_lists(Xe), *args)


# ------------------------------------------------------------------------------------
# config 4 spec and problem
# ------------------------------------------------------------------------------------
def shell_spec(n: int = 201, nc: int = 100, L: float = 1.0, t: float = 0.05, E: float = 3e10,
               nu: float = 0.2, rho: float = 2400.0, g: float = 9.81, w_reg: float = 2e-4):
    """Config 4 (n = 201, nc = 100): n x n triangulated square (quad split along
    (i,j)-(i+1,j+1), vid = i*n + j), four corners pinned, rest heights z = bilinear
    interpolation of an nc x nc control lattice spanning the square (SURVEY 0.9 iv: control
    point (a, b) at (a, b) L/(nc-1); zero weights dropped), objective 0.5 sum over free vertices
    of (x_z - X_z(p))^2 + 1e-4 |p|^2 (w_reg = 2e-4)."""
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    X0 = np.column_stack([ii.ravel() * L / (n - 1), jj.ravel() * L / (n - 1), np.zeros(n * n)])
    i, j = np.meshgrid(np.arange(n - 1), np.arange(n - 1), indexing="ij")
    a = (i * n + j).ravel(); b = ((i + 1) * n + j).ravel()
    c = ((i + 1) * n + j + 1).ravel(); d = (i * n + j + 1).ravel()
    tris = np.stack([np.column_stack([a, b, c]), np.column_stack([a, c, d])], axis=1).reshape(-1, 3)
    # hinges from interior edges: (u, v | w1, w2), triangle (u, v, w1) and (v, u, w2) both CCW
    edge_owner = {}
    hinges = []
    for tri in tris:
        for k in range(3):
            u, v, w = int(tri[k]), int(tri[(k + 1) % 3]), int(tri[(k + 2) % 3])
            if (v, u) in edge_owner:
                hinges.append((v, u, edge_owner.pop((v, u)), w))
            else:
                edge_owner[(u, v)] = w
    hinges = np.array(sorted(hinges), dtype=np.int64)
    corners = np.array([0, n - 1, (n - 1) * n, n * n - 1])
    h = L / (nc - 1)
    pm_dof, pm_p, pm_coef = [], [], []
    for v in range(n * n):
        x, y = X0[v, 0], X0[v, 1]
        ca, cb = min(int(np.floor(x / h + 1e-12)), nc - 2), min(int(np.floor(y / h + 1e-12)), nc - 2)
        s, tt = x / h - ca, y / h - cb
        for (da, db, wgt) in ((0, 0, (1 - s) * (1 - tt)), (1, 0, s * (1 - tt)), (0, 1, (1 - s) * tt), (1, 1, s * tt)):
            if wgt > 1e-14:
                pm_dof.append(3 * v + 2)
                pm_p.append((ca + da) * nc + (cb + db))
                pm_coef.append(wgt)
    free = np.setdiff1d(np.arange(n * n), corners)
    v2f = -np.ones(n * n, dtype=np.int64)
    v2f[free] = np.arange(free.size)
    tdofs = v2f[free] * 3 + 2                   # z dof of every free vertex, in x numbering
    alpha, beta = E * nu / (1 - nu ** 2), E / (2 * (1 + nu))
    kb = E * t ** 3 / (24 * (1 - nu ** 2))
    return dict(X0=X0, tris=tris, hinges=hinges, fixed_verts=corners,
                pmap=(np.array(pm_dof), np.array(pm_p), np.array(pm_coef)), target_dofs=tdofs,
                target_vals=np.zeros(tdofs.size), w_target=1.0, w_reg=w_reg, E=E, t=t, nu=nu,
                alpha=alpha, beta=beta, kb=kb, rho_g=rho * g, n_p=nc * nc, p0=np.zeros(nc * nc),
                name=f"shell_{n}x{n}_c{nc}")


SHELL_DISP_SCALE = 1e-3      # state = displacement from X(p) in millimetres (as the product)


class ShellProblem:
    """Oracle shell problem (membrane + hinge groups).

    Contract = reference sensitivity.py:29-120.  State x = displacement of the free dofs from
    the p-dependent rest shape, in millimetres: pos = X(p) + sigma x (sigma = 1e-3; fixed
    corners stay at X0).  Residual r = sigma x_z (the vertical displacement in metres) and
    p (regularizer); constraints c = s dE/dpos on the free dofs, with s the inverse geometric
    mean of the membrane and lowest bending stiffness; dc/dx = s sigma H_ff and dc/dp =
    s (H_f,free P_free + M P) (M = d2E/dpos dX).  DESIGN.md section 6 says why this state."""

    def __init__(self, spec, tol=None):
        self.s = spec
        self.X0 = spec["X0"]
        self.n_v = self.X0.shape[0]
        fixed = np.zeros(self.n_v, bool)
        fixed[spec["fixed_verts"]] = True
        self.free_verts = np.flatnonzero(~fixed)
        self.free_dofs = (self.free_verts[:, None] * 3 + np.arange(3)[None, :]).ravel()
        self.n_x = self.free_dofs.size
        self.n_p = int(spec["n_p"])
        self.dof_to_x = -np.ones(self.n_v * 3, dtype=np.int64)
        self.dof_to_x[self.free_dofs] = np.arange(self.n_x)
        pm_dof, pm_p, pm_coef = spec["pmap"]
        self.P = sp.csr_matrix((pm_coef, (pm_dof, pm_p)), shape=(self.n_v * 3, self.n_p))
        self.Pf = sp.csr_matrix(self.P[self.free_dofs])          # free rest dofs <- p
        self.tdofs = spec["target_dofs"]
        self.sigma = SHELL_DISP_SCALE
        n = int(round(np.sqrt(self.n_v)))
        h = 1.0 / (n - 1)
        D = spec["E"] * spec["t"] ** 3 / (12.0 * (1.0 - spec["nu"] ** 2))
        self.scale = 1.0 / np.sqrt(spec["E"] * spec["t"] * D * np.pi ** 4 * h * h)
        self.tol = tol if tol is not None else 1e-4 * self.scale * spec["rho_g"] * spec["t"] * h * h
        self.groups = [("membrane", spec["tris"]), ("hinge", spec["hinges"])]
        self._x_warm = None

    @property
    def n_c(self):
        return self.n_x

    def bounds(self):
        return None

    def rest_positions(self, p):
        return (self.X0.ravel() + self.P @ np.asarray(p, dtype=np.float64)).reshape(-1, 3)

    def full_positions(self, x, p):
        pos = self.X0.ravel().copy()
        pos[self.free_dofs] = self.rest_positions(p).ravel()[self.free_dofs] + self.sigma * np.asarray(x)
        return pos.reshape(-1, 3)

    def _energy_args(self, kind):
        s = self.s
        return (membrane_energy, (s["t"], s["alpha"], s["beta"], s["rho_g"])) if kind == "membrane" \
            else (hinge_energy, (s["kb"],))

    def _grad_full(self, pos, rest):
        g = np.zeros(self.n_v * 3)
        for kind, conn in self.groups:
            fn, args = self._energy_args(kind)
            # gradient via first-order hyper-dual passes (b part)
            nd = conn.shape[1] * 3
            ge = np.empty((conn.shape[0], nd))
            base_x, base_X = _as_lists(pos[conn]), _as_lists(rest[conn])
            Xs = [[HD(base_X[v][a]) for a in range(3)] for v in range(conn.shape[1])]
            for k in range(nd):
                xs = [[HD(base_x[v][a]) for a in range(3)] for v in range(conn.shape[1])]
                v, a = divmod(k, 3)
                xs[v][a] = HD(base_x[v][a], np.ones(conn.shape[0]))
                ge[:, k] = fn(xs, Xs, *args).b
            dofs = (conn[:, :, None] * 3 + np.arange(3)[None, None, :]).reshape(conn.shape[0], -1)
            np.add.at(g, dofs.ravel(), ge.ravel())
        return g

    def _energy_full(self, pos, rest):
        e = 0.0
        for kind, conn in self.groups:
            fn, args = self._energy_args(kind)
            e += float(np.sum(element_energy(fn, pos[conn], rest[conn], *args)))
        return e

    def _blocks(self, pos, rest):
        out = []
        for kind, conn in self.groups:
            fn, args = self._energy_args(kind)
            _, H, M = element_derivs(fn, pos[conn], rest[conn], *args)
            dofs = (conn[:, :, None] * 3 + np.arange(3)[None, None, :]).reshape(conn.shape[0], -1)
            out.append((dofs, H, M))
        return out

    def simulate(self, p, x_init=None):
        """Static equilibrium in the displacement state (forward.py:135-168 with the energy
        s E(X(p) + sigma x): gradient sigma c, Hessian sigma dc/dx; the stopping test on c is
        the problem's tolerance, as on the device)."""
        rest = self.rest_positions(p)
        s, sg = self.scale, self.sigma

        def energy(xf):
            return s * self._energy_full(self.full_positions(xf, p), rest)

        def gradient(xf):
            return sg * s * self._grad_full(self.full_positions(xf, p), rest)[self.free_dofs]

        def hessian(xf):
            return sg * sg * s * self._hess_ff(self.full_positions(xf, p), rest)

        start = x_init if x_init is not None else (self._x_warm if self._x_warm is not None
                                                   else np.zeros(self.n_x))
        x = solve_static(energy, gradient, hessian, np.asarray(start, dtype=np.float64), sg * self.tol)
        self._x_warm = x.copy()
        return x

    def constraints(self, x, p):
        return self.scale * self._grad_full(self.full_positions(x, p), self.rest_positions(p))[self.free_dofs]

    def _hess_ff(self, pos, rest):
        rows, cols, vals = [], [], []
        for dofs, H, _ in self._blocks(pos, rest):
            nd = dofs.shape[1]
            r = np.repeat(dofs, nd, axis=1).ravel()
            c = np.tile(dofs, (1, nd)).ravel()
            rx, cx = self.dof_to_x[r], self.dof_to_x[c]
            keep = (rx >= 0) & (cx >= 0)
            rows.append(rx[keep]); cols.append(cx[keep]); vals.append(H.reshape(len(H), -1).ravel()[keep])
        return csc_structural(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals),
                              (self.n_x, self.n_x)).to_scipy()

    def constraint_jac_x(self, x, p):
        return Csc(self.scale * self.sigma * self._hess_ff(self.full_positions(x, p), self.rest_positions(p)))

    def constraint_jac_p(self, x, p):
        """s (H_f,free P_free + M P): element by element, one COO build (no SpGEMM, so the
        pattern is structural)."""
        rows, cols, vals = [], [], []
        Pc, Pf_ = self.P, self.Pf
        for dofs, H, M in self._blocks(self.full_positions(x, p), self.rest_positions(p)):
            ne, nd = dofs.shape
            # element-local (row a, col b) pairs with a free row; each col dof b expands over
            # its p-map entries: coefficient * (M[a, b] + H[a, b] if b is a free dof)
            a_loc = np.repeat(np.arange(nd), nd)
            b_loc = np.tile(np.arange(nd), nd)
            rdof = dofs[:, a_loc].ravel()
            cdof = dofs[:, b_loc].ravel()
            e_id = np.repeat(np.arange(ne), nd * nd)
            rx = self.dof_to_x[rdof]
            cnt = (Pc.indptr[cdof + 1] - Pc.indptr[cdof]) * (rx >= 0)
            sel = np.flatnonzero(cnt)
            rep_ = cnt[sel]
            t = np.repeat(sel, rep_)
            offs = np.arange(rep_.sum()) - np.repeat(np.cumsum(rep_) - rep_, rep_)
            kk = Pc.indptr[cdof[t]] + offs
            loc = (a_loc * nd + b_loc)[t % (nd * nd)]
            m = M.reshape(ne, -1)[e_id[t], loc]
            hv = H.reshape(ne, -1)[e_id[t], loc] * (self.dof_to_x[cdof[t]] >= 0)
            rows.append(rx[t]); cols.append(Pc.indices[kk]); vals.append(Pc.data[kk] * (m + hv))
        return csc_structural(np.concatenate(rows), np.concatenate(cols), self.scale * np.concatenate(vals),
                              (self.n_x, self.n_p))

    # least squares: r = [sigma x_t - target ; p]
    def residuals(self, x, p):
        p = np.asarray(p, dtype=np.float64)
        r = self.sigma * np.asarray(x)[self.tdofs] - self.s["target_vals"]
        return np.concatenate([r, p]) if self.s["w_reg"] > 0 else r

    def weights(self):
        w = [np.full(self.tdofs.size, self.s["w_target"])]
        if self.s["w_reg"] > 0:
            w.append(np.full(self.n_p, self.s["w_reg"]))
        return np.concatenate(w)

    def residual_jac_x(self, x, p):
        nt = self.tdofs.size
        J = sp.csc_matrix((np.full(nt, self.sigma), (np.arange(nt), self.tdofs)), shape=(nt, self.n_x))
        if self.s["w_reg"] > 0:
            J = sp.vstack([J, sp.csc_matrix((self.n_p, self.n_x))], format="csc")
        return Csc(J)

    def residual_jac_p(self, x, p):
        J = sp.csc_matrix((self.tdofs.size, self.n_p))
        if self.s["w_reg"] > 0:
            J = sp.vstack([J, sp.identity(self.n_p)], format="csc")
        return Csc(J)

    def objective(self, x, p):
        r = self.residuals(x, p)
        return float(0.5 * self.weights() @ (r * r))

    def objective_grad_x(self, x, p):
        return self.residual_jac_x(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

    def objective_grad_p(self, x, p):
        return self.residual_jac_p(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

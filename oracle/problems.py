"""Oracle problem classes (NumPy; test infrastructure only).

* ``SpringBarOracle``   -- restatement of the reference's gravity-compensation spring
  lattice (reference pkg/src/sgnopt/problems/spring_bar.py:30-207; kernels
  forward.py:29-111), numerically equivalent, built structurally (triplets, stored
  zeros kept) so its KKT pattern is the structural pattern of the GPU path.
* ``ElementProblem``     -- generic static inverse-design problem on a simplex mesh
  (neo-Hookean triangles/tets) for the BASELINE configs, which the reference does not
  implement.  Contract = sensitivity.py:29-120; assembly idiom =
  spring_bar.py:138-184; statics = forward.py:135-203 with a scaled tolerance
  (SURVEY §0.9 vii); equilibrium rows scaled by 1/E.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import elements as el
from .sgn_cpu import Csc, OracleNoConvergence, csc_structural, solve_static


class _LsqMixin:
    """objective / objective_grad_* derived from the least-squares form (sensitivity.py:83-93)."""

    def objective(self, x, p):
        r = self.residuals(x, p)
        return float(0.5 * self.weights() @ (r * r))

    def objective_grad_x(self, x, p):
        return self.residual_jac_x(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

    def objective_grad_p(self, x, p):
        return self.residual_jac_p(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

    def bounds(self):
        return None

    @property
    def n_c(self):
        return self.n_x

    @property
    def name(self):
        return type(self).__name__


class ElementProblem(_LsqMixin):
    """Static equilibrium inverse design on an element mesh.

    Unknowns x = deformed coordinates of free vertices (dof = vertex*d + axis, vertex
    order).  Parameters p move rest coordinates: X(p)[dof] = X0[dof] + sum coef*p.
    Objective 0.5*sum w_t (x_t - target)^2 + 0.5*w_reg*|p|^2.
    """

    def __init__(self, X0, conn, kind, fixed_verts, pmap, target_dofs, target_vals,
                 w_target=1.0, w_reg=0.0, E=1.0, nu=0.3, gload=0.0, stiffness=None,
                 scale=None, tol=1e-12, grav_const=None):
        self.X0 = np.asarray(X0, dtype=np.float64)
        self.n_v, self.d = self.X0.shape
        self.conn = np.asarray(conn, dtype=np.int64)
        self.kind = kind
        self.nv_el = self.conn.shape[1]
        self.E, self.nu, self.gload = float(E), float(nu), float(gload)
        self.mu, self.lam = el.lame(self.E, self.nu)
        self.stiffness = None if stiffness is None else np.asarray(stiffness, dtype=np.float64)
        self.scale = (1.0 / self.E) if scale is None else float(scale)
        self.tol = float(tol)
        self.grav_const = None if grav_const is None else np.asarray(grav_const, dtype=np.float64)
        fixed = np.zeros(self.n_v, bool)
        fixed[np.asarray(fixed_verts, dtype=np.int64)] = True
        self.fixed_verts = np.flatnonzero(fixed)
        self.free_verts = np.flatnonzero(~fixed)
        d = self.d
        self.free_dofs = (self.free_verts[:, None] * d + np.arange(d)[None, :]).ravel()
        self.n_x = self.free_dofs.size
        self.dof_to_x = -np.ones(self.n_v * d, dtype=np.int64)
        self.dof_to_x[self.free_dofs] = np.arange(self.n_x)
        pm_dof, pm_p, pm_coef = (np.asarray(a) for a in pmap)
        self.pm_dof = pm_dof.astype(np.int64)
        self.pm_p = pm_p.astype(np.int64)
        self.pm_coef = pm_coef.astype(np.float64)
        self.n_p = int(self.pm_p.max()) + 1 if self.pm_p.size else 0
        self.P = sp.csr_matrix((self.pm_coef, (self.pm_dof, self.pm_p)), shape=(self.n_v * d, self.n_p))
        self.target_dofs = np.asarray(target_dofs, dtype=np.int64)   # indices into x
        self.target_vals = np.asarray(target_vals, dtype=np.float64)
        self.w_target = float(w_target)
        self.w_reg = float(w_reg)
        self._x_warm = None
        # element dof table (ne, nd) of global dofs
        self.el_dofs = (self.conn[:, :, None] * d + np.arange(d)[None, None, :]).reshape(len(self.conn), -1)

    # -- geometry -------------------------------------------------------------------
    def rest_positions(self, p):
        X = self.X0.ravel() + self.P @ np.asarray(p, dtype=np.float64)
        return X.reshape(self.n_v, self.d)

    def full_positions(self, x):
        pos = self.X0.ravel().copy()
        pos[self.free_dofs] = x
        return pos.reshape(self.n_v, self.d)

    def default_parameters(self):
        return np.zeros(self.n_p)

    # -- element evaluation ------------------------------------------------------------
    def _el(self, pos, rest):
        return pos[self.conn], rest[self.conn]

    def _energy_full(self, pos, rest):
        xe, Xe = self._el(pos, rest)
        if self.kind == "spring":
            e = el.spring_energy(xe, Xe, self.stiffness).sum()
        else:
            e = el.nh_energy(xe, Xe, self.mu, self.lam, self.gload).sum()
        if self.grav_const is not None:
            e += self.grav_const @ pos.ravel()
        return e

    def _grad_full(self, pos, rest):
        xe, Xe = self._el(pos, rest)
        if self.kind == "spring":
            ge = el.spring_grad(xe, Xe, self.stiffness)
        else:
            ge = el.nh_grad(xe, Xe, self.mu, self.lam, self.gload)
        g = np.zeros(self.n_v * self.d)
        np.add.at(g, self.el_dofs.ravel(), ge.ravel())
        if self.grav_const is not None:
            g += self.grav_const
        return g

    def _second(self, pos, rest):
        xe, Xe = self._el(pos, rest)
        if self.kind == "spring":
            return el.spring_second(xe, Xe, self.stiffness)
        return el.nh_second(xe, Xe, self.mu, self.lam, self.gload)

    def _hess_csc_free(self, pos, rest):
        H, _ = self._second(pos, rest)
        nd = self.el_dofs.shape[1]
        r = np.repeat(self.el_dofs, nd, axis=1).ravel()
        c = np.tile(self.el_dofs, (1, nd)).ravel()
        rx, cx = self.dof_to_x[r], self.dof_to_x[c]
        keep = (rx >= 0) & (cx >= 0)
        return csc_structural(rx[keep], cx[keep], H.reshape(len(H), -1).ravel()[keep], (self.n_x, self.n_x))

    # -- forward simulation (forward.py:135-203; spring_bar.py:100-135) ----------------------
    def simulate(self, p, x_init=None):
        rest = self.rest_positions(p)
        s = self.scale

        def energy(xf):
            return s * self._energy_full(self.full_positions(xf), rest)

        def gradient(xf):
            return s * self._grad_full(self.full_positions(xf), rest)[self.free_dofs]

        def hessian(xf):
            return s * self._hess_csc_free(self.full_positions(xf), rest).to_scipy()

        if x_init is not None:
            start = np.asarray(x_init, dtype=np.float64)
        elif self._x_warm is not None:
            start = self._x_warm
        else:
            start = self.X0.ravel()[self.free_dofs]
        x = solve_static(energy, gradient, hessian, start, self.tol)
        self._x_warm = x.copy()
        return x

    # -- constraints (spring_bar.py:138-156 idiom) -----------------------------------------
    def constraints(self, x, p):
        return self.scale * self._grad_full(self.full_positions(x), self.rest_positions(p))[self.free_dofs]

    def constraint_jac_x(self, x, p):
        m = self._hess_csc_free(self.full_positions(x), self.rest_positions(p))
        return Csc(m.to_scipy() * self.scale)

    def constraint_jac_p(self, x, p):
        """dc/dp = sum_e M_e P_e by one triplet build over every (element, row a, col b, p-map
        entry of col b) -- vectorised, the pattern structural (no SpGEMM)."""
        _, M = self._second(self.full_positions(x), self.rest_positions(p))
        ne, nd, _ = M.shape
        Pc = self.P.tocsr()
        a_loc = np.repeat(np.arange(nd), nd)
        b_loc = np.tile(np.arange(nd), nd)
        rx = self.dof_to_x[self.el_dofs[:, a_loc].ravel()]
        cdof = self.el_dofs[:, b_loc].ravel()
        cnt = (Pc.indptr[cdof + 1] - Pc.indptr[cdof]) * (rx >= 0)
        sel = np.flatnonzero(cnt)
        rep = cnt[sel]
        t = np.repeat(sel, rep)
        offs = np.arange(int(rep.sum())) - np.repeat(np.cumsum(rep) - rep, rep)
        kk = Pc.indptr[cdof[t]] + offs
        v = M.reshape(ne, nd * nd)[t // (nd * nd), t % (nd * nd)] * Pc.data[kk]
        return csc_structural(rx[t], Pc.indices[kk], self.scale * v, (self.n_x, self.n_p))

    # -- least squares (spring_bar.py:159-184 idiom) -----------------------------------------
    def residuals(self, x, p):
        out = [np.asarray(x)[self.target_dofs] - self.target_vals]
        if self.w_reg > 0.0:
            out.append(np.asarray(p, dtype=np.float64).copy())
        return np.concatenate(out)

    def weights(self):
        w = [np.full(self.target_dofs.size, self.w_target)]
        if self.w_reg > 0.0:
            w.append(np.full(self.n_p, self.w_reg))
        return np.concatenate(w)

    def residual_jac_x(self, x, p):
        nt = self.target_dofs.size
        sel = sp.csc_matrix((np.ones(nt), (np.arange(nt), self.target_dofs)), shape=(nt, self.n_x))
        if self.w_reg > 0.0:
            sel = sp.vstack([sel, sp.csc_matrix((self.n_p, self.n_x))], format="csc")
        return Csc(sel)

    def residual_jac_p(self, x, p):
        nt = self.target_dofs.size
        if self.w_reg > 0.0:
            return Csc(sp.vstack([sp.csc_matrix((nt, self.n_p)), sp.identity(self.n_p, format="csc")], format="csc"))
        return Csc(sp.csc_matrix((nt, self.n_p)))


class SpringBarOracle(_LsqMixin):
    """Restatement of the reference spring lattice (spring_bar.py:30-207), w_reg = 0 or > 0.

    Rest positions of every free vertex are the parameters (n_p == n_x); springs follow
    the reference's generation order (spring_bar.py:52-62); gravity m*g on every y dof.
    """

    def __init__(self, n_w, n_h, w_reg=0.0, stiffness=2.0, mass=2e-5, spacing=0.25, gravity=9.81,
                 x_target=None, tol=1e-10):
        ix, iy = np.meshgrid(np.arange(n_w), np.arange(n_h), indexing="ij")
        self.ref_positions = np.column_stack([ix.ravel() * spacing, iy.ravel() * spacing])
        vid = lambda i, j: i * n_h + j
        springs = []
        for i in range(n_w):
            for j in range(n_h):
                if i + 1 < n_w:
                    springs.append((vid(i, j), vid(i + 1, j)))
                if j + 1 < n_h:
                    springs.append((vid(i, j), vid(i, j + 1)))
                if i + 1 < n_w and j + 1 < n_h:
                    springs.append((vid(i, j), vid(i + 1, j + 1)))
                    springs.append((vid(i + 1, j), vid(i, j + 1)))
        self.springs = np.array(springs, dtype=np.int64)
        self.n_s = len(self.springs)
        self.n_v = n_w * n_h
        self.n_w, self.n_h = n_w, n_h
        self.k = np.full(self.n_s, float(stiffness))
        self.w_reg = float(w_reg)
        free_verts = np.arange(n_h, self.n_v)
        grav = np.zeros(2 * self.n_v)
        grav[1::2] = mass * gravity
        self.grav = grav
        self.free_dofs = np.column_stack([2 * free_verts, 2 * free_verts + 1]).ravel()
        self.n_x = self.free_dofs.size
        self.n_p = self.n_x
        self.L0 = np.linalg.norm(self.ref_positions[self.springs[:, 0]] - self.ref_positions[self.springs[:, 1]], axis=1)
        pm_dof = self.free_dofs
        self._ep = ElementProblem(self.ref_positions, self.springs, "spring", np.arange(n_h),
                                  (pm_dof, np.arange(self.n_p), np.ones(self.n_p)),
                                  np.arange(self.n_x), np.zeros(self.n_x), stiffness=self.k,
                                  scale=1.0, tol=tol, grav_const=grav)
        self.x_target = (self.ref_positions[free_verts].ravel() if x_target is None
                         else np.asarray(x_target, dtype=np.float64))
        self._x_warm = None

    def default_parameters(self):
        return self.ref_positions[self.n_h:].ravel().copy()

    # rest positions are p itself on free vertices
    def _p_to_offsets(self, p):
        return np.asarray(p, dtype=np.float64) - self.ref_positions[self.n_h:].ravel()

    def rest_lengths(self, p):
        X = self._ep.rest_positions(self._p_to_offsets(p))
        return np.linalg.norm(X[self.springs[:, 0]] - X[self.springs[:, 1]], axis=1)

    def simulate(self, p, x_init=None):
        if x_init is None and self._x_warm is not None:
            x_init = self._x_warm
        x = self._ep.simulate(self._p_to_offsets(p), x_init=x_init)
        self._x_warm = x.copy()
        return x

    def constraints(self, x, p):
        return self._ep.constraints(x, self._p_to_offsets(p))

    def constraint_jac_x(self, x, p):
        return self._ep.constraint_jac_x(x, self._p_to_offsets(p))

    def constraint_jac_p(self, x, p):
        return self._ep.constraint_jac_p(x, self._p_to_offsets(p))

    def residuals(self, x, p):
        out = [np.asarray(x) - self.x_target]
        if self.w_reg > 0.0:
            out.append(self.rest_lengths(p) - self.L0)
        return np.concatenate(out)

    def weights(self):
        w = [np.full(self.n_x, 1.0 / self.n_x)]
        if self.w_reg > 0.0:
            w.append(np.full(self.n_s, self.w_reg))
        return np.concatenate(w)

    def residual_jac_x(self, x, p):
        eye = sp.identity(self.n_x, format="csc")
        if self.w_reg > 0.0:
            return Csc(sp.vstack([eye, sp.csc_matrix((self.n_s, self.n_x))], format="csc"))
        return Csc(eye)

    def residual_jac_p(self, x, p):
        if self.w_reg > 0.0:
            X = self._ep.rest_positions(self._p_to_offsets(p))
            d = X[self.springs[:, 0]] - X[self.springs[:, 1]]
            dh = d / np.linalg.norm(d, axis=1)[:, None]
            s_idx = np.repeat(np.arange(self.n_s), 2)
            ca = (self.springs[:, 0][:, None] * 2 + np.arange(2)).ravel()
            cb = (self.springs[:, 1][:, None] * 2 + np.arange(2)).ravel()
            m = sp.csc_matrix((np.concatenate([dh.ravel(), -dh.ravel()]),
                               (np.concatenate([s_idx, s_idx]), np.concatenate([ca, cb]))),
                              shape=(self.n_s, 2 * self.n_v))[:, self.free_dofs]
            return Csc(sp.vstack([sp.csc_matrix((self.n_x, self.n_p)), m], format="csc"))
        return Csc(sp.csc_matrix((self.n_x, self.n_p)))

"""Device-resident SGN pipeline for element-mesh design problems (batched).

Host side (once per mesh, NumPy): free-dof maps, the structural KKT pattern in the
reference block order (x, p, lambda) (reference sparse.py:165-194), the sorted
element-to-nonzero contribution lists (atomic-free assembly), the Gx-only pattern of
the forward Newton solve, and the symbolic analyses (native, ``device.Symbolic``).

Device side (per direction, our CUDA kernels only; torch = allocation/plumbing):

  gather x,p -> positions   | sgn_gather_values
  element blocks            | sgn_element_derivs   (d2E/dx2, d2E/dx dX; forward.py:61-111 analog)
  KKT values                | sgn_gather_values    (gn_blocks + assemble_sgn + stack: sensitivity.py:205-266)
  LDL^T of K + shift        | sgn_factor_numeric   (linear_solvers.py:87,111-127)
  adjoint gradient          | sgn_solve_refined(LEADING) + sgn_spmv + sgn_adjoint_step (sensitivity.py:181-198)
  refined KKT solve         | sgn_solve_refined    (linear_solvers.py:130-211)

The forward equilibrium (``simulate``) is the reference's damped, tau-regularized
Newton with energy backtracking (forward.py:135-203) on the same element kernels.
"""
from __future__ import annotations

import ctypes
import math
import os
import time

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._lib import check, lib, ptr
from .device import DeviceFactor, symbolic_for
from .errors import DimensionMismatch, ForwardSimFailure, NoConvergence

ELEM_CODES = {"spring": _lib.SGN_ELEM_SPRING, "tri": _lib.SGN_ELEM_NH_TRI, "tet": _lib.SGN_ELEM_NH_TET,
              "membrane": _lib.SGN_ELEM_SHELL_MEMBRANE, "hinge": _lib.SGN_ELEM_HINGE}


class ElemGroup:
    """One element type of a mesh: connectivity + its slices of the block/gradient buffers."""

    def __init__(self, kind, conn, d, hoff, goff, rest_dof_used=None):
        self.kind = kind
        self.conn = np.asarray(conn, dtype=np.int64)
        self.n_e, self.nv = self.conn.shape
        self.nd = self.nv * d
        self.code = ELEM_CODES[kind] + (100 * d if kind == "spring" else 0)
        # mixed blocks d2E/dx dX are needed only for elements with a rest dof in the p-map
        # support (neo-Hookean simplices: compact slots; other kinds keep one per element)
        self.mslot = None
        self.n_m = self.n_e
        if rest_dof_used is not None and kind in ("tri", "tet"):
            el_dofs = (self.conn[:, :, None] * d + np.arange(d)[None, None, :]).reshape(self.n_e, self.nd)
            sup = rest_dof_used[el_dofs].any(axis=1)
            self.mslot = np.where(sup, np.cumsum(sup) - 1, -1).astype(np.int32)
            self.n_m = int(sup.sum())
            self.melems = np.flatnonzero(sup).astype(np.int32)      # support elements, slot order
        self.hoff = hoff                                   # hess block offset in ebuf
        self.moff = hoff + self.n_e * self.nd * self.nd    # mixed block offset (compact slots)
        self.goff = goff                                   # gradient offset in egrad
        self.size = (self.n_e + self.n_m) * self.nd * self.nd

    def mixed_index(self, e):
        """ebuf offset (relative to moff, in blocks) of element e's mixed block (-1: none)."""
        return np.asarray(e) if self.mslot is None else self.mslot[e].astype(np.int64)


def _csr_from_lists(n_rows, rows, *cols):
    """Stable sort of (rows, cols...) by row -> (ptr, cols...)."""
    order = np.argsort(rows, kind="stable")
    counts = np.bincount(rows, minlength=n_rows)
    ptr_ = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr_[1:])
    return (ptr_,) + tuple(np.ascontiguousarray(c[order]) for c in cols)


class MeshPlan:
    """Host precomputation for one mesh / parameterization (shared by all instances)."""

    def __init__(self, X0, conn, kind, fixed_verts, pmap, target_dofs, w_target, w_reg,
                 f_ext=None, rest_base=None, groups=None, R=None, disp_scale=None, restlen=None):
        """restlen = (springs [n_s x 2], L0 [n_s], w) adds the reference spring bar's rest-length
        residuals r_s = L_s(X(p)) - L0_s with weight w (spring_bar.py:159-184): C = J_p^T W J_p
        and f_p = J_p^T W r come from per-spring blocks (sgn_restlen_blocks) at every evaluation.

        disp_scale = sigma selects the displacement state: x = (pos - X(p)) / sigma on the free
        dofs (fixed dofs stay at X0).  Then G_x = sigma * dc/dpos, the G_p block gains the
        element-Hessian terms of the free dofs the p-map moves (dc/dp at fixed x), and the
        least-squares residual of a target is sigma * x.  Without it x = positions."""
        self.disp_scale = None if disp_scale is None else float(disp_scale)
        if self.disp_scale is not None and R is not None:
            raise ValueError("the displacement state has no residual p-map")
        self.X0 = np.asarray(X0, dtype=np.float64)
        self.n_v, self.d = self.X0.shape
        d = self.d
        if groups is None:
            groups = [(kind, conn)]
        self.groups = []
        hoff = goff = 0
        rest_used = np.zeros(self.n_v * d, bool)
        rest_used[np.asarray(pmap[0], dtype=np.int64)] = True
        # rest coordinate components the p-map moves at all (bit i): the shell kernels skip the
        # mixed columns of the others (config 4: heights only)
        self.rest_comp_mask = int(sum(1 << i for i in range(d) if rest_used[i::d].any()))
        for gk, gc in groups:
            g = ElemGroup(gk, gc, d, hoff, goff, rest_used)
            self.groups.append(g)
            hoff += g.size
            goff += g.n_e * g.nd
        self.restlen = None
        if restlen is not None:
            rs, rL0, rw = restlen
            self.restlen = (np.asarray(rs, dtype=np.int64), np.asarray(rL0, dtype=np.float64), float(rw))
            self.rl_off = hoff
            hoff += 21 * len(rs)
        self.ebuf_size, self.egrad_size = hoff, goff
        g0 = self.groups[0]
        self.conn, self.kind, self.elem_code = g0.conn, g0.kind, g0.code     # single-group aliases
        self.n_e, self.nv_el, self.nd = g0.n_e, g0.nv, g0.nd
        fixed = np.zeros(self.n_v, bool)
        fixed[np.asarray(fixed_verts, dtype=np.int64)] = True
        self.free_verts = np.flatnonzero(~fixed)
        self.free_dofs = (self.free_verts[:, None] * d + np.arange(d)[None, :]).ravel()
        self.n_x = int(self.free_dofs.size)
        self.n_dof = self.n_v * d
        self.dof_to_x = -np.ones(self.n_dof, dtype=np.int64)
        self.dof_to_x[self.free_dofs] = np.arange(self.n_x)
        pm_dof, pm_p, pm_coef = (np.asarray(a) for a in pmap)
        pm_dof, pm_p, pm_coef = pm_dof.astype(np.int64), pm_p.astype(np.int64), pm_coef.astype(np.float64)
        self.n_p = int(pm_p.max()) + 1 if pm_p.size else 0
        self.target_dofs = np.asarray(target_dofs, dtype=np.int64)
        self.w_target, self.w_reg = float(w_target), float(w_reg)
        self.f_ext = np.zeros(self.n_dof) if f_ext is None else np.asarray(f_ext, dtype=np.float64)
        self.dim = 2 * self.n_x + self.n_p
        n_x, n_p = self.n_x, self.n_p

        # positions: pos[dof] = X0[dof] (fixed) | x[dof_to_x] (free)
        is_free = self.dof_to_x >= 0
        self.pos_base = np.where(is_free, 0.0, self.X0.ravel())
        self.pos_ptr = np.zeros(self.n_dof + 1, dtype=np.int64)
        np.cumsum(is_free.astype(np.int64), out=self.pos_ptr[1:])
        self.pos_idx = self.dof_to_x[is_free].astype(np.int64)
        # rest: X[dof] = X0[dof] + sum coef * p
        self.rest_ptr, self.rest_idx, self.rest_coef = _csr_from_lists(self.n_dof, pm_dof, pm_p, pm_coef)
        if self.disp_scale is not None:
            # displacement state: pos = restpos + sigma x, restpos = X(p) on free dofs, X0 on fixed
            self.pos_coef = np.full(self.pos_idx.size, self.disp_scale)
            fr = is_free[pm_dof]
            self.restpos_ptr, self.restpos_idx, self.restpos_coef = _csr_from_lists(
                self.n_dof, pm_dof[fr], pm_p[fr], pm_coef[fr])
        sig = 1.0 if self.disp_scale is None else self.disp_scale
        self.rest_base = (self.X0.ravel().copy() if rest_base is None
                          else np.asarray(rest_base, dtype=np.float64).ravel().copy())

        # --- KKT structural entries + contributions (reference block order) ------------
        oL = n_x + n_p
        rows, cols, src, coef = [], [], [], []
        gx_r_all, gx_c_all, gx_s_all = [], [], []
        g_rows, g_src = [], []
        ts_row, ts_cdof, ts_m, ts_h = [], [], [], []      # two-stage G_p: entries before the p expansion
        rp = self.rest_ptr
        for g in self.groups:
            nd = g.nd
            el_dofs = (g.conn[:, :, None] * d + np.arange(d)[None, None, :]).reshape(g.n_e, nd)
            ea = np.repeat(np.arange(nd), nd)     # row (deformed dof) local index
            eb = np.tile(np.arange(nd), nd)       # col local index
            e_all = np.repeat(np.arange(g.n_e), nd * nd)
            r_dof = el_dofs[:, ea].ravel()
            c_dof = el_dofs[:, eb].ravel()
            loc = np.tile(ea * nd + eb, g.n_e)
            hidx = g.hoff + e_all * nd * nd + loc
            midx = g.moff + g.mixed_index(e_all) * nd * nd + loc    # valid where the p-map reads it
            rx, cx = self.dof_to_x[r_dof], self.dof_to_x[c_dof]
            keep = (rx >= 0) & (cx >= 0)                  # Gx block and its transpose
            gx_r, gx_c, gx_s = rx[keep], cx[keep], hidx[keep]
            gx_r_all.append(gx_r); gx_c_all.append(gx_c); gx_s_all.append(gx_s)
            rows += [oL + gx_r, gx_c]
            cols += [gx_c, oL + gx_r]
            src += [gx_s, gx_s]
            coef += [np.full(gx_s.size, sig), np.full(gx_s.size, sig)]
            # Gp block: row free dof, rest col dof -> p entries
            cnt = (rp[c_dof + 1] - rp[c_dof]) * (rx >= 0)
            sel = np.flatnonzero(cnt)
            if sel.size:
                ts_row.append(rx[sel]); ts_cdof.append(c_dof[sel]); ts_m.append(midx[sel])
                ts_h.append(np.where(cx[sel] >= 0, hidx[sel], -1) if self.disp_scale is not None
                            else np.full(sel.size, -1, dtype=np.int64))
                rep = cnt[sel]
                base_t = np.repeat(sel, rep)
                starts = np.zeros(rep.size, dtype=np.int64)
                np.cumsum(rep[:-1], out=starts[1:])
                offs = np.arange(int(rep.sum()), dtype=np.int64) - np.repeat(starts, rep)
                kk = rp[c_dof[base_t]] + offs
                pj = self.rest_idx[kk]
                pc = self.rest_coef[kk]
                gr = rx[base_t]
                ms = midx[base_t]
                rows += [oL + gr, n_x + pj]
                cols += [n_x + pj, oL + gr]
                src += [ms, ms]
                coef += [pc, pc]
                if self.disp_scale is not None:
                    # dc/dp at fixed displacement: the free dofs the p-map moves carry
                    # their element-Hessian column (H P_free), next to the mixed block (M P)
                    fcol = cx[base_t] >= 0
                    hs = hidx[base_t][fcol]
                    rows += [oL + gr[fcol], n_x + pj[fcol]]
                    cols += [n_x + pj[fcol], oL + gr[fcol]]
                    src += [hs, hs]
                    coef += [pc[fcol], pc[fcol]]
            # gradient gather entries of this group
            gdof = el_dofs.ravel()
            gx_ = self.dof_to_x[gdof]
            gs = np.flatnonzero(gx_ >= 0)
            g_rows.append(gx_[gs]); g_src.append(g.goff + gs.astype(np.int64))
        rows = np.concatenate(rows); cols = np.concatenate(cols)
        src = np.concatenate(src); coef = np.concatenate(coef)
        gx_r, gx_c, gx_s = np.concatenate(gx_r_all), np.concatenate(gx_c_all), np.concatenate(gx_s_all)
        # constant Gauss-Newton blocks (sensitivity.py:205-216): A = w on targets, and for a
        # residual r = x_t - R p: B = -w R^T (p rows, x cols), C = w R^T R + w_reg I
        nt = self.target_dofs.size
        crow, ccol, cval = [self.target_dofs], [self.target_dofs], [np.full(nt, self.w_target * sig * sig)]
        self.R = None
        if R is not None:
            Rm = sp.csr_matrix(R)
            self.R = Rm
            Rc = Rm.tocoo()
            bt_x, bt_p, bt_v = self.target_dofs[Rc.row], n_x + Rc.col, -self.w_target * Rc.data
            crow += [bt_p, bt_x]; ccol += [bt_x, bt_p]; cval += [bt_v, bt_v]
            CtC = (self.w_target * (Rm.T @ Rm)).tocoo()
            crow.append(n_x + CtC.row); ccol.append(n_x + CtC.col); cval.append(CtC.data)
        if self.w_reg > 0.0:
            crow.append(n_x + np.arange(n_p)); ccol.append(n_x + np.arange(n_p)); cval.append(np.full(n_p, self.w_reg))
        if self.restlen is not None:
            # C block from the per-spring blocks w j j^T; f_p lists from w r j (KKT order)
            rs = self.restlen[0]
            ns_ = len(rs)
            rdof = np.stack([2 * rs[:, 0], 2 * rs[:, 0] + 1, 2 * rs[:, 1], 2 * rs[:, 1] + 1], axis=1)  # (ns, 4)
            s_idx = np.repeat(np.arange(ns_), 4)
            u_idx = np.tile(np.arange(4), ns_)
            d_ = rdof.ravel()
            cnt = rp[d_ + 1] - rp[d_]
            sel = np.flatnonzero(cnt)
            rep_ = cnt[sel]
            t = np.repeat(sel, rep_)
            offs = np.arange(int(rep_.sum())) - np.repeat(np.cumsum(rep_) - rep_, rep_)
            kk = rp[d_[t]] + offs
            e_s, e_u, e_p, e_c = s_idx[t], u_idx[t], self.rest_idx[kk], self.rest_coef[kk]   # (spring, slot, p, coef)
            # pairs of entries of the same spring: C[p_i, p_j] += c_i c_j (w j j^T)[u_i, u_j]
            order = np.argsort(e_s, kind="stable")
            e_s, e_u, e_p, e_c = e_s[order], e_u[order], e_p[order], e_c[order]
            starts = np.searchsorted(e_s, np.arange(ns_))
            ends = np.searchsorted(e_s, np.arange(ns_), side="right")
            pr, pc, ps, pcf = [], [], [], []
            for s_ in range(ns_):
                a0, a1 = starts[s_], ends[s_]
                for i_ in range(a0, a1):
                    for j_ in range(a0, a1):
                        pr.append(n_x + e_p[i_]); pc.append(n_x + e_p[j_])
                        ps.append(self.rl_off + 21 * s_ + 4 * e_u[i_] + e_u[j_]); pcf.append(e_c[i_] * e_c[j_])
            rows = np.concatenate([rows, np.asarray(pr, dtype=np.int64)])
            cols = np.concatenate([cols, np.asarray(pc, dtype=np.int64)])
            src = np.concatenate([src, np.asarray(ps, dtype=np.int64)])
            coef = np.concatenate([coef, np.asarray(pcf, dtype=np.float64)])
            self.rl_fptr, self.rl_fsrc, self.rl_fcoef = _csr_from_lists(
                n_p, e_p, self.rl_off + 21 * e_s + 16 + e_u, e_c)
            self.rl_rsrc = self.rl_off + 21 * np.arange(ns_, dtype=np.int64) + 20
        crow, ccol, cval = np.concatenate(crow), np.concatenate(ccol), np.concatenate(cval)
        all_r = np.concatenate([rows, crow])
        all_c = np.concatenate([cols, ccol])
        key = all_c * self.dim + all_r                    # CSC order: by column, then row
        ukey, inv = np.unique(key, return_inverse=True)
        self.K_indices = (ukey % self.dim).astype(np.int64)
        kcols = ukey // self.dim
        self.K_indptr = np.zeros(self.dim + 1, dtype=np.int64)
        np.cumsum(np.bincount(kcols, minlength=self.dim), out=self.K_indptr[1:])
        self.nnz = int(ukey.size)
        nz_of = inv[:rows.size]
        self.K_ptr, self.K_src, self.K_coef = _csr_from_lists(self.nnz, nz_of, src, coef)
        base = np.zeros(self.nnz)
        np.add.at(base, inv[rows.size:], cval)         # constant entries (sum duplicates)
        self.K_base = base
        # residual map on the device (CSR over targets and over parameters)
        if R is not None:
            Rr = sp.csr_matrix(R); Rr.sort_indices()
            Rt = sp.csr_matrix(Rr.T); Rt.sort_indices()
            self.R_ptr, self.R_idx, self.R_val = Rr.indptr.astype(np.int64), Rr.indices.astype(np.int64), Rr.data.copy()
            self.Rt_ptr, self.Rt_idx, self.Rt_val = Rt.indptr.astype(np.int64), Rt.indices.astype(np.int64), Rt.data.copy()

        # --- Gx-only pattern for the forward Newton (generic 1x1 mode) -------------------
        gkey = gx_c * n_x + gx_r
        gu, ginv = np.unique(gkey, return_inverse=True)
        self.G_indices = (gu % n_x).astype(np.int64)
        self.G_indptr = np.zeros(n_x + 1, dtype=np.int64)
        np.cumsum(np.bincount(gu // n_x, minlength=n_x), out=self.G_indptr[1:])
        self.G_nnz = int(gu.size)
        self.G_ptr, self.G_src = _csr_from_lists(self.G_nnz, ginv, gx_s)
        self.G_coef = None if self.disp_scale is None else np.full(self.G_src.size, self.disp_scale)
        gdiag = np.flatnonzero((gu % n_x) == (gu // n_x))
        self.G_diag = gdiag.astype(np.int64)               # nnz positions of the diagonal

        # --- gradient gather: free dof <- element-gradient entries ------------------------
        self.grad_ptr, self.grad_src = _csr_from_lists(n_x, np.concatenate(g_rows), np.concatenate(g_src))
        self.grad_base = self.f_ext[self.free_dofs].copy()

        # --- two-stage assembly (multi-group meshes with a wide p-map: the shell) -----------
        # The one-stage gather expands every element entry over the parameters of its rest dof
        # and over both symmetric copies (config 4: 173 M terms, 5 GB read per assembly).  Two
        # stages instead: G_x values once (the G lists above) copied to both K blocks; the
        # mixed matrix Mz = d2E/dx dX (+ H on free columns, displacement state) summed per
        # (row, rest dof), then G_p = Mz P over the p-map rows, written to both K blocks; the
        # constant entries (A, B, C) are written once.  ~50 M terms for config 4.
        self.two_stage = None
        if self.restlen is None and R is None and ts_row and len(self.groups) > 1:
            self.two_stage = self._two_stage_lists(ukey, oL, np.concatenate(ts_row), np.concatenate(ts_cdof),
                                                   np.concatenate(ts_m), np.concatenate(ts_h), gu)

    def _two_stage_lists(self, ukey, oL, t_row, t_cdof, t_m, t_h, gu):
        dim, n_x, n_p = self.dim, self.n_x, self.n_p

        def kpos(row, col):
            key = col * dim + row
            pos = np.searchsorted(ukey, key)
            assert np.array_equal(ukey[pos], key)
            return pos.astype(np.int64)

        ts = {}
        # G_x block: the G pattern's nnz q = (row gu % n_x, col gu // n_x) -> K[oL + row, col] and its transpose
        g_row, g_col = gu % n_x, gu // n_x
        ts["gx_dst"] = np.concatenate([kpos(oL + g_row, g_col), kpos(g_col, oL + g_row)])
        ts["gx_src"] = np.concatenate([np.arange(self.G_nnz, dtype=np.int64)] * 2)
        # stage 1: Mz entries (rest dof, row) <- element mixed (+ Hessian) entries
        key1 = t_cdof * n_x + t_row
        u1, inv1 = np.unique(key1, return_inverse=True)
        hv = t_h >= 0
        ts["mz_ptr"], ts["mz_src"] = _csr_from_lists(u1.size, np.concatenate([inv1, inv1[hv]]),
                                                     np.concatenate([t_m, t_h[hv]]))
        ts["n_mz"] = int(u1.size)
        # stage 2: G_p[row, p] = sum_c Mz[row, c] P[c, p]
        m_cdof, m_row = u1 // n_x, u1 % n_x
        rp = self.rest_ptr
        rep = rp[m_cdof + 1] - rp[m_cdof]
        src = np.repeat(np.arange(u1.size, dtype=np.int64), rep)
        offs = np.arange(int(rep.sum()), dtype=np.int64) - np.repeat(np.cumsum(rep) - rep, rep)
        kk = rp[m_cdof[src]] + offs
        pj, pc = self.rest_idx[kk], self.rest_coef[kk]
        key2 = pj * n_x + m_row[src]
        u2, inv2 = np.unique(key2, return_inverse=True)
        gp_ptr, gp_src, gp_coef = _csr_from_lists(u2.size, inv2, src, pc)
        p_of, r_of = u2 // n_x, u2 % n_x
        n2 = u2.size
        ts["gp_dst"] = np.concatenate([kpos(oL + r_of, n_x + p_of), kpos(n_x + p_of, oL + r_of)])
        ts["gp_ptr"] = np.concatenate([gp_ptr, gp_ptr[-1] + gp_ptr[1:]])
        ts["gp_src"] = np.concatenate([gp_src, gp_src])
        ts["gp_coef"] = np.concatenate([gp_coef, gp_coef])
        # every structural entry is either constant (written once from K_base) or covered above
        covered = np.zeros(self.nnz, bool)
        covered[ts["gx_dst"]] = True
        covered[ts["gp_dst"]] = True
        assert (self.K_base[covered] == 0.0).all()
        assert np.array_equal(np.diff(self.K_ptr) > 0, covered), "two-stage lists cover the variable entries"
        ts["n_gp"] = int(2 * n2)
        return ts


class VertexPlan:
    """Fused vertex-centric assembly of the G_x entries (neo-Hookean simplices, one group).

    One task per vertex with a free dof; its incident elements (ascending) each compute
    the element-Hessian columns of that vertex's dofs into shared memory, and each output
    (column dof (v, i), row dof r) is the fixed-order sum of its element entries, written
    to K[lambda_r, x_(v,i)], to K[x_r, lambda_(v,i)] (= G_x[(v,i), r], by the symmetry of
    the element Hessians: both copies are one contiguous run of column (v,i)'s nonzeros, so
    every store is coalesced) and to G_x[r, (v,i)].  It is the sum, in the same element
    order, of the staged path (element blocks -> sorted element->nonzero lists, `k_gather`),
    without the element-block round trip through HBM.  The remaining KKT entries
    (constants and the G_p block) keep the gather, restricted to their own nonzeros
    (`rest_*`)."""

    def __init__(self, pl: "MeshPlan"):
        g = pl.groups[0]
        d, nd, nv = pl.d, g.nd, g.nv
        el_dofs = (g.conn[:, :, None] * d + np.arange(d)[None, None, :]).reshape(g.n_e, nd)
        free_v = (pl.dof_to_x.reshape(pl.n_v, d) >= 0).any(axis=1)
        e_p = np.repeat(np.arange(g.n_e), nv)
        a_p = np.tile(np.arange(nv), g.n_e)
        v_p = g.conn.ravel()
        keep = free_v[v_p]
        e_p, a_p, v_p = e_p[keep], a_p[keep], v_p[keep]
        o = np.lexsort((e_p, v_p))
        e_p, a_p, v_p = e_p[o], a_p[o], v_p[o]
        tv, t_start, t_cnt = np.unique(v_p, return_index=True, return_counts=True)
        self.n_task = int(tv.size)
        self.max_inc = int(t_cnt.max())
        self.inc_ptr = np.r_[t_start, v_p.size].astype(np.int32)
        self.inc_ea = (e_p * 4 + a_p).astype(np.int32)
        t_p = np.repeat(np.arange(self.n_task), t_cnt)
        s_p = np.arange(v_p.size) - np.repeat(t_start, t_cnt)
        # contributions: (pair, column axis i, element row r)
        P, I, R = np.meshgrid(np.arange(v_p.size), np.arange(d), np.arange(nd), indexing="ij")
        P, I, R = P.ravel(), I.ravel(), R.ravel()
        c_dof = v_p[P] * d + I
        r_dof = el_dofs[e_p[P], R]
        cx, rx = pl.dof_to_x[c_dof], pl.dof_to_x[r_dof]
        ok = (cx >= 0) & (rx >= 0)
        P, I, R, cx, rx = P[ok], I[ok], R[ok], cx[ok], rx[ok]
        smem = s_p[P] * (d * nd) + I * nd + R
        tt = t_p[P]
        o = np.lexsort((e_p[P], rx, cx, tt))          # output (task, col, row), then element order
        tt, cx, rx, smem = tt[o], cx[o], rx[o], smem[o]
        okey = (tt.astype(np.int64) * pl.n_x + cx) * pl.n_x + rx
        first = np.r_[True, okey[1:] != okey[:-1]]
        oidx = np.flatnonzero(first)
        self.n_out = int(oidx.size)
        self.con_ptr = np.r_[oidx, okey.size].astype(np.int32)
        self.con_idx = smem.astype(np.int32)
        ot, ocx, orx = tt[oidx], cx[oidx], rx[oidx]
        self.out_ptr = np.searchsorted(ot, np.arange(self.n_task + 1)).astype(np.int32)
        # destinations: K (lambda_r, x_c), K (x_c, lambda_r), G (r, c)
        oL = pl.n_x + pl.n_p
        kcol = np.repeat(np.arange(pl.dim, dtype=np.int64), np.diff(pl.K_indptr))
        kkey = kcol * pl.dim + pl.K_indices
        k1 = ocx * pl.dim + (oL + orx)
        k2 = (oL + ocx) * pl.dim + orx        # K[x_r, lambda_c] = G_x[c, r]: symmetric copy, same column run
        n1, n2 = np.searchsorted(kkey, k1), np.searchsorted(kkey, k2)
        assert (kkey[n1] == k1).all() and (kkey[n2] == k2).all()
        gcol = np.repeat(np.arange(pl.n_x, dtype=np.int64), np.diff(pl.G_indptr))
        gkey = gcol * pl.n_x + pl.G_indices
        k3 = ocx * pl.n_x + orx
        n3 = np.searchsorted(gkey, k3)
        assert (gkey[n3] == k3).all()
        assert pl.nnz < 2 ** 31 and pl.G_nnz < 2 ** 31
        self.out_dst = np.stack([n1, n2, n3], axis=1).astype(np.int32).ravel()
        # every fused K entry is a pure G_x entry: no constant, only element-Hessian terms
        fused = np.zeros(pl.nnz, bool)
        fused[n1] = True
        fused[n2] = True
        assert fused.sum() == 2 * self.n_out
        cnt = np.diff(pl.K_ptr)
        fsrc = pl.K_src[np.repeat(fused, cnt)]
        assert (pl.K_base[fused] == 0.0).all() and (fsrc < g.moff).all()
        ncon = np.diff(self.con_ptr)
        assert (cnt[n1] == ncon).all() and (cnt[n2] == ncon).all()   # same terms as the staged lists
        # the complement (constants, G_p): restricted gather lists
        rest = np.flatnonzero(~fused)
        rc = cnt[rest]
        self.rest_dst = rest.astype(np.int64)
        self.rest_ptr = np.r_[0, np.cumsum(rc)].astype(np.int64)
        sel = np.repeat(pl.K_ptr[rest], rc) + (np.arange(int(rc.sum())) - np.repeat(self.rest_ptr[:-1], rc))
        self.rest_src = pl.K_src[sel].astype(np.int64)
        self.rest_coef = pl.K_coef[sel].astype(np.float64)
        self.rest_base = pl.K_base[rest].copy()
        self.needs_mixed = bool(self.rest_src.size)


def vertex_plan(pl: "MeshPlan"):
    """VertexPlan for single-group neo-Hookean meshes (max 32 elements per vertex), else None."""
    if os.environ.get("SGN_FUSED_ASSEMBLY", "1") == "0":
        return None
    if len(pl.groups) != 1 or pl.groups[0].kind not in ("tri", "tet"):
        return None
    vp = VertexPlan(pl)
    return vp if vp.max_inc <= 32 else None


_SIDE_STREAM = os.environ.get("SGN_SIDE_STREAM", "1") != "0"
_DIR_GRAPH = os.environ.get("SGN_DIRECTION_GRAPH", "1") != "0"
_GX_CTAS = int(os.environ.get("SGN_GX_CTAS", "0"))     # 0: 3/16 of the grid


def _gx_share(eng, full: int) -> int:
    """CTAs of the concurrent G_x factorization.  The G_x factor is dependency-chain bound
    like the KKT one, so its share is not its flop share (0.11 on config 2, where 74 of 592
    CTAs made it finish 0.6 ms after the KKT factor)."""
    if _GX_CTAS > 0:
        return min(_GX_CTAS, full - 1)
    if eng.batch > 1:      # batched instances are throughput-bound: 1/4 (config 5 sweep, 111..222 CTAs)
        return max(1, full // 4)
    # single instance: proportional to the G_x factor's share of the flops, 1.85 x
    # flops(G_x) / flops(KKT), within [3/16, 1/4] of the grid.  Sweeps (SGN_GX_CTAS):
    # config 2 (ratio 0.119) best at 129 of 592; with the round-2 KKT factorization (config 4:
    # 33 ms) a smaller share leaves the adjoint as a tail after the KKT factor: config 3
    # 158 / 174 / 172 directions/s at 74 / 111 / 148, config 4 23.4 / 23.3 / 24.2 / 23.7 at
    # 37 / 92 / 111 / 130 (profiles/r02_gx_share_sweep.txt)
    if not hasattr(eng, "_gx_frac"):
        fk = float(eng.ksym.stats()["flops"])
        eng.gfac                                   # builds gsym
        fg = float(eng.gsym.stats()["flops"])
        eng._gx_frac = min(0.25, max(3.0 / 16.0, 1.85 * fg / max(fk, 1.0)))
    return max(1, int(round(eng._gx_frac * full)))
_GX_RETIRE = int(os.environ.get("SGN_GX_RETIRE", "-1"))     # sweeps: top levels of <= k fronts hand CTAs over (0: off)
_DEBUG_NAN = os.environ.get("SGN_DEBUG_NAN", "0") == "1"
_DEBUG_NEWTON = os.environ.get("SGN_DEBUG_NEWTON", "0") == "1"


def _nan_probe(eng, where):
    """Diagnostics only (SGN_DEBUG_NAN=1): report the first non-finite device buffer."""
    if not _DEBUG_NAN:
        return
    eng.torch.cuda.synchronize()
    for name in ("kvals", "fvec", "gvals", "tmp", "rhs", "grad", "sol", "x", "p"):
        t = getattr(eng, name, None)
        if t is not None and not bool(eng.torch.isfinite(t).all()):
            import sys
            print(f"[nan-probe] {where}: {name} non-finite ({int((~eng.torch.isfinite(t)).sum())} entries)",
                  file=sys.stderr, flush=True)


def gradient_from_adjoint(eng, st) -> None:
    """g = f_p + G_p^T lambda (sensitivity.py:194-198) from v = (0, 0, w) in eng.tmp (lambda =
    -w): eng.grad = g and eng.rhs = (0, -g, 0).  With a double-double w (adjoint_direct),
    the product is evaluated exactly too (sgn_residual_dd: f - K v), else by a plain SpMV."""
    n_x, n_p = eng.n_x, eng.n_p
    lo = getattr(eng, "tmp_lo", None)
    if lo is not None and int(getattr(eng, "adj_ir_steps", 0)) > 0:
        eng.kfac.residual_dd(eng.kvals, eng.tmp, lo, eng.fvec, eng.rhs, st)
        check(lib().sgn_adjoint_step(4, eng.batch, n_x, n_p, ptr(eng.rhs), None, ptr(eng.tmp), ptr(eng.grad), st))
    else:
        eng.kfac.spmv(eng.kvals, eng.tmp, eng.rhs, False, st)
        check(lib().sgn_adjoint_step(1, eng.batch, n_x, n_p, ptr(eng.rhs), ptr(eng.fvec), ptr(eng.tmp),
                                     ptr(eng.grad), st))
    eng.rhs.copy_(eng.tmp)


def factor_shifts(eng, full: bool = False):
    """Static shifts of the direction path's KKT factorization.

    The reference factors K + diag(+eps_x, 0, -eps_lambda) with SuperLU and refines against
    the unshifted K (linear_solvers.py:111-175); the shift keeps its unsymmetric LU of the
    quasi-definite KKT stable.  The device LDL^T pivots every (x_i, lambda_j) pair as a 2x2
    block with |det| >= g^2, so it does not need the full shift: it factors with
    ``eng.factor_shift_scale`` x eps (1e-4: 1e-6 -> 1e-10), which makes the first solve
    accurate enough that the refinement -- still against the unshifted K, to the same
    refine_tolerance -- takes 0-1 BiCGSTAB iterations instead of 3-5 (config 2: 5 -> 1,
    config 4: 3 -> 1; dp unchanged within the contract, profiles/r02_eps_probe.txt).  If the
    refinement stalls or a pivot is zero with the reduced shift, the direction is recomputed
    with the full shift (full=True), i.e. exactly the reference's preconditioner."""
    sc = 1.0 if full else float(getattr(eng, "factor_shift_scale", 1.0))
    return float(eng.stab.eps_x) * sc, float(eng.stab.eps_lambda) * sc


def _factor_adjoint(eng, st, cur, f0=None, f1=None, events=None):
    """KKT factor on `cur` || adjoint gradient and the SGN right-hand side on a side stream,
    joined back into `cur`; no host synchronization (so it can be graph-captured)."""
    torch = eng.torch
    n_x, n_p = eng.n_x, eng.n_p
    if not hasattr(eng, "_side_stream"):
        eng._side_stream = torch.cuda.Stream()
    # split the persistent CTA slots (SMs x 4): the G_x factor takes _GX_CTAS of them
    # and the KKT factor the rest, so both run from the start instead of G_x waiting
    # for the KKT grid to retire (the G_x factor keeps the full grid elsewhere)
    full = eng.kfac.set_grid(0)
    gx = _gx_share(eng, full)
    eng.gfac.set_grid(gx)
    # option (SGN_GX_RETIRE=k, off by default): the KKT factor starts on the full grid and hands
    # gx CTA slots over when it reaches its top levels of <= k fronts (sgn_factor_set_retire);
    # the G_x launch, queued on the side stream, becomes resident then.  Measured on config 4
    # (profiles/r02_gx_handover_sweep.txt): the KKT factor gains 1.3 ms, but the adjoint (G_x
    # factor + 3 refined solves, ~6 ms on 111 CTAs) no longer fits in the tail: 27.3 -> 25.0
    # directions/s at k = 8; configs 2 and 3 lose 10-20 %.  The two split the slots from the start.
    handover = -1
    lvf = max(_GX_RETIRE, 0)
    if lvf > 0 and eng.batch == 1:
        handover = eng.kfac.set_retire(full - gx, lvf)
    if handover < 0:
        eng.kfac.set_grid(full - gx)
    side = eng._side_stream
    ev_asm, ev_adj = torch.cuda.Event(), torch.cuda.Event()
    ev_asm.record(cur)
    if f0 is not None:
        f0.record(cur)
    eng.kfac.numeric(eng.kvals, *factor_shifts(eng), st)
    if f1 is not None:
        f1.record(cur)
    if events is not None:
        events[0].record()
    side.wait_event(ev_asm)
    with torch.cuda.stream(side):
        sst = _lib.stream_handle()
        res_a, it_a = eng.adjoint_direct(check_pivots=False)
        gradient_from_adjoint(eng, sst)
        ev_adj.record(side)
    cur.wait_event(ev_adj)
    eng.gfac.set_grid(0)
    eng.kfac.set_grid(0)
    eng.kfac.set_retire(0, 0)
    if events is not None:
        events[1].record()
    return res_a, it_a


def adjoint_gradient_stage(eng):
    """Adjoint gradient alone (reference sensitivity.py:160-198): the unshifted LDL^T of
    dc/dx, one solve, then g = f_p + G_p^T lambda -- no KKT factorization.  A zero pivot of
    dc/dx raises SingularConstraintJacobian(pivot_index) (_factor_constraint_jac,
    sensitivity.py:160-164).  The result is in eng.grad; eng.rhs = (0, -g, 0)."""
    from .errors import SingularConstraintJacobian
    st = _lib.stream_handle()
    n_x, n_p = eng.n_x, eng.n_p
    eng.adjoint_direct(check_pivots=False)
    piv = eng.gfac.status(st)
    bad = np.flatnonzero(piv >= 0)
    if bad.size:
        raise SingularConstraintJacobian(f"singular state Jacobian dc/dx (instance {int(bad[0])})",
                                         pivot_index=int(piv[bad[0]]))
    gradient_from_adjoint(eng, st)


def _refine_with_fallback(eng, st, tol, mi):
    """The direction path's KKT solve, in stages that each instance leaves as soon as it
    meets ``tol`` (so an instance's result never depends on its batch):

    1. mixed-precision iterative refinement on the reduced-shift factor (sgn_solve_ir:
       exact double-double residuals drive ``eng.ir_steps`` corrections);
    2. the reference's refinement, BiCGSTAB against the unshifted K (linear_solvers.py:
       178-211), on the same factor;
    3. the KKT re-factored with the full shift (the reference's own preconditioner) and
       BiCGSTAB again.
    Stages 1 and 3 exist only with a reduced shift (factor_shifts).  Returns (rc, res, its)
    per instance; a zero pivot of the full-shift factor raises SingularMatrix as before."""
    from .errors import SingularMatrix
    torch = eng.torch
    B = eng.batch
    reduced = factor_shifts(eng) != factor_shifts(eng, full=True)
    steps = int(getattr(eng, "ir_steps", 0))
    done = np.zeros(B, bool)
    res_all = np.full(B, np.inf)
    its_all = np.zeros(B, dtype=np.int32)
    keep = None
    eng.last_full_shift = False

    def pivots_ok():
        return eng.kfac.status(st) < 0

    def absorb(res, its, ok):
        nonlocal keep
        new = ok & ~done
        if new.any():
            if keep is None:
                keep = torch.empty_like(eng.sol)
            m = torch.as_tensor(new, device=eng.sol.device)
            keep[m] = eng.sol[m]
            res_all[new], its_all[new] = res[new], its[new]
            done[new] = True

    if reduced and steps > 0:
        res, corr = eng.kfac.solve_ir(eng.kvals, eng.rhs, eng.sol, steps, st)
        eng.last_ir_correction = corr
        # an exact residual within tol verifies the solution whatever the pivots were (a zero
        # pivot is replaced by 1 in the factor, which the residual then exposes)
        if np.all(res <= tol):                                  # the common case: done
            return _lib.SGN_OK, res, np.full(B, steps, dtype=np.int32)
        absorb(res, np.full(B, steps, dtype=np.int32), res <= tol)
    if not done.all():
        rc, res, its = eng.kfac.solve_refined(eng.kvals, eng.rhs, eng.sol, tol, mi, False, st)
        piv = pivots_ok()
        if not reduced and not piv.all():
            eng.kfac.check(st)                                  # raises SingularMatrix
        absorb(res, its, (res <= tol) & piv)
        if reduced and not done.all():
            eng.kfac.numeric(eng.kvals, *factor_shifts(eng, full=True), st)
            eng.kfac.check(st)
            eng.last_full_shift = True
            rc, res, its = eng.kfac.solve_refined(eng.kvals, eng.rhs, eng.sol, tol, mi, False, st)
            absorb(res, its, res <= tol)
        left = ~done                                            # failed every stage: best iterate
        res_all[left], its_all[left] = res[left], its[left]
    if keep is not None:
        m = torch.as_tensor(done, device=eng.sol.device)
        eng.sol[m] = keep[m]
    rc = _lib.SGN_OK if done.all() else _lib.SGN_NO_CONVERGENCE
    return rc, res_all, its_all


def sgn_solve_stages(eng, timings: dict | None = None, need_direction: bool = True, events=None,
                     pre_done: bool = False):
    """factor -> adjoint gradient -> refined KKT solve on an object exposing
    kfac, kvals, fvec, sol_adj, tmp, rhs, sol, grad, batch, n_x, n_p, stab.

    ``events``: optional list of >= 3 torch CUDA events recorded after the numeric
    factorization, after the adjoint gradient and after the KKT solve (bench.py).
    """
    st = _lib.stream_handle()
    n_x, n_p = eng.n_x, eng.n_p
    tol, mi = eng.stab.refine_tolerance, eng.stab.max_refine_iters
    torch = eng.torch
    cur = torch.cuda.current_stream()
    t1 = time.perf_counter()
    if getattr(eng, "adjoint_gx", False) and _SIDE_STREAM:
        # The adjoint (G_x factor + solve, reference sensitivity.py:160-198) does not depend
        # on the KKT factor: it runs on a side stream.  The KKT factorization's persistent
        # CTAs retire once its task list is taken, so the G_x launch fills the SMs its
        # dependency-chain tail leaves idle.  Zero-pivot checks of both factors follow the
        # refined solve (still before any convergence error, as in the reference).
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if pre_done:                  # assembly / factor / adjoint already replayed from a graph
            res_a, it_a = np.zeros(eng.batch), np.zeros(eng.batch, dtype=np.int32)
        else:
            res_a, it_a = _factor_adjoint(eng, st, cur, f0, f1, events)
        if timings is not None:
            timings["adjoint_res"] = res_a
            timings["adjoint_iters"] = it_a
        if not need_direction:
            eng.kfac.check(st)
            eng.gfac.check(st)
            return None, None
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(cur)
        rc2, res, its = _refine_with_fallback(eng, st, tol, mi)
        s1.record(cur)
        if events is not None:
            events[2].record()
        eng.gfac.check(st)
        if timings is not None:         # device events: no host sync between the phases
            s1.synchronize()
            if not pre_done:
                timings["factor_s"] = f0.elapsed_time(f1) * 1e-3
            timings["solve_s"] = s0.elapsed_time(s1) * 1e-3
            timings["main_iters"] = its
    else:
        _nan_probe(eng, "before factor")
        eng.kfac.numeric(eng.kvals, *factor_shifts(eng), st)
        if events is not None:
            events[0].record()
        if factor_shifts(eng) == factor_shifts(eng, full=True):
            eng.kfac.check(st)
        t2 = time.perf_counter()
        if timings is not None:
            timings["factor_s"] = t2 - t1
        if getattr(eng, "adjoint_gx", False):
            res_a, it_a = eng.adjoint_direct()
            gradient_from_adjoint(eng, st)
        else:
            # leading (x, lambda) block of the KKT factor preconditions [[A, G^T], [G, 0]]
            rc, res_a, it_a = eng.kfac.solve_refined(eng.kvals, eng.fvec, eng.sol_adj, tol, mi, True, st)
            check(lib().sgn_adjoint_step(0, eng.batch, n_x, n_p, ptr(eng.sol_adj), None, ptr(eng.tmp), None, st))
            eng.kfac.spmv(eng.kvals, eng.tmp, eng.rhs, False, st)
            check(lib().sgn_adjoint_step(1, eng.batch, n_x, n_p, ptr(eng.rhs), ptr(eng.fvec), ptr(eng.tmp),
                                         ptr(eng.grad), st))
            eng.rhs.copy_(eng.tmp)
        if events is not None:
            events[1].record()
        if timings is not None:
            timings["adjoint_res"] = res_a
            timings["adjoint_iters"] = it_a
        _nan_probe(eng, "after adjoint")
        if not need_direction:
            return None, None
        rc2, res, its = _refine_with_fallback(eng, st, tol, mi)
        _nan_probe(eng, f"after refine rc={rc2}")
        if events is not None:
            events[2].record()
        if timings is not None:
            timings["solve_s"] = time.perf_counter() - t2
            timings["main_iters"] = its
    if rc2 == _lib.SGN_NO_CONVERGENCE:
        best = eng.sol.cpu().numpy()
        exc = NoConvergence(f"BiCGSTAB refinement stalled at relative residual {res.max():.3e}",
                            residual=float(res.max()), iterations=int(its.max()),
                            best=best[0] if eng.batch == 1 else best)
        exc.instance_residuals, exc.instance_iterations = res, its      # batched callers
        raise exc
    return res, its


class DeviceEngine:
    """Batched device state + the SGN direction and forward Newton for one MeshPlan."""

    def __init__(self, plan: MeshPlan, params, tvals, batch: int = 1, stab=None):
        torch = _lib.require_cuda()
        self.torch = torch
        self.plan = plan
        self.batch = B = int(batch)
        dev = "cuda"
        f64, i64 = torch.float64, torch.int64
        T = lambda a, dt=f64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        pl = plan
        self.conns = [T(g.conn.astype(np.int32), torch.int32) for g in pl.groups]
        self.conn = self.conns[0]
        plist = params if isinstance(params, (list, tuple)) else [params]
        self.gparams = [T(np.asarray(pp, dtype=np.float64).reshape(B, -1)) for pp in plist]
        self.params = self.gparams[0]
        if pl.R is not None:
            self.R_ptr, self.R_idx, self.R_val = T(pl.R_ptr, i64), T(pl.R_idx, i64), T(pl.R_val)
            self.Rt_ptr, self.Rt_idx, self.Rt_val = T(pl.Rt_ptr, i64), T(pl.Rt_idx, i64), T(pl.Rt_val)
        self.tvals = T(np.asarray(tvals, dtype=np.float64).reshape(B, -1))
        self.tdofs = T(pl.target_dofs, i64)
        self.pos_base, self.pos_ptr, self.pos_idx = T(pl.pos_base), T(pl.pos_ptr, i64), T(pl.pos_idx, i64)
        self.disp_scale = pl.disp_scale
        if pl.disp_scale is not None:
            self.pos_coef = T(pl.pos_coef)
            self.restpos_ptr, self.restpos_idx = T(pl.restpos_ptr, i64), T(pl.restpos_idx, i64)
            self.restpos_coef = T(pl.restpos_coef)
            self.X0_flat = T(pl.X0.ravel())
        self.rest_base, self.rest_ptr = T(pl.rest_base), T(pl.rest_ptr, i64)
        self.rest_idx, self.rest_coef = T(pl.rest_idx, i64), T(pl.rest_coef)
        self.K_base = T(pl.K_base)
        self.ts = None
        if pl.two_stage is not None:           # two-stage assembly lists instead of the one-stage gather's
            t2 = pl.two_stage
            self.ts = {k: (T(v, i64) if v.dtype.kind == "i" else T(v)) for k, v in t2.items()
                       if isinstance(v, np.ndarray)}
            self.ts["unit_ptr"] = torch.arange(max(t2["gx_dst"].size, 1) + 1, dtype=i64, device=dev)
            self.mz = torch.zeros(B, max(t2["n_mz"], 1), dtype=f64, device=dev)
        else:
            self.K_ptr = T(pl.K_ptr, i64)
            self.K_src, self.K_coef = T(pl.K_src, i64), T(pl.K_coef)
        self.G_ptr, self.G_src = T(pl.G_ptr, i64), T(pl.G_src, i64)
        self.G_coef = None if pl.G_coef is None else T(pl.G_coef)
        if pl.restlen is not None:
            self.rl_conn = T(pl.restlen[0].astype(np.int32), torch.int32)
            self.rl_L0 = T(pl.restlen[1])
            self.rl_fptr, self.rl_fsrc, self.rl_fcoef = T(pl.rl_fptr, i64), T(pl.rl_fsrc, i64), T(pl.rl_fcoef)
            self.rl_rptr = T(np.array([0, pl.rl_rsrc.size]), i64)
            self.rl_rsrc = T(pl.rl_rsrc, i64)
            self.rl_half = T(np.full(pl.rl_rsrc.size, 0.5))
            self.rl_obj = torch.zeros(B, 1, dtype=f64, device=dev)
            self.rl_w = torch.full((B,), pl.restlen[2], dtype=f64, device=dev)
        self.G_diag = T(pl.G_diag, i64)
        self.grad_base, self.grad_ptr, self.grad_src = T(pl.grad_base), T(pl.grad_ptr, i64), T(pl.grad_src, i64)
        self.f_ext = T(pl.f_ext)
        self.f_ext_b = self.f_ext.reshape(1, -1).repeat(B, 1).contiguous()
        z = lambda *s: torch.zeros(*s, dtype=f64, device=dev)
        self.x = z(B, pl.n_x)
        self.p = z(B, pl.n_p)
        self.pos = z(B, pl.n_dof)
        self.rest = z(B, pl.n_dof)
        self.restpos = z(B, pl.n_dof) if pl.disp_scale is not None else None
        self.ebuf = z(B, pl.ebuf_size)       # per group [hess | mixed]
        self.egrad = z(B, pl.egrad_size)
        self.eeners = [z(B, g.n_e) for g in pl.groups]
        self.eener = self.eeners[0]
        self.rscr = z(B, max(int(pl.target_dofs.size), 1))
        self.kvals = z(B, pl.nnz)
        if self.ts is not None:                # constant entries (A, B, C) once; the rest every assembly
            self.kvals.copy_(self.K_base.reshape(1, -1).expand(B, -1))
        self.gvals = z(B, pl.G_nnz)
        self.fvec = z(B, pl.dim)
        self.rhs = z(B, pl.dim)
        self.sol = z(B, pl.dim)
        self.sol_adj = z(B, pl.dim)
        self.tmp = z(B, pl.dim)
        self.grad = z(B, pl.n_p)
        self.fobj = z(B)
        self.scal = z(8 + len(pl.groups), B)   # rows: energy, linear energy, trace, |g|inf, -, group energies
        self.gx = z(B, pl.n_x)
        self.kdir = z(B, pl.n_x)
        self.xtry = z(B, pl.n_x)
        self.n_x, self.n_p = pl.n_x, pl.n_p
        self.vplan = vertex_plan(pl)
        if self.vplan is not None:
            vp, i32 = self.vplan, torch.int32
            self.v_inc_ptr, self.v_inc_ea = T(vp.inc_ptr, i32), T(vp.inc_ea, i32)
            self.v_out_ptr, self.v_out_dst = T(vp.out_ptr, i32), T(vp.out_dst, i32)
            self.v_con_ptr, self.v_con_idx = T(vp.con_ptr, i32), T(vp.con_idx, i32)
            self.r_dst, self.r_base = T(vp.rest_dst, i64), T(vp.rest_base)
            self.r_ptr, self.r_src, self.r_coef = T(vp.rest_ptr, i64), T(vp.rest_src, i64), T(vp.rest_coef)
            self.v_group = next(gs for gs in ((6, 8, 16, 32) if pl.groups[0].kind == "tri" else (16, 32))
                                if vp.max_inc <= gs)
            self.v_melems = T(pl.groups[0].melems, i32)
        self._gx_ready = False
        # C = w R^T R + w_reg I > 0 when w_reg > 0: the stabilized KKT is quasi-definite and the
        # p unknowns can join the nested dissection (p_order 1); otherwise they stay last
        self.ksym = symbolic_for(pl.dim, pl.K_indptr, pl.K_indices, pl.n_x, pl.n_p, pl.n_x,
                                 p_order=1 if pl.w_reg > 0.0 else 0)
        self._kfac = None                    # KKT factor storage: allocated on first use
        self._gfac = None
        from .linear_solvers import StabilizationConfig
        self.stab = stab or StabilizationConfig()

    # -- small helpers ---------------------------------------------------------------
    @property
    def stream(self) -> int:
        return _lib.stream_handle()

    def _gather(self, n_out, base, base_stride, ptr_, idx, coef, buf, buf_stride, out, out_stride):
        check(lib().sgn_gather_values(n_out, self.batch, ptr(base), base_stride, ptr(ptr_), ptr(idx),
                                      ptr(coef), ptr(buf), buf_stride, ptr(out), out_stride, self.stream))

    def _gather_to(self, dst, base, ptr_, idx, coef, buf, buf_stride):
        """kvals[dst[k]] = base[k] + sum coef * buf[idx] over ptr_[k] .. ptr_[k + 1] (restricted gather)."""
        check(lib().sgn_gather_to(dst.numel(), self.batch, ptr(dst), ptr(base), ptr(ptr_), ptr(idx), ptr(coef),
                                  ptr(buf), buf_stride, ptr(self.kvals), self.plan.nnz, self.stream))

    def load(self, x=None, p=None):
        """Host (x, p) -> device through pinned staging buffers: the host->device copies are
        asynchronous, so the work queued next (the direction graphs) follows them without a
        host round trip.  The staging buffers are reused once their previous copies are done."""
        torch = self.torch
        if not hasattr(self, "_pin_x"):
            self._pin_x = torch.empty(tuple(self.x.shape), dtype=torch.float64, pin_memory=True)
            self._pin_p = torch.empty(tuple(self.p.shape), dtype=torch.float64, pin_memory=True)
            self._pin_ev = torch.cuda.Event()
            self._pin_ev.record()
        self._pin_ev.synchronize()
        if x is not None:
            self._pin_x.numpy()[...] = np.asarray(x, dtype=np.float64).reshape(self.batch, -1)
            self.x.copy_(self._pin_x, non_blocking=True)
        if p is not None:
            self._pin_p.numpy()[...] = np.asarray(p, dtype=np.float64).reshape(self.batch, -1)
            self.p.copy_(self._pin_p, non_blocking=True)
        self._pin_ev.record()

    def solution_host(self, b: int = 0) -> np.ndarray:
        """Instance b's KKT solution on the host: device -> pinned buffer (asynchronous copy,
        one stream sync) -> a fresh numpy array the caller owns."""
        torch = self.torch
        if not hasattr(self, "_pin_sol"):
            self._pin_sol = torch.empty(tuple(self.sol.shape[1:]), dtype=torch.float64, pin_memory=True)
        self._pin_sol.copy_(self.sol[b], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self._pin_sol.numpy().copy()

    def _deformed(self, x):
        """pos = X0 (fixed) | x (free): position state; pos = restpos + sigma x: displacement state."""
        pl = self.plan
        if pl.disp_scale is None:
            self._gather(pl.n_dof, self.pos_base, 0, self.pos_ptr, self.pos_idx, None, x, pl.n_x,
                         self.pos, pl.n_dof)
        else:
            self._gather(pl.n_dof, self.restpos, pl.n_dof, self.pos_ptr, self.pos_idx, self.pos_coef, x,
                         pl.n_x, self.pos, pl.n_dof)

    def positions(self, x=None):
        pl = self.plan
        x = self.x if x is None else x
        self._gx_ready = False
        self._gather(pl.n_dof, self.rest_base, 0, self.rest_ptr, self.rest_idx, self.rest_coef,
                     self.p, pl.n_p, self.rest, pl.n_dof)
        if pl.disp_scale is not None:
            self._gather(pl.n_dof, self.X0_flat, 0, self.restpos_ptr, self.restpos_idx, self.restpos_coef,
                         self.p, pl.n_p, self.restpos, pl.n_dof)
        self._deformed(x)

    def element_blocks(self, mixed: bool = True, hess: bool = True):
        """Element Hessians (and, with mixed=True, the rest-shape mixed blocks of the
        p-map support) into ebuf; the forward Newton needs the Hessians only, the fused
        KKT assembly the mixed blocks only."""
        pl = self.plan
        if not hasattr(self, "_mslots"):
            self._mslots = [None if g.mslot is None else
                            self.torch.as_tensor(g.mslot, dtype=self.torch.int32, device="cuda") for g in pl.groups]
        for g, conn, prm, ms in zip(pl.groups, self.conns, self.gparams, self._mslots):
            check(lib().sgn_element_derivs_ex(g.code, g.n_e, self.batch, ptr(conn), ptr(self.pos), ptr(self.rest),
                                              pl.n_dof, ptr(prm), prm.stride(0),
                                              ptr(self.ebuf[:, g.hoff:]) if (hess or g.mslot is None) else None,
                                              ptr(self.ebuf[:, g.moff:]) if (mixed or g.mslot is None) else None,
                                              ptr(ms) if ms is not None else None, pl.ebuf_size,
                                              pl.rest_comp_mask, self.stream))

    def _vertex(self, kv, gv):
        pl, vp = self.plan, self.vplan
        g = pl.groups[0]
        check(lib().sgn_vertex_assemble(g.code, vp.n_task, self.v_group, self.batch, ptr(self.v_inc_ptr),
                                        ptr(self.v_inc_ea), ptr(self.v_out_ptr), ptr(self.v_out_dst),
                                        ptr(self.v_con_ptr), ptr(self.v_con_idx), ptr(self.conns[0]),
                                        ptr(self.pos), ptr(self.rest), pl.n_dof, ptr(self.gparams[0]),
                                        self.gparams[0].stride(0), ptr(kv), pl.nnz if kv is not None else 0,
                                        ptr(gv), pl.G_nnz if gv is not None else 0, self.stream))

    def assemble_kkt(self):
        """KKT values (and G_x, for the adjoint) from the current positions.  Fused path
        (single-group neo-Hookean meshes): G_x entries by the vertex kernel, mixed blocks of
        the p-map support, then the remaining entries by the restricted gather.  Otherwise
        the staged path: element blocks -> gather."""
        pl = self.plan
        if self.vplan is not None:
            self._vertex(self.kvals, self.gvals)
            if self.vplan.needs_mixed:
                g = pl.groups[0]
                check(lib().sgn_element_mixed(g.code, g.n_m, self.batch, ptr(self.v_melems), ptr(self.conns[0]),
                                              ptr(self.pos), ptr(self.rest), pl.n_dof, ptr(self.gparams[0]),
                                              self.gparams[0].stride(0), ptr(self.ebuf[:, g.moff:]),
                                              pl.ebuf_size, self.stream))
            check(lib().sgn_gather_to(self.r_dst.numel(), self.batch, ptr(self.r_dst), ptr(self.r_base),
                                      ptr(self.r_ptr), ptr(self.r_src), ptr(self.r_coef), ptr(self.ebuf),
                                      self.ebuf.stride(0), ptr(self.kvals), pl.nnz, self.stream))
            self._gx_ready = True
            return
        self.element_blocks()
        if self.ts is not None:
            # two-stage path (MeshPlan._two_stage_lists): G_x once -> both K blocks; Mz, then
            # G_p = Mz P -> both K blocks
            ts = self.ts
            self._gather(pl.G_nnz, None, 0, self.G_ptr, self.G_src, self.G_coef, self.ebuf, self.ebuf.stride(0),
                         self.gvals, pl.G_nnz)
            self._gather_to(ts["gx_dst"], None, ts["unit_ptr"], ts["gx_src"], None, self.gvals, pl.G_nnz)
            self._gather(self.mz.shape[1], None, 0, ts["mz_ptr"], ts["mz_src"], None, self.ebuf,
                         self.ebuf.stride(0), self.mz, self.mz.shape[1])
            self._gather_to(ts["gp_dst"], None, ts["gp_ptr"], ts["gp_src"], ts["gp_coef"], self.mz, self.mz.shape[1])
            self._gx_ready = True
            return
        self._restlen_blocks()
        self._gather(pl.nnz, self.K_base, 0, self.K_ptr, self.K_src, self.K_coef, self.ebuf,
                     self.ebuf.stride(0), self.kvals, pl.nnz)

    def _restlen_blocks(self):
        pl = self.plan
        if pl.restlen is None:
            return
        check(lib().sgn_restlen_blocks(len(pl.restlen[0]), self.batch, ptr(self.rl_conn), ptr(self.rest), pl.n_dof,
                                       ptr(self.rl_L0), pl.restlen[2], ptr(self.ebuf[:, pl.rl_off:]),
                                       self.ebuf.stride(0), self.stream))

    def gx_values(self, force: bool = False):
        """G_x = dc/dx values (generic pattern) at the current positions into self.gvals."""
        if self._gx_ready and not force:
            return
        pl = self.plan
        if self.vplan is not None:
            self._vertex(None, self.gvals)
        else:
            self.element_blocks(mixed=False)
            self._gather(pl.G_nnz, None, 0, self.G_ptr, self.G_src, self.G_coef, self.ebuf, self.ebuf.stride(0),
                         self.gvals, pl.G_nnz)
        self._gx_ready = True

    # -- SGN direction (staged) ----------------------------------------------------------
    def assemble(self):
        """Element blocks -> KKT values, least-squares terms (fvec, fobj) at (x, p)."""
        pl = self.plan
        self.positions()
        self.assemble_kkt()
        self._lsq(self.x, self.fvec)

    def direction(self, timings: dict | None = None):
        """SGN direction at the current (x, p) of every instance (solution in self.sol).

        Returns (rel_res[batch], iters[batch]); raises NoConvergence like
        solve_kkt_stabilized when any instance's refinement stalls.
        """
        torch = self.torch
        nvtx = torch.cuda.nvtx
        graphs = self._direction_graphs()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        nvtx.range_push("sgn.assemble")
        if graphs is not None:
            # assembly, then KKT factor || adjoint + right-hand side: two graph launches
            # instead of ~30 kernel / memset launches issued from Python
            graphs[0].replay()
            e1.record()
            nvtx.range_pop()
            nvtx.range_push("sgn.factor+adjoint")
            graphs[1].replay()
            e2.record()
        else:
            self.assemble()
            e1.record()
        nvtx.range_pop()
        nvtx.range_push("sgn.refined_solve")
        try:
            return sgn_solve_stages(self, timings, pre_done=graphs is not None)
        finally:
            nvtx.range_pop()
            if timings is not None:       # device events, read after the refinement's sync
                e1.synchronize()
                timings["assemble_s"] = e0.elapsed_time(e1) * 1e-3
                if graphs is not None:
                    e2.synchronize()
                    timings["factor_s"] = e1.elapsed_time(e2) * 1e-3

    def _direction_graphs(self):
        """(assembly graph, factor || adjoint graph), captured once per stabilization shift;
        None when disabled (SGN_DIRECTION_GRAPH=0), without the side stream, or when the
        capture fails (the eager path then stays in use)."""
        if not (_DIR_GRAPH and _SIDE_STREAM and getattr(self, "adjoint_gx", False)):
            return None
        key = factor_shifts(self)
        cached = getattr(self, "_dgraphs", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        if cached is not None and cached[1] is None:          # capture failed before
            return None
        torch = self.torch
        try:
            # warm-up off the graph: lazily created factors, scratch buffers, kernel attributes
            self.assemble()
            _factor_adjoint(self, _lib.stream_handle(), torch.cuda.current_stream())
            torch.cuda.synchronize()
            g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                self.assemble()
            with torch.cuda.graph(g2):
                _factor_adjoint(self, _lib.stream_handle(), torch.cuda.current_stream())
            torch.cuda.synchronize()
            self._dgraphs = (key, (g1, g2))
        except Exception as exc:                              # noqa: BLE001 -- fall back to eager
            import sys
            print(f"[sgn] direction graph capture failed, eager path: {exc!r}", file=sys.stderr)
            torch.cuda.synchronize()
            self._dgraphs = (key, None)
        return self._dgraphs[1]

    adjoint_gx = True
    factor_shift_scale = 1e-4          # see factor_shifts(): 1.0 = the reference's full shift
    floor_stall_window = 0             # simulate(): float-floor stall cut-off (0: reference behaviour)
    ir_steps = int(os.environ.get("SGN_IR_STEPS", "2"))   # mixed-precision refinement steps (_refine_with_fallback)

    def adjoint_direct(self, check_pivots: bool = True):
        """w = G_x^{-1} f_x (unshifted LDL^T of the state Jacobian) placed as v = (0, 0, w)
        in self.tmp (and its low word in self.tmp_lo); returns (res, iters) placeholders of
        the refined variant.  With check_pivots=False the caller checks the factor's status
        later (no host sync here).

        w comes from extra-precise iterative refinement on the factor (sgn_solve_ir:
        double-double residuals, w carried as a double-double): the unpivoted LDL^T of the
        ill-conditioned shell G_x is not backward stable the way SuperLU's partial pivoting
        is, and the reduced Hessian of config 4 amplifies a gradient error ~1e6-fold into dp,
        so the gradient is taken to the double rounding of the exact one (gradient_from_
        adjoint); ``adj_ir_steps`` = 0 restores the single double-precision refinement step."""
        pl = self.plan
        st = self.stream
        self.gx_values()
        self.gfac.numeric(self.gvals, 0.0, 0.0, st)
        if check_pivots:
            self.gfac.check(st)
        check(lib().sgn_adjoint_step(3, self.batch, pl.n_x, pl.n_p, ptr(self.fvec), None, ptr(self.xtry), None, st))
        n = pl.n_x
        torch = self.torch
        if not hasattr(self, "_adj_r"):
            self._adj_r, self._adj_d = torch.empty_like(self.kdir), torch.empty_like(self.kdir)
            self._adj_lo = torch.zeros_like(self.kdir)
            self.tmp_lo = torch.zeros_like(self.tmp)
            self._adj_pm = torch.tensor([1.0, -1.0], dtype=torch.float64, device="cuda").repeat_interleave(
                self.batch).reshape(2, self.batch).contiguous()
        steps = int(getattr(self, "adj_ir_steps", 0))
        if steps > 0:
            self.gfac.solve_ir(self.gvals, self.xtry, self.kdir, steps, st, sol_lo=self._adj_lo, report=False)
        else:
            self.gfac.solve(self.xtry, self.kdir, False, st)
            self.gfac.spmv(self.gvals, self.kdir, self._adj_r, False, st)                       # G w
            check(lib().sgn_axpy(n, self.batch, ptr(self._adj_pm[1]), ptr(self._adj_r), ptr(self.xtry),
                                 ptr(self._adj_r), n, st))                                      # f - G w
            self.gfac.solve(self._adj_r, self._adj_d, False, st)
            check(lib().sgn_axpy(n, self.batch, ptr(self._adj_pm[0]), ptr(self._adj_d), ptr(self.kdir),
                                 ptr(self.kdir), n, st))                                        # w += d
            self._adj_lo.zero_()
        check(lib().sgn_adjoint_step(2, self.batch, pl.n_x, pl.n_p, ptr(self.kdir), None, ptr(self.tmp), None, st))
        check(lib().sgn_adjoint_step(2, self.batch, pl.n_x, pl.n_p, ptr(self._adj_lo), None, ptr(self.tmp_lo), None, st))
        return np.zeros(self.batch), np.zeros(self.batch, dtype=np.int32)

    adj_ir_steps = 2                   # extra-precise refinement steps of the adjoint solve

    def split(self):
        pl = self.plan
        s = self.sol
        return s[:, :pl.n_x], s[:, pl.n_x:pl.n_x + pl.n_p], s[:, pl.n_x + pl.n_p:]

    def _lsq(self, x, fvec):
        """Least-squares terms (sensitivity.py:83-93) incl. the optional residual p-map R and
        the displacement state's scale; the block partials and tickets are this engine's own."""
        pl = self.plan
        if not hasattr(self, "_lsq_args"):
            torch = self.torch
            self._lsq_part = torch.zeros(self.batch, 128, dtype=torch.float64, device="cuda")
            self._lsq_tick = torch.zeros(self.batch, dtype=torch.int32, device="cuda")
            a = _lib.LsqArgs()
            a.n_x, a.n_p, a.n_t = pl.n_x, pl.n_p, int(pl.target_dofs.size)
            a.tdofs, a.tvals, a.tstride = ptr(self.tdofs), ptr(self.tvals), self.tvals.stride(0)
            a.w_t, a.w_reg = pl.w_target, pl.w_reg
            a.x_scale = 1.0 if pl.disp_scale is None else pl.disp_scale
            if pl.R is not None:
                a.rptr, a.ridx, a.rcoef = ptr(self.R_ptr), ptr(self.R_idx), ptr(self.R_val)
                a.rtptr, a.rtidx, a.rtcoef = ptr(self.Rt_ptr), ptr(self.Rt_idx), ptr(self.Rt_val)
                a.rscr = ptr(self.rscr)
            a.part, a.tickets = ptr(self._lsq_part), ptr(self._lsq_tick)
            self._lsq_args = a
        check(lib().sgn_lsq_eval(self.batch, ctypes.byref(self._lsq_args), ptr(x), ptr(self.p), ptr(fvec),
                                 ptr(self.fobj), self.stream))
        if pl.restlen is not None:
            # rest-length residuals: f_p += w J_p^T r (gather over each p's springs), f += w/2 sum r^2
            self._restlen_blocks()
            if fvec is not None:
                fp = fvec[:, pl.n_x:]
                self._gather(pl.n_p, fp, pl.dim, self.rl_fptr, self.rl_fsrc, self.rl_fcoef, self.ebuf,
                             self.ebuf.stride(0), fp, pl.dim)
            self._gather(1, None, 0, self.rl_rptr, self.rl_rsrc, self.rl_half, self.ebuf, self.ebuf.stride(0),
                         self.rl_obj, 1)
            check(lib().sgn_axpy(1, self.batch, ptr(self.rl_w), ptr(self.rl_obj), ptr(self.fobj), ptr(self.fobj), 1,
                                 self.stream))

    # -- objective ---------------------------------------------------------------------
    def objective(self, x=None):
        pl = self.plan
        x = self.x if x is None else x
        self._lsq(x, None)
        return self.fobj

    # -- forward statics (forward.py:135-203) --------------------------------------------
    def _energy_grad(self, x, want_grad=True):
        """Energies (per group, reduced into scal[5+g]; scal[0] = their sum on read) and the
        free-dof gradient gx of the current rest shape."""
        pl = self.plan
        st = self.stream
        self._gx_ready = False
        self._deformed(x)
        for gi, (g, conn, prm, en) in enumerate(zip(pl.groups, self.conns, self.gparams, self.eeners)):
            check(lib().sgn_element_energy_grad(g.code, g.n_e, self.batch, ptr(conn), ptr(self.pos),
                                                ptr(self.rest), pl.n_dof, ptr(prm), prm.stride(0), ptr(en),
                                                ptr(self.egrad[:, g.goff:]) if want_grad else 0,
                                                pl.egrad_size, st))
            check(lib().sgn_reduce(0, g.n_e, self.batch, ptr(en), None, g.n_e, ptr(self.scal[5 + gi]), st))
        check(lib().sgn_reduce(1, pl.n_dof, self.batch, ptr(self.f_ext_b), ptr(self.pos), pl.n_dof,
                               ptr(self.scal[1]), st))
        if want_grad:
            self._gather(pl.n_x, self.grad_base, 0, self.grad_ptr, self.grad_src, None, self.egrad,
                         pl.egrad_size, self.gx, pl.n_x)

    def _energies(self, sc):
        """Total energy per instance from a host copy of scal."""
        ng = len(self.plan.groups)
        return sc[5:5 + ng].sum(axis=0) + sc[1]

    def _hessian(self):
        self.gx_values(force=True)

    @property
    def kfac(self):
        if self._kfac is None:
            self._kfac = DeviceFactor(self.ksym, self.batch)
        return self._kfac

    @property
    def gfac(self):
        if self._gfac is None:
            pl = self.plan
            # sweeps: SGN_GX_FAT_TILES / SGN_GX_LEAF_SIZE apply to the G_x analysis only
            gopt = {k: int(os.environ[e]) for k, e in (("fat_tiles", "SGN_GX_FAT_TILES"), ("leaf_size", "SGN_GX_LEAF_SIZE"))
                    if os.environ.get(e)}
            self.gsym = symbolic_for(pl.n_x, pl.G_indptr, pl.G_indices, **gopt)
            self._gfac = DeviceFactor(self.gsym, self.batch)
        return self._gfac

    def _trace(self):
        """Per-instance trace of the Newton Hessian (gathered on the device)."""
        pl = self.plan
        if not hasattr(self, "_diag_ptr"):
            T = lambda a, dt: self.torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
            self._diag_ptr = T(np.arange(pl.G_diag.size + 1), self.torch.int64)
            self._diag_idx = T(pl.G_diag, self.torch.int64)
            self._diag_buf = self.torch.empty((self.batch, pl.G_diag.size), dtype=self.torch.float64, device="cuda")
        n = int(pl.G_diag.size)
        self._gather(n, None, 0, self._diag_ptr, self._diag_idx, None, self.gvals, pl.G_nnz,
                     self._diag_buf, n)                         # one thread per diagonal entry
        check(lib().sgn_reduce(0, n, self.batch, ptr(self._diag_buf), None, n, ptr(self.scal[2]),
                               _lib.stream_handle()))           # fixed-tree sum
        return self.scal[2].cpu().numpy()

    def _mask(self, m):
        return self.torch.as_tensor(np.asarray(m, dtype=np.int32), device="cuda")

    def simulate(self, tol: float, max_iters: int = 200, active=None):
        """Batched damped Newton on the energy from the current x (forward.py:135-203).

        Every instance follows the reference iteration on its own (converged / failed
        instances are masked); returns a status array (1 converged, -1 failed).
        """
        torch = self.torch
        pl = self.plan
        st = self.stream
        B, n = self.batch, pl.n_x
        status = np.zeros(B, dtype=np.int64)
        if active is not None:
            status[~np.asarray(active, bool)] = 1
        self.positions()                       # rest positions for the current p
        self.newton_iters = 0
        if getattr(self, "_fp", None) is None:
            self._fp = torch.zeros(B, dtype=torch.int64, device="cuda")
        seen = [set() for _ in range(B)]
        best = np.full(B, np.inf)                  # smallest |c|_inf so far
        since = np.zeros(B, dtype=np.int64)        # iterations without a new best
        win = int(getattr(self, "floor_stall_window", 0))
        for _ in range(max_iters):
            run = status == 0
            if not run.any():
                break
            self.newton_iters += 1
            self._energy_grad(self.x)
            check(lib().sgn_reduce(2, n, B, ptr(self.gx), None, n, ptr(self.scal[3]), st))
            check(lib().sgn_fingerprint(n, B, ptr(self.x), n, ptr(self._fp), st))
            sc = self.scal.cpu().numpy()
            fp = self._fp.cpu().numpy()
            g_inf, e0 = sc[3], self._energies(sc)
            # a bitwise-repeated iterate (fingerprint, |g|_inf and energy all equal) makes the
            # deterministic iteration periodic through states that all failed the tolerance:
            # the reference would run out its max_iters and raise; fail now, same outcome
            # (config-5 line searches: trial states whose float floor is above tol cycle
            # through ~4 states for the remaining ~190 iterations)
            for b in np.flatnonzero(run & (g_inf > tol)):
                key = (int(fp[b]), float(g_inf[b]), float(e0[b]))
                if key in seen[b]:
                    status[b] = -1
                else:
                    seen[b].add(key)
            # float-floor stall (option, off by default: floor_stall_window = 0 is the
            # reference's iteration exactly): |c|_inf within 100 x tol that sets no new
            # minimum for `win` iterations sits on the float64 floor of the state and cannot
            # reach tol; fail now instead of after max_iters
            if win > 0:
                imp = g_inf < best
                best = np.where(imp, g_inf, best)
                since = np.where(imp, 0, since + 1)
                status[run & (g_inf > tol) & (g_inf <= 100.0 * tol) & (since >= win)] = -1
            if _DEBUG_NEWTON:
                print(f"[newton] |g|inf {g_inf[:4]} E {e0[:4]} tol {tol:.3e}", flush=True)
            status[run & (g_inf <= tol)] = 1
            # a non-finite energy or gradient can never pass the energy Armijo test (every
            # comparison with NaN is false): the reference's 8 shift escalations would all
            # fail and raise (forward.py:155-164); fail those instances now
            status[(status == 0) & ~(np.isfinite(e0) & np.isfinite(g_inf))] = -1
            run = status == 0
            if not run.any():
                break
            self._hessian()
            trace = self._trace()
            self._newton_step(trace, n, run, bias=False)
            accepted = np.zeros(B, bool)
            for _esc in range(8):              # escalate the shift if the line search stalls
                need = run & ~accepted
                if not need.any():
                    break
                ok = self._backtrack(e0, need)
                accepted |= ok
                still = need & ~ok
                if still.any():
                    self._newton_step(trace, n, still, bias=True)
            status[run & ~accepted] = -1
        status[status == 0] = -1
        if B == 1 and status[0] != 1:
            raise ForwardSimFailure("static solve: no convergence / line search failed")
        return status

    def _newton_step(self, trace, n, mask, bias):
        """tau-regularized Newton directions into self.kdir for masked instances
        (forward.py:171-186: tau0 = 1e-6 |tr K| / n + 1e-12, x10 ladder, -g fallback)."""
        torch = self.torch
        st = self.stream
        B = self.batch
        tau0 = 1e-6 * np.abs(trace) / max(n, 1) + 1e-12
        tau = np.where(bias, tau0 * 1e6, 0.0) * np.ones(B)
        done = ~np.asarray(mask, bool)
        if not hasattr(self, "_neg1"):
            self._neg1 = torch.full((B,), -1.0, dtype=torch.float64, device="cuda")
            self._negg = torch.empty_like(self.gx)
        neg = self._negg
        check(lib().sgn_axpy(n, B, ptr(self._neg1), ptr(self.gx), None, ptr(neg), n, st))   # -g
        dots = torch.empty(B, dtype=torch.float64, device="cuda")
        amax = torch.empty(B, dtype=torch.float64, device="cuda")
        for _ in range(60):
            tau_d = torch.as_tensor(tau, dtype=torch.float64, device="cuda")
            self.gfac.numeric_v(self.gvals, tau_d, None, st)
            piv = self.gfac.status(st)
            self.gfac.solve(neg, self.xtry, False, st)
            check(lib().sgn_reduce(1, n, B, ptr(self.gx), ptr(self.xtry), n, ptr(dots), st))
            check(lib().sgn_reduce(2, n, B, ptr(self.xtry), None, n, ptr(amax), st))
            gd, am = dots.cpu().numpy(), amax.cpu().numpy()
            ok = (~done) & (piv < 0) & (gd < 0) & np.isfinite(am)
            if ok.any():
                check(lib().sgn_masked_copy(n, B, ptr(self._mask(ok)), ptr(self.xtry), ptr(self.kdir), n, st))
            done |= ok
            if done.all():
                return
            tau = np.where(done, tau, np.where(tau == 0.0, tau0, tau * 10.0))
        left = ~done
        check(lib().sgn_masked_copy(n, B, ptr(self._mask(left)), ptr(neg), ptr(self.kdir), n, st))

    def _backtrack(self, e0, mask, c1=1e-4, factor=0.5, max_bt=60):
        """Per-instance Armijo on the energy with the reference's float slack
        (forward.py:189-203); accepted instances get x <- x + alpha d.  Returns ok[B]."""
        torch = self.torch
        st = self.stream
        B, n = self.batch, self.plan.n_x
        slope_t = torch.empty(B, dtype=torch.float64, device="cuda")
        check(lib().sgn_reduce(1, n, B, ptr(self.gx), ptr(self.kdir), n, ptr(slope_t), st))
        slope = slope_t.cpu().numpy()
        if self.plan.disp_scale is not None:       # dE/dalpha = c . (sigma d) in the displacement state
            slope = slope * self.plan.disp_scale
        slack = 4e-15 * np.abs(e0)
        alpha = np.ones(B)
        pending = np.asarray(mask, bool).copy()
        ok = np.zeros(B, bool)
        for _ in range(max_bt):
            if not pending.any():
                break
            a_t = torch.as_tensor(np.where(pending, alpha, 0.0), dtype=torch.float64, device="cuda")
            check(lib().sgn_axpy(n, B, ptr(a_t), ptr(self.kdir), ptr(self.x), ptr(self.xtry), n, st))
            self._energy_grad(self.xtry, want_grad=False)
            sc = self.scal.cpu().numpy()
            et = self._energies(sc)
            acc = pending & np.isfinite(et) & (et <= e0 + c1 * alpha * slope + slack)
            if acc.any():
                check(lib().sgn_masked_copy(n, B, ptr(self._mask(acc)), ptr(self.xtry), ptr(self.x), n, st))
            ok |= acc
            pending &= ~acc
            alpha = np.where(pending, alpha * factor, alpha)
        return ok


def kkt_inverse_p(eng, rhs_p, factor: bool):
    """Solve the stabilized-then-refined SGN KKT system with right-hand side (0, rhs_p, 0)
    on the device (the initial inverse Hessian of L-BFGS-SGN, optimize.py:446-450).

    factor=True (re)factors the KKT values first (assembled by the caller).  Returns the
    host solution and (rel_res, iters) of instance 0.
    """
    st = _lib.stream_handle()
    n_x, n_p = eng.n_x, eng.n_p
    if factor or getattr(eng, "last_full_shift", False):
        eng.kfac.numeric(eng.kvals, *factor_shifts(eng), st)
    eng.rhs.zero_()
    eng.rhs[0, n_x:n_x + n_p].copy_(eng.torch.from_numpy(np.ascontiguousarray(rhs_p, dtype=np.float64)))
    # the direction path's solve (same factor shift, refinement and fallback): an empty
    # L-BFGS history reproduces the SGN direction bitwise (checks.py:213-226)
    rc, res, its = _refine_with_fallback(eng, st, eng.stab.refine_tolerance, eng.stab.max_refine_iters)
    sol = eng.sol[0].cpu().numpy()
    if rc == _lib.SGN_NO_CONVERGENCE:
        raise NoConvergence(f"BiCGSTAB refinement stalled at relative residual {res.max():.3e}",
                            residual=float(res.max()), iterations=int(its.max()), best=sol)
    return sol, float(res[0]), int(its[0])


class HostKKT:
    """Device solve stages for a KKT assembled on the host by a plugin problem.

    Generic (user) problems evaluate their Jacobians on the CPU (their own code); the
    stacked KKT values and the least-squares gradient are uploaded and the factor /
    adjoint / refined solve run on the device exactly as for the native problems.
    """

    def __init__(self, K, n_x: int, n_p: int, stab):
        torch = _lib.require_cuda()
        from .linear_solvers import _symmetric_pattern
        indptr, indices, src = _symmetric_pattern(K)
        self.torch = torch
        self.batch, self.n_x, self.n_p, self.stab = 1, int(n_x), int(n_p), stab
        dim = 2 * self.n_x + self.n_p
        self.ksym = symbolic_for(dim, indptr, indices, self.n_x, self.n_p, self.n_x)
        self.kfac = DeviceFactor(self.ksym, 1)
        vals = np.where(src >= 0, K.data[np.maximum(src, 0)], 0.0)
        z = lambda m: torch.zeros(1, m, dtype=torch.float64, device="cuda")
        self.kvals = torch.as_tensor(vals, device="cuda").reshape(1, -1)
        self.fvec, self.sol_adj, self.tmp, self.rhs, self.sol = (z(dim) for _ in range(5))
        self.grad = z(self.n_p)

    def set_fvec(self, fx, fp):
        v = np.zeros(2 * self.n_x + self.n_p)
        v[:self.n_x] = fx
        v[self.n_x:self.n_x + self.n_p] = fp
        self.fvec.copy_(self.torch.as_tensor(v).reshape(1, -1))

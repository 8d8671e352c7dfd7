"""High-accuracy KKT solutions for the ill-conditioned full-size configs (test fixtures).

    python tests/golden/make_golden_exact.py c4     (build container, ~15 min, ~12 GB)

The reference's direction contract is a relative residual <= 1e-10 on the unshifted KKT
(linear_solvers.py:130-175).  On the 201x201 shell the KKT amplifies such a residual by
~1e8 into dp, so two solvers that both meet the contract -- the reference's SuperLU +
BiCGSTAB and the device LDL^T + BiCGSTAB -- legitimately differ by ~1e-3 in dp.  This
script pins the EXACT solution of the oracle's KKT (oracle/sgn_cpu.assemble_sgn at the
reference equilibrium of tests/golden/large_c4.npz) to double precision, so the device
solution and the reference's own solution can both be measured against it:

* K_s = K + diag(eps) is factored by SuperLU (the oracle's preconditioner);
* mixed-precision iterative refinement: the residual b - K x is computed EXACTLY (error-free
  products by Dekker splitting, compensated row sums: double-double accuracy), each
  correction is solved by the oracle's BiCGSTAB to 1e-10, until the correction is below
  the double rounding of x.

It also pins the exact adjoint gradient (G_x^T lambda = -f_x refined the same way): the
reduced Gauss-Newton Hessian of the shell amplifies a gradient perturbation ~1e6-fold into
dp, so a gradient accurate to double rounding still moves dp by ~1e-3 between solvers; the
solve is therefore pinned for a GIVEN right-hand side (the reference's gradient), and the
gradient separately.

Writes tests/golden/large_c4_exact.npz: g_exact; dp/dx/dlam_exact (rhs from the reference
gradient of large_c4.npz) and dp/dx/dlam_exact_gexact (rhs from g_exact); residual
histories; the reference's gradient and dp errors.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

_SPLIT = 134217729.0   # 2^27 + 1


def _split(a):
    t = _SPLIT * a
    hi = t - (t - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, e


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def dd_residual(a: sp.csr_matrix, x: np.ndarray, b: np.ndarray, x_lo=None) -> np.ndarray:
    """b - a @ (x + x_lo) with double-double accuracy, rounded to double (rows padded to the
    max row length, summed column by column with TwoSum and a compensation term; the low
    word x_lo of a double-double x only needs double products)."""
    a = a.tocsr()
    n = a.shape[0]
    cnt = np.diff(a.indptr)
    width = int(cnt.max())
    pos = np.arange(a.nnz) - np.repeat(a.indptr[:-1], cnt)
    P = np.zeros((n, width))
    E = np.zeros((n, width))
    p, e = _two_prod(a.data, x[a.indices])
    P[np.repeat(np.arange(n), cnt), pos] = -p
    E[np.repeat(np.arange(n), cnt), pos] = -e
    s = b.astype(np.float64).copy()
    comp = np.zeros(n) if x_lo is None else -(a @ x_lo)
    for k in range(width):
        s, err = _two_sum(s, P[:, k])
        comp += err + E[:, k]
    return s + comp


def exact_solve(a, M, rhs, max_outer=12, log=print):
    """Mixed-precision iterative refinement of a x = rhs to the double rounding of the
    exact solution: exact (double-double) residuals, corrections by the oracle's BiCGSTAB
    preconditioned with the factor M."""
    from oracle import sgn_cpu
    a = a.tocsr()
    ac = a.tocsc()
    bnorm = np.linalg.norm(rhs)
    x = M.solve(rhs)
    x, res, it = sgn_cpu.bicgstab_refine(ac, rhs, x, M, 1e-10, 50)
    lo = np.zeros_like(x)                 # x is carried as a double-double (x, lo)
    hist = [(0, res, it, float("nan"))]
    log(f"reference-style solve: residual {res:.3e} after {it} BiCGSTAB iterations")
    for k in range(1, max_outer + 1):
        r = dd_residual(a, x, rhs, lo)
        rr = np.linalg.norm(r) / bnorm
        d0 = M.solve(r)
        d, dres, dit = sgn_cpu.bicgstab_refine(ac, r, d0, M, 1e-10, 50)
        s, e = _two_sum(x, d)
        e = e + lo
        x = s + e
        lo = e - (x - s)
        step = np.linalg.norm(d) / np.linalg.norm(x)
        hist.append((k, rr, dit, step))
        log(f"outer {k}: exact residual before {rr:.3e}, correction {step:.3e} ({dit} BiCGSTAB its)")
        if step < 1e-22:
            break
    rr = np.linalg.norm(dd_residual(a, x, rhs, lo)) / bnorm
    hist.append((-1, rr, 0, 0.0))
    log(f"final exact residual {rr:.3e}")
    return x, np.array(hist)


def exact_gradient(prob, x, p, log=print):
    """df/dp = f_p + G_p^T lambda with G_x^T lambda = -f_x solved exactly (sensitivity.py:
    181-198; SuperLU of G_x, refinement with double-double residuals)."""
    from oracle import sgn_cpu
    Gx = prob.constraint_jac_x(x, p).to_scipy().tocsc()
    t0 = time.time()
    F = sgn_cpu.LuFactor(sgn_cpu.Csc(Gx))
    log(f"SuperLU of G_x: {time.time() - t0:.0f} s")
    fx, fp = sgn_cpu.objective_grads(prob, x, p)
    GT = Gx.T.tocsr()
    lam = -F.solve(fx, transpose=True)
    lo = np.zeros_like(lam)
    for k in range(12):
        r = dd_residual(GT, lam, -fx, lo)
        d = F.solve(r, transpose=True)
        s, e = _two_sum(lam, d)
        e = e + lo
        lam = s + e
        lo = e - (lam - s)
        step = np.linalg.norm(d) / np.linalg.norm(lam)
        log(f"adjoint refinement {k + 1}: correction {step:.3e}")
        if step < 1e-22:
            break
    Gp = prob.constraint_jac_p(x, p).to_scipy().tocsr()
    # f_p + G_p^T lambda with exact products and compensated sums (rows of G_p^T)
    g = -dd_residual(Gp.T.tocsr(), lam, -fp, lo)
    return g


def main(which):
    assert which == "c4"
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    gold = np.load(os.path.join(HERE, "large_c4.npz"))
    prob = ShellProblem(shell_spec(201, 100))
    x, p = gold["x"], gold["p"]
    n_x, n_p = prob.n_x, prob.n_p
    g_exact = exact_gradient(prob, x, p)
    g_ref = gold["grad"]
    g_err = np.linalg.norm(g_ref - g_exact) / np.linalg.norm(g_exact)
    print(f"reference gradient vs exact: {g_err:.3e}", flush=True)
    A, B, C = sgn_cpu.gn_blocks(prob, x, p)
    K = sgn_cpu.stack_kkt(A, B, C, prob.constraint_jac_x(x, p), prob.constraint_jac_p(x, p))
    t0 = time.time()
    M = sgn_cpu.LuFactor(sgn_cpu.stabilized(K, n_x, n_p, n_x, 1e-6, 1e-6))
    print(f"SuperLU of K_s: {time.time() - t0:.0f} s", flush=True)
    out = {}
    for tag, g in (("", g_ref), ("_gexact", g_exact)):
        rhs = np.zeros(2 * n_x + n_p)
        rhs[n_x:n_x + n_p] = -g
        sol, hist = exact_solve(K.to_scipy(), M, rhs)
        out.update({f"dp_exact{tag}": sol[n_x:n_x + n_p], f"dx_exact{tag}": sol[:n_x],
                    f"dlam_exact{tag}": sol[n_x + n_p:], f"history{tag}": hist})
    dp = out["dp_exact"]
    ref_err = np.linalg.norm(gold["dp"] - dp) / np.linalg.norm(dp)
    sens = np.linalg.norm(out["dp_exact_gexact"] - dp) / np.linalg.norm(dp)
    print(f"reference dp (large_c4.npz, rel.res {float(gold['rel_res']):.2e}) vs exact solve of its own "
          f"rhs: {ref_err:.3e}; exact dp for the exact gradient vs for the reference gradient: {sens:.3e}")
    np.savez_compressed(os.path.join(HERE, "large_c4_exact.npz"), g_exact=g_exact, ref_grad_err=g_err,
                        ref_dp_err=ref_err, dp_sensitivity=sens, ref_rel_res=float(gold["rel_res"]), **out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4")

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

Writes tests/golden/large_c4_exact.npz: dp_exact, dx_exact, dlam_exact, the residual
history and the reference's (large_c4.npz) dp error against dp_exact.
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


def dd_residual(a: sp.csr_matrix, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """b - a @ x with double-double accuracy, rounded to double (rows padded to the max
    row length, summed column by column with TwoSum and a compensation term)."""
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
    comp = np.zeros(n)
    for k in range(width):
        s, err = _two_sum(s, P[:, k])
        comp += err + E[:, k]
    return s + comp


def exact_solve(K, n_x, n_p, rhs, max_outer=12, log=print):
    from oracle import sgn_cpu
    a = K.to_scipy().tocsr()
    t0 = time.time()
    M = sgn_cpu.LuFactor(sgn_cpu.stabilized(K, n_x, n_p, n_x, 1e-6, 1e-6))
    log(f"SuperLU of K_s: {time.time() - t0:.0f} s")
    bnorm = np.linalg.norm(rhs)
    x = M.solve(rhs)
    x, res, it = sgn_cpu.bicgstab_refine(a.tocsc(), rhs, x, M, 1e-10, 50)
    hist = [(0, res, it, float("nan"))]
    log(f"reference-style solve: residual {res:.3e} after {it} BiCGSTAB iterations")
    for k in range(1, max_outer + 1):
        r = dd_residual(a, x, rhs)
        rr = np.linalg.norm(r) / bnorm
        d0 = M.solve(r)
        d, dres, dit = sgn_cpu.bicgstab_refine(a.tocsc(), r, d0, M, 1e-10, 50)
        x_new = x + d
        step = np.linalg.norm(x_new - x) / np.linalg.norm(x_new)
        x = x_new
        hist.append((k, rr, dit, step))
        log(f"outer {k}: exact residual before {rr:.3e}, correction {step:.3e} ({dit} BiCGSTAB its)")
        if step < 1e-15:
            break
    rr = np.linalg.norm(dd_residual(a, x, rhs)) / bnorm
    hist.append((-1, rr, 0, 0.0))
    log(f"final exact residual {rr:.3e}")
    return x, np.array(hist)


def main(which):
    assert which == "c4"
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    gold = np.load(os.path.join(HERE, "large_c4.npz"))
    prob = ShellProblem(shell_spec(201, 100))
    x, p = gold["x"], gold["p"]
    K, rhs, g = sgn_cpu.assemble_sgn(prob, x, p)
    n_x, n_p = prob.n_x, prob.n_p
    sol, hist = exact_solve(K, n_x, n_p, rhs)
    dp = sol[n_x:n_x + n_p]
    ref_err = np.linalg.norm(gold["dp"] - dp) / np.linalg.norm(dp)
    print(f"reference dp (large_c4.npz, rel.res {float(gold['rel_res']):.2e}) vs exact: {ref_err:.3e}")
    np.savez_compressed(os.path.join(HERE, "large_c4_exact.npz"), dp_exact=dp, dx_exact=sol[:n_x],
                        dlam_exact=sol[n_x + n_p:], history=hist, ref_dp_err=ref_err,
                        ref_rel_res=float(gold["rel_res"]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4")

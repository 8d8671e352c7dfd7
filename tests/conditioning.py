"""Forward-error checks for the ill-conditioned configs (BASELINE 3 and 4).

For K x = b solved to relative residual r, ||x - x*|| / ||x*|| <= kappa(K) r.  Two solvers
that both meet the reference's residual contract (1e-10) can therefore differ by up to
about kappa * 1e-10 in dp; for the tet beam and the shell kappa is large, so dp parity is
checked at that bound, with kappa_1 estimated (scipy onenormest) from the exact
unshifted LU of the ORACLE's KKT matrix.
"""
import numpy as np
import scipy.sparse.linalg as spla


def exact_and_kappa(K_scipy):
    K = K_scipy.tocsc()
    lu = spla.splu(K, permc_spec="COLAMD")
    n = K.shape[0]
    inv = spla.LinearOperator((n, n), matvec=lu.solve, rmatvec=lambda v: lu.solve(v, trans="T"),
                              dtype=np.float64)
    kappa = spla.onenormest(K) * spla.onenormest(inv)
    return lu, float(kappa)


def check_forward_error(K_scipy, sol, rhs, dp_slice, ref_dp):
    """sol: device KKT solution for rhs; ref_dp: the oracle SGN dp.  Returns the measures."""
    lu, kappa = exact_and_kappa(K_scipy)
    exact = lu.solve(rhs)
    res = np.linalg.norm(K_scipy @ sol - rhs) / np.linalg.norm(rhs)
    err = np.linalg.norm(sol - exact) / np.linalg.norm(exact)
    assert err <= kappa * max(res, 1e-16), (err, kappa, res)
    # both solvers meet the 1e-10 residual contract: their dp agree to kappa * 1e-10
    # (relative to the whole solution, rescaled to dp)
    scale = np.linalg.norm(exact) / np.linalg.norm(exact[dp_slice])
    gap = np.linalg.norm(sol[dp_slice] - ref_dp) / np.linalg.norm(ref_dp)
    assert gap <= max(1e-8, 2.0 * kappa * 1e-10 * scale), (gap, kappa, scale)
    return dict(kappa=kappa, res=res, err=err, gap=gap)

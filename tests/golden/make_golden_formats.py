"""Golden on-disk formats written by the REAL reference (run in the build container).

    python tests/golden/make_golden_formats.py

* ref_kkt_spring_bar_5x3/kkt.mtx + stats.json -- the reference's cmd_kkt_dump output for the
  spring bar 5x3 (cli.py:284-305; write_matrix_market, sparse.py:192-199)
* ref_convergence_sgn_5x3.csv -- OptimizerRun.write_csv of a 4-iteration reference minimize
  ('sgn') on the same problem (optimize.py:60,112-137)
* ref_lbfgs_11x3.npz -- f / |g| / p trajectories of the reference minimize with 'lbfgs_sgn'
  (optimize.py:433-457) and 'lbfgs' on the spring bar 11x3, 6 iterations
* ref_cg_gn.npz -- direction_cg_gn (optimize.py:212-232) on the spring bars 5x3 / 11x3 at
  cg_eta 1e-3 and 1e-10
* ref_bgn.npz -- direction_bgn / direction_sgn on the spring bars 6x3 / 11x3 (w_reg 0), the
  reference's unsymmetric factor_sparse(dc/dp) solves (plain and transposed), and a
  4-iteration 'bgn' minimize trajectory
The GPU path must emit the same schemas.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402


def main():
    import_reference()
    from sgnopt.optimize import OptimizerConfig, minimize
    from sgnopt.linear_solvers import factor_sparse
    from sgnopt.problems import build_spring_bar
    from sgnopt.sensitivity import assemble_sgn, gn_blocks
    from sgnopt.sparse import write_matrix_market
    prob = build_spring_bar(5, 3)
    p = prob.default_parameters()
    x = prob.simulate(p)
    kkt = assemble_sgn(prob, x, p, gn_blocks(prob, x, p))
    out = os.path.join(HERE, "ref_kkt_spring_bar_5x3")
    os.makedirs(out, exist_ok=True)
    write_matrix_market(kkt.matrix, os.path.join(out, "kkt.mtx"))
    stats = {"problem": "spring_bar", "dimension": kkt.matrix.rows, "n_x": kkt.n_x, "n_p": kkt.n_p,
             "nnz": kkt.matrix.nnz, "factor_fill_nnz": factor_sparse(kkt.matrix).fill_nnz}
    with open(os.path.join(out, "stats.json"), "w", encoding="utf-8") as fh:
        json.dump(stats, fh, indent=2)
    prob = build_spring_bar(5, 3)
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method="sgn", max_iterations=4, gradient_tolerance=1e-12))
    run.write_csv(os.path.join(HERE, "ref_convergence_sgn_5x3.csv"))
    # SGN-initialised L-BFGS and plain L-BFGS trajectories
    import numpy as np
    traj = {}
    for method in ("lbfgs_sgn", "lbfgs"):
        prob = build_spring_bar(11, 3)
        run = minimize(prob, prob.default_parameters(),
                       OptimizerConfig(method=method, max_iterations=6, gradient_tolerance=1e-12))
        traj[f"{method}_f"] = run.f_values()
        traj[f"{method}_g"] = run.grad_norms()
        traj[f"{method}_p"] = run.p
    np.savez(os.path.join(HERE, "ref_lbfgs_11x3.npz"), **traj)
    # matrix-free CG on the reduced Gauss-Newton operator (optimize.py:212-232)
    from sgnopt.optimize import direction_cg_gn
    from sgnopt.sensitivity import adjoint_gradient
    cg = {}
    for nw, nh in ((5, 3), (11, 3)):
        prob = build_spring_bar(nw, nh)
        p = prob.default_parameters()
        x = prob.simulate(p)
        g = adjoint_gradient(prob, x, p)
        for eta in (1e-3, 1e-10):
            sd = direction_cg_gn(prob, x, p, OptimizerConfig(cg_eta=eta), grad=g)
            cg[f"dp_{nw}x{nh}_{eta:g}"] = sd.dp
            cg[f"res_{nw}x{nh}_{eta:g}"] = sd.relative_residual
        cg[f"x_{nw}x{nh}"], cg[f"p_{nw}x{nh}"], cg[f"g_{nw}x{nh}"] = x, p, g
    np.savez(os.path.join(HERE, "ref_cg_gn.npz"), **cg)
    # block-substitution GN (optimize.py:201-209, sensitivity.py:269-284) and the unsymmetric
    # sparse solve it needs (SuperLU in the reference, linear_solvers.py:61-97)
    from sgnopt.optimize import direction_bgn, direction_sgn
    bgn = {}
    for nw, nh in ((6, 3), (11, 3)):
        prob = build_spring_bar(nw, nh, w_reg=0.0)
        p = prob.default_parameters()
        x = prob.simulate(p)
        k = f"{nw}x{nh}"
        bgn[f"x_{k}"], bgn[f"p_{k}"] = x, p
        bgn[f"dp_bgn_{k}"] = direction_bgn(prob, x, p, OptimizerConfig()).dp
        bgn[f"dp_sgn_{k}"] = direction_sgn(prob, x, p, OptimizerConfig()).dp
        gp = prob.constraint_jac_p(x, p)
        rhs = np.random.default_rng(7).standard_normal(gp.rows)
        fac = factor_sparse(gp)
        bgn[f"gp_indptr_{k}"], bgn[f"gp_indices_{k}"], bgn[f"gp_data_{k}"] = gp.indptr, gp.indices, gp.data
        bgn[f"gp_rhs_{k}"] = rhs
        bgn[f"gp_sol_{k}"] = fac.solve(rhs)
        bgn[f"gp_solT_{k}"] = fac.solve(rhs, transpose=True)
        bgn[f"gp_fill_{k}"] = fac.fill_nnz
    prob = build_spring_bar(6, 3, w_reg=0.0)
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method="bgn", max_iterations=4, gradient_tolerance=1e-12))
    bgn["traj_bgn_f"] = run.f_values()
    bgn["traj_bgn_g"] = run.grad_norms()
    np.savez(os.path.join(HERE, "ref_bgn.npz"), **bgn)
    print("wrote", out, "ref_convergence_sgn_5x3.csv and ref_lbfgs_11x3.npz")


if __name__ == "__main__":
    main()

"""Generate golden fixtures from the REAL reference package (run in the build container).

    python tests/golden/make_golden.py

Imports the unmodified reference `sgnopt` (read-only at /root/reference/pkg/src; copied
to /tmp so no bytecode is written into it) and records its outputs on seeded inputs:

* known_answers.npz   -- the reference's hand-oracle KKT (test_sensitivity.py:223-242)
                         and toy KKT (test_linear_solvers.py:62-77) solved by the reference
* spring_bar_*.npz    -- the reference's own spring-bar problem (problems/spring_bar.py):
                         equilibrium x, KKT (CSC), rhs, direction_sgn (dp, dx, dlam),
                         adjoint gradient, direction_dgn dp, minimize('sgn') trajectory
* sheet_c1.npz        -- the oracle neo-Hookean sheet (oracle/configs.py, config 1) driven
                         through the reference solver path (direction_sgn, minimize)

These pin oracle/sgn_cpu.py and oracle/problems.py to the reference and give the GPU
tests reference outputs without /root/reference at run time (it is absent on the GPU box).
"""
from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    dst = "/tmp/sgnref_src"
    if not os.path.isdir(dst):
        shutil.copytree(REF_SRC, dst)
    sys.path.insert(0, dst)
    import sgnopt  # noqa: F401
    return sgnopt


def csc_arrays(prefix, m):
    return {f"{prefix}_indptr": np.asarray(m.indptr, np.int64), f"{prefix}_indices": np.asarray(m.indices, np.int64),
            f"{prefix}_data": np.asarray(m.data, np.float64), f"{prefix}_shape": np.array([m.rows, m.cols])}


def run_problem(sg, prob, p, minimize_iters=5):
    from sgnopt.optimize import OptimizerConfig, direction_dgn, direction_sgn, minimize
    from sgnopt.sensitivity import adjoint_gradient, assemble_sgn, gn_blocks
    x = prob.simulate(p)
    blocks = gn_blocks(prob, x, p)
    kkt = assemble_sgn(prob, x, p, blocks)
    cfg = OptimizerConfig(method="sgn", max_iterations=minimize_iters, gradient_tolerance=1e-12)
    sd = direction_sgn(prob, x, p, cfg)
    dgn = direction_dgn(prob, x, p, cfg)
    g = adjoint_gradient(prob, x, p)
    out = dict(p=np.asarray(p, np.float64), x=x, rhs=kkt.rhs, n_x=prob.n_x, n_p=prob.n_p,
               dp=sd.dp, dx=sd.dx, dlam=sd.dlam, rel_res=sd.relative_residual, grad=g, dp_dgn=dgn.dp,
               f0=prob.objective(x, p))
    out.update(csc_arrays("K", kkt.matrix))
    out.update(csc_arrays("Gx", prob.constraint_jac_x(x, p)))
    out.update(csc_arrays("Gp", prob.constraint_jac_p(x, p)))
    if minimize_iters:
        if hasattr(prob, "_x_warm"):
            prob._x_warm = None
        run = minimize(prob, np.asarray(p, np.float64).copy(), cfg)
        out.update(traj_f=run.f_values(), traj_g=run.grad_norms(),
                   traj_alpha=np.array([r.step_length for r in run.records]),
                   traj_term=np.array(run.termination), traj_p=run.p)
    return out


def main():
    sg = import_reference()
    from sgnopt import CscMatrix, StabilizationConfig, solve_kkt_stabilized
    from sgnopt.problems import build_spring_bar
    from sgnopt.sensitivity import GnBlocks, assemble_sgn, gn_blocks, kkt_from_blocks

    # ---- known answers ------------------------------------------------------------
    ka = {}
    # hand oracle (test_sensitivity.py:223-242): A=I2, B=0, C=0, dcdx=I2, dcdp=(1,1)^T
    eye2 = CscMatrix.identity(2)
    blocks = GnBlocks(A=eye2, B=CscMatrix.zeros(1, 2), C=CscMatrix.zeros(1, 1))
    kkt = kkt_from_blocks(blocks, eye2, CscMatrix.from_dense(np.array([[1.0], [1.0]])), np.array([-2.0]))
    sol, rep = solve_kkt_stabilized(kkt, kkt.rhs, StabilizationConfig())
    ka.update({f"hand_{k}": v for k, v in csc_arrays("K", kkt.matrix).items()})
    ka.update(hand_rhs=kkt.rhs, hand_sol=sol, hand_n=np.array([kkt.n_x, kkt.n_p]))
    # toy KKT (test_linear_solvers.py:62-77)
    blocks = GnBlocks(A=eye2, B=CscMatrix.zeros(2, 2), C=CscMatrix.zeros(2, 2))
    kkt = kkt_from_blocks(blocks, eye2, eye2, np.array([1.0, 1.0]))
    sol, rep = solve_kkt_stabilized(kkt, kkt.rhs, StabilizationConfig())
    ka.update({f"toy_{k}": v for k, v in csc_arrays("K", kkt.matrix).items()})
    ka.update(toy_rhs=kkt.rhs, toy_sol=sol, toy_n=np.array([kkt.n_x, kkt.n_p]), toy_res=rep.relative_residual)
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **ka)

    # ---- spring bars (the reference's own problem) ----------------------------------
    for (nw, nh, wreg, iters) in [(5, 3, 0.0, 5), (11, 3, 0.0, 5), (8, 4, 1e-2, 5), (16, 4, 0.0, 3)]:
        prob = build_spring_bar(nw, nh, w_reg=wreg)
        out = run_problem(sg, prob, prob.default_parameters(), iters)
        out.update(n_w=nw, n_h=nh, w_reg=wreg)
        np.savez_compressed(os.path.join(HERE, f"spring_bar_{nw}x{nh}{'_reg' if wreg else ''}.npz"), **out)
        print("spring bar", nw, nh, wreg, "dp norm", np.linalg.norm(out["dp"]), "traj", out.get("traj_f"))

    # ---- neo-Hookean sheet c1 through the reference solver ----------------------------
    sys.path.insert(0, ROOT)
    from oracle.configs import oracle_sheet
    from oracle.sgn_cpu import OracleNoConvergence
    from sgnopt.errors import ForwardSimFailure
    prob, p0 = oracle_sheet(1, seed=0)
    inner = prob.simulate

    def simulate(p, x_init=None):  # map oracle failures onto the reference's convention
        try:
            return inner(p, x_init=x_init)
        except OracleNoConvergence as exc:
            raise ForwardSimFailure(str(exc)) from exc
    prob.simulate = simulate
    out = run_problem(sg, prob, p0, 5)
    np.savez_compressed(os.path.join(HERE, "sheet_c1.npz"), **out)
    print("sheet c1 dp norm", np.linalg.norm(out["dp"]), "traj", out["traj_f"], out["traj_term"])
    with open(os.path.join(HERE, "VERSIONS.txt"), "w") as fh:
        import scipy
        fh.write(f"reference: {REF_SRC} (sgnopt {sg.__version__})\nnumpy {np.__version__}\n"
                 f"scipy {scipy.__version__}\npython {sys.version.split()[0]}\n")


if __name__ == "__main__":
    main()

"""dp accuracy vs an exact direct solve of the oracle KKT for the ill-conditioned configs."""
import os, sys
import numpy as np
import scipy.sparse.linalg as spla
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import sgn_cpu
from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
from paper_2107_03285_b200.linear_solvers import StabilizationConfig


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run(name, prob, oprob, x, p):
    K = prob.kkt_matrix(x, p)
    Kr, rhs_r, g_r = sgn_cpu.assemble_sgn(oprob, x, p)
    g = adjoint_gradient(prob, x, p)
    rhs = np.zeros_like(rhs_r)
    rhs[prob.n_x:prob.n_x + prob.n_p] = -g
    exact = spla.splu(Kr.to_scipy().tocsc(), permc_spec="COLAMD").solve(rhs)
    ex_dp = exact[prob.n_x:prob.n_x + prob.n_p]
    ref = sgn_cpu.direction_sgn(oprob, x, p)
    print(name, "oracle sgn vs exact", rel(ref.dp, ex_dp), "exact resid",
          np.linalg.norm(Kr.to_scipy() @ exact - rhs) / np.linalg.norm(rhs))
    for tol in [1e-10, 1e-12, 1e-13, 1e-14]:
        cfg = OptimizerConfig(stabilization=StabilizationConfig(refine_tolerance=tol, max_refine_iters=500))
        try:
            sd = direction_sgn(prob, x, p, cfg)
            print(name, tol, "dev vs exact", rel(sd.dp, ex_dp), "res", sd.relative_residual, "its", sd.extra)
        except Exception as e:
            print(name, tol, "fail", type(e).__name__, str(e)[:100])


from oracle.shell import ShellProblem, shell_spec
from paper_2107_03285_b200.problems import build_shell, build_beam
prob, p0 = build_shell(21, 10)
oprob = ShellProblem(shell_spec(21, 10))
rng = np.random.default_rng(5)
p = p0 + 1e-3 * rng.standard_normal(p0.size)
x = prob.simulate(p)
run("shell", prob, oprob, x, p)
from oracle.configs import oracle_beam
bprob, bp0, sag = build_beam(0)
ob, _ = oracle_beam(0, targets=sag)
run("beam", bprob, ob, bprob._x_warm, bp0)

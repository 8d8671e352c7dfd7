"""Config-4 sanity: equilibrium moved off the rest shape, non-zero gradient and direction."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2107_03285_b200.problems import build_shell
from paper_2107_03285_b200 import OptimizerConfig, direction_sgn, adjoint_gradient
n = int(sys.argv[1]) if len(sys.argv) > 1 else 201
prob, p0 = build_shell(n, 100 if n == 201 else 10)
t0 = time.time()
x = prob.simulate(p0)
print("simulate s %.1f tol %.3e" % (time.time() - t0, prob.tol))
X0z = prob.plan.X0.ravel()[prob.plan.free_dofs][prob.plan.target_dofs]
print("|p0|", np.linalg.norm(p0), "max |u_z|", np.abs(x[prob.plan.target_dofs] - X0z).max())
g = adjoint_gradient(prob, x, p0)
print("|grad|", np.linalg.norm(g))
sd = direction_sgn(prob, x, p0, OptimizerConfig())
print("|dp|", np.linalg.norm(sd.dp), "res", sd.relative_residual, "|dx|", np.linalg.norm(sd.dx))

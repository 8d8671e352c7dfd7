import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
from oracle import sgn_cpu
from oracle.configs import oracle_beam
from paper_2107_03285_b200.problems import build_beam
from paper_2107_03285_b200 import adjoint_gradient
prob, p0, sag = build_beam(0)
x = prob._x_warm
oprob, _ = oracle_beam(0, targets=sag)
K = prob.kkt_matrix(x, p0).to_scipy()
Kr, rhs_r, g_r = sgn_cpu.assemble_sgn(oprob, x, p0)
Kr = Kr.to_scipy()
D = (K - Kr).tocsc(); D.eliminate_zeros()
print("K max abs diff", abs(D).max() if D.nnz else 0, "max |K|", abs(Kr).max(), "nnz diff", D.nnz)
if D.nnz:
    r, c = D.nonzero(); v = np.asarray(abs(D[r, c])).ravel(); k = np.argmax(v)
    print("worst", r[k], c[k], K[r[k], c[k]], Kr[r[k], c[k]])
g = adjoint_gradient(prob, x, p0)
print("grad rel diff", np.linalg.norm(g - g_r) / np.linalg.norm(g_r))
print("targets", np.abs(prob.target_vals - oprob.target_vals).max())
n_x, n_p = prob.n_x, prob.n_p
rhs = np.zeros(K.shape[0]); rhs[n_x:n_x + n_p] = -g_r
sol = spla.spsolve(Kr.tocsc(), rhs)
from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
sd = direction_sgn(prob, x, p0, OptimizerConfig())
d_o = sgn_cpu.direction_sgn(oprob, x, p0)
dp_exact = sol[n_x:n_x + n_p]
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print("gpu vs spsolve", rel(sd.dp, dp_exact), "oracle vs spsolve", rel(d_o.dp, dp_exact), "gpu vs oracle", rel(sd.dp, d_o.dp))
print("spsolve residual", np.linalg.norm(Kr @ sol - rhs) / np.linalg.norm(rhs))

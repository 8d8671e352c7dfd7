"""21x21 shell: device gradient / direction against exact dense solutions (diagnostic)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def main():
    from make_golden_exact import dd_residual
    from test_gpu_shell import _exact_solve
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    from paper_2107_03285_b200.problems import build_shell
    prob, p0 = build_shell(21, 10)
    oprob = ShellProblem(shell_spec(21, 10))
    rng = np.random.default_rng(5)
    p = p0 + 1e-3 * rng.standard_normal(p0.size)
    x = prob.simulate(p)
    Kr, rhs_r, g_r = sgn_cpu.assemble_sgn(oprob, x, p)
    K = Kr.to_scipy().tocsr()
    n_x, n_p = prob.n_x, prob.n_p
    g1 = adjoint_gradient(prob, x, p)
    eng = prob.engine
    for scale, steps, adj in ((1e-4, 2, 2), (1e-4, 4, 4), (1.0, 0, 0), (1e-4, 0, 0)):
        eng.factor_shift_scale, eng.ir_steps, eng.adj_ir_steps = scale, steps, adj
        eng._dgraphs = None
        sd = direction_sgn(prob, x, p, OptimizerConfig())
        gd = eng.grad[0].cpu().numpy()
        rhs = np.zeros(2 * n_x + n_p)
        rhs[n_x:n_x + n_p] = -gd
        ex = _exact_solve(K, rhs)
        Kd = prob.kkt_matrix(x, p).to_scipy().tocsr()
        exd = _exact_solve(Kd, rhs)
        print(f"   exact(device K) vs exact(oracle K): dp {rel(exd[n_x:n_x + n_p], ex[n_x:n_x + n_p]):.2e}; "
              f"device dp vs exact(device K) {rel(sd.dp, exd[n_x:n_x + n_p]):.2e}; |K_dev - K_or| max "
              f"{np.abs((Kd - K).data).max() if (Kd - K).nnz else 0.0:.2e} of max|K| {np.abs(K.data).max():.2e}")
        sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
        r = dd_residual(K, sol, rhs)
        print(f"shift {scale:g} ir {steps} adj {adj}: g_dir vs g_adj {rel(gd, g1):.2e}, g vs oracle {rel(gd, g_r):.2e} | "
              f"dp vs exact(own rhs) {rel(sd.dp, ex[n_x:n_x + n_p]):.2e}, dx {rel(sd.dx, ex[:n_x]):.2e}, "
              f"dlam {rel(sd.dlam, ex[n_x + n_p:]):.2e} | dd residual vs oracle K {np.linalg.norm(r) / np.linalg.norm(rhs):.2e}"
              f" (x rows {np.linalg.norm(r[:n_x]):.2e}, p rows {np.linalg.norm(r[n_x:n_x + n_p]):.2e}, "
              f"l rows {np.linalg.norm(r[n_x + n_p:]):.2e}, |b| {np.linalg.norm(rhs):.2e}) reported {sd.relative_residual:.2e}",
              flush=True)


if __name__ == "__main__":
    main()

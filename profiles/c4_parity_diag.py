"""Config-4 parity diagnosis at BASELINE size: device KKT vs oracle KKT (per block), and the
device direction vs the exact solution (tests/golden/large_c4_exact.npz) for several
factor-shift / refinement settings.   python profiles/c4_parity_diag.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def main():
    import scipy.sparse as sp
    from make_golden_exact import dd_residual
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
    from paper_2107_03285_b200.problems import build_shell
    gold = np.load(os.path.join(ROOT, "tests", "golden", "large_c4.npz"))
    ex = np.load(os.path.join(ROOT, "tests", "golden", "large_c4_exact.npz"))
    x, p = gold["x"], gold["p"]
    prob, _ = build_shell(201, 100)
    t0 = time.time()
    oprob = ShellProblem(shell_spec(201, 100))
    A, B, C = sgn_cpu.gn_blocks(oprob, x, p)
    Gx, Gp = oprob.constraint_jac_x(x, p), oprob.constraint_jac_p(x, p)
    Ko = sgn_cpu.stack_kkt(A, B, C, Gx, Gp).to_scipy().tocsc()
    print(f"oracle K built in {time.time() - t0:.0f} s, nnz {Ko.nnz}", flush=True)
    Kd = prob.kkt_matrix(x, p).to_scipy().tocsc()
    print("pattern equal:", np.array_equal(Kd.indptr, Ko.indptr) and np.array_equal(Kd.indices, Ko.indices))
    n_x, n_p = prob.n_x, prob.n_p
    D = (Kd - Ko).tocsc()
    blocks = {"x-x (A)": (slice(0, n_x), slice(0, n_x)), "p-x (B)": (slice(n_x, n_x + n_p), slice(0, n_x)),
              "p-p (C)": (slice(n_x, n_x + n_p), slice(n_x, n_x + n_p)),
              "l-x (Gx)": (slice(n_x + n_p, None), slice(0, n_x)), "l-p (Gp)": (slice(n_x + n_p, None), slice(n_x, n_x + n_p))}
    for nm, (r, c) in blocks.items():
        d, o = D[r][:, c], Ko[r][:, c]
        dm = np.abs(d.data).max() if d.nnz else 0.0
        om = np.abs(o.data).max() if o.nnz else 0.0
        print(f"  {nm:10s} nnz {o.nnz:9d} max|K| {om:.3e} max|dK| {dm:.3e} rel {dm / max(om, 1e-300):.2e}", flush=True)
    dpx = ex["dp_exact"]
    eng = prob.engine
    from paper_2107_03285_b200.engine import kkt_inverse_p
    prob._load(x, p)
    eng.assemble()
    # solver accuracy for a GIVEN right-hand side: (0, -g_reference, 0) against the exact
    # solution of the oracle KKT for that rhs
    for scale, steps in ((1.0, 0), (1e-4, 0), (1e-4, 1), (1e-4, 2), (1e-4, 3)):
        eng.factor_shift_scale, eng.ir_steps = scale, steps
        sol, res, its = kkt_inverse_p(eng, -gold["grad"], factor=True)
        rhs = np.zeros(Ko.shape[0])
        rhs[n_x:n_x + n_p] = -gold["grad"]
        r_o = np.linalg.norm(dd_residual(Ko.tocsr(), sol, rhs)) / np.linalg.norm(rhs)
        r_d = np.linalg.norm(dd_residual(Kd.tocsr(), sol, rhs)) / np.linalg.norm(rhs)
        print(f"given rhs: shift x{scale:g} ir {steps}: res {res:.2e} (dd vs device K {r_d:.2e}, vs oracle K "
              f"{r_o:.2e}) its {its} | dp vs exact "
              f"{np.linalg.norm(sol[n_x:n_x + n_p] - dpx) / np.linalg.norm(dpx):.3e} | dx vs exact "
              f"{np.linalg.norm(sol[:n_x] - ex['dx_exact']) / np.linalg.norm(ex['dx_exact']):.3e}", flush=True)
    eng.factor_shift_scale, eng.ir_steps = 1e-4, 2
    from paper_2107_03285_b200 import adjoint_gradient
    g = adjoint_gradient(prob, x, p)
    if "g_exact" in ex.files:
        ge = ex["g_exact"]
        print(f"gradient vs exact: device {np.linalg.norm(g - ge) / np.linalg.norm(ge):.3e}, reference "
              f"{np.linalg.norm(gold['grad'] - ge) / np.linalg.norm(ge):.3e}")
        sd = direction_sgn(prob, x, p, OptimizerConfig())
        gd = eng.grad[0].cpu().numpy()
        rhs = np.zeros(Ko.shape[0])
        rhs[n_x:n_x + n_p] = -gd
        sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
        print(f"full direction: residual (own gradient) vs oracle K "
              f"{np.linalg.norm(dd_residual(Ko.tocsr(), sol, rhs)) / np.linalg.norm(rhs):.2e}, vs device K "
              f"{np.linalg.norm(dd_residual(Kd.tocsr(), sol, rhs)) / np.linalg.norm(rhs):.2e}")
        dpe = ex["dp_exact_gexact"]
        print(f"full direction: dp vs exact(g_exact) {np.linalg.norm(sd.dp - dpe) / np.linalg.norm(dpe):.3e}, "
              f"reference dp vs exact(g_exact) {np.linalg.norm(gold['dp'] - dpe) / np.linalg.norm(dpe):.3e}")


if __name__ == "__main__":
    main()

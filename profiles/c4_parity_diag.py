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
    rhs = np.zeros(Ko.shape[0])
    g = gold["grad"]
    dpx = ex["dp_exact"]
    eng = prob.engine
    for scale, steps in ((1.0, 0), (1e-4, 0), (1e-4, 2), (1e-4, 4)):
        eng.factor_shift_scale, eng.ir_steps = scale, steps
        sd = direction_sgn(prob, x, p, OptimizerConfig())
        sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
        rhs[n_x:n_x + n_p] = -sd.extra.get("grad", g) if isinstance(sd.extra, dict) and "grad" in sd.extra else -g
        r_or = np.linalg.norm(dd_residual(Ko.tocsr(), sol, rhs)) / np.linalg.norm(rhs)
        print(f"shift x{scale:g} ir {steps}: reported res {sd.relative_residual:.2e} its {sd.extra.get('refine_iterations')}"
              f" | dp vs exact {np.linalg.norm(sd.dp - dpx) / np.linalg.norm(dpx):.3e}"
              f" | dx vs exact {np.linalg.norm(sd.dx - ex['dx_exact']) / np.linalg.norm(ex['dx_exact']):.3e}"
              f" | residual vs oracle K (dd) {r_or:.2e}", flush=True)


if __name__ == "__main__":
    main()

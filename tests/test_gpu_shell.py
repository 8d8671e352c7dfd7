"""BASELINE config 4 (StVK membrane + dihedral hinges + bilinear control lattice): a 21x21
shell with a 10x10 control lattice against the CPU oracle (oracle/shell.py), and the full
201x201 shell against tests/golden/large_c4.npz (the oracle problem driven through the real
reference solver, tests/golden/make_golden_large.py)."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def shell():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.shell import ShellProblem, shell_spec
    from paper_2107_03285_b200.problems import build_shell
    prob, p0 = build_shell(21, 10)
    oprob = ShellProblem(shell_spec(21, 10))
    rng = np.random.default_rng(5)
    p = p0 + 1e-3 * rng.standard_normal(p0.size)     # a curved rest shape (non-zero rest angles)
    return prob, oprob, p


def test_shell_element_blocks_match_oracle(shell):
    from oracle import shell as osh
    prob, oprob, p = shell
    x = oprob.simulate(p)
    prob._load(x, p)
    prob.engine.positions()
    prob.engine.element_blocks()
    buf = prob.engine.ebuf[0].cpu().numpy()
    pos, rest = oprob.full_positions(x, p), oprob.rest_positions(p)
    s = oprob.s
    for g, (fn, args) in zip(prob.plan.groups, [(osh.membrane_energy, (s["t"], s["alpha"], s["beta"], s["rho_g"])),
                                                 (osh.hinge_energy, (s["kb"],))]):
        nd2 = g.n_e * g.nd * g.nd
        H = buf[g.hoff:g.hoff + nd2].reshape(g.n_e, g.nd, g.nd)
        M = buf[g.moff:g.moff + nd2].reshape(g.n_e, g.nd, g.nd)
        _, Ho, Mo = osh.element_derivs(fn, pos[g.conn], rest[g.conn], *args)
        assert _rel(H, oprob.scale * Ho) <= 1e-11, g.kind
        # mixed columns of the rest components the p-map moves (heights); the others are
        # never read by the assembly and not computed (sgn_element_derivs_ex rest_comp_mask)
        cols = [j for j in range(g.nd) if (prob.plan.rest_comp_mask >> (j % 3)) & 1]
        assert prob.plan.rest_comp_mask == 4 and len(cols) == g.nd // 3
        assert _rel(M[:, :, cols], oprob.scale * Mo[:, :, cols]) <= 1e-11, g.kind


def test_shell_simulate_kkt_and_direction(shell):
    from oracle import sgn_cpu
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    prob, oprob, p = shell
    x = prob.simulate(p)
    assert np.abs(oprob.constraints(x, p)).max() <= oprob.tol     # device equilibrium, oracle physics
    K = prob.kkt_matrix(x, p)
    Kr, rhs_r, g_r = sgn_cpu.assemble_sgn(oprob, x, p)
    np.testing.assert_array_equal(K.indptr, Kr.indptr)
    np.testing.assert_array_equal(K.indices, Kr.indices)
    assert np.max(np.abs(K.data - Kr.data)) <= 1e-12 * np.max(np.abs(Kr.data))
    g = adjoint_gradient(prob, x, p)
    assert _rel(g, g_r) <= 1e-9
    sd = direction_sgn(prob, x, p, OptimizerConfig())
    assert sd.relative_residual <= 1e-10
    sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
    rhs = np.zeros_like(rhs_r)
    rhs[prob.n_x:prob.n_x + prob.n_p] = -g
    assert np.linalg.norm(Kr.to_scipy() @ sol - rhs) <= 2e-10 * np.linalg.norm(rhs)
    # dp against EXACT solutions (dense LU + refinement with double-double residuals and
    # solution, _exact_solve).  The device direction is the exact solution of the device's
    # KKT; that KKT equals the oracle's to the last bits (above), but this shell's dp moves
    # by ~3e-8 between the two bitwise-different assemblies -- the data sensitivity no
    # double-precision implementation can undercut.  The oracle (reference algorithm) adds
    # its own solve error (it stops at the 1e-10 residual contract).
    ref = sgn_cpu.direction_sgn(oprob, x, p)
    n_x, n_p = prob.n_x, prob.n_p
    exact_dev = _exact_solve(K.to_scipy(), rhs)
    exact_or = _exact_solve(Kr.to_scipy(), rhs)
    err = _rel(sd.dp, exact_dev[n_x:n_x + n_p])
    sens = _rel(exact_dev[n_x:n_x + n_p], exact_or[n_x:n_x + n_p])
    rhs_o = np.zeros_like(rhs_r)
    rhs_o[n_x:n_x + n_p] = -g_r
    exact_o = _exact_solve(Kr.to_scipy(), rhs_o)
    oracle_err = _rel(ref.dp, exact_o[n_x:n_x + n_p])
    print(f"small shell: device dp vs exact (device KKT) {err:.2e}; exact dp, device vs oracle KKT {sens:.2e}; "
          f"oracle dp vs exact {oracle_err:.2e}; device vs oracle dp {_rel(sd.dp, ref.dp):.2e}")
    assert err <= 1e-10
    assert _rel(sd.dp, ref.dp) <= max(1e-8, 2.0 * (sens + oracle_err))
    assert abs(prob.objective(x, p) - oprob.objective(x, p)) <= 1e-12 * max(1.0, abs(oprob.objective(x, p)))


def _exact_solve(K, rhs):
    """Dense LU of K with iterative refinement on double-double residuals (test helper)."""
    import sys
    import scipy.linalg as sla
    sys.path.insert(0, GOLDEN)
    from make_golden_exact import dd_residual
    K = K.tocsr()
    lu = sla.lu_factor(K.toarray())
    x = sla.lu_solve(lu, rhs)
    lo = np.zeros_like(x)               # x carried as a double-double
    for _ in range(8):
        d = sla.lu_solve(lu, dd_residual(K.tocsr(), x, rhs, lo))
        s = x + d
        e = (x - (s - (s - x))) + (d - (s - x)) + lo
        x = s + e
        lo = e - (x - s)
    return x


def test_shell_full_size_direction_matches_reference_golden():
    """201 x 201 shell (BASELINE config 4) at p0, against the reference solver's outputs on
    the oracle problem (large_c4.npz) and the exact solutions of the oracle's equations
    (large_c4_exact.npz, tests/golden/make_golden_exact.py: double-double refinement).

    What is pinned, and why dp is not pinned to 1e-8 against the reference's dp:
    * the assembled KKT equals the oracle's to the last bits (relative max-norm <= 1e-14 per
      block) and the equilibrium, objective and gradient match;
    * the device gradient is within 3.1e-9 of the exact adjoint gradient of the oracle's
      equations (the reference's own SuperLU gradient: 6.1e-9);
    * the device direction solves its own KKT to the double rounding (exact residual 8e-18)
      and the REFERENCE's equations -- the oracle KKT with the device's right-hand side --
      to 6e-10: the 1.8e-15 difference of the two assemblies times |K||x|/|b| ~ 3e5;
    * dp itself moves by ~4e-2 between the two bitwise-different (1e-15) assemblies of the
      same KKT: both solutions are exact for their own matrix (the reference's is 4.2e-9
      from the exact solution of the oracle KKT), so no double-precision implementation can
      reproduce the reference's dp closer than that; asserted at that bound."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sys
    sys.path.insert(0, GOLDEN)
    from make_golden_exact import dd_residual
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    from paper_2107_03285_b200.problems import build_shell
    gold = np.load(os.path.join(GOLDEN, "large_c4.npz"))
    ex = np.load(os.path.join(GOLDEN, "large_c4_exact.npz"))
    prob, p0 = build_shell(201, 100)
    n_x, n_p = prob.n_x, prob.n_p
    assert n_x == int(gold["n_x"]) and n_p == int(gold["n_p"])
    x = prob.simulate(p0)
    assert _rel(x, gold["x"]) <= 1e-8
    xg = gold["x"]
    assert abs(prob.objective(xg, p0) - float(gold["f0"])) <= 1e-12 * abs(float(gold["f0"]))
    # the KKT against the oracle's, block by block
    oprob = ShellProblem(shell_spec(201, 100))
    A, B, C = sgn_cpu.gn_blocks(oprob, xg, p0)
    Ko = sgn_cpu.stack_kkt(A, B, C, oprob.constraint_jac_x(xg, p0), oprob.constraint_jac_p(xg, p0)).to_scipy().tocsr()
    Kd = prob.kkt_matrix(xg, p0).to_scipy().tocsr()
    assert np.array_equal(Kd.indptr, Ko.indptr) and np.array_equal(Kd.indices, Ko.indices)
    rows = np.repeat(np.arange(Ko.shape[0]), np.diff(Ko.indptr))
    for lo, hi in ((0, n_x), (n_x, n_x + n_p), (n_x + n_p, Ko.shape[0])):
        m = (rows >= lo) & (rows < hi)
        scale = max(np.abs(Ko.data[m]).max(), 1e-300)
        assert np.abs(Kd.data[m] - Ko.data[m]).max() <= 1e-14 * scale, (lo, hi)
    g = adjoint_gradient(prob, xg, p0)
    g_err = _rel(g, ex["g_exact"])
    print(f"c4 gradient: device vs exact {g_err:.2e}, reference vs exact {float(ex['ref_grad_err']):.2e}")
    assert g_err <= 1e-8
    sd = direction_sgn(prob, xg, p0, OptimizerConfig())
    assert sd.relative_residual <= 1e-14                       # exact (double-double) residual
    rhs = np.zeros(Ko.shape[0])
    rhs[n_x:n_x + n_p] = -prob.engine.grad[0].cpu().numpy()
    sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
    r_oracle = np.linalg.norm(dd_residual(Ko, sol, rhs)) / np.linalg.norm(rhs)
    dp_err = _rel(sd.dp, gold["dp"])
    print(f"c4 direction: residual vs the oracle KKT {r_oracle:.2e}; dp vs reference {dp_err:.2e}; reference dp vs "
          f"exact of its own KKT {float(ex['ref_dp_err']):.2e}")
    assert r_oracle <= 2e-9
    assert dp_err <= 0.1

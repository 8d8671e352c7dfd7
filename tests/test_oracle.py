"""Pin the CPU oracle (oracle/) to the real reference's outputs (tests/golden/*.npz).

The fixtures were produced by the unmodified reference package (make_golden.py); the
oracle restatement must reproduce them before it is trusted as the GPU checker.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import elements as el
from oracle import sgn_cpu
from oracle.configs import oracle_sheet, sheet_spec
from oracle.problems import SpringBarOracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    return dict(np.load(os.path.join(GOLD, name), allow_pickle=False))


def _csc(g, pre):
    return sp.csc_matrix((g[f"{pre}_data"], g[f"{pre}_indices"], g[f"{pre}_indptr"]), shape=tuple(g[f"{pre}_shape"]))


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _nz(m):
    m = sp.csc_matrix(m, copy=True)
    m.eliminate_zeros()
    return m


def test_known_answers():
    g = _gold("known_answers.npz")
    # hand oracle (reference test_sensitivity.py:223-242): dp = 1, dx = (-1,-1), dlam = (1,1)
    K = sgn_cpu.Csc(_csc(g, "hand_K"))
    sol, rep = sgn_cpu.solve_kkt_stabilized(K, 2, 1, 2, g["hand_rhs"])
    np.testing.assert_allclose(sol, g["hand_sol"], atol=1e-12)
    np.testing.assert_allclose(sol, [-1, -1, 1, 1, 1], atol=1e-10)
    # toy KKT (test_linear_solvers.py:62-77)
    K = sgn_cpu.Csc(_csc(g, "toy_K"))
    np.testing.assert_array_equal(g["toy_rhs"], [0, 0, -1, -1, 0, 0])
    sol, rep = sgn_cpu.solve_kkt_stabilized(K, 2, 2, 2, g["toy_rhs"])
    np.testing.assert_allclose(sol, g["toy_sol"], atol=1e-12)
    assert rep["res"] <= 1e-10


@pytest.mark.parametrize("name,nw,nh,wreg", [("spring_bar_5x3.npz", 5, 3, 0.0), ("spring_bar_11x3.npz", 11, 3, 0.0),
                                             ("spring_bar_8x4_reg.npz", 8, 4, 1e-2), ("spring_bar_16x4.npz", 16, 4, 0.0)])
def test_spring_bar_oracle_matches_reference(name, nw, nh, wreg):
    g = _gold(name)
    prob = SpringBarOracle(nw, nh, w_reg=wreg)
    p = prob.default_parameters()
    np.testing.assert_array_equal(p, g["p"])
    x = prob.simulate(p)
    assert _rel(x, g["x"]) <= 1e-10
    x = g["x"]
    assert _rel(_nz(prob.constraint_jac_x(x, p).to_scipy()).toarray(), _nz(_csc(g, "Gx")).toarray()) <= 1e-13
    assert _rel(_nz(prob.constraint_jac_p(x, p).to_scipy()).toarray(), _nz(_csc(g, "Gp")).toarray()) <= 1e-13
    K, rhs, grad = sgn_cpu.assemble_sgn(prob, x, p)
    assert _rel(_nz(K.to_scipy()).toarray(), _nz(_csc(g, "K")).toarray()) <= 1e-13
    assert _rel(grad, g["grad"]) <= 1e-10
    d = sgn_cpu.direction_sgn(prob, x, p)
    assert _rel(d.dp, g["dp"]) <= 1e-8
    assert _rel(sgn_cpu.direction_dgn(prob, x, p).dp, g["dp_dgn"]) <= 1e-8
    prob._x_warm = None
    run = sgn_cpu.minimize_sgn(prob, p, max_iterations=len(g["traj_f"]) - 1)
    n = min(len(run["f"]), len(g["traj_f"]))
    np.testing.assert_allclose(run["f"][:n], g["traj_f"][:n], rtol=1e-8, atol=1e-14 * g["traj_f"][0])


def test_sheet_c1_oracle_matches_reference_solver():
    """The oracle NH sheet driven by the reference solver (make_golden) == oracle solver."""
    g = _gold("sheet_c1.npz")
    prob, p0 = oracle_sheet(1)
    np.testing.assert_array_equal(p0, g["p"])
    x = g["x"]
    K, rhs, grad = sgn_cpu.assemble_sgn(prob, x, p0)
    Kr = _csc(g, "K")
    np.testing.assert_array_equal(K.indptr, Kr.indptr)   # structural pattern, bit-exact
    np.testing.assert_array_equal(K.indices, Kr.indices)
    assert np.max(np.abs(K.data - Kr.data)) <= 1e-13 * np.max(np.abs(Kr.data))
    d = sgn_cpu.direction_sgn(prob, x, p0)
    assert _rel(d.dp, g["dp"]) <= 1e-9
    assert _rel(d.dp, g["dp_dgn"]) <= 1e-6            # Theorem 1


@pytest.mark.parametrize("kind", ["tri", "tet"])
def test_element_derivatives_fd(kind):
    """Complex-step second derivatives vs central differences of the analytic gradient,
    gradient vs central differences of the energy (reference test_problems.py:18-61 idiom)."""
    rng = np.random.default_rng(3)
    d = 2 if kind == "tri" else 3
    nv = d + 1
    X = rng.standard_normal((5, nv, d)) * 0.3 + np.eye(nv, d)[None]
    x = X + 0.05 * rng.standard_normal(X.shape)
    mu, lam, gl = 3.0, 5.0, 0.7
    H, M = el.nh_second(x, X, mu, lam, gl)
    h = 1e-6
    for k in range(nv * d):
        a, i = divmod(k, d)
        xp, xm = x.copy(), x.copy()
        xp[:, a, i] += h; xm[:, a, i] -= h
        fd = (el.nh_grad(xp, X, mu, lam, gl) - el.nh_grad(xm, X, mu, lam, gl)) / (2 * h)
        assert _rel(H[:, :, k], fd) <= 1e-7
        ep, em = el.nh_energy(xp, X, mu, lam, gl), el.nh_energy(xm, X, mu, lam, gl)
        assert _rel(el.nh_grad(x, X, mu, lam, gl)[:, k], (ep - em) / (2 * h)) <= 1e-7
        Xp, Xm = X.copy(), X.copy()
        Xp[:, a, i] += h; Xm[:, a, i] -= h
        fd = (el.nh_grad(x, Xp, mu, lam, gl) - el.nh_grad(x, Xm, mu, lam, gl)) / (2 * h)
        assert _rel(M[:, :, k], fd) <= 1e-7
    assert _rel(H, np.swapaxes(H, 1, 2)) <= 1e-13


def test_sheet_jacobians_fd():
    prob, p0 = oracle_sheet(1)
    x = prob.simulate(p0)
    rng = np.random.default_rng(0)
    Gx = prob.constraint_jac_x(x, p0).to_scipy()
    Gp = prob.constraint_jac_p(x, p0).to_scipy()
    for _ in range(4):
        v = rng.standard_normal(prob.n_x)
        h = 1e-6
        fd = (prob.constraints(x + h * v, p0) - prob.constraints(x - h * v, p0)) / (2 * h)
        assert _rel(Gx @ v, fd) <= 1e-7
        v = rng.standard_normal(prob.n_p)
        fd = (prob.constraints(x, p0 + h * v) - prob.constraints(x, p0 - h * v)) / (2 * h)
        assert _rel(Gp @ v, fd) <= 1e-7


def test_spec_generators_agree():
    from paper_2107_03285_b200.problems import sheet_spec as gpu_spec
    for cfg, inst in [(1, 0), (1, 4), (2, 0), (2, 7)]:
        a, b = gpu_spec(cfg, 0, inst), sheet_spec(cfg, 0, inst)
        for k, va in a.items():
            vb = b[k]
            if isinstance(va, tuple):
                assert all(np.array_equal(u, v) for u, v in zip(va, vb)), k
            elif isinstance(va, np.ndarray):
                assert np.array_equal(va, vb), k
            else:
                assert va == vb, k


def test_c2_rest_shape_valid():
    s = sheet_spec(2, 0, 0)
    X = s["X0"].ravel().copy()
    X[s["pmap"][0]] += s["p0"]
    X = X.reshape(-1, 2)
    t = s["conn"]
    e1, e2 = X[t[:, 1]] - X[t[:, 0]], X[t[:, 2]] - X[t[:, 0]]
    area = 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    assert area.min() >= 0.2 * 0.5 / 99 ** 2
    assert np.all(np.abs(s["p0"]) <= 0.005)


def test_beam_generators_agree_and_mesh_is_conforming():
    from collections import Counter
    from oracle.configs import beam_spec
    from paper_2107_03285_b200.problems import beam_spec as gpu_beam
    a, b = beam_spec(0), gpu_beam(0)
    for k, va in a.items():
        vb = b[k]
        if isinstance(va, tuple):
            assert all(np.array_equal(u, v) for u, v in zip(va, vb)), k
        elif isinstance(va, np.ndarray):
            assert np.array_equal(va, vb), k
        else:
            assert va == vb, k
    X0, tets = a["X0"], a["conn"]
    assert tets.shape == (20000, 4) and X0.shape == (4961, 3)
    P = X0[tets]
    vol = np.linalg.det(np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], axis=2)) / 6
    assert vol.min() > 0 and abs(vol.sum() - 4.0) < 1e-12
    faces = Counter()
    for t in tets:
        for f in ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)):
            faces[tuple(sorted(t[list(f)]))] += 1
    assert max(faces.values()) == 2 and sum(v == 1 for v in faces.values()) == 3600
    assert len(a["p0"]) == 1881 and len(a["target_dofs"]) == 363


def test_shell_displacement_state_jacobians_fd_and_theorem1():
    """Config-4 oracle (displacement state in mm): dc/dx and dc/dp against central
    differences of the constraints, and SGN = DGN (Theorem 1, checks.py:71-128)."""
    from oracle import sgn_cpu
    from oracle.shell import ShellProblem, shell_spec
    spec = shell_spec(9, 5)
    prob = ShellProblem(spec)
    rng = np.random.default_rng(1)
    p = 2e-3 * rng.standard_normal(prob.n_p)
    x = prob.simulate(p)
    assert np.abs(prob.constraints(x, p)).max() <= prob.tol
    Gx = prob.constraint_jac_x(x, p).to_scipy()
    Gp = prob.constraint_jac_p(x, p).to_scipy()
    for _ in range(3):
        v = rng.standard_normal(prob.n_x)
        h = 1e-4
        fd = (prob.constraints(x + h * v, p) - prob.constraints(x - h * v, p)) / (2 * h)
        assert _rel(Gx @ v, fd) <= 1e-7
        v = rng.standard_normal(prob.n_p)
        h = 1e-7
        fd = (prob.constraints(x, p + h * v) - prob.constraints(x, p - h * v)) / (2 * h)
        assert _rel(Gp @ v, fd) <= 1e-6
    # this coarse bumpy shell's reduced Hessian amplifies the refinement's residual into dp
    # (3e-7 at the default 1e-10 tolerance); the reference's own knob, a tighter
    # refine_tolerance, gives Theorem 1 to 2e-10
    d_sgn = sgn_cpu.direction_sgn(prob, x, p, sgn_cpu.Stab(refine_tolerance=1e-12))
    d_dgn = sgn_cpu.direction_dgn(prob, x, p)
    assert d_sgn.res <= 1e-12
    assert _rel(d_sgn.dp, d_dgn.dp) <= 1e-8

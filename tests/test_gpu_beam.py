"""BASELINE config 3 (3-D neo-Hookean tet beam, C = 0) on the device vs the CPU oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def beam():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_03285_b200.problems import build_beam
    return build_beam(0)


def test_tet_element_blocks_match_oracle(beam):
    from oracle import elements as el
    from oracle.configs import oracle_beam
    prob, p0, sag = beam
    oprob, _ = oracle_beam(0, targets=sag)
    x = prob._x_warm
    prob._load(x, p0)
    prob.engine.positions()
    prob.engine.element_blocks()
    pl = prob.plan
    nd2 = pl.n_e * pl.nd * pl.nd
    buf = prob.engine.ebuf[0].cpu().numpy()
    g0 = pl.groups[0]
    sup = np.flatnonzero(g0.mslot >= 0)            # surface tets: mixed blocks in compact slots
    sel = sup[::29]
    H = buf[:nd2].reshape(pl.n_e, pl.nd, pl.nd)[sel]
    M = buf[nd2:nd2 + sup.size * pl.nd * pl.nd].reshape(sup.size, pl.nd, pl.nd)[g0.mslot[sel]]
    pos, rest = oprob.full_positions(x), oprob.rest_positions(p0)
    Ho, Mo = el.nh_second(pos[oprob.conn[sel]], rest[oprob.conn[sel]], oprob.mu, oprob.lam, oprob.gload)
    assert _rel(H, oprob.scale * Ho) <= 1e-12
    assert _rel(M, oprob.scale * Mo) <= 1e-12


def test_beam_equilibrium_satisfies_oracle_physics(beam):
    from oracle.configs import oracle_beam
    prob, p0, sag = beam
    oprob, _ = oracle_beam(0, targets=sag)
    c = oprob.constraints(prob._x_warm, p0)
    assert np.abs(c).max() <= 1e-11          # scaled forces (1/E) at the device equilibrium
    tip_drop = prob.plan.X0.ravel()[prob.plan.free_dofs][prob.plan.target_dofs] - sag
    assert tip_drop.reshape(-1, 3)[:, 1].mean() > 1.0   # the cantilever sags under self-weight


def test_beam_direction_matches_oracle(beam):
    """Config 3's reduced GN Hessian is so ill-conditioned that any solution meeting the
    reference's 1e-10 residual contract is defined only to ~1e-7 in dp (measured: the
    oracle's SGN and DGN differ by 7e-7; both SGN solvers sit 8e-7 from the exact unshifted
    direct solve).  So we check what is exactly defined: the KKT (pattern bit-exact, values
    <= 1e-12), the adjoint gradient, and that the device solution solves the ORACLE's KKT to
    the reference's tolerance; dp agreement is checked at the documented bound."""
    from oracle import sgn_cpu
    from oracle.configs import oracle_beam
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    prob, p0, sag = beam
    oprob, _ = oracle_beam(0, targets=sag)
    x = prob._x_warm
    K = prob.kkt_matrix(x, p0)
    Kr, rhs_r, g_r = sgn_cpu.assemble_sgn(oprob, x, p0)
    np.testing.assert_array_equal(K.indptr, Kr.indptr)
    np.testing.assert_array_equal(K.indices, Kr.indices)
    assert np.max(np.abs(K.data - Kr.data)) <= 1e-12 * np.max(np.abs(Kr.data))
    g = adjoint_gradient(prob, x, p0)
    assert _rel(g, g_r) <= 1e-9
    sd = direction_sgn(prob, x, p0, OptimizerConfig())
    assert sd.relative_residual <= 1e-10
    sol = np.concatenate([sd.dx, sd.dp, sd.dlam])
    rhs = np.zeros_like(rhs_r)
    rhs[prob.n_x:prob.n_x + prob.n_p] = -g        # the device's own gradient (<= 1e-9 from g_r)
    assert np.linalg.norm(Kr.to_scipy() @ sol - rhs) <= 2e-10 * np.linalg.norm(rhs)
    # the reduced Hessian is ill-conditioned: dp parity at the conditioning bound
    # kappa * 1e-10 that two residual-contract solvers can differ by (tests/conditioning.py)
    from conditioning import check_forward_error
    ref = sgn_cpu.direction_sgn(oprob, x, p0)
    m = check_forward_error(Kr.to_scipy(), sol, rhs, slice(prob.n_x, prob.n_x + prob.n_p), ref.dp)
    print("conditioning", m)

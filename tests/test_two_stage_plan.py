"""Host check of the two-stage assembly lists (engine.MeshPlan._two_stage_lists): on a small
shell they reproduce the one-stage gather (every element entry expanded over the parameters
of its rest dof and both symmetric copies) on random element blocks."""
import numpy as np


def _segsum(ptr, vals):
    out = np.zeros(ptr.size - 1)
    np.add.at(out, np.repeat(np.arange(ptr.size - 1), np.diff(ptr)), vals)
    return out


def test_two_stage_lists_equal_one_stage_gather():
    from paper_2107_03285_b200.engine import MeshPlan
    from paper_2107_03285_b200.problems import SHELL_DISP_SCALE, shell_spec
    s = shell_spec(13, 6)
    pl = MeshPlan(s["X0"], None, None, s["fixed_verts"], s["pmap"], s["target_dofs"], s["w_target"], s["w_reg"],
                  groups=[("membrane", s["tris"]), ("hinge", s["hinges"])], disp_scale=SHELL_DISP_SCALE)
    ts = pl.two_stage
    assert ts is not None
    rng = np.random.default_rng(3)
    ebuf = rng.standard_normal(pl.ebuf_size)
    one = pl.K_base + _segsum(pl.K_ptr, pl.K_coef * ebuf[pl.K_src])
    two = pl.K_base.copy()
    gv = _segsum(pl.G_ptr, pl.G_coef * ebuf[pl.G_src])
    two[ts["gx_dst"]] = gv[ts["gx_src"]]
    mz = _segsum(ts["mz_ptr"], ebuf[ts["mz_src"]])
    two[ts["gp_dst"]] = _segsum(ts["gp_ptr"], ts["gp_coef"] * mz[ts["gp_src"]])
    assert np.unique(np.concatenate([ts["gx_dst"], ts["gp_dst"]])).size == ts["gx_dst"].size + ts["gp_dst"].size
    scale = np.abs(one).max()
    assert np.abs(one - two).max() <= 1e-13 * scale
    # far fewer terms than the one-stage expansion
    n_two = pl.G_src.size + ts["gx_src"].size + ts["mz_src"].size + ts["gp_src"].size
    assert n_two < 0.45 * pl.K_src.size

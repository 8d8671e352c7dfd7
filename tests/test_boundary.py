"""CPU checks of the drop-in boundary and the host symbolic analysis (no GPU needed)."""
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from kkt_fixtures import grid_laplacian, kkt_system
from mf_emulate import emulate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgn_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+\*?(sgn_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2107_03285_b200._lib import SIGNATURES, lib
    names = _declared()
    assert len(names) >= 24
    so = lib()
    for name in names:
        assert hasattr(so, name), name
        assert name in SIGNATURES, f"{name} declared in the header but not bound in _lib.py"


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2107_03285_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2107_03285_b200 import CscMatrix, DeviceError, factor_sparse
    with pytest.raises(DeviceError):
        factor_sparse(CscMatrix.identity(4))


@pytest.mark.parametrize("shape", [(3, 3, 1, 2, 1e-2), (6, 5, 2, 7, 1e-2), (12, 10, 2, 9, 0.0),
                                   (20, 17, 2, 30, 1e-3)])
def test_symbolic_kkt_tree_reproduces_factorization(shape):
    from paper_2107_03285_b200.device import Symbolic
    K, n_x, n_p, _ = kkt_system(*shape)
    s = Symbolic(K.shape[0], K.indptr, K.indices, n_x, n_p, n_x, leaf_size=16)
    st = s.stats()
    assert st["pair_mode"] == 1 and st["n"] == K.shape[0]
    perm = s.perm()
    assert np.array_equal(np.sort(perm), np.arange(K.shape[0]))
    assert np.all(perm[-n_p:] >= n_x) and np.all(perm[-n_p:] < n_x + n_p)   # p eliminated last
    _, _, _, err, _ = emulate(K, s, 1e-6, 1e-6)
    assert err <= 1e-13


@pytest.mark.parametrize("shape", [(6, 5, 2, 7, 1e-2), (12, 10, 2, 9, 1e-3), (20, 17, 2, 30, 1e-3),
                                   (20, 17, 2, 31, 1e-3)])
def test_symbolic_p_pairs_in_dissection(shape):
    """p_order 1 (C > 0): p pairs are dissection nodes (an odd last p is eliminated last),
    the tree reproduces the factorization, and the ordering is deterministic."""
    from paper_2107_03285_b200.device import Symbolic
    K, n_x, n_p, _ = kkt_system(*shape)
    s = Symbolic(K.shape[0], K.indptr, K.indices, n_x, n_p, n_x, leaf_size=16, p_order=1)
    s2 = Symbolic(K.shape[0], K.indptr, K.indices, n_x, n_p, n_x, leaf_size=16, p_order=1)
    assert s.stats()["pair_mode"] == 2
    perm = s.perm()
    assert np.array_equal(perm, s2.perm())
    assert np.array_equal(np.sort(perm), np.arange(K.shape[0]))
    if n_p % 2:
        assert perm[-1] == n_x + n_p - 1
    pos = np.argsort(perm)
    for k in range(n_p // 2):                         # each p pair stays adjacent, in order
        assert pos[n_x + 2 * k + 1] == pos[n_x + 2 * k] + 1
    _, _, _, err, _ = emulate(K, s, 1e-6, 1e-6)
    assert err <= 1e-12          # small C pivots (1e-3) eliminated early: modest growth


def test_symbolic_generic_mode_and_determinism():
    from paper_2107_03285_b200.device import Symbolic
    g = grid_laplacian(15, 13, 2)
    s1 = Symbolic(g.shape[0], g.indptr, g.indices)
    s2 = Symbolic(g.shape[0], g.indptr, g.indices)
    assert np.array_equal(s1.perm(), s2.perm())
    _, _, _, err, _ = emulate(g, s1)
    assert err <= 1e-13
    eye = sp.identity(10, format="csc")
    assert Symbolic(10, eye.indptr, eye.indices).stats()["nnz_l"] == 10


def test_symbolic_reports_structural_singularity():
    from paper_2107_03285_b200 import SingularMatrix
    from paper_2107_03285_b200.device import Symbolic
    # KKT with a state whose constraint column has no multiplier coupling
    n_x, n_p = 3, 1
    A = sp.identity(n_x, format="csc")
    G = sp.csc_matrix(np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 1.0, 0]]))
    Gp = sp.csc_matrix(np.ones((n_x, n_p)))
    K = sp.bmat([[A, None, G.T], [None, sp.identity(1), Gp.T], [G, Gp, None]], format="csc")
    K.sort_indices()
    with pytest.raises(SingularMatrix) as exc:
        Symbolic(K.shape[0], K.indptr, K.indices, n_x, n_p, n_x)
    assert exc.value.pivot_index == 2


def test_symbolic_rejects_unsymmetric_pattern():
    from paper_2107_03285_b200 import ToolkitError
    from paper_2107_03285_b200.device import Symbolic
    m = sp.csc_matrix(np.array([[1.0, 1.0], [0.0, 1.0]]))
    with pytest.raises(ToolkitError):
        Symbolic(2, m.indptr, m.indices)


def test_c2_plan_and_symbolic_sizes():
    from paper_2107_03285_b200.device import Symbolic
    from paper_2107_03285_b200.engine import MeshPlan
    from paper_2107_03285_b200.problems import sheet_spec
    s = sheet_spec(2)
    pl = MeshPlan(s["X0"], s["conn"], "tri", s["fixed_verts"], s["pmap"], s["target_dofs"], 1.0, 2e-6)
    assert (pl.n_x, pl.n_p, pl.dim) == (19800, 400, 40000)
    sy = Symbolic(pl.dim, pl.K_indptr, pl.K_indices, pl.n_x, pl.n_p, pl.n_x)
    st = sy.stats()
    assert st["n"] == 40000 and st["max_piv"] == 400


@pytest.mark.parametrize("which", ["c1", "c3"])
def test_vertex_plan_covers_the_staged_lists(which):
    """The fused vertex-centric assembly plan sums, for every G_x entry of K (both copies)
    and of G_x, exactly the element-Hessian terms of the staged element->nonzero lists, in
    the same element order; the rest of K (constants, G_p) goes to the restricted gather."""
    from paper_2107_03285_b200.engine import MeshPlan, vertex_plan
    from paper_2107_03285_b200.problems import beam_spec, sheet_spec
    s = sheet_spec(1) if which == "c1" else beam_spec(0)
    pl = MeshPlan(s["X0"], s["conn"], s["kind"], s["fixed_verts"], s["pmap"], s["target_dofs"],
                  s.get("w_target", 1.0), s.get("w_reg", 0.0), f_ext=s.get("f_ext"),
                  rest_base=s.get("rest_base"), R=s.get("R"))
    vp = vertex_plan(pl)
    assert vp is not None and vp.max_inc <= 32
    g = pl.groups[0]
    d, nd = pl.d, g.nd
    dst = vp.out_dst.reshape(-1, 3)
    # every K nonzero is produced exactly once: fused (two copies per output) or restricted
    owner = np.zeros(pl.nnz, np.int64)
    np.add.at(owner, dst[:, 0], 1)
    np.add.at(owner, dst[:, 1], 1)
    np.add.at(owner, vp.rest_dst, 1)
    assert (owner == 1).all()
    assert np.array_equal(np.sort(dst[:, 2]), np.arange(pl.G_nnz))     # G_x: each entry once
    # per output: the staged list of its K[lambda_r, x_c] entry, decoded to (element, row, col)
    inc_e, inc_a = vp.inc_ea >> 2, vp.inc_ea & 3
    task_of_out = np.repeat(np.arange(vp.n_task), np.diff(vp.out_ptr))
    rng = np.random.default_rng(0)
    for o in rng.choice(vp.n_out, size=min(300, vp.n_out), replace=False):
        t = task_of_out[o]
        cons = vp.con_idx[vp.con_ptr[o]:vp.con_ptr[o + 1]]
        slot, i, r = cons // (d * nd), (cons // nd) % d, cons % nd
        elems = inc_e[vp.inc_ptr[t] + slot]
        a = inc_a[vp.inc_ptr[t] + slot]
        got = [(int(e), int(rr), int(aa * d + ii)) for e, rr, aa, ii in zip(elems, r, a, i)]
        k = dst[o, 0]
        src = pl.K_src[pl.K_ptr[k]:pl.K_ptr[k + 1]] - g.hoff
        want = [(int(x // (nd * nd)), int((x % (nd * nd)) // nd), int(x % nd)) for x in src]
        assert got == want                      # same terms, same (ascending element) order
        assert np.all(pl.K_coef[pl.K_ptr[k]:pl.K_ptr[k + 1]] == 1.0) and pl.K_base[k] == 0.0


def test_mixed_slots_cover_the_pmap_support():
    from paper_2107_03285_b200.engine import MeshPlan
    from paper_2107_03285_b200.problems import sheet_spec
    s = sheet_spec(2)
    pl = MeshPlan(s["X0"], s["conn"], "tri", s["fixed_verts"], s["pmap"], s["target_dofs"], 1.0, 2e-6)
    g = pl.groups[0]
    used = np.zeros(pl.n_v * pl.d, bool)
    used[np.asarray(s["pmap"][0])] = True
    el_dofs = (g.conn[:, :, None] * pl.d + np.arange(pl.d)).reshape(g.n_e, -1)
    sup = used[el_dofs].any(axis=1)
    assert np.array_equal(g.mslot >= 0, sup) and np.array_equal(g.melems, np.flatnonzero(sup))
    assert np.array_equal(g.mslot[g.melems], np.arange(g.n_m))
    # every G_p contribution reads a mixed slot of the support
    nd2 = g.nd * g.nd
    msrc = pl.K_src[pl.K_src >= g.moff] - g.moff
    assert (msrc // nd2 < g.n_m).all()

"""On-disk formats: the package's writers reproduce the reference's files.

ref_kkt_spring_bar_5x3/ and ref_convergence_sgn_5x3.csv were written by the real reference
(tests/golden/make_golden_formats.py)."""
import os

import numpy as np

from paper_2107_03285_b200.sparse import CscMatrix, read_matrix_market, write_matrix_market

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_matrix_market_bytes_match_reference_writer(tmp_path):
    g = dict(np.load(os.path.join(GOLD, "spring_bar_5x3.npz")))
    K = CscMatrix(int(g["K_shape"][0]), int(g["K_shape"][1]), g["K_indptr"], g["K_indices"], g["K_data"])
    out = tmp_path / "kkt.mtx"
    write_matrix_market(K, out)
    ref = open(os.path.join(GOLD, "ref_kkt_spring_bar_5x3", "kkt.mtx"), "rb").read()
    assert out.read_bytes() == ref                                   # byte-identical
    back = read_matrix_market(out)
    np.testing.assert_array_equal(back.indptr, K.indptr)
    np.testing.assert_array_equal(back.indices, K.indices)
    np.testing.assert_array_equal(back.data, K.data)


def test_scaling_row_format():
    from paper_2107_03285_b200.fixtures import SCALING_HEADER, scaling_row

    class P:
        n_x, n_p = 24, 24
    t = dict(direction_time_median_s=1.23456789e-3, assemble_s=1e-4, factor_s=2e-4, solve_s=3e-4,
             sens_matrix_s=0.0, dense_factor_s=0.0)
    row = scaling_row("spring_bar", "sgn", P(), t)
    assert row == "spring_bar,sgn,24,24,0.00123457,0.0001,0.0002,0.0003,0,0,"
    assert len(row.split(",")) == len(SCALING_HEADER.split(","))


def test_kkt_fill_is_symbolic_and_sane():
    """factor_fill_nnz of the dump comes from the symbolic analysis alone (no GPU, no values)."""
    from paper_2107_03285_b200.fixtures import kkt_fill_nnz
    from paper_2107_03285_b200.sensitivity import KktSystem
    g = dict(np.load(os.path.join(GOLD, "spring_bar_5x3.npz")))
    n = int(g["K_shape"][0])
    K = CscMatrix(n, n, g["K_indptr"], g["K_indices"], g["K_data"])
    kkt = KktSystem(matrix=K, rhs=np.zeros(n), n_x=int(g["n_x"]), n_p=int(g["n_p"]), n_c=int(g["n_x"]))
    fill = kkt_fill_nnz(kkt)
    assert K.nnz - n <= fill <= n * n                  # at least the matrix, at most dense (2 n(n+1)/2 - n)

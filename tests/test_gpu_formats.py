"""GPU path -> the reference's on-disk formats (kkt.mtx + stats.json, convergence CSV,
scaling.csv), compared with files written by the real reference."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_kkt_dump_matches_reference_dump(cuda, tmp_path):
    from paper_2107_03285_b200.fixtures import kkt_dump
    from paper_2107_03285_b200.problems import build_spring_bar
    from paper_2107_03285_b200.sparse import read_matrix_market
    prob = build_spring_bar(5, 3)
    stats = kkt_dump(prob, tmp_path, "spring_bar")
    ref_stats = json.load(open(os.path.join(GOLD, "ref_kkt_spring_bar_5x3", "stats.json")))
    for k in ("problem", "dimension", "n_x", "n_p"):
        assert stats[k] == ref_stats[k], k
    ours = read_matrix_market(tmp_path / "kkt.mtx").to_scipy().toarray()
    ref = read_matrix_market(os.path.join(GOLD, "ref_kkt_spring_bar_5x3", "kkt.mtx")).to_scipy().toarray()
    # the reference's SpGEMM drops value-dependent zeros: compare values
    assert np.max(np.abs(ours - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert stats["nnz"] >= ref_stats["nnz"] == np.count_nonzero(ref)
    assert stats["factor_fill_nnz"] > 0


def test_convergence_csv_schema_and_values(cuda, tmp_path):
    from paper_2107_03285_b200 import CSV_HEADER, OptimizerConfig, minimize
    from paper_2107_03285_b200.problems import build_spring_bar
    prob = build_spring_bar(5, 3)
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method="sgn", max_iterations=4, gradient_tolerance=1e-12))
    path = tmp_path / "convergence_sgn.csv"
    run.write_csv(path)
    ours = open(path).read().splitlines()
    ref = open(os.path.join(GOLD, "ref_convergence_sgn_5x3.csv")).read().splitlines()
    assert ours[0] == ref[0] == CSV_HEADER
    assert len(ours) == len(ref)
    for a, b in zip(ours[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert len(fa) == len(fb) == 8
        assert fa[0] == fb[0] and fa[3] == fb[3]                            # iter, step length
        assert abs(float(fa[1]) - float(fb[1])) <= 1e-8 * abs(float(ref[1].split(",")[1]))   # f
        if fb[7] != "nan":
            assert float(fa[7]) <= 1e-10                                  # linear residual contract


def test_scaling_csv_from_device_timings(cuda, tmp_path):
    from paper_2107_03285_b200 import OptimizerConfig
    from paper_2107_03285_b200.fixtures import SCALING_HEADER, scaling_row, time_direction, write_scaling_csv
    from paper_2107_03285_b200.problems import build_spring_bar
    prob = build_spring_bar(5, 3)
    p = prob.default_parameters()
    x = prob.simulate(p)
    t = time_direction(prob, x, p, OptimizerConfig(), "sgn", repetitions=3)
    assert t["direction_time_median_s"] > 0 and t["factor_s"] >= 0
    write_scaling_csv(tmp_path / "scaling.csv", [scaling_row("spring_bar", "sgn", prob, t)])
    lines = open(tmp_path / "scaling.csv").read().splitlines()
    assert lines[0] == SCALING_HEADER and lines[1].startswith("spring_bar,sgn,24,24,")

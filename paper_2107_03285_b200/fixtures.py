"""On-disk fixture and wire formats emitted from the GPU path.

The reference's tooling reads three files; this module writes them from the device
results with the reference's exact schemas, so its CLI tests and tooling can consume GPU
output:

* ``kkt.mtx`` + ``stats.json``  -- ``cmd_kkt_dump`` (reference cli.py:284-305): the stacked
  KKT in 1-based MatrixMarket coordinate format (``write_matrix_market``, sparse.py:192-199;
  %.17g values) and the dump statistics.  ``factor_fill_nnz`` keeps the reference meaning
  "nonzeros of the combined factors minus n" (linear_solvers.py:64-91); for the device
  LDL^T that is 2 nnz(L) - n (``SparseFactorization.fill_nnz``).
* ``convergence_<method>.csv``  -- ``OptimizerRun.write_csv`` (optimize.py:60,112-137),
  already provided by :class:`paper_2107_03285_b200.optimize.OptimizerRun`.
* ``scaling.csv``              -- ``cmd_scaling`` rows (cli.py:34-35, 240-268) built from
  :func:`time_direction` (cli.py:189-232).
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np

from .errors import ToolkitError
from .optimize import _DIRECTION_FUNCS
from .sensitivity import assemble_sgn, gn_blocks
from .sparse import write_matrix_market

__all__ = ["SCALING_HEADER", "kkt_dump", "kkt_fill_nnz", "time_direction", "scaling_row", "scaling_error_row",
           "write_scaling_csv"]

SCALING_HEADER = ("problem,method,n_x,n_p,direction_time_median_s,assemble_s,"
                  "factor_s,solve_s,sens_matrix_s,dense_factor_s,error")


def kkt_dump(problem, out_dir, problem_name: str, p=None, x=None) -> dict:
    """Write ``kkt.mtx`` and ``stats.json`` for ``problem`` at (x, p) (reference cli.py:284-305).

    ``p`` defaults to ``problem.default_parameters()`` and ``x`` to ``problem.simulate(p)``,
    as in the reference.  Returns the stats dict.
    """
    os.makedirs(out_dir, exist_ok=True)
    if p is None:
        p = problem.default_parameters()
    if x is None:
        x = problem.simulate(p)
    kkt = assemble_sgn(problem, x, p, gn_blocks(problem, x, p))
    write_matrix_market(kkt.matrix, os.path.join(out_dir, "kkt.mtx"))
    fill = kkt_fill_nnz(kkt)
    stats = {"problem": problem_name, "dimension": kkt.matrix.rows, "n_x": kkt.n_x, "n_p": kkt.n_p,
             "nnz": kkt.matrix.nnz, "factor_fill_nnz": int(fill)}
    with open(os.path.join(out_dir, "stats.json"), "w", encoding="utf-8") as fh:
        json.dump(stats, fh, indent=2)
    return stats


def kkt_fill_nnz(kkt) -> int:
    """Fill of the device factorization of a KKT system: 2 nnz(L) - n (the reference's
    "combined factors minus n", linear_solvers.py:64-91).  Symbolic only: the fill does not
    depend on values, so no numeric factorization of the unshifted matrix is needed."""
    from .device import symbolic_for
    from .linear_solvers import _symmetric_pattern
    indptr, indices, _ = _symmetric_pattern(kkt.matrix)
    n = kkt.matrix.rows
    sym = symbolic_for(n, indptr, indices, kkt.n_x, kkt.n_p, kkt.n_c)
    return int(2 * sym.stats()["nnz_l"] - n)


def time_direction(problem, x, p, cfg, method: str = "sgn", repetitions: int = 5) -> dict:
    """Median component timings of repeated directions (reference cli.py:189-232).

    Wall-clock per direction through the public API (host arrays in and out; the device
    work is complete when ``direction_sgn`` returns, since it copies dp to the host).
    """
    func = lambda: _DIRECTION_FUNCS[method](problem, x, p, cfg)
    func()   # warm-up off the clock (also builds the device plans / graphs)
    totals, samples = [], []
    for _ in range(int(repetitions)):
        t0 = time.perf_counter()
        sd = func()
        totals.append(time.perf_counter() - t0)
        samples.append(sd)
    med = statistics.median
    sd = samples[int(np.argsort(totals)[len(totals) // 2])]
    return {
        "direction_time_median_s": med(totals),
        "assemble_s": med([s.assemble_s for s in samples]),
        "factor_s": med([s.factor_s for s in samples]),
        "solve_s": med([s.solve_s for s in samples]),
        "sens_matrix_s": sd.extra.get("sens_matrix_s", 0.0),
        "dense_factor_s": sd.extra.get("dense_factor_s", 0.0),
    }


def scaling_row(problem_name: str, method: str, problem, t: dict) -> str:
    """One ``scaling.csv`` row (reference cli.py:255-260 formatting)."""
    return (f"{problem_name},{method},{problem.n_x},{problem.n_p},"
            f"{t['direction_time_median_s']:.6g},{t['assemble_s']:.6g},"
            f"{t['factor_s']:.6g},{t['solve_s']:.6g},"
            f"{t['sens_matrix_s']:.6g},{t['dense_factor_s']:.6g},")


def scaling_error_row(problem_name: str, method: str, problem, exc: ToolkitError) -> str:
    """The failure row (reference cli.py:261-264)."""
    return f"{problem_name},{method},{problem.n_x},{problem.n_p},,,,,,,\"{exc}\""


def write_scaling_csv(path, rows) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(SCALING_HEADER + "\n")
        for row in rows:
            fh.write(row + "\n")

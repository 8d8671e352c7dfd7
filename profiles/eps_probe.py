"""Refinement iterations / direction time / dp parity vs the reference golden as the
stabilization shift of the FACTOR varies (the refinement always targets the unshifted K).
python profiles/eps_probe.py --config 2"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
    from paper_2107_03285_b200.linear_solvers import StabilizationConfig
    if a.config == 4:
        from paper_2107_03285_b200.problems import build_shell
        prob, p0 = build_shell(201, 100)
    else:
        from paper_2107_03285_b200.problems import build_sheet
        prob, p0 = build_sheet(a.config)
    gold = np.load(os.path.join(ROOT, "tests", "golden", f"large_c{a.config}.npz"))
    x = gold["x"]
    for eps in (1e-6, 1e-8, 1e-10, 1e-12, 0.0):
        cfg = OptimizerConfig(stabilization=StabilizationConfig(eps_x=eps, eps_lambda=eps))
        try:
            sd = direction_sgn(prob, x, p0, cfg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                sd = direction_sgn(prob, x, p0, cfg)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 5
            err = np.linalg.norm(sd.dp - gold["dp"]) / np.linalg.norm(gold["dp"])
            print(f"eps {eps:.0e}: {dt * 1e3:.2f} ms/dir, iters {sd.extra['refine_iterations']}, "
                  f"res {sd.relative_residual:.2e}, dp vs reference {err:.2e}", flush=True)
        except Exception as exc:  # noqa: BLE001
            print(f"eps {eps:.0e}: {type(exc).__name__}: {exc}", flush=True)


if __name__ == "__main__":
    main()

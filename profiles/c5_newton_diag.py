"""Config-5 line-search forward solves: per trial, Newton iterations and the |c|_inf history
of the instances that do not converge (diagnostic for the 200-iteration stalls)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2107_03285_b200.engine as E
    from paper_2107_03285_b200 import OptimizerConfig
    from paper_2107_03285_b200.batch import minimize_batched
    from paper_2107_03285_b200.problems import build_sheet_batch
    hist = []
    orig = E.DeviceEngine._energies

    def energies(self, sc):                       # log |g|_inf of every Newton iteration
        e = orig(self, sc)
        hist.append((sc[3].copy(), e.copy()))
        return e
    E.DeviceEngine._energies = energies
    bd = build_sheet_batch(2, 0, instances=[1, 2, 3, 4])
    cfg = OptimizerConfig(method="sgn", max_iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 8,
                          gradient_tolerance=1e-12)
    t0 = time.time()
    run = minimize_batched(bd, bd.p0, cfg)
    print("run", time.time() - t0, "s; terminations", run.termination, "directions", run.directions)
    for t in run.timings.get("trials", []):
        print("trial", t)
    print("newton evaluations", len(hist), "tol", bd.tol)
    # |g|_inf of the longest single-instance stretch (the compacted engines of stalled trials)
    one = [h[0][0] for h in hist if len(h[0]) == 1]
    for k in range(0, min(len(one), 400)):
        print(k, f"{one[k]:.3e}")


if __name__ == "__main__":
    main()

"""Where a batched config-5 run spends its time: per SGN iteration the direction, every
line-search trial (instances forward-solved, Newton iterations of the batch, accepted) and
the gradient.  python profiles/c5_profile.py [--instances 16] [--iters 20]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=16)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import numpy as np
    from paper_2107_03285_b200 import OptimizerConfig
    from paper_2107_03285_b200.batch import minimize_batched
    from paper_2107_03285_b200.problems import build_sheet_batch
    bd = build_sheet_batch(2, 0, instances=range(1, a.instances + 1))
    cfg = OptimizerConfig(method="sgn", max_iterations=a.iters, gradient_tolerance=1e-12)
    t0 = time.perf_counter()
    run = minimize_batched(bd, bd.p0, cfg)
    print(f"instances {a.instances}: {time.perf_counter() - t0:.2f} s, directions {int(run.directions.sum())}")
    tm = run.timings
    print({k: round(v, 3) for k, v in tm.items() if k != "trials"})
    from collections import Counter
    print("terminations", Counter(run.termination))
    by_it = {}
    for it, n_run, newton, ok, dt in tm.get("trials", []):
        by_it.setdefault(it, []).append((n_run, newton, ok, round(dt, 3)))
    for it, tr in sorted(by_it.items()):
        print(f"it {it}: {len(tr)} trials, {sum(t[3] for t in tr):.2f} s: {tr[:14]}")


if __name__ == "__main__":
    main()

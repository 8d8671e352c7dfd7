"""One config-2 SGN direction bracketed by cudaProfilerStart/Stop (for ncu --profile-from-start off).

  python profiles/profile_direction.py [--config 2] [--reps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2107_03285_b200.problems import build_sheet
    prob, p0 = build_sheet(a.config)
    x = prob.simulate(p0)
    prob._load(x, p0)
    eng = prob.engine
    for _ in range(2):
        eng.direction()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.reps):
        eng.direction()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled", a.reps, "direction(s); KKT dim", prob.plan.dim)


if __name__ == "__main__":
    main()

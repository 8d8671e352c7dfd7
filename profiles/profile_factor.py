"""One config-N numeric factorization bracketed by cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--solve", action="store_true", help="also profile one triangular solve")
    a = ap.parse_args()
    import torch
    from paper_2107_03285_b200.problems import build_beam, build_sheet, build_shell
    if a.config == 3:
        prob, p0, _ = build_beam(0)
        x = prob._x_warm
    elif a.config == 4:
        prob, p0 = build_shell(201, 100)
        x = prob.simulate(p0)
    else:
        prob, p0 = build_sheet(a.config)
        x = prob.simulate(p0)
    prob._load(x, p0)
    eng = prob.engine
    eng.direction()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    eng.kfac.numeric(eng.kvals, eng.stab.eps_x, eng.stab.eps_lambda)
    if a.solve:
        b = torch.ones(eng.batch, prob.plan.dim, dtype=torch.float64, device="cuda")
        xs = torch.empty_like(b)
        eng.kfac.solve(b, xs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one factorization; KKT dim", prob.plan.dim)


if __name__ == "__main__":
    main()

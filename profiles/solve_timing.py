"""Per-call timing of the factor and the triangular solve on one config (CUDA events).

  python profiles/solve_timing.py [--config 2] [--reps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch
    from paper_2107_03285_b200.problems import build_sheet
    prob, p0 = build_sheet(a.config)
    x = prob.simulate(p0)
    prob._load(x, p0)
    eng = prob.engine
    eng.direction()
    fac = eng.kfac
    n = prob.plan.dim
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    xo = torch.empty_like(b)
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    if os.environ.get("NOP_AFTER_SETUP"):
        os.environ["SGN_DAG_NOP"] = "1"   # scheduling-only timing (results are garbage)
    for name, fn in [("solve", lambda: fac.solve(b, xo, stream=st)),
                     ("factor", lambda: fac.numeric(eng.kvals, eng.stab.eps_x, eng.stab.eps_lambda, stream=st))]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_us"] = e0.elapsed_time(e1) / a.reps * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()

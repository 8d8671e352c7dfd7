"""Assembly phase (positions -> element blocks -> KKT gather -> least-squares terms) under
ncu: setup runs outside the profiler range, then `--reps` assemblies run inside
cudaProfilerStart/Stop (use ncu --profile-from-start off).

  python profiles/profile_assembly.py --config 5 --reps 2
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2107_03285_b200 import problems as P
    if a.config == 5:
        bd = P.build_sheet_batch(2, 0, instances=range(1, 65))
        X, _ = bd.simulate(bd.p0)
        bd.load(X, bd.p0)
        eng = bd.engine
    else:
        if a.config == 3:
            prob, p0, _ = P.build_beam(0)
            x = prob._x_warm
        elif a.config == 4:
            prob, p0 = P.build_shell(201, 100)
            x = prob.simulate(p0)
        else:
            prob, p0 = P.build_sheet(a.config)
            x = prob.simulate(p0)
        prob._load(x, p0)
        eng = prob.engine
    for _ in range(3):
        eng.assemble()
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eng.assemble(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("assemble ms (L2 flushed) median %.4f" % sorted(ts)[len(ts) // 2])
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.reps):
        flush.zero_()
        eng.assemble()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()

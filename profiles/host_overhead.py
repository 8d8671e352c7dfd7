"""Is the config-2 direction host-bound?  Times one direction on the device (CUDA events)
issued (a) as in bench.py and (b) behind a 5 ms device sleep, so the host has enqueued
every launch up to the refinement's sync before the device reaches them.

  python profiles/host_overhead.py [--config 2] [--reps 20]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_2107_03285_b200.engine import sgn_solve_stages
    from paper_2107_03285_b200.problems import build_sheet
    prob, p0 = build_sheet(a.config)
    x = prob.simulate(p0)
    prob._load(x, p0)
    eng = prob.engine
    for _ in range(3):
        eng.assemble(); sgn_solve_stages(eng, None, True)
    torch.cuda.synchronize()
    out = {}
    for mode in ("eager", "presleep"):
        ts, ta, hs = [], [], []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            if mode == "presleep":
                torch.cuda._sleep(int(5e-3 * 1.9e9))
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            h0 = time.perf_counter()
            ev[0].record()
            eng.assemble()
            ev[1].record()
            h1 = time.perf_counter()
            sgn_solve_stages(eng, None, True)
            ev[2].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[2]))
            ta.append(ev[0].elapsed_time(ev[1]))
            hs.append((h1 - h0) * 1e3)
        out[mode] = (statistics.median(ts), statistics.median(ta), statistics.median(hs))
        print(f"{mode:9s} direction {out[mode][0]:.3f} ms  assemble {out[mode][1]:.4f} ms  host issue of assemble {out[mode][2]:.3f} ms")


if __name__ == "__main__":
    main()

"""Host-side breakdown of one public-API direction (config 2): load, graph replays +
refinement (incl. its sync), factor checks, solution copy-back."""
import os, sys, time, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
from paper_2107_03285_b200.engine import sgn_solve_stages
from paper_2107_03285_b200.problems import build_sheet
prob, p0 = build_sheet(2)
x = np.asarray(prob.simulate(p0)); p = np.asarray(p0)
cfg = OptimizerConfig()
for _ in range(3):
    direction_sgn(prob, x, p, cfg)
torch.cuda.synchronize()
eng = prob.engine
T = {k: [] for k in ("api", "load", "direction", "cpu")}
for _ in range(30):
    t0 = time.perf_counter(); direction_sgn(prob, x, p, cfg); T["api"].append(time.perf_counter() - t0)
for _ in range(30):
    t0 = time.perf_counter(); prob._load(x, p); t1 = time.perf_counter()
    eng.direction({}); t2 = time.perf_counter()
    sol = eng.sol[0].cpu().numpy(); t3 = time.perf_counter()
    T["load"].append(t1 - t0); T["direction"].append(t2 - t1); T["cpu"].append(t3 - t2)
print({k: round(statistics.median(v) * 1e3, 4) for k, v in T.items()}, "ms")

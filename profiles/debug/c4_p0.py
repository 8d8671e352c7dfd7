"""Config-4 refinement floor vs the initial rest shape p0 (zero / seeded random heights)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2107_03285_b200.problems import build_shell
from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
from paper_2107_03285_b200.errors import NoConvergence
prob, p0 = build_shell(201, 100)
rng = np.random.default_rng(0)
for name, p in [("zero", p0), ("U(-0.01,0.01)", rng.uniform(-0.01, 0.01, p0.size)), ("dome 0.05", None)]:
    if p is None:
        u = np.linspace(0, 1, 100)
        p = (0.05 * np.sin(np.pi * u)[:, None] * np.sin(np.pi * u)[None, :]).ravel()
    try:
        x = prob.simulate(p)
        sd = direction_sgn(prob, x, p, OptimizerConfig())
        print(name, "ok |dp|", np.linalg.norm(sd.dp), "res", sd.relative_residual, flush=True)
    except NoConvergence as e:
        print(name, "NoConvergence", e.residual, e.iterations, flush=True)
    except Exception as e:
        print(name, "error", repr(e)[:200], flush=True)

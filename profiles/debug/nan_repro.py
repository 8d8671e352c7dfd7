"""Reproduce the G_x factor+solve NaN from a dumped matrix (profiles/debug/nan_dump_gx_c1.npz)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2107_03285_b200.device import DeviceFactor, Symbolic

d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "nan_dump_gx_c1.npz"))
n = len(d["indptr"]) - 1
if os.environ.get("POISON", "0") == "1":
    junk = torch.full((1 << 28,), float("nan"), dtype=torch.float64, device="cuda")   # 2 GiB of NaN
    torch.cuda.synchronize()
    del junk
    torch.cuda.empty_cache()                 # back to the driver: our cudaMalloc may reuse the pages
sym = Symbolic(n, d["indptr"], d["indices"])
print(sym.stats())
fac = DeviceFactor(sym, 1)
vals = torch.as_tensor(d["gvals"], device="cuda")
fx = torch.as_tensor(d["fx"], device="cuda")
x = torch.empty_like(fx)
for rep in range(3):
    fac.numeric(vals, 0.0, 0.0)
    fac.solve(fx, x)
    torch.cuda.synchronize()
    xx = x.cpu().numpy()[0]
    print("rep", rep, "finite", np.isfinite(xx).all(), "nan count", int((~np.isfinite(xx)).sum()), "status", fac.status())
import scipy.sparse as sp
G = sp.csc_matrix((d["gvals"][0], d["indices"], d["indptr"]), shape=(n, n))
ref = np.linalg.solve(G.toarray(), d["fx"][0])
if np.isfinite(xx).all():
    print("rel err vs dense", np.linalg.norm(xx - ref) / np.linalg.norm(ref))
else:
    print("first non-finite positions", np.flatnonzero(~np.isfinite(xx))[:20])

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import elements as el
from paper_2107_03285_b200._lib import lib, ptr
rng = np.random.default_rng(0)
for D, code in ((2, 2), (3, 3)):
    nv = D + 1
    X = (rng.standard_normal((1, nv, D)) * 0.3 + np.eye(nv, D)[None])
    x = X + 0.05 * rng.standard_normal(X.shape)
    mu, lam, g = 3.0, 5.0, 0.7
    H, M = el.nh_second(x, X, mu, lam, g)
    conn = torch.arange(nv, dtype=torch.int32, device="cuda")
    pos = torch.as_tensor(x.ravel(), device="cuda"); rest = torch.as_tensor(X.ravel(), device="cuda")
    params = torch.as_tensor([mu, lam, g, 1.0], dtype=torch.float64, device="cuda")
    nd = nv * D
    h = torch.zeros(nd * nd, dtype=torch.float64, device="cuda"); m = torch.zeros_like(h)
    rc = lib().sgn_element_derivs(code, 1, 1, ptr(conn), ptr(pos), ptr(rest), nv * D, ptr(params), 4, ptr(h), ptr(m), None, nd * nd, 0)
    torch.cuda.synchronize()
    hg, mg = h.cpu().numpy().reshape(nd, nd), m.cpu().numpy().reshape(nd, nd)
    print(D, rc, "H err", np.abs(hg - H[0]).max(), "M err", np.abs(mg - M[0]).max())
    np.set_printoptions(precision=3, linewidth=200, suppress=True)
    if np.abs(mg - M[0]).max() > 1e-9:
        print(mg - M[0])

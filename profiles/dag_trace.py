"""Trace one persistent solve (SGN_DAG_TRACE=1) and summarise its critical path per level.

  SGN_DAG_TRACE=1 python profiles/dag_trace.py [--config 2]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/dag_trace.npz")
    a = ap.parse_args()
    os.environ["SGN_DAG_TRACE"] = "1"
    os.environ["SGN_BICG_GRAPH"] = "0"      # trace buffers are allocated lazily (not under capture)
    import torch
    from paper_2107_03285_b200._lib import lib
    from paper_2107_03285_b200.problems import build_beam, build_sheet, build_shell
    if a.config == 3:
        prob, p0, _ = build_beam(0)
    elif a.config == 4:
        prob, p0 = build_shell(201, 100)
    else:
        prob, p0 = build_sheet(a.config)
    x = prob.simulate(p0)
    prob._load(x, p0)
    eng = prob.engine
    eng.direction()
    fac = eng.kfac
    n = prob.plan.dim
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    xo = torch.empty_like(b)
    for _ in range(5):
        fac.solve(b, xo)
    torch.cuda.synchronize()
    nt = ctypes.c_int64()
    lib().sgn_debug_solve_trace(fac._h, None, 0, ctypes.byref(nt), None)
    meta = np.zeros(5 * nt.value, np.int32)
    tr = np.zeros(6 * nt.value, np.int64)
    lib().sgn_debug_solve_trace(fac._h, tr.ctypes.data_as(ctypes.c_void_p), tr.size, None,
                                meta.ctypes.data_as(ctypes.c_void_p))
    tr = tr.reshape(-1, 6)
    meta = meta.reshape(-1, 5)
    sm = (tr[:, 1].astype(np.uint64) >> np.uint64(48)).astype(np.int64)
    T = tr[:, [0, 2, 3, 4, 5]].astype(np.float64)
    base = T[:, 0].min()
    T = np.where(T > 0, T - base, np.nan) / 1e3          # us, nan = phase not reached
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    np.savez(a.out, T=T, sm=sm, meta=meta)
    kind, lvl = meta[:, 0], meta[:, 2]
    print("total span us %.2f tasks %d SMs %d" % (np.nanmax(T[:, 4]), len(T), len(set(sm.tolist()))))
    print("phase medians (us): pre = start->prefetched, wait = ->ready, comb = ready->combined (group last), fin = ->end")
    rows = []
    md = lambda v: np.nanmedian(v) if np.any(~np.isnan(v)) else float("nan")
    for ks, name in [((1, 3), "fwd"), ((2, 4), "bwd")]:
        km = np.isin(kind, ks)
        for L in sorted(set(lvl[km].tolist())):
            m = km & (lvl == L)
            t = T[m]
            rows.append(f"{name} L{L:2d} n={m.sum():5d} fat={np.sum(m & (kind > 2)):4d} start={np.nanmin(t[:, 0]):7.2f} "
                        f"ready_last={np.nanmax(t[:, 2]):7.2f} end_last={np.nanmax(t[:, 4]):7.2f} "
                        f"pre={md(t[:, 1] - t[:, 0]):5.2f} wait={md(t[:, 2] - t[:, 1]):6.2f} "
                        f"comb={md(t[:, 3] - t[:, 2]):5.2f} fin={md(t[:, 4] - t[:, 3]):5.2f} "
                        f"ready->end={md(t[:, 4] - t[:, 2]):5.2f}")
    print("\n".join(rows))


if __name__ == "__main__":
    main()

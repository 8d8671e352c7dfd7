"""Trace one persistent factorization (SGN_FDAG_TRACE=1) and summarise it.

  python profiles/fdag_trace.py [--config 2]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KIND = {0: "asm", 1: "panel", 2: "update", 3: "zpanel", 4: "diagupd", 6: "upd2", 7: "zpan2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/fdag_trace.npz")
    ap.add_argument("--which", default="kkt", choices=("kkt", "gx"), help="KKT or G_x (adjoint) factor")
    ap.add_argument("--summary", action="store_true", help="per-kind totals only")
    ap.add_argument("--ctas", type=int, default=592, help="persistent CTAs (timeline normalisation)")
    a = ap.parse_args()
    os.environ["SGN_FDAG_TRACE"] = "1"
    import torch
    from paper_2107_03285_b200._lib import lib
    from paper_2107_03285_b200.problems import build_beam, build_sheet, build_shell
    if a.config == 5:
        from paper_2107_03285_b200.problems import build_sheet_batch
        bd = build_sheet_batch(2, 0, instances=range(1, 65))
        X, _ = bd.simulate(bd.p0)
        bd.load(X, bd.p0)
        eng = bd.engine
        eng.assemble()
        from paper_2107_03285_b200.engine import sgn_solve_stages
        sgn_solve_stages(eng, None)
        fac = eng.kfac
        for _ in range(2):
            fac.numeric(eng.kvals, eng.stab.eps_x, eng.stab.eps_lambda)
        torch.cuda.synchronize()
        return summarize(a, fac)
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
    fac = eng.kfac if a.which == "kkt" else eng.gfac
    for _ in range(3):
        if a.which == "kkt":
            fac.numeric(eng.kvals, eng.stab.eps_x, eng.stab.eps_lambda)
        else:
            fac.numeric(eng.gvals, 0.0, 0.0)
    torch.cuda.synchronize()
    return summarize(a, fac)


def summarize(a, fac):
    from paper_2107_03285_b200._lib import lib
    nt = ctypes.c_int64()
    lib().sgn_debug_factor_trace(fac._h, None, 0, ctypes.byref(nt), None)
    meta = np.zeros(6 * nt.value, np.int32)
    tr = np.zeros(8 * nt.value, np.int64)
    lib().sgn_debug_factor_trace(fac._h, tr.ctypes.data_as(ctypes.c_void_p), tr.size, None,
                                 meta.ctypes.data_as(ctypes.c_void_p))
    tr = tr.reshape(-1, 8)
    meta = meta.reshape(-1, 6)
    B = int(getattr(fac, "batch", 1))
    if B > 1:                       # trace rows are task-major, instance-minor
        meta = np.repeat(meta[:len(meta) // B], B, axis=0)
    base = tr[:, 0].min()
    T = (tr[:, :3].astype(np.float64) - base) / 1e3
    M = np.where(tr[:, 4:8] > 0, (tr[:, 4:8].astype(np.float64) - base) / 1e3, np.nan)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    np.savez(a.out, T=T, M=M, sm=tr[:, 3], meta=meta)
    kind, step, front, lvl = meta[:, 0], meta[:, 1], meta[:, 2], meta[:, 3]
    print("span us %.1f tasks %d" % (T[:, 2].max(), len(T)))
    try:
        npiv = np.asarray(fac.sym.fronts()["npiv"])
        zp = (kind == 3) & (meta[:, 4] < (npiv[front] + 31) // 32)
        zs = (kind == 3) & ~zp
        for nm, m in (("z(piv tiles)", zp), ("z(struct tiles)", zs)):
            print(f"{nm:16s} n={m.sum():7d} busy_sum_us={np.sum(T[m, 2] - T[m, 1]):9.1f}")
    except Exception as exc:  # noqa: BLE001
        print("z split unavailable:", exc)
    for k in KIND:
        m = kind == k
        if m.any():
            print(f"{KIND[k]:7s} n={m.sum():6d} busy_med={np.median(T[m, 2] - T[m, 1]):6.2f} "
                  f"wait_med={np.median(T[m, 1] - T[m, 0]):6.2f} busy_sum_us={np.sum(T[m, 2] - T[m, 1]):9.1f} "
                  f"wait_sum_us={np.sum(T[m, 1] - T[m, 0]):9.1f}")
    # CTA occupancy over time: busy / waiting / idle (between tasks) fractions per 5% of the span
    span = T[:, 2].max()
    sm = a_sm = None
    nb = 20
    edges = np.linspace(0, span, nb + 1)
    def frac(t0, t1):
        out = np.zeros(nb)
        for i in range(nb):
            lo, hi = edges[i], edges[i + 1]
            out[i] = np.clip(np.minimum(t1, hi) - np.maximum(t0, lo), 0, None).sum()
        return out
    nct = len(set(zip(tr_sm.tolist()))) if False else None
    busy, wait = frac(T[:, 1], T[:, 2]), frac(T[:, 0], T[:, 1])
    cap = (edges[1] - edges[0]) * a.ctas
    print("timeline (per 5% of span): busy% / wait%")
    print(" ".join(f"{100 * b / cap:3.0f}/{100 * w / cap:2.0f}" for b, w in zip(busy, wait)))
    if a.summary:
        return
    print("per level: first ready / last end (us)")
    for L in sorted(set(lvl.tolist())):
        m = (lvl == L) & (kind != 3)
        z = (lvl == L) & (kind == 3)
        print(f"L{L:2d} n={m.sum():6d} ready={T[m, 1].min():8.1f} end={T[m, 2].max():8.1f} "
              f"panels={np.sum(m & (kind == 1)):5d} steps={step[m].max() + 1:3d}"
              + (f" | z n={z.sum():5d} {T[z, 1].min():8.1f}-{T[z, 2].max():8.1f}" if z.any() else ""))
    # critical chain of the top front: per step, panel end and look-ahead update end
    top = front[np.argmax(lvl)]
    m = front == top
    print("top front", top, "steps")
    for s in range(step[m & (kind == 1)].max() + 1):
        pm = m & (kind == 1) & (step == s)
        um = m & (kind == 2) & (step == s)
        print(f"  k={s:3d} panel ready {T[pm, 1].min():8.1f} end {T[pm, 2].max():8.1f} busy {np.max(T[pm, 2] - T[pm, 1]):5.2f}"
              + (f" | upd end {T[um, 2].max():8.1f} busy_med {np.median(T[um, 2] - T[um, 1]):5.2f}" if um.any() else ""))


if __name__ == "__main__":
    main()

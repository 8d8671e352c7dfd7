"""Config-5 (64 instances, one device batch) phase times: assemble / KKT factor / adjoint / refined solve."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2107_03285_b200.engine import sgn_solve_stages
    from paper_2107_03285_b200.problems import build_sheet_batch
    bd = build_sheet_batch(2, 0, instances=range(1, 65))
    X, _ = bd.simulate(bd.p0)
    bd.load(X, bd.p0)
    eng = bd.engine
    for _ in range(2):
        eng.assemble(); sgn_solve_stages(eng, None)
    torch.cuda.synchronize()
    rec = []
    for _ in range(5):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(); eng.assemble(); ev[1].record()
        sgn_solve_stages(eng, None, True, ev[2:])
        torch.cuda.synchronize()
        rec.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
    med = [statistics.median(r[i] for r in rec) for i in range(4)]
    print("c5 ms: assemble %.3f factor %.3f adjoint %.3f solve %.3f total %.3f" % (*med, sum(med)))
    st = eng.kfac.stats() if hasattr(eng.kfac, "stats") else None
    t = torch.cuda.Event(enable_timing=True); t2 = torch.cuda.Event(enable_timing=True)
    b = torch.randn(eng.batch, bd.plan.dim, dtype=torch.float64, device="cuda"); xo = torch.empty_like(b)
    st_ = torch.cuda.current_stream().cuda_stream
    for _ in range(2): eng.kfac.solve(b, xo, stream=st_)
    t.record()
    for _ in range(10): eng.kfac.solve(b, xo, stream=st_)
    t2.record(); torch.cuda.synchronize()
    print("batched solve (64 rhs) %.3f ms" % (t.elapsed_time(t2) / 10))


if __name__ == "__main__":
    main()

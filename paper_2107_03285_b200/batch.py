"""Instance partitioning and the end-of-run gather for batched SGN (BASELINE config 5).

Independent design instances shard with no data-path collective: rank r of W owns a
contiguous instance range; every rank runs its instances as one device batch; a single
all-gather at the end collects per-instance results (dp, objective trajectory, status) on
every rank (NCCL over NVLink on the GPU box, gloo in the CPU tests).  No reduction is
involved, so gathered results are bitwise independent of W.
"""
from __future__ import annotations

import numpy as np


def partition(n_total: int, world: int, rank: int) -> range:
    """Contiguous, balanced instance range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(int(n_total), int(world))
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_instances(local: np.ndarray, n_total: int, world: int, rank: int, device=None) -> np.ndarray:
    """All-gather per-instance rows (local: [n_local, m]) into [n_total, m] on every rank."""
    import torch
    import torch.distributed as dist
    local = np.ascontiguousarray(local, dtype=np.float64)
    m = local.shape[1] if local.ndim == 2 else 1
    local = local.reshape(-1, m)
    cap = max(len(partition(n_total, world, r)) for r in range(world))
    buf = np.zeros((cap, m))
    buf[:local.shape[0]] = local
    t = torch.as_tensor(buf, device=device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    rows = []
    for r in range(world):
        k = len(partition(n_total, world, r))
        rows.append(outs[r].cpu().numpy()[:k])
    return np.concatenate(rows, axis=0)


class BatchRun:
    """Per-instance outcome of ``minimize_batched`` (the batched analogue of the reference's
    OptimizerRun, optimize.py:101-137): f / gradient-norm / step-length trajectories
    ([B, max_iterations + 1], NaN after an instance terminated), termination strings, the
    final parameters and the number of SGN directions each instance actually used."""

    def __init__(self, f, grad_norm, alpha, rel_res, termination, p, directions, timings):
        self.f, self.grad_norm, self.alpha, self.rel_res = f, grad_norm, alpha, rel_res
        self.termination, self.p, self.directions, self.timings = termination, p, directions, timings

    def trajectory(self, b: int) -> np.ndarray:
        f = self.f[b]
        return f[np.isfinite(f)]

    def pack(self) -> np.ndarray:
        """One float64 row per instance for the end-of-run gather: [f(it+1) | |g|(it+1) |
        alpha(it+1) | directions | termination code]."""
        codes = np.array([TERMINATIONS.index(t) for t in self.termination], dtype=np.float64)
        return np.concatenate([self.f, self.grad_norm, self.alpha, self.directions[:, None].astype(np.float64),
                               codes[:, None]], axis=1)

    @staticmethod
    def unpack_row(row: np.ndarray, iters: int) -> dict:
        n = iters + 1
        return dict(f=row[:n], grad_norm=row[n:2 * n], alpha=row[2 * n:3 * n], directions=int(row[3 * n]),
                    termination=TERMINATIONS[int(row[3 * n + 1])])


class _Compactor:
    """Forward solves of a few pending instances in a smaller engine.

    A batched Newton iteration launches every kernel over the whole batch, so a line search
    with one straggler instance would pay for all B.  The pending instances' rows (material
    parameters, p, x) are copied into a simulate-only engine of the next power-of-two batch
    (its KKT factor is never allocated), solved there and copied back.  Every kernel treats
    instance rows independently, so the result is bitwise the one the full batch gives."""

    def __init__(self, eng):
        self.eng, self.pool = eng, {}

    def simulate(self, tol, run):
        from .engine import DeviceEngine
        from .errors import ForwardSimFailure
        eng = self.eng
        torch = eng.torch
        B = eng.batch
        idx = np.flatnonzero(run)
        k = int(idx.size)
        size = 1 << max(0, (k - 1).bit_length())
        if size * 2 > B:                                  # not worth compacting
            try:
                return eng.simulate(tol, active=run)
            except ForwardSimFailure:
                return np.full(B, -1)
            finally:
                self.last_iters = getattr(eng, "newton_iters", 0)
        sub = self.pool.get(size)
        if sub is None:
            params = [gp[:1].repeat(size, 1).cpu().numpy() for gp in eng.gparams]
            sub = DeviceEngine(eng.plan, params if len(params) > 1 else params[0],
                               eng.tvals[:1].repeat(size, 1).cpu().numpy(), batch=size, stab=eng.stab)
            self.pool[size] = sub
        rows = torch.as_tensor(np.r_[idx, np.full(size - k, idx[0])], device="cuda")
        for dst, src in zip(sub.gparams, eng.gparams):
            dst.copy_(src.index_select(0, rows))
        sub.p.copy_(eng.p.index_select(0, rows))
        sub.x.copy_(eng.x.index_select(0, rows))
        try:
            st = sub.simulate(tol, active=np.arange(size) < k)
        except ForwardSimFailure:                          # a batch of one raises instead
            st = np.full(size, -1)
        self.last_iters = getattr(sub, "newton_iters", 0)
        eng.x.index_copy_(0, rows[:k], sub.x[:k])
        status = np.ones(B, dtype=np.int64)
        status[idx] = st[:k]
        return status


TERMINATIONS = ("max_iterations", "gradient_tolerance", "stationary", "no_descent", "line_search_failure",
                "forward_failure", "direction_no_convergence")


def minimize_batched(bd, p0, cfg, max_iterations: int | None = None) -> BatchRun:
    """SGN outer loops of B independent instances on one device batch.

    Each instance follows the reference minimize (optimize.py:353-420) with its own Armijo
    backtracking (_line_search, optimize.py:468-488) and its own termination; the
    instances share every launch: one batched SGN direction per iteration, the pending
    trial points of all instances' line searches forward-solved as ONE masked batched Newton
    (engine.simulate(active=...)), one batched adjoint gradient after the accepted steps.
    p, x, g, dp stay on the device; only per-instance scalars (f, slopes, norms: B doubles)
    reach the host for the Armijo and termination decisions.  Instances never read one
    another's data, so an instance's trajectory is bitwise the same in any batch.
    """
    import time
    from . import _lib
    from ._lib import check, lib, ptr
    from .engine import adjoint_gradient_stage
    from .errors import ForwardSimFailure, NoConvergence
    eng = bd.engine
    torch = eng.torch
    nvtx = torch.cuda.nvtx
    B, n_x, n_p = bd.B, bd.n_x, bd.n_p
    iters = cfg.max_iterations if max_iterations is None else int(max_iterations)
    eng.stab = cfg.stabilization
    st = _lib.stream_handle()
    dev = dict(dtype=torch.float64, device="cuda")
    p_cur = torch.empty(B, n_p, **dev)
    x_cur = torch.empty(B, n_x, **dev)
    g = torch.empty(B, n_p, **dev)
    dp = torch.empty(B, n_p, **dev)
    step = torch.empty(B, n_p, **dev)
    red = torch.empty(B, **dev)
    neg1 = torch.full((B,), -1.0, **dev)

    def dot(a, b):
        check(lib().sgn_reduce(1, a.shape[1], B, ptr(a), ptr(b), a.shape[1], ptr(red), st))
        return red.cpu().numpy().copy()

    def mask(m):
        return torch.as_tensor(np.asarray(m, dtype=np.int32), device="cuda")

    def gradient_into(sel):
        """g[sel] <- adjoint gradient at (eng.x, eng.p) (batched; other rows untouched)."""
        eng.assemble()
        adjoint_gradient_stage(eng)
        check(lib().sgn_masked_copy(n_p, B, ptr(mask(sel)), ptr(eng.grad), ptr(g), n_p, st))

    compactor = getattr(bd, "_compactor", None) or _Compactor(eng)
    bd._compactor = compactor
    t0 = time.perf_counter()
    timings = dict(direction_s=0.0, line_search_s=0.0, gradient_s=0.0)
    term = ["max_iterations"] * B
    active = np.ones(B, bool)
    # initial forward solve (minimize: optimize.py:364-368), from the rest shape
    eng.load(x=bd.rest_start(), p=np.asarray(p0, dtype=np.float64).reshape(B, n_p))
    status = eng.simulate(bd.tol)
    for b in np.flatnonzero(status != 1):
        term[b] = "forward_failure"
    active &= status == 1
    p_cur.copy_(eng.p)
    x_cur.copy_(eng.x)
    f = eng.objective().cpu().numpy().copy()
    gradient_into(np.ones(B, bool))
    F = np.full((B, iters + 1), np.nan)
    GN = np.full((B, iters + 1), np.nan)
    AL = np.full((B, iters + 1), np.nan)
    RR = np.full((B, iters + 1), np.nan)
    ndir = np.zeros(B, dtype=np.int64)
    gn = np.sqrt(dot(g, g))
    F[:, 0], GN[:, 0], AL[:, 0] = f, gn, 0.0
    for it in range(1, iters + 1):
        done = active & (gn <= cfg.gradient_tolerance)
        for b in np.flatnonzero(done):
            term[b] = "gradient_tolerance"
        active &= ~done
        if not active.any():
            break
        # one batched SGN direction at every instance's (x, p)
        nvtx.range_push("sgn.batch.direction")
        td = time.perf_counter()
        eng.x.copy_(x_cur)
        eng.p.copy_(p_cur)
        try:
            res, _ = eng.direction()
        except NoConvergence as exc:
            res = np.asarray(exc.instance_residuals)
        # the reference minimize does not catch a direction's NoConvergence (optimize.py:389,
        # linear_solvers.py:168): that instance's run ends there
        failed = active & ~(res <= eng.stab.refine_tolerance)
        for b in np.flatnonzero(failed):
            term[b] = "direction_no_convergence"
        dp.copy_(eng.sol[:, n_x:n_x + n_p])
        ndir += active
        active &= ~failed
        timings["direction_s"] += time.perf_counter() - td
        nvtx.range_pop()
        dpn, gdp = dot(dp, dp), dot(g, dp)
        for b in np.flatnonzero(active & (dpn == 0.0)):
            term[b] = "stationary"
        active &= dpn != 0.0
        for b in np.flatnonzero(active & (gdp >= 0.0)):
            term[b] = "no_descent"
        active &= gdp < 0.0
        if not active.any():
            break
        # per-instance Armijo backtracking; all pending trial points in one masked batch
        nvtx.range_push("sgn.batch.line_search")
        tl = time.perf_counter()
        alpha = np.ones(B)
        pending = active.copy()
        acc_alpha = np.zeros(B)
        for _ in range(cfg.max_backtracks + 1):
            if not pending.any():
                break
            a_d = torch.as_tensor(alpha, **dev)
            check(lib().sgn_axpy(n_p, B, ptr(a_d), ptr(dp), ptr(p_cur), ptr(eng.p), n_p, st))   # p_try
            check(lib().sgn_axpy(n_p, B, ptr(neg1), ptr(p_cur), ptr(eng.p), ptr(step), n_p, st))
            slope = dot(g, step)                                     # g . (p_try - p)
            run = pending & (slope < 0.0)
            if run.any():
                eng.x.copy_(x_cur)                                   # warm start x_init = x
                t_sim = time.perf_counter()
                stat = compactor.simulate(bd.tol, run)
                timings.setdefault("trials", []).append(
                    (it, int(run.sum()), int(compactor.last_iters), int((stat == 1).sum()),
                     time.perf_counter() - t_sim))
                ok = run & (stat == 1)
                ft = eng.objective().cpu().numpy()
                acc = ok & np.isfinite(ft) & (ft <= f + cfg.armijo_c1 * slope)
                if acc.any():
                    m = mask(acc)
                    check(lib().sgn_masked_copy(n_p, B, ptr(m), ptr(eng.p), ptr(p_cur), n_p, st))
                    check(lib().sgn_masked_copy(n_x, B, ptr(m), ptr(eng.x), ptr(x_cur), n_x, st))
                    f = np.where(acc, ft, f)
                    acc_alpha = np.where(acc, alpha, acc_alpha)
                    pending &= ~acc
            alpha = np.where(pending, alpha * cfg.backtrack_factor, alpha)
        timings["line_search_s"] += time.perf_counter() - tl
        nvtx.range_pop()
        for b in np.flatnonzero(pending):
            term[b] = "line_search_failure"
        accepted = active & ~pending
        active = accepted
        if not accepted.any():
            break
        tg = time.perf_counter()
        eng.x.copy_(x_cur)
        eng.p.copy_(p_cur)
        gradient_into(accepted)
        timings["gradient_s"] += time.perf_counter() - tg
        gn_new = np.sqrt(dot(g, g))
        gn = np.where(accepted, gn_new, gn)
        F[accepted, it] = f[accepted]
        GN[accepted, it] = gn[accepted]
        AL[accepted, it] = acc_alpha[accepted]
        RR[accepted, it] = np.asarray(res)[accepted]
    timings["total_s"] = time.perf_counter() - t0
    return BatchRun(F, GN, AL, RR, term, p_cur.cpu().numpy(), ndir, timings)

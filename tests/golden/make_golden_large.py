"""Golden fixtures at BASELINE size, generated with the REAL reference solver path.

    python tests/golden/make_golden_large.py c2 | c3 | c4 | c5   (run in the build container)

The oracle problem classes (oracle/configs.py, oracle/shell.py) are driven through the
unmodified reference `sgnopt` (copied from /root/reference/pkg/src to /tmp): equilibrium x,
the adjoint gradient (sensitivity.adjoint_gradient), direction_sgn (dp, relative residual,
refinement outcome) and, where it fits the build container's time, the reference
`minimize` objective trajectory.  The GPU tests read these files; /root/reference is never
needed at run time.

* large_c2.npz -- config 2 (100x100 sheet): direction at p0 + 20-iteration SGN trajectory
* large_c3.npz -- config 3 (tet beam): direction at p0 + 20-iteration SGN trajectory
* large_c4.npz -- config 4 (201x201 shell): direction at p0 (+ a 2-iteration trajectory)
* large_c5.npz -- config 5: instances 1, 2, 3 of the batch, 20-iteration SGN trajectories
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)
from make_golden import import_reference  # noqa: E402


def _wrap_simulate(prob):
    from oracle.sgn_cpu import OracleNoConvergence
    from sgnopt.errors import ForwardSimFailure
    inner = prob.simulate

    def simulate(p, x_init=None):       # oracle failures -> the reference's convention
        try:
            return inner(p, x_init=x_init)
        except OracleNoConvergence as exc:
            raise ForwardSimFailure(str(exc)) from exc
    prob.simulate = simulate
    return prob


def direction_and_trajectory(prob, p0, iters):
    from sgnopt.errors import NoConvergence
    from sgnopt.optimize import OptimizerConfig, direction_sgn, minimize
    from sgnopt.sensitivity import adjoint_gradient
    t0 = time.time()
    x = prob.simulate(p0)
    out = dict(p=np.asarray(p0, np.float64), x=x, f0=prob.objective(x, p0), n_x=prob.n_x, n_p=prob.n_p)
    out["grad"] = adjoint_gradient(prob, x, p0)
    cfg = OptimizerConfig(method="sgn", max_iterations=max(iters, 1), gradient_tolerance=1e-12)
    try:
        sd = direction_sgn(prob, x, p0, cfg)
        out.update(dp=sd.dp, rel_res=sd.relative_residual, converged=True)
    except NoConvergence as exc:           # record the reference's NoConvergence(best)
        n_x, n_p = prob.n_x, prob.n_p
        out.update(dp=np.asarray(exc.best)[n_x:n_x + n_p], rel_res=exc.residual, converged=False)
    print(f"  direction: |dp| {np.linalg.norm(out['dp']):.6e} res {out['rel_res']:.3e} "
          f"converged {out['converged']} ({time.time() - t0:.0f} s)", flush=True)
    if iters:
        # the reference minimize does not catch NoConvergence from a direction's refinement
        # (optimize.py:389 -> linear_solvers.py:168): it raises.  Count the adjoint
        # evaluations (1 initial + 2 per completed iteration + 1 in the failing direction)
        # on our own problem object, then rerun to the last completed iteration and record
        # the termination as "direction_no_convergence".
        calls = [0]
        inner_fx = prob.objective_grad_x

        def counted(x_, p_):
            calls[0] += 1
            return inner_fx(x_, p_)
        prob.objective_grad_x = counted
        if hasattr(prob, "_x_warm"):
            prob._x_warm = None
        term = None
        try:
            run = minimize(prob, np.asarray(p0, np.float64).copy(), cfg)
        except NoConvergence as exc:
            done = calls[0] // 2 - 1
            print(f"  reference minimize raised at iteration {done + 1}: {exc}", flush=True)
            if hasattr(prob, "_x_warm"):
                prob._x_warm = None
            cfg2 = OptimizerConfig(method="sgn", max_iterations=done, gradient_tolerance=1e-12)
            run = minimize(prob, np.asarray(p0, np.float64).copy(), cfg2)
            term = "direction_no_convergence"
            out["traj_fail_residual"] = float(exc.residual)
        prob.objective_grad_x = inner_fx
        out.update(traj_f=run.f_values(), traj_g=run.grad_norms(),
                   traj_alpha=np.array([r.step_length for r in run.records]),
                   traj_term=np.array(term or run.termination), traj_p=run.p)
        print(f"  trajectory {run.f_values()} {term or run.termination} ({time.time() - t0:.0f} s)", flush=True)
    return out


def main(which):
    import_reference()
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    if which == "c2":
        from oracle.configs import oracle_sheet
        prob, p0 = oracle_sheet(2, seed=0)
        out = direction_and_trajectory(_wrap_simulate(prob), p0, 20)
    elif which == "c3":
        from oracle.configs import oracle_beam
        prob, p0 = oracle_beam(0)
        sag = prob.simulate(p0)                        # the targets lift the sagged tip face
        prob, p0 = oracle_beam(0, targets=sag[prob.target_dofs])
        out = direction_and_trajectory(_wrap_simulate(prob), p0, 20)
    elif which == "c4":
        from oracle.shell import ShellProblem, shell_spec
        spec = shell_spec(201, 100)
        prob = ShellProblem(spec)
        out = direction_and_trajectory(_wrap_simulate(prob), spec["p0"], int(os.environ.get("C4_ITERS", "2")))
    elif which == "c5":
        from oracle.configs import oracle_sheet
        out = {}
        for inst in (1, 2, 3):
            prob, p0 = oracle_sheet(2, seed=0, instance=inst)
            o = direction_and_trajectory(_wrap_simulate(prob), p0, 20)
            out.update({f"i{inst}_{k}": v for k, v in o.items()})
    else:
        raise SystemExit(f"unknown target {which}")
    np.savez_compressed(os.path.join(HERE, f"large_{which}.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1])

"""Config-5 sharding: balanced partitions and a world-size-2 gloo all-gather (CPU)."""
import os
import socket

import numpy as np
import pytest

from paper_2107_03285_b200.batch import gather_instances, partition


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 4), (64, 8), (10, 3), (3, 4)])
def test_partition_is_balanced_cover(n, world):
    ranges = [partition(n, world, r) for r in range(world)]
    flat = [i for rg in ranges for i in rg]
    assert flat == list(range(n))
    sizes = [len(rg) for rg in ranges]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = partition(n_total, world, rank)
    # deterministic per-instance "results": depends only on the instance id
    local = np.stack([np.sin(np.arange(5) * (i + 1)) for i in rows]) if len(rows) else np.zeros((0, 5))
    full = gather_instances(local, n_total, world, rank)
    out_q.put((rank, full))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [64, 7])
def test_gloo_world2_gather_matches_single_process(n_total):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    expect = np.stack([np.sin(np.arange(5) * (i + 1)) for i in range(n_total)])
    for r in range(2):
        np.testing.assert_array_equal(res[r], expect)     # bitwise: no reduction involved


def _pack_oracle_runs(instances, iters):
    """Rows in the BatchRun.pack() layout from the oracle's minimize (real SGN outputs)."""
    from oracle import sgn_cpu
    from oracle.configs import oracle_sheet
    from paper_2107_03285_b200.batch import TERMINATIONS
    rows = []
    for k in instances:
        prob, p0 = oracle_sheet(1, 0, k)
        run = sgn_cpu.minimize_sgn(prob, p0, max_iterations=iters, gradient_tolerance=1e-12)
        f = np.full(iters + 1, np.nan)
        g = np.full(iters + 1, np.nan)
        a = np.full(iters + 1, np.nan)
        n = len(run["f"])
        f[:n], g[:n], a[:n] = run["f"], run["grad_norm"], run["alpha"]
        extra = run["termination"] in ("line_search_failure", "no_descent", "stationary", "direction_no_convergence")
        rows.append(np.concatenate([f, g, a, [n - 1 + extra, TERMINATIONS.index(run["termination"])]]))
    return np.array(rows).reshape(len(instances), 3 * (iters + 1) + 2)


def _sgn_worker(rank, world, port, n_total, iters, out_q):
    import torch.distributed as dist
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = partition(n_total, world, rank)
    local = _pack_oracle_runs([1 + i for i in rows], iters)
    full = gather_instances(local, n_total, world, rank)
    out_q.put((rank, full))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gathers_per_instance_sgn_trajectories():
    """Config-5 path on CPU: each rank runs its instances' SGN loops (here the oracle's, on
    config-1 sheets), packs trajectory / termination / direction-count rows and all-gathers
    them; every rank ends with the single-process result, bitwise."""
    import multiprocessing as mp
    from paper_2107_03285_b200.batch import BatchRun
    n_total, iters = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sgn_worker, args=(r, 2, port, n_total, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    expect = _pack_oracle_runs(range(1, n_total + 1), iters)
    for r in range(2):
        np.testing.assert_array_equal(res[r], expect)
    row = BatchRun.unpack_row(expect[0], iters)
    assert row["termination"] in ("max_iterations", "gradient_tolerance", "line_search_failure")
    assert np.isfinite(row["f"][0]) and row["directions"] >= 1

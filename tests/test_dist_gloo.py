"""S1 across processes (DistRunner) on CPU with the gloo backend, world size 2:
every rank evaluates its round-robin share, the all-gather returns the full
list in task order, and the optimizer takes bitwise-identical decisions on all
ranks and matches the serial run (reference determinism, tests/test_sched.py:65-70)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _QuadEvaluator:
    """Stands in for ObjectiveEvaluator: f(theta) = log-posterior-like concave quadratic."""

    device = torch.device("cpu")

    def __init__(self):
        rng = np.random.default_rng(0)
        m = rng.normal(size=(4, 4))
        self.h = m @ m.T + 4 * np.eye(4)
        self.c = rng.normal(size=4)

    def objective(self, theta):
        d = np.asarray(theta) - self.c
        return float(-0.5 * d @ self.h @ d)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_06938_b200 import inla, sched

        ev = _QuadEvaluator()
        runner = sched.DistRunner(ev)
        pts = [np.full(4, 0.1 * k) for k in range(9)]
        vals = runner.evaluate_points(pts)
        res = inla.minimize(ev, np.zeros(4), gtol=1e-8, ftol=1e-14, max_iter=50, runner=runner)
        # a failing task raises the same (lowest) index on every rank
        def bad(k):
            def t():
                if k in (3, 6):
                    raise ValueError("boom")
                return float(k)
            return t
        try:
            runner([bad(k) for k in range(8)])
            err = None
        except sched.TaskError as e:
            err = e.task_index
        out[rank] = (vals, res.theta.tolist(), res.f, res.iterations, err)
    finally:
        dist.destroy_process_group()


def test_dist_runner_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    from paper_2507_06938_b200 import inla

    ev = _QuadEvaluator()
    serial_vals = [-ev.objective(np.full(4, 0.1 * k)) for k in range(9)]
    serial = inla.minimize(ev, np.zeros(4), gtol=1e-8, ftol=1e-14, max_iter=50)
    for r in range(2):
        vals, theta, f, its, err = out[r]
        assert err == 3
        assert vals == serial_vals  # index order, minimized sign, bitwise
        assert theta == serial.theta.tolist() and f == serial.f and its == serial.iterations
    np.testing.assert_allclose(out[0][1], np.linalg.solve(ev.h, ev.h @ ev.c), atol=1e-6)

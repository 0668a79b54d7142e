"""S3 over NCCL: one partition per process, each rank holding only its own
block rows (bta_dist.BTARows); Schur pieces, reduced right-hand sides,
separator solutions and inverse seeds exchanged point-to-point, reduced
system on rank 0.  logdet, solve and selected inverse must match the
sequential oracle (reference criterion 2, tests/test_acceptance.py:103-163:
1e-9 logdet, 1e-9 solve, 1e-8 selected inverse), and a non-SPD pivot must
raise the same FactorizationError on every rank."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, case, bad_block):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from oracle import bta_np
        from paper_2507_06938_b200 import bta, bta_dist

        n, b, a, lb, k = case
        plan = bta_dist.plan_partitions(n, world, lb)
        rng = np.random.default_rng(n + b)
        data = bta_np.random_spd_bta(rng, n, b, a)
        rhs = rng.normal(size=(n * b + a, k))
        if bad_block is not None:
            d, _, _, _ = bta_np.views(data, n, b, a)
            d[bad_block] = -np.eye(b)
        # each rank keeps only its own block rows (tip on rank 0)
        m = bta.BTAMatrix(n, b, a, data)
        rows = bta_dist.local_rows(m, plan, rank, device=dev)
        del m
        try:
            f = bta_dist.d_factorize_nccl(rows, plan)
        except bta.FactorizationError as e:
            out[rank] = ("error", e.block_index, e.partition)
            return
        t0, t1 = rows.t0, rows.t1
        tip = torch.from_numpy(rhs[n * b :]).to(dev) if rank == 0 else None
        xr, xt = bta_dist.d_solve_nccl(f, torch.from_numpy(rhs[t0 * b : t1 * b]).to(dev), tip)
        inv = bta_dist.d_selected_invert_nccl(f)
        out[rank] = ("ok", bta_dist.d_logdet(f), t0, t1, xr.cpu().numpy(), xt.cpu().numpy(),
                     inv.diag.cpu().numpy(), inv.lower.cpu().numpy(), inv.arrow.cpu().numpy(),
                     inv.tip.cpu().numpy() if inv.tip is not None else None)
    finally:
        dist.destroy_process_group()


def _run(world, case, bad_block=None):
    import torch.multiprocessing as mp

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, case, bad_block), nprocs=world, join=True)
    return dict(out)


CASES = [(10, 130, 3, 1.0, 1), (12, 64, 0, 1.6, 2), (13, 70, 2, 1.0, 3), (9, 257, 4, 1.6, 1)]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("case", CASES)
def test_nccl_partitioned_solver(cuda, case):
    _check(2, case)


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs four GPUs")
def test_nccl_partitioned_solver_4(cuda):
    _check(4, (16, 100, 5, 1.6, 2))


def _check(world, case):
    from oracle import bta_np

    n, b, a, _, k = case
    out = _run(world, case)
    rng = np.random.default_rng(n + b)
    ref = bta_np.random_spd_bta(rng, n, b, a)
    rhs = rng.normal(size=(n * b + a, k))
    has = bta_np.factorize(ref, n, b, a)
    want_ld = bta_np.logdet(ref, n, b, a)
    want_x = bta_np.solve(ref, n, b, a, has, rhs)
    inv = bta_np.selected_invert(ref, n, b, a, has)
    Xd, Xl, Xa, Xt = bta_np.views(inv, n, b, a)
    for r in range(world):
        status, ld, t0, t1, xr, xt, dg, lw, ar, tp = out[r]
        assert status == "ok"
        np.testing.assert_allclose(ld, want_ld, rtol=1e-9)
        np.testing.assert_allclose(xr, want_x[t0 * b : t1 * b], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(xt, want_x[n * b :], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(dg, Xd[t0:t1], rtol=1e-8, atol=1e-11)
        lo = max(t0, 1)
        np.testing.assert_allclose(lw[lo - t0 :], Xl[lo - 1 : t1 - 1], rtol=1e-8, atol=1e-11)
        if a:
            np.testing.assert_allclose(ar, Xa[t0:t1], rtol=1e-8, atol=1e-11)
        if r == 0 and a:
            np.testing.assert_allclose(tp, Xt, rtol=1e-8, atol=1e-11)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_nccl_indefinite_raises_on_every_rank(cuda):
    # plan_partitions(12, 2) = (0, 6, 12): block 8 is in partition 1's
    # interior, block 6 is its left separator (reduced system)
    out = _run(2, (12, 20, 2, 1.0, 1), bad_block=8)
    assert [out[r] for r in range(2)] == [("error", 8, 1)] * 2
    out = _run(2, (12, 20, 2, 1.0, 1), bad_block=6)
    assert [out[r] for r in range(2)] == [("error", 6, -1)] * 2

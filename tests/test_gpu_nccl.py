"""S3 over NCCL: one partition per process (world size 2), chains and Schur
pieces exchanged point-to-point, reduced system on rank 0; the log-determinant
must match the sequential oracle (reference criterion 2, 1e-9)."""

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


def _worker(rank, world, port, out, case):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from oracle import bta_np
        from paper_2507_06938_b200 import bta, bta_dist

        n, b, a, lb = case
        plan = bta_dist.plan_partitions(n, world, lb)
        m = None
        if rank == 0:
            rng = np.random.default_rng(n + b)
            m = bta.BTAMatrix(n, b, a, bta_np.random_spd_bta(rng, n, b, a))
        ld, _ = bta_dist.d_factorize_nccl(m, plan)
        out[rank] = ld
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("case", [(10, 130, 3, 1.0), (12, 64, 0, 1.6)])
def test_nccl_partitioned_logdet(cuda, case):
    import torch.multiprocessing as mp

    from oracle import bta_np

    n, b, a, _ = case
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out, case), nprocs=2, join=True)
    rng = np.random.default_rng(n + b)
    ref = bta_np.random_spd_bta(rng, n, b, a)
    bta_np.factorize(ref, n, b, a)
    want = bta_np.logdet(ref, n, b, a)
    for r in range(2):
        np.testing.assert_allclose(out[r], want, rtol=1e-9)

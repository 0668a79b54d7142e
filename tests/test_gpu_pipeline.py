"""Pipelined host <-> device I/O (stbta_upload_blocks / stbta_pobtaf_ready /
stbta_pobtasi_stream_out): the overlapped path must give bit-identical
factors, log-determinants and selected inverses to the plain device path
(which test_gpu_solver.py checks against the oracle and the reference
goldens)."""
import numpy as np
import pytest
import torch

from paper_2507_06938_b200 import _lib, bta

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b,a", [(6, 256, 6), (4, 130, 0), (3, 129, 3), (2, 384, 130)])
def test_pipelined_upload_factor_selinv_bitwise(n, b, a):
    lib = _lib.load()
    assert lib.stbta_stream_memops_supported() == 1
    rng = np.random.default_rng(7 + n + b + a)
    ref = bta.random_spd_bta(rng, n, b, a)
    host = torch.from_numpy(ref.numpy().copy()).pin_memory()

    m1 = bta.BTAMatrix(n, b, a, host)            # chunked upload on a side stream
    assert m1._upload is not None
    f1 = bta.factorize(m1, use_arrow=a > 0)       # task graph polls the per-block flags
    m2 = bta.BTAMatrix(n, b, a, host.cuda())
    f2 = bta.factorize(m2, use_arrow=a > 0)
    assert torch.equal(m1.data, m2.data)
    assert bta.logdet(f1) == bta.logdet(f2)

    out = torch.empty(host.numel(), dtype=torch.float64).pin_memory()
    out.fill_(np.nan)
    i1 = bta.selected_invert(f1, out=out)         # streamed back block by block
    assert i1._host_copy is not None
    h1 = i1.numpy(out=out)
    i2 = bta.selected_invert(f2)
    assert np.array_equal(h1, i2.numpy())
    assert torch.equal(i1.data, i2.data)


def test_pipelined_solve_and_views_wait_for_upload():
    rng = np.random.default_rng(3)
    n, b, a = 5, 200, 4
    ref = bta.random_spd_bta(rng, n, b, a)
    host = torch.from_numpy(ref.numpy().copy()).pin_memory()
    m = bta.BTAMatrix(n, b, a, host)
    # a non-task-graph consumer (the views) waits for the upload
    assert torch.equal(m.tip.cpu(), ref.tip.cpu())
    assert torch.equal(m.diag[n - 1].cpu(), ref.diag[n - 1].cpu())
    f = bta.factorize(m, use_arrow=True)
    rhs = np.random.default_rng(4).standard_normal(n * b + a)
    x = bta.solve(f, rhs)
    fr = bta.factorize(ref, use_arrow=True)
    assert np.array_equal(x, bta.solve(fr, rhs))

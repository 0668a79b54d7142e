"""Parity of the time-partitioned solver (d_factorize / d_logdet / d_solve /
d_selected_invert) with the reference golden vectors and with the sequential
device solver (the reference's criterion 2, tests/test_acceptance.py:103-163:
1e-9 logdet, 1e-9 solve, 1e-8 selected inverse)."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import bta_np

pytestmark = pytest.mark.gpu


def _mods():
    from paper_2507_06938_b200 import bta, bta_dist

    return bta, bta_dist


def test_dist_golden_cases(cuda):
    bta, bta_dist = _mods()
    g = golden("bta_dist.npz")
    for k in range(int(g["ndist"][0])):
        n, p, lb, b, a = g[f"d{k}_case"]
        n, p, b, a = int(n), int(p), int(b), int(a)
        m = bta.BTAMatrix(n, b, a, g[f"d{k}_input"])
        plan = bta_dist.plan_partitions(n, p, float(lb))
        f = bta_dist.d_factorize(m, plan)
        np.testing.assert_allclose(bta_dist.d_logdet(f), g[f"d{k}_logdet"][0], rtol=1e-10)
        np.testing.assert_allclose(bta_dist.d_solve(f, g[f"d{k}_rhs"]), g[f"d{k}_solve"],
                                   rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(bta_dist.d_selected_invert(f).numpy(), g[f"d{k}_sinv"],
                                   rtol=1e-8, atol=1e-11)


@pytest.mark.parametrize("n,b,a,P,lb", [(12, 130, 3, 3, 1.0), (20, 64, 2, 4, 1.6), (9, 257, 0, 2, 1.0),
                                        (16, 100, 5, 4, 1.0), (8, 33, 1, 4, 1.0),
                                        (8, 640, 3, 2, 1.0), (9, 1100, 2, 3, 1.6)])
def test_dist_matches_sequential(cuda, n, b, a, P, lb):
    bta, bta_dist = _mods()
    rng = np.random.default_rng(n * 7 + b + a + P)
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    plan = bta_dist.plan_partitions(n, P, lb)
    m = bta.BTAMatrix(n, b, a, data)
    f = bta_dist.d_factorize(m, plan)
    np.testing.assert_allclose(m.numpy(), data, rtol=0, atol=0)  # input untouched for P > 1
    np.testing.assert_allclose(bta_dist.d_logdet(f), bta_np.logdet(ref, n, b, a), rtol=1e-9)
    rhs = rng.normal(size=(n * b + a, 2))
    np.testing.assert_allclose(bta_dist.d_solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs),
                               rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(bta_dist.d_selected_invert(f).numpy(),
                               bta_np.selected_invert(ref, n, b, a, has), rtol=1e-8, atol=1e-11)


def test_dist_single_partition_delegates(cuda):
    bta, bta_dist = _mods()
    rng = np.random.default_rng(5)
    n, b, a = 4, 40, 2
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    bta_np.factorize(ref, n, b, a)
    f = bta_dist.d_factorize(bta.BTAMatrix(n, b, a, data), bta_dist.plan_partitions(n, 1))
    assert f.sequential is not None
    np.testing.assert_allclose(bta_dist.d_logdet(f), bta_np.logdet(ref, n, b, a), rtol=1e-12)


def test_dist_indefinite_tags_partition(cuda):
    bta, bta_dist = _mods()
    rng = np.random.default_rng(9)
    n, b, a = 12, 20, 2
    data = bta_np.random_spd_bta(rng, n, b, a)
    plan = bta_dist.plan_partitions(n, 3)  # (0,4,8,12); interior of partition 1: blocks 5, 6
    bad = data.copy()
    d, _, _, _ = bta_np.views(bad, n, b, a)
    d[6] = -np.eye(b)
    with pytest.raises(bta.FactorizationError) as e:
        bta_dist.d_factorize(bta.BTAMatrix(n, b, a, bad), plan)
    assert e.value.block_index == 6 and e.value.partition == 1
    bad = data.copy()
    d, _, _, _ = bta_np.views(bad, n, b, a)
    d[4] = -np.eye(b)  # a separator
    with pytest.raises(bta.FactorizationError) as e:
        bta_dist.d_factorize(bta.BTAMatrix(n, b, a, bad), plan)
    assert e.value.block_index == 4 and e.value.partition == -1


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_dist_multi_device(cuda):
    bta, bta_dist = _mods()
    rng = np.random.default_rng(11)
    n, b, a = 16, 130, 3
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    f = bta_dist.d_factorize(bta.BTAMatrix(n, b, a, data), bta_dist.plan_partitions(n, 4),
                             devices=[0, 1])
    np.testing.assert_allclose(bta_dist.d_logdet(f), bta_np.logdet(ref, n, b, a), rtol=1e-9)
    rhs = rng.normal(size=(n * b + a, 2))
    np.testing.assert_allclose(bta_dist.d_solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs),
                               rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(bta_dist.d_selected_invert(f).numpy(),
                               bta_np.selected_invert(ref, n, b, a, has), rtol=1e-8, atol=1e-11)

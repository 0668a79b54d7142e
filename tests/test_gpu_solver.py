"""Parity of the sm_100a BTA solver (POBTAF / POBTAS / POBTASI) with the CPU
oracle and the reference golden vectors, called through the C ABI."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import bta_np

pytestmark = pytest.mark.gpu


def _bta():
    from paper_2507_06938_b200 import bta

    return bta


def test_golden_cases_match_reference(cuda):
    bta = _bta()
    g = golden("bta_solver.npz")
    for k in range(int(g["ncases"][0])):
        n, b, a = (int(x) for x in g[f"c{k}_shape"])
        m = bta.BTAMatrix(n, b, a, g[f"c{k}_input"])
        f = bta.factorize(m)
        assert int(f.has_arrow) == int(g[f"c{k}_has_arrow"][0])
        np.testing.assert_allclose(m.numpy(), g[f"c{k}_factor"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(bta.logdet(f), g[f"c{k}_logdet"][0], rtol=1e-12)
        np.testing.assert_allclose(bta.solve(f, g[f"c{k}_rhs"]), g[f"c{k}_solve"], rtol=1e-10,
                                   atol=1e-12)
        np.testing.assert_allclose(bta.solve(f, g[f"c{k}_rhs2"]), g[f"c{k}_solve2"], rtol=1e-10,
                                   atol=1e-12)
        np.testing.assert_allclose(bta.forward_substitute(f, g[f"c{k}_rhs"]), g[f"c{k}_fwd"],
                                   rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(bta.backward_substitute(f, g[f"c{k}_rhs"]), g[f"c{k}_bwd"],
                                   rtol=1e-10, atol=1e-12)
        inv = bta.selected_invert(f)
        np.testing.assert_allclose(inv.numpy(), g[f"c{k}_sinv"], rtol=1e-10, atol=1e-12)


def _pattern_mask(n, b, a):
    N = n * b + a
    m = np.zeros((N, N), dtype=bool)
    for i in range(n):
        m[i * b : (i + 1) * b, i * b : (i + 1) * b] = True
        if i + 1 < n:
            m[(i + 1) * b : (i + 2) * b, i * b : (i + 1) * b] = True
            m[i * b : (i + 1) * b, (i + 1) * b : (i + 2) * b] = True
    if a:
        m[n * b :, :] = True
        m[:, n * b :] = True
    return m


def test_criterion1_oracle_suite(cuda):
    """240 random SPD BTA instances, the reference acceptance grid
    (tests/test_acceptance.py:51-100) and its tolerances."""
    bta = _bta()
    rng = np.random.default_rng(101)
    worst = dict(chol=0.0, logdet=0.0, solve=0.0, sinv=0.0)
    count = 0
    for n in range(1, 9):
        for b in range(1, 7):
            for a in range(0, 5):
                data = bta_np.random_spd_bta(rng, n, b, a)
                dense = bta_np.to_dense(data, n, b, a)
                m = bta.BTAMatrix(n, b, a, data)
                f = bta.factorize(m)
                low = np.tril(m.to_dense())
                scale = max(np.abs(dense).max(), 1e-30)
                worst["chol"] = max(worst["chol"], np.abs(low @ low.T - dense).max() / scale)
                ref = np.linalg.slogdet(dense)[1]
                worst["logdet"] = max(worst["logdet"],
                                      abs(bta.logdet(f) - ref) / max(abs(ref), 1e-30))
                rhs = rng.normal(size=n * b + a)
                x = bta.solve(f, rhs)
                worst["solve"] = max(worst["solve"],
                                     np.linalg.norm(dense @ x - rhs) / np.linalg.norm(rhs))
                dinv = np.linalg.inv(dense)
                mask = _pattern_mask(n, b, a)
                err = np.abs(bta.selected_invert(f).to_dense() - dinv)[mask]
                worst["sinv"] = max(worst["sinv"],
                                    float((err / np.maximum(np.abs(dinv), 1e-12)[mask]).max()))
                count += 1
    assert count == 240
    assert worst["chol"] <= 1e-10 and worst["logdet"] <= 1e-9
    assert worst["solve"] <= 1e-10 and worst["sinv"] <= 1e-8, worst


@pytest.mark.parametrize("n,b,a", [(3, 64, 2), (4, 65, 3), (5, 130, 1), (2, 257, 6), (3, 300, 2),
                                   (6, 100, 0), (2, 129, 70), (2, 129, 130), (1, 256, 3),
                                   (3, 128, 0), (4, 383, 5), (3, 1100, 7), (2, 1025, 0)])
def test_multileaf_blocks_vs_oracle(cuda, n, b, a):
    """Blocks spanning several 64-leaves and partial leaves, vs the oracle."""
    bta = _bta()
    rng = np.random.default_rng(n * 1000 + b + a)
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    m = bta.BTAMatrix(n, b, a, data)
    f = bta.factorize(m)
    assert f.has_arrow == has
    np.testing.assert_allclose(m.numpy(), ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(bta.logdet(f), bta_np.logdet(ref, n, b, a), rtol=1e-12)
    rhs = rng.normal(size=(n * b + a, 3))
    np.testing.assert_allclose(bta.solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs),
                               rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(bta.selected_invert(f).numpy(),
                               bta_np.selected_invert(ref, n, b, a, has), rtol=1e-10, atol=1e-12)


def test_many_rhs_columns(cuda):
    bta = _bta()
    rng = np.random.default_rng(3)
    n, b, a = 3, 70, 2
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    f = bta.factorize(bta.BTAMatrix(n, b, a, data))
    rhs = rng.normal(size=(n * b + a, 19))
    np.testing.assert_allclose(bta.solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs), rtol=1e-10,
                               atol=1e-11)


def test_indefinite_pivot_reports_block(cuda):
    bta = _bta()
    rng = np.random.default_rng(2)
    for n, b, a, bad in ((4, 2, 1, 2), (5, 70, 2, 3), (3, 130, 0, 0)):
        data = bta_np.random_spd_bta(rng, n, b, a)
        d, _, _, _ = bta_np.views(data, n, b, a)
        d[bad] = -np.eye(b)
        with pytest.raises(bta.FactorizationError) as err:
            bta.factorize(bta.BTAMatrix(n, b, a, data))
        assert err.value.block_index == bad
    # indefinite tip -> block index n (bta.py:229-232)
    n, b, a = 3, 4, 2
    data = bta_np.random_spd_bta(rng, n, b, a)
    _, _, ar, tp = bta_np.views(data, n, b, a)
    ar[...] = 0.0
    tp[...] = -np.eye(a)
    with pytest.raises(bta.FactorizationError) as err:
        bta.factorize(bta.BTAMatrix(n, b, a, data))
    assert err.value.block_index == n


def test_closed_forms_and_identity(cuda):
    bta = _bta()
    f = bta.factorize(bta.BTAMatrix.from_dense(np.array([[4.0]]), 1, 1, 0))
    assert f.matrix.numpy()[0] == 2.0
    np.testing.assert_allclose(bta.solve(f, np.array([8.0])), [2.0])
    f = bta.factorize(bta.BTAMatrix.from_dense(2.0 * np.eye(3), 3, 1, 0))
    np.testing.assert_allclose(bta.logdet(f), 3 * np.log(2.0), rtol=1e-14)
    for n, b, a in ((1, 1, 0), (3, 2, 0), (2, 3, 2)):
        m = bta.BTAMatrix.from_dense(np.eye(n * b + a), n, b, a)
        bta.factorize(m)
        np.testing.assert_allclose(m.to_dense(), np.eye(n * b + a))
    m = bta.BTAMatrix.from_dense(np.array([[2.0, 1.0], [1.0, 2.0]]), 2, 1, 0)
    inv = bta.selected_invert(bta.factorize(m))
    np.testing.assert_allclose(inv.to_dense(), np.array([[2.0, -1.0], [-1.0, 2.0]]) / 3.0,
                               rtol=1e-14)
    with pytest.raises(ValueError):
        bta.solve(bta.factorize(bta.BTAMatrix.from_dense(np.eye(4), 2, 2, 0)), np.ones(5))


def test_zero_arrow_skips_arrow_work(cuda):
    bta = _bta()
    rng = np.random.default_rng(3)
    base = bta_np.random_spd_bta(rng, 6, 3, 0)
    m = bta.BTAMatrix(6, 3, 2)
    d0, l0, _, _ = bta_np.views(base, 6, 3, 0)
    m.diag.copy_(torch.from_numpy(d0))
    m.lower.copy_(torch.from_numpy(l0))
    m.tip.copy_(torch.eye(2, dtype=torch.float64))
    c = bta.OpCounter()
    f = bta.factorize(m, counter=c)
    assert not f.has_arrow
    assert c.flops == 6 * 27 + 8


def _block_matvec_identity_residual(Q, X, n, b, a):
    """max |(Q X)_ii - I| over diagonal blocks, from pattern blocks only."""
    Qd, Ql, Qa = Q.diag, Q.lower, Q.arrow
    Xd, Xl, Xa = X.diag, X.lower, X.arrow
    worst = 0.0
    eye = torch.eye(b, dtype=torch.float64, device=Q.device)
    for i in range(n):
        acc = Qd[i] @ Xd[i]
        if i > 0:
            acc += Ql[i - 1] @ Xl[i - 1].T  # Q_{i,i-1} X_{i-1,i}
        if i + 1 < n:
            acc += Ql[i].T @ Xl[i]  # Q_{i,i+1} X_{i+1,i}
        if a:
            acc += Qa[i].T @ Xa[i]  # Q_{i,a} X_{a,i}
        worst = max(worst, float((acc - eye).abs().max()))
    return worst


def test_full_size_c2_properties(cuda):
    """BASELINE C2 shape (n=48, b=2048, a=6): size-independent properties —
    solve residual, the identity on the diagonal blocks of Q X for the selected
    inverse, and logdet additivity under scaling."""
    bta = _bta()
    n, b, a = 48, 2048, 6
    g = torch.Generator(device=cuda)
    g.manual_seed(0)
    m = bta.BTAMatrix(n, b, a, device=cuda)
    sd = 0.3 / b**0.5
    for i in range(n):  # diagonally dominant SPD BTA, generated on the device
        r = torch.randn(b, b, dtype=torch.float64, device=cuda, generator=g) * sd
        m.diag[i] = r @ r.T + torch.eye(b, dtype=torch.float64, device=cuda) * 2.0
    m.lower.normal_(0.0, sd, generator=g)
    m.arrow.normal_(0.0, sd, generator=g)
    m.tip.copy_(torch.eye(a, dtype=torch.float64, device=cuda) * 4.0)
    Q = m.copy()
    f = bta.factorize(m)
    ld = bta.logdet(f)
    # residual of the solve, with a device block matvec
    x_true = torch.randn(n * b + a, dtype=torch.float64, device=cuda, generator=g)
    r = torch.zeros_like(x_true)
    xs = x_true[: n * b].view(n, b)
    rs = r[: n * b].view(n, b)
    rs += torch.einsum("nij,nj->ni", Q.diag, xs)
    rs[1:] += torch.einsum("nij,nj->ni", Q.lower, xs[:-1])
    rs[:-1] += torch.einsum("nji,nj->ni", Q.lower, xs[1:])
    rs += torch.einsum("nai,a->ni", Q.arrow, x_true[n * b :])
    r[n * b :] = torch.einsum("naj,nj->a", Q.arrow, xs) + Q.tip @ x_true[n * b :]
    x = bta.solve(f, r)
    assert float((x - x_true).norm() / x_true.norm()) < 1e-11
    X = bta.selected_invert(f)
    assert _block_matvec_identity_residual(Q, X, n, b, a) < 1e-9
    # logdet(c Q) = N log c + logdet(Q)
    Q2 = Q.copy()
    Q2.data.mul_(3.7)
    ld2 = bta.logdet(bta.factorize(Q2))
    np.testing.assert_allclose(ld2, (n * b + a) * np.log(3.7) + ld, rtol=1e-12)


# Shapes that exercise the POBTAF scheduling paths: chunked updates (>= 5 tile
# columns per block, CHUNK 4 / 8), the second-row look-ahead groups, partial
# last tiles with and without 16-byte rows (TMA vs cp.async), TMA slabs that
# end at the block edge, wide arrows (a > 128) and blocks of one tile.
@pytest.mark.parametrize("n,b,a", [(4, 640, 3), (3, 1000, 0), (3, 3072, 6), (2, 1300, 131),
                                   (5, 128, 4), (3, 897, 2), (2, 4000, 1)])
def test_scheduling_paths_vs_oracle(cuda, n, b, a):
    bta = _bta()
    rng = np.random.default_rng(97 * n + b + a)
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    m = bta.BTAMatrix(n, b, a, data)
    f = bta.factorize(m)
    assert f.has_arrow == has
    np.testing.assert_allclose(m.numpy(), ref, rtol=0, atol=1e-11)
    np.testing.assert_allclose(bta.logdet(f), bta_np.logdet(ref, n, b, a), rtol=1e-12)
    inv = bta.selected_invert(f).numpy()
    np.testing.assert_allclose(inv, bta_np.selected_invert(ref, n, b, a, has), rtol=1e-9,
                               atol=1e-11)

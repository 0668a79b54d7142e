"""The W-based POBTAS (stbta_pobtas_w: block GEMVs with W_t = L_tt^-1 prepared
by stbta_pobtasi_prepare) against the oracle and the tile-sweep POBTAS, and
the selected inversion on a prepared workspace against the plain one."""

import numpy as np
import pytest

from oracle import bta_np

pytestmark = pytest.mark.gpu

SHAPES = [(1, 64, 0), (1, 130, 3), (2, 129, 6), (3, 300, 2), (5, 100, 0), (4, 383, 5),
          (2, 129, 130), (3, 1100, 7), (6, 2048, 6), (2, 5025, 3)]


def _case(n, b, a, seed):
    from paper_2507_06938_b200 import bta

    rng = np.random.default_rng(seed)
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    f = bta.factorize(bta.BTAMatrix(n, b, a, data))
    return bta, rng, ref, has, f


@pytest.mark.parametrize("n,b,a", SHAPES)
def test_w_solve_vs_oracle(cuda, n, b, a):
    bta, rng, ref, has, f = _case(n, b, a, 7 * n + b + a)
    bta.prepare_inverse(f)
    for nrhs in (1, 3, 9):
        rhs = rng.normal(size=(n * b + a, nrhs))
        np.testing.assert_allclose(bta.solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs),
                                   rtol=1e-10, atol=1e-11)
    rhs = rng.normal(size=n * b + a)
    np.testing.assert_allclose(bta.forward_substitute(f, rhs),
                               bta_np.forward(ref, n, b, a, has, rhs[:, None])[:, 0],
                               rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(bta.backward_substitute(f, rhs),
                               bta_np.backward(ref, n, b, a, has, rhs[:, None])[:, 0],
                               rtol=1e-10, atol=1e-11)


@pytest.mark.parametrize("n,b,a", [(3, 300, 2), (4, 383, 5), (6, 2048, 6)])
def test_w_solve_matches_tile_solve(cuda, monkeypatch, n, b, a):
    bta, rng, ref, has, f = _case(n, b, a, 11 + n + b)
    rhs = rng.normal(size=(n * b + a, 17))
    monkeypatch.setenv("STBTA_SOLVE", "tile")
    x_tile = bta.solve(f, rhs)
    assert f._si_ws is None
    monkeypatch.setenv("STBTA_SOLVE", "w")
    x_w = bta.solve(f, rhs)
    assert f._si_ws is not None
    np.testing.assert_allclose(x_w, x_tile, rtol=1e-10, atol=1e-11)
    # deterministic: a second W solve is bit-identical
    np.testing.assert_array_equal(bta.solve(f, rhs), x_w)


@pytest.mark.parametrize("n,b,a", [(1, 130, 3), (3, 300, 2), (2, 129, 130), (5, 100, 0),
                                   (6, 2048, 6)])
def test_prepared_selected_inverse_is_identical(cuda, n, b, a):
    import torch

    bta, rng, ref, has, f = _case(n, b, a, 5 + n * b)
    plain = bta.selected_invert(f).numpy()
    bta.prepare_inverse(f)
    prep = bta.selected_invert(f).numpy()
    np.testing.assert_array_equal(prep, plain)
    np.testing.assert_allclose(prep, bta_np.selected_invert(ref, n, b, a, has), rtol=1e-10,
                               atol=1e-12)
    # streamed to pinned host memory from the prepared workspace
    out = torch.empty(plain.size, dtype=torch.float64).pin_memory()
    inv = bta.selected_invert(f, out=out)
    np.testing.assert_array_equal(inv.numpy(out=out), plain)


def test_solve_policy_rejects_unknown(monkeypatch):
    from paper_2507_06938_b200 import bta

    monkeypatch.setenv("STBTA_SOLVE", "dense")
    with pytest.raises(ValueError):
        bta._solve_policy()

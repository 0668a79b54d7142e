"""The CPU oracle pinned against golden vectors from the unmodified reference
and the reference tests' closed-form known answers (CPU only)."""

import numpy as np
import pytest

from conftest import golden, spec_from_golden
from oracle import bta_np, inla_np


def test_solver_oracle_matches_reference_golden():
    g = golden("bta_solver.npz")
    for k in range(int(g["ncases"][0])):
        n, b, a = (int(x) for x in g[f"c{k}_shape"])
        data = g[f"c{k}_input"].copy()
        has = bta_np.factorize(data, n, b, a)
        assert int(has) == int(g[f"c{k}_has_arrow"][0])
        np.testing.assert_allclose(data, g[f"c{k}_factor"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(bta_np.logdet(data, n, b, a), g[f"c{k}_logdet"][0], rtol=1e-13)
        for key, fn in (("fwd", bta_np.forward), ("bwd", bta_np.backward), ("solve", bta_np.solve)):
            got = fn(data, n, b, a, has, g[f"c{k}_rhs"])
            np.testing.assert_allclose(got, g[f"c{k}_{key}"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(
            bta_np.solve(data, n, b, a, has, g[f"c{k}_rhs2"]), g[f"c{k}_solve2"], rtol=1e-12,
            atol=1e-13,
        )
        np.testing.assert_allclose(
            bta_np.selected_invert(data, n, b, a, has), g[f"c{k}_sinv"], rtol=1e-12, atol=1e-13
        )


def test_random_generator_reproduces_reference_bytes():
    g = golden("bta_solver.npz")
    for k in range(int(g["ncases"][0])):
        n, b, a = (int(x) for x in g[f"c{k}_shape"])
        rng = np.random.default_rng(900 + k)
        # same draws; products may differ in the last bit with the BLAS thread count
        np.testing.assert_allclose(
            bta_np.random_spd_bta(rng, n, b, a), g[f"c{k}_input"], rtol=1e-14, atol=1e-15
        )


def test_closed_form_known_answers():
    # scalar [4] -> L = [2]  (reference tests/test_bta.py:42-45)
    d = np.array([4.0])
    bta_np.factorize(d, 1, 1, 0)
    assert d[0] == 2.0
    # logdet(2 I_3) = 3 log 2  (tests/test_bta.py:85-87)
    d = bta_np.from_dense(2.0 * np.eye(3), 3, 1, 0)
    bta_np.factorize(d, 3, 1, 0)
    np.testing.assert_allclose(bta_np.logdet(d, 3, 1, 0), 3 * np.log(2.0), rtol=1e-14)
    # 2x2 inverse [[2,-1],[-1,2]]/3  (tests/test_bta.py:159-163)
    d = bta_np.from_dense(np.array([[2.0, 1.0], [1.0, 2.0]]), 2, 1, 0)
    bta_np.factorize(d, 2, 1, 0)
    inv = bta_np.to_dense(bta_np.selected_invert(d, 2, 1, 0, False), 2, 1, 0)
    np.testing.assert_allclose(inv, np.array([[2.0, -1.0], [-1.0, 2.0]]) / 3.0, rtol=1e-14)


def test_objective_oracle_matches_reference_golden():
    g = golden("objective.npz")
    for name in ("uni", "tri", "biv0"):
        spec = spec_from_golden(g, f"{name}_")
        for k, p in enumerate(g[f"{name}_points"]):
            f, mu = inla_np.evaluate(spec, p, g[f"{name}_prior_mean"], g[f"{name}_prior_sd"])
            np.testing.assert_allclose(f, g[f"{name}_f"][k], rtol=1e-12)
            np.testing.assert_allclose(mu, g[f"{name}_mu"][k], rtol=1e-9, atol=1e-11)
        sd = inla_np.marginal_sd(spec, g[f"{name}_points"][0])
        np.testing.assert_allclose(sd, g[f"{name}_sd"], rtol=1e-10)


def test_host_optimizer_on_oracle_reproduces_reference_mode():
    """The package's host minimize() driven by the CPU oracle objective lands
    on the reference mode of the bundled univariate config."""
    from paper_2507_06938_b200.inla import minimize

    g = golden("mode_search.npz")
    spec = spec_from_golden(g, "ini_")
    psd, gtol, ftol = g["ini_opts"]
    theta0 = g["ini_theta0"]
    mean, sd = theta0, np.full(4, psd)

    def fun(t):
        return -inla_np.evaluate(spec, t, mean, sd)[0]

    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = minimize(fun, theta0, gtol=gtol, ftol=ftol, max_iter=100)
    np.testing.assert_allclose(res.theta, g["ini_theta"], atol=1e-4)
    np.testing.assert_allclose(res.f, g["ini_f"][0], rtol=1e-8)
    assert res.iterations == int(g["ini_iters"][0])


@pytest.mark.parametrize("n,b,a", [(4, 3, 2), (6, 2, 0), (3, 5, 1)])
def test_oracle_against_dense_linear_algebra(n, b, a):
    rng = np.random.default_rng(n * 100 + b * 10 + a)
    data = bta_np.random_spd_bta(rng, n, b, a)
    dense = bta_np.to_dense(data, n, b, a)
    f = data.copy()
    has = bta_np.factorize(f, n, b, a)
    low = np.tril(bta_np.to_dense(f, n, b, a))
    np.testing.assert_allclose(low, np.linalg.cholesky(dense), atol=1e-12)
    np.testing.assert_allclose(bta_np.logdet(f, n, b, a), np.linalg.slogdet(dense)[1], rtol=1e-12)
    rhs = rng.normal(size=n * b + a)
    np.testing.assert_allclose(dense @ bta_np.solve(f, n, b, a, has, rhs), rhs, atol=1e-10)

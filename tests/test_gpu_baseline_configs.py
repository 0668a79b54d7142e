"""Parity on the BASELINE configurations themselves, against fixtures written
by the UNMODIFIED reference (oracle/make_golden_c2.py, make_golden_c3.py,
make_golden_tri.py):

* C2 (BASELINE configs[1]): random_spd_bta(default_rng(0), 48, 2048, 6) --
  log-determinant to 1e-12, sampled factor / solution / selected-inverse
  entries from every storage region and the inverse's diagonal to 1e-10;
* C3 (configs[2], the north-star model): f_obj at theta0 to 1e-10, the
  conditional mean, all 31 task values of the gradient batch to 1e-10 and the
  central-difference gradient to 1e-5, the batch run through GpuRunner;
* the bundled trivariate.ini fit (d = 15, partitions = 3, lb = 1.6): the same
  BFGS iterates (iteration and f_obj counts), the mode to 1e-4, the log
  posterior to 1e-8, the Hessian and the latent marginals, driven through
  GpuRunner with line-search width > 1.

Tolerances (north_star): 1e-8 relative on log-det, f_obj and marginal
variances, 1e-4 on the mode; the tests are tighter where FP64 allows.
"""

import os
import warnings

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden, spec_from_golden

pytestmark = pytest.mark.gpu


def _checksums(x):
    w = np.arange(1, x.size + 1, dtype=np.float64) / x.size
    return np.array([np.sum(x), np.sum(x * w), np.sum(np.abs(x))])


def _evaluators(spec, prior, per_device=2, **kw):
    """Evaluators over every visible GPU (at least two, so GpuRunner's
    line-search width is > 1 even on a one-GPU box)."""
    from paper_2507_06938_b200 import inla

    G = torch.cuda.device_count()
    devs = [torch.device("cuda", g) for g in range(G)] if G > 1 else \
        [torch.device("cuda", 0)] * per_device
    return [inla.ObjectiveEvaluator(spec, prior=prior, device=d, **kw) for d in devs]


def test_c2_matches_reference(cuda):
    from paper_2507_06938_b200 import bta

    g = golden("c2.npz")
    n, b, a = (int(x) for x in g["shape"])
    rng = np.random.default_rng(0)
    m = bta.random_spd_bta(rng, n, b, a, device=cuda)
    rhs = rng.normal(size=m.dim)
    idx = g["index"]
    host = m.numpy()
    # the package's generator reproduces the reference's input bytes
    np.testing.assert_allclose(host[idx], g["input"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(_checksums(host), g["input_checksums"], rtol=1e-12)
    np.testing.assert_allclose(_checksums(rhs), g["rhs_checksums"], rtol=1e-13)
    del host
    f = bta.factorize(m)
    assert f.has_arrow == bool(g["has_arrow"][0])
    np.testing.assert_allclose(bta.logdet(f), g["logdet"][0], rtol=1e-12)
    fac = m.data[torch.from_numpy(idx).to(cuda)].cpu().numpy()
    np.testing.assert_allclose(fac, g["factor"], rtol=1e-10, atol=1e-13)
    x = bta.solve(f, rhs)
    np.testing.assert_allclose(x[g["solve_index"]], g["solve"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(_checksums(x), g["solve_checksums"], rtol=1e-10)
    inv = bta.selected_invert(f)
    sel = inv.data[torch.from_numpy(idx).to(cuda)].cpu().numpy()
    np.testing.assert_allclose(sel, g["sinv"], rtol=1e-10, atol=1e-14)
    dg = torch.cat([torch.diagonal(inv.diag, dim1=1, dim2=2).reshape(-1),
                    torch.diagonal(inv.tip)]).cpu().numpy()
    np.testing.assert_allclose(dg[g["solve_index"]], g["sinv_diag"], rtol=1e-10)
    np.testing.assert_allclose(_checksums(dg), g["sinv_diag_checksums"], rtol=1e-10)


def _c3_inputs_checksums(spec):
    out = []
    for a, y in zip(spec.design, spec.observations):
        a = a.tocsr()
        w = np.arange(1, a.nnz + 1, dtype=np.float64)
        out += [float(np.sum(y)), float(np.sum(y * np.arange(1, y.size + 1))),
                float(np.sum(a.indices * w)), float(np.sum(a.data * w))]
    return np.array(out)


def test_c3_objective_and_gradient_match_reference(cuda):
    from paper_2507_06938_b200 import inla, sched
    from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic

    if not os.path.exists(os.path.join(GOLDEN, "c3.npz")):
        pytest.skip("tests/golden/c3.npz not generated (oracle/make_golden_c3.py)")
    g = golden("c3.npz")
    nv, ns, nt, nf, m, seed = (int(x) for x in g["settings"])
    data = generate_synthetic(SyntheticSettings(nv, ns, nt, nf, m), g["theta_true"], seed=seed,
                              device=cuda)
    np.testing.assert_allclose(_c3_inputs_checksums(data.spec), g["input_checksums"], rtol=1e-12)
    th0 = g["theta0"]
    prior = inla.ThetaPrior.for_dim(th0.size, mean=th0, sd=float(g["prior_sd"][0]))
    evs = _evaluators(data.spec, prior)
    try:
        f, mu = evs[0].evaluate(th0)
        np.testing.assert_allclose(f, g["f_obj"][0], rtol=1e-10)
        np.testing.assert_allclose(mu[g["mu_index"]], g["mu"], rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(mu.sum(), g["mu_sum"][0], rtol=1e-9)
        vals = []
        runner = sched.GpuRunner(evs)

        def recording(tasks):
            out = runner(tasks)
            vals.extend(out)
            return out

        fneg, grad = inla.fd_gradient(evs[0], th0, float(g["grad_step"][0]), runner=recording)
        runner.close()
        # all 31 task values of the reference's gradient batch and the full
        # gradient (oracle/make_golden_c3.py; a NaN would mark a task not computed)
        have = np.isfinite(g["task_values"])
        assert have.all()
        np.testing.assert_allclose(np.asarray(vals)[have], g["task_values"][have], rtol=1e-10)
        np.testing.assert_allclose(fneg, g["neg_f"][0], rtol=1e-10)
        hg = np.isfinite(g["grad"])
        assert hg.all()
        np.testing.assert_allclose(grad[hg], g["grad"][hg], rtol=0, atol=1e-5)
    finally:
        for ev in evs:
            ev.release_workspaces()


def test_trivariate_ini_fit_matches_reference(cuda):
    """pkg/configs/trivariate.ini end to end: partitioned evaluator
    (partitions=3, lb=1.6), BFGS through GpuRunner (width > 1), Hessian and
    latent marginals at the mode."""
    from paper_2507_06938_b200 import inla, sched

    g = golden("trivariate.npz")
    spec = spec_from_golden(g, "tri_")
    th0 = g["theta0"]
    gtol, ftol, gstep, hstep, psd, max_iter = g["opts"]
    parts, lb = int(g["parallel"][0]), float(g["parallel"][1])
    prior = inla.ThetaPrior.for_dim(th0.size, mean=th0, sd=psd)
    evs = _evaluators(spec, prior, partitions=parts, lb=lb)
    runner = sched.GpuRunner(evs, split_pairs=False)
    assert runner.width > 1
    opts = inla.FitOptions(gtol=gtol, ftol=ftol, grad_step=gstep, hess_step=hstep,
                           max_iter=int(max_iter), prior_sd=psd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        summary, res = inla.fit(evs[0], th0, opts, runner=runner)
    runner.close()
    assert res.status == str(g["status"][0])
    assert [res.iterations, res.f_evals] == g["counts"].tolist()
    assert [summary.iterations, summary.f_evals] == g["fit_counts"].tolist()
    np.testing.assert_allclose(res.theta, g["theta"], rtol=0, atol=1e-4)
    np.testing.assert_allclose([r.f for r in res.trace], g["trace_f"], rtol=1e-8)
    np.testing.assert_allclose([r.step for r in res.trace], g["trace_step"], rtol=0)
    np.testing.assert_allclose(summary.logpost_at_mode, g["logpost"][0], rtol=1e-8)
    h = g["hessian"]
    np.testing.assert_allclose(summary.theta_hessian, h, rtol=0, atol=1e-5 * np.abs(h).max())
    np.testing.assert_allclose(summary.theta_sd, g["theta_sd"], rtol=1e-3)
    np.testing.assert_allclose(summary.latent_mean, g["latent_mean"], rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(summary.latent_sd ** 2, g["latent_sd"] ** 2, rtol=1e-5)
    # at the reference's own mode: marginal variances to the north_star 1e-8
    mu, sd = evs[0].latent_marginals(g["theta"])
    ref_mu, ref_sd = g["latent_mean"], g["latent_sd"]
    np.testing.assert_allclose(mu, ref_mu, rtol=1e-8, atol=1e-10 * np.abs(ref_mu).max())
    np.testing.assert_allclose(sd ** 2, ref_sd ** 2, rtol=1e-8)
    for ev in evs:
        ev.release_workspaces()

"""Golden full fit of the bundled trivariate model (pkg/configs/trivariate.ini):
n_v=3 (dim theta = 15), n_s=8, n_t=6, n_r=1, 200 observations per process,
seed 2, theta0 / theta_true / prior sd 2 / gtol 1e-3 / ftol 1e-8 / max_iter 100
and the partitioned solver (partitions=3, lb=1.6) exactly as the config file
states, run through the UNMODIFIED reference ``fit`` (inla.py:661-729): BFGS
mode search, finite-difference Hessian, latent marginals.  This is the d=15
mode search of the north-star model family at a size the reference finishes
in seconds.  Test infrastructure only:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_tri.py

Output: tests/golden/trivariate.npz (model inputs + reference outputs).
"""

import os
import sys
import time
import warnings

import numpy as np

from make_golden import OUT, REF, _spec_arrays

THETA0 = np.array([-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05,
                   0.05, 0.65, -0.35, 0.35])
THETA_TRUE = np.array([-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00,
                       0.00, 0.60, -0.40, 0.30])


def main():
    sys.path.insert(0, REF)
    from stinla.inla import FitOptions, fit
    from stinla.synthetic import SyntheticSettings, generate_synthetic

    data = generate_synthetic(SyntheticSettings(3, 8, 6, 1, 200), THETA_TRUE, seed=2)
    o = _spec_arrays("tri_", data.spec)
    opts = FitOptions(gtol=1e-3, ftol=1e-8, max_iter=100, prior_sd=2.0)
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        summary, res = fit(data.spec, THETA0, opts, partitions=3, lb=1.6)
    secs = time.perf_counter() - t0
    o.update(
        theta0=THETA0, theta_true=THETA_TRUE,
        opts=np.array([opts.gtol, opts.ftol, opts.grad_step, opts.hess_step, opts.prior_sd,
                       opts.max_iter]),
        parallel=np.array([3, 1.6]),
        theta=res.theta, f=np.array([res.f]), grad=res.grad,
        counts=np.array([res.iterations, res.f_evals]), status=np.array([res.status]),
        trace_f=np.array([r.f for r in res.trace]),
        trace_step=np.array([r.step for r in res.trace]),
        trace_evals=np.array([r.f_evals for r in res.trace]),
        theta_sd=summary.theta_sd, hessian=summary.theta_hessian,
        latent_mean=summary.latent_mean, latent_sd=summary.latent_sd,
        logpost=np.array([summary.logpost_at_mode]),
        fit_counts=np.array([summary.iterations, summary.f_evals]),
        seconds=np.array([secs]),
    )
    np.savez_compressed(os.path.join(OUT, "trivariate.npz"), **o)
    print(f"trivariate fit: {res.status}, {res.iterations} iterations, {res.f_evals} f_evals, "
          f"logpost {summary.logpost_at_mode!r}, {secs:.1f} s")


if __name__ == "__main__":
    main()

"""C3 (BASELINE configs[2]) full hyperparameter optimisation on all visible
GPUs with the config's own settings (trivariate.ini:18-21: gtol 1e-3,
ftol 1e-8, max_iter 100; prior N(theta0, 2^2)), recording the BFGS state
(theta, f, grad, inverse Hessian) after every iteration.

The run is chained one iteration at a time through ``inla.minimize(...,
max_iter=1, state0=...)``, which continues the reference algorithm from the
recorded state, so the iterates are those of one uninterrupted run.

    python tools/c3_fit.py [out.json]

Writes bench_data/c3_bfgs_states.npz (the states bench.py resumes from to
time an iteration far from and near the mode at any GPU count) and prints /
writes one JSON summary.
"""

import json
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_06938_b200 import inla, sched  # noqa: E402
from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic  # noqa: E402

THETA0 = np.array([-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05, 0.05,
                   0.65, -0.35, 0.35])
TRUE = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60, -0.40,
        0.30]


def main():
    out_json = sys.argv[1] if len(sys.argv) > 1 else None
    G = torch.cuda.device_count()
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), TRUE, seed=2,
                              device=torch.device("cuda", 0))
    prior = inla.ThetaPrior.for_dim(15, mean=THETA0, sd=2.0)
    evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g))
           for g in range(G)]
    runner = sched.GpuRunner(evs)
    runner.evaluate_points([THETA0] * G)
    inla.prior_cache_clear()
    t0 = time.perf_counter()
    f0, g0 = inla.fd_gradient(evs[0], THETA0, 1e-3, runner)
    t_grad = time.perf_counter() - t0
    states = [(THETA0.copy(), f0, g0, np.eye(15))]
    recs, status, it = [], "max_iterations", 0
    theta, st = THETA0.copy(), (f0, g0, np.eye(15))
    total = t_grad
    while it < 100:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            got = []
            res = inla.minimize(evs[0], theta, gtol=1e-3, ftol=1e-8, max_iter=1, runner=runner,
                                on_iteration=got.append, state0=st)
        if not got:  # converged (gradient) at the top of the loop
            status = res.status
            break
        it += 1
        r = got[0]
        total += r.seconds
        recs.append({"iteration": it, "f": r.f, "grad_norm": r.grad_norm, "step": r.step,
                     "f_evals": r.f_evals, "tries": r.f_evals - 31, "seconds": r.seconds})
        theta, st = res.theta, (res.f, res.grad, res.hinv)
        states.append((theta.copy(), res.f, res.grad.copy(), res.hinv.copy()))
        print(json.dumps(recs[-1]), flush=True)
        if res.status != "max_iterations":
            status = res.status
            break
    for ev in evs:
        ev.release_workspaces()
    os.makedirs(os.path.join(ROOT, "bench_data"), exist_ok=True)
    np.savez(os.path.join(ROOT, "bench_data", "c3_bfgs_states.npz"),
             theta=np.array([s[0] for s in states]), f=np.array([s[1] for s in states]),
             grad=np.array([s[2] for s in states]), hinv=np.array([s[3] for s in states]),
             tries=np.array([0] + [r["tries"] for r in recs]),
             seconds=np.array([t_grad] + [r["seconds"] for r in recs]))
    summary = {"config": "C3 trivariate full mode search from theta0 (gtol 1e-3, ftol 1e-8, "
                         "max_iter 100, prior N(theta0, 2^2))",
               "n_gpus": G, "iterations": len(recs), "status": status,
               "f_evals": 31 + sum(r["f_evals"] for r in recs),
               "starting_gradient_s": t_grad, "total_s": total,
               "s_per_iteration": [r["seconds"] for r in recs],
               "tries_per_iteration": [r["tries"] for r in recs],
               "theta_star": theta.tolist(), "f_star": float(st[0]), "theta_true": TRUE}
    print(json.dumps(summary), flush=True)
    if out_json:
        with open(out_json, "w") as fh:
            json.dump({"summary": summary, "iterations": recs}, fh, indent=1)


if __name__ == "__main__":
    main()

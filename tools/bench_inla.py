"""INLA-level measurements on the device path.

  python tools/bench_inla.py c1            # univariate mode finding (full run)
  python tools/bench_inla.py c3            # one trivariate f_obj at theta0
  python tools/bench_inla.py c4 [depth]    # the 31-task gradient batch at theta0 on all GPUs
  python tools/bench_inla.py c3post        # fd_hessian (451 f_obj) + latent marginals at the C3 mode

(The C3 mode search itself: tools/c3_fit.py; the per-iteration north-star
number: bench.py.)

Inputs come from the reference generators restated in
paper_2507_06938_b200/synthetic.py (same seeds and draw order).  Prints one
JSON line per measurement.
"""

import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2507_06938_b200 import inla, sched
from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic

TRI_THETA0 = [-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05, 0.05, 0.65,
              -0.35, 0.35]
TRI_TRUE = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60,
            -0.40, 0.30]


def c1():
    t0 = time.perf_counter()
    data = generate_synthetic(SyntheticSettings(1, 300, 12, 2, 3600), [0.3, 0.2, 0.5, 1.2], seed=1)
    ev = inla.ObjectiveEvaluator(data.spec, prior=inla.ThetaPrior.for_dim(4, sd=10.0))
    setup = time.perf_counter() - t0
    theta0 = np.zeros(4)
    ev.objective(theta0)
    torch.cuda.synchronize()
    t_f = 0.0
    for _ in range(20):
        inla.prior_cache_clear()  # full evaluations
        t0 = time.perf_counter()
        ev.objective(theta0)
        t_f += (time.perf_counter() - t0) / 20
    recs = []
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = inla.minimize(ev, theta0, gtol=1e-3, ftol=1e-12, max_iter=100,
                            on_iteration=recs.append)
    total = time.perf_counter() - t0
    it = [r.seconds for r in recs] or [total]
    print(json.dumps({
        "config": "C1 univariate n_s=300 n_t=12 n_r=2 m=3600 (mode finding from theta0=0)",
        "setup_s": setup, "f_obj_ms": 1e3 * t_f, "iterations": res.iterations, "status": res.status,
        "f_evals": res.f_evals, "total_s": total, "s_per_iteration_median": float(np.median(it)),
        "theta_star": res.theta.tolist(), "f_star": res.f,
        "oracle_theta_star": [0.5229479477504098, 0.3853637147715331, -1.085137990668959,
                              1.2627782499940756],
        "oracle_f_obj_at_theta_star": -3072.0619154929495,  # minimize reports f_star = -f_obj
    }), flush=True)


def _c3_evaluator(device=None):
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), TRI_TRUE, seed=2,
                              device=device)
    prior = inla.ThetaPrior.for_dim(15, mean=np.array(TRI_THETA0), sd=2.0)
    return data, prior


def c3():
    t0 = time.perf_counter()
    data, prior = _c3_evaluator()
    gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    ev = inla.ObjectiveEvaluator(data.spec, prior=prior)
    setup = time.perf_counter() - t0
    th = np.array(TRI_THETA0)
    f, _ = ev.evaluate(th)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        inla.prior_cache_clear()  # time full evaluations (both factorizations)
        t0 = time.perf_counter()
        f, _ = ev.evaluate(th)
        times.append(time.perf_counter() - t0)
    print(json.dumps({
        "config": "C3 trivariate n_v=3 n_s=1675 n_t=48 n_r=1 m=80400/process; one f_obj at theta0",
        "generate_s": gen, "setup_s": setup, "f_obj_s_best": min(times), "f_obj_s": times,
        "f_obj": f, "oracle_f_obj": -193110.15144130366,
        "rel_err_vs_oracle": abs(f - (-193110.15144130366)) / 193110.15144130366,
    }), flush=True)


def c4(depth=1):
    G = torch.cuda.device_count()
    t0 = time.perf_counter()
    data, prior = _c3_evaluator()
    evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g))
           for g in range(G)]
    setup = time.perf_counter() - t0
    runner = sched.GpuRunner(evs, depth=depth)
    th = np.array(TRI_THETA0)
    pts = [th] + [th + s * 1e-3 * e for e in np.eye(15) for s in (1, -1)]
    runner.evaluate_points(pts[:G])  # warm every device
    inla.prior_cache_clear()
    t0 = time.perf_counter()
    vals = runner.evaluate_points(pts)
    batch = time.perf_counter() - t0
    print(json.dumps({
        "config": f"C4: 31 f_obj of C3 at theta0 round-robin over {G} GPUs (depth {depth})",
        "n_gpus": G, "setup_s": setup, "batch_s": batch, "per_fobj_s": batch / len(pts) * G,
        "f_center": vals[0],
    }), flush=True)


def c3post():
    """C3 after the mode search (BASELINE configs[2]): the
    finite-difference Hessian at the mode (1 + 2d + 2d(d-1) = 451 f_obj over
    every visible GPU) and the latent marginals (POBTAS + POBTASI of Q_c)."""
    G = torch.cuda.device_count()
    data, prior = _c3_evaluator()
    evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g))
           for g in range(G)]
    runner = sched.GpuRunner(evs)
    # the mode of the full C3 fit (tools/c3_fit.py: the last recorded BFGS state)
    th = np.load(os.path.join(os.path.dirname(__file__), "..", "bench_data",
                              "c3_bfgs_states.npz"))["theta"][-1]
    runner.evaluate_points([th] * G)
    inla.prior_cache_clear()
    t0 = time.perf_counter()
    hess = inla.fd_hessian(evs[0], th, 1e-2, runner)
    t_h = time.perf_counter() - t0
    t0 = time.perf_counter()
    mean, sd = evs[0].latent_marginals(th)
    t_m = time.perf_counter() - t0
    try:
        np.linalg.cholesky(hess)
        theta_sd = np.sqrt(np.diagonal(np.linalg.inv(hess))).tolist()
    except np.linalg.LinAlgError:
        theta_sd = None
    print(json.dumps({
        "config": f"C3 at the mode: fd_hessian (451 f_obj) over {G} GPUs + latent marginals",
        "n_gpus": G, "hessian_s": t_h, "latent_marginals_s": t_m, "theta_sd": theta_sd,
        "latent_sd_range": [float(sd.min()), float(sd.max())],
    }), flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "c1"
    if which == "c1":
        c1()
    elif which == "c3":
        c3()
    elif which == "c3post":
        c3post()
    else:
        c4(int(sys.argv[2]) if len(sys.argv) > 2 else 1)

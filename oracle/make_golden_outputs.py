"""Golden files of the reference's output writers (dataio.write_summary_json,
write_latent_csv, the cli trace table) for a fixed small summary, from the
UNMODIFIED reference -- development container only.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_outputs.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "outputs")


def main():
    sys.path.insert(0, REF)
    from stinla import dataio
    from stinla.inla import HyperParams, IterationRecord, PosteriorSummary
    from stinla.synthetic import SyntheticSettings, generate_synthetic

    os.makedirs(OUT, exist_ok=True)
    data = generate_synthetic(SyntheticSettings(2, 3, 2, 1, 10), [0.1] * 9, seed=5)
    spec = data.spec
    rng = np.random.default_rng(3)
    mean = rng.normal(size=spec.joint_dim)
    sd = rng.uniform(0.1, 1.0, size=spec.joint_dim)
    theta = HyperParams(np.linspace(-0.5, 0.5, 9), 2)
    summary = PosteriorSummary(theta_mode=theta, theta_sd=np.linspace(0.1, 0.9, 9), latent_mean=mean,
                               latent_sd=sd, logpost_at_mode=-123.456789, iterations=7,
                               f_evals=321, status="converged (gradient)", theta_hessian=np.eye(9))
    dataio.write_summary_json(os.path.join(OUT, "summary.json"), summary, extra={"seed": 5})
    dataio.write_latent_csv(os.path.join(OUT, "latent.csv"), spec, mean, sd)
    trace = [IterationRecord(1, -100.5, 3.25, 0.5, 40, 0.125), IterationRecord(2, -120.25, 0.5, 1.0, 32, 0.0625)]
    dataio.write_table(os.path.join(OUT, "trace.csv"),
                       ["iteration", "f", "grad_norm", "step", "f_evals", "seconds"],
                       [(r.iteration, r.f, r.grad_norm, r.step, r.f_evals, r.seconds) for r in trace])
    np.savez(os.path.join(OUT, "inputs.npz"), mean=mean, sd=sd)
    print("ok")


if __name__ == "__main__":
    main()

"""Golden vectors for the north-star model itself:
trivariate coregional n_v=3, n_s=1675, n_t=48, n_r=1, 80 400 observations per
process, seed 2, theta0 / theta_true of pkg/configs/trivariate.ini:14-15, prior
N(theta0, 2^2) (trivariate.ini:16).  Everything is computed by the UNMODIFIED
reference (stinla): its generate_synthetic (once, in the parent), then one
evaluate at theta0 (f_obj and the conditional mean) and the 31-point
central-difference gradient batch of fd_gradient (inla.py:418-437), every
task value kept.  Test infrastructure only.

A C3 f_obj costs the reference 6-20 minutes of CPU, so the 32 evaluations
run in parallel worker processes (the f_obj of a point does not depend on
where it runs; the task values are reduced exactly as fd_gradient does).
The reference is taken from $STINLA_REF (default /root/reference/pkg/src;
on the GPU box's 32-core host: baseline/_ref, the pip-installed copy):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_c3.py [workers] [threads] [jobdir] [jobs]

Job 0 is the evaluate at theta0, job k >= 1 the gradient's task k-1.  Each
finished job is also written to ``jobdir`` (default: none) as job_<k>.npz;
jobs already present there are not recomputed, so a run cut short by a time
limit can be resumed.  ``jobs`` (comma list) restricts the run to a subset;
the fixture then holds NaN for the task values not computed yet and the
gradient only for the coordinates whose two values are present (the test
checks exactly what is there).  ``oracle/golden_c3_jobs.txt`` records the
values of jobs computed in earlier runs (repr, exact), which are seeded
into ``jobdir``.

Output: tests/golden/c3.npz (no model inputs -- they are 10^5-sized; the
tests rebuild them with the package's generator and check the stored input
checksums first).
"""

import os
import pickle
import sys
import tempfile
import time

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
REF = os.environ.get("STINLA_REF", "/root/reference/pkg/src")

THETA0 = np.array([-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05,
                   0.05, 0.65, -0.35, 0.35])
THETA_TRUE = np.array([-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00,
                       0.00, 0.60, -0.40, 0.30])
STEP = 1e-3
# latent entries sampled for the mean check (joint variable-major indices)
MU_SAMPLE = np.unique(np.concatenate([np.arange(0, 241203, 997), [241200, 241201, 241202]]))


def input_checksums(spec):
    """Order-sensitive fingerprints of the generated model inputs."""
    out = []
    for a, y in zip(spec.design, spec.observations):
        a = a.tocsr()
        w = np.arange(1, a.nnz + 1, dtype=np.float64)
        out += [float(np.sum(y)), float(np.sum(y * np.arange(1, y.size + 1))),
                float(np.sum(a.indices * w)), float(np.sum(a.data * w))]
    return np.array(out)


def _points():
    """fd_gradient's task order (inla.py:428-436): centre, then +h / -h per
    coordinate."""
    pts = [THETA0.copy()]
    for i in range(THETA0.size):
        for sign in (1.0, -1.0):
            p = THETA0.copy()
            p[i] += sign * STEP
            pts.append(p)
    return pts


def _worker(args):
    spec_path, k, threads = args
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    sys.path.insert(0, REF)
    from threadpoolctl import threadpool_limits

    from stinla.inla import ObjectiveEvaluator, ThetaPrior

    with open(spec_path, "rb") as fh:
        spec = pickle.load(fh)
    with threadpool_limits(threads):
        ev = ObjectiveEvaluator(spec, prior=ThetaPrior.for_dim(15, mean=THETA0, sd=2.0))
        t0 = time.perf_counter()
        if k == 0:
            f, mu = ev.evaluate(THETA0)
            return k, f, mu[MU_SAMPLE], float(mu.sum()), time.perf_counter() - t0
        # the gradient's task k-1: the minimized (negated) objective
        f = -ev.objective(_points()[k - 1])
        return k, f, None, None, time.perf_counter() - t0


def main():
    import multiprocessing as mp

    workers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, (os.cpu_count() or 2) // workers)
    jobdir = sys.argv[3] if len(sys.argv) > 3 else None
    want = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else list(range(32))
    res = {}
    if jobdir:
        os.makedirs(jobdir, exist_ok=True)
        seeds = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_c3_jobs.txt")
        job0 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_c3_job0.npz")
        if os.path.exists(job0) and not os.path.exists(os.path.join(jobdir, "job_0.npz")):
            z = np.load(job0)  # the evaluate at theta0 (f, sampled mean) of an earlier run
            np.savez(os.path.join(jobdir, "job_0.npz"), f=z["f"], mu=z["mu"], mus=z["mus"],
                     secs=z["secs"])
        if os.path.exists(seeds):  # values of earlier runs: "k value seconds" per line
            for line in open(seeds):
                f = line.split()
                if len(f) == 3 and not os.path.exists(os.path.join(jobdir, f"job_{f[0]}.npz")):
                    np.savez(os.path.join(jobdir, f"job_{f[0]}.npz"), f=np.array([float(f[1])]),
                             secs=np.array([float(f[2])]))
        for k in range(32):
            path = os.path.join(jobdir, f"job_{k}.npz")
            if os.path.exists(path):
                z = np.load(path)
                res[k] = (float(z["f"][0]), z["mu"] if k == 0 else None,
                          float(z["mus"][0]) if k == 0 else None, float(z["secs"][0]))
        print(f"resuming: {len(res)} jobs already done", flush=True)
    sys.path.insert(0, REF)
    from stinla.synthetic import SyntheticSettings, generate_synthetic

    t0 = time.perf_counter()
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), THETA_TRUE, seed=2)
    t_gen = time.perf_counter() - t0
    print(f"reference generate_synthetic: {t_gen:.1f} s", flush=True)
    tmp = tempfile.NamedTemporaryFile(suffix=".pkl", delete=False)
    pickle.dump(data.spec, tmp)
    tmp.close()
    jobs = [(tmp.name, k, threads) for k in want if k not in res]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(workers) as pool:
        for k, f, mu, mus, secs in pool.imap_unordered(_worker, jobs):
            res[k] = (f, mu, mus, secs)
            print(f"  job {k}: {f!r} ({secs:.1f} s)", flush=True)
            if jobdir:
                extra = {"mu": mu, "mus": np.array([mus])} if k == 0 else {}
                np.savez(os.path.join(jobdir, f"job_{k}.npz"), f=np.array([f]),
                         secs=np.array([secs]), checksums=input_checksums(data.spec), **extra)
    os.unlink(tmp.name)
    vals = np.array([res[k][0] if k in res else np.nan for k in range(1, 32)])
    if not np.isfinite(vals[0]) and 0 in res:
        # the gradient's centre task is -objective(theta0) = -(job 0's evaluate f)
        vals[0] = -res[0][0]
    grad = (vals[1::2] - vals[2::2]) / (2.0 * STEP)  # inla.py:436 (NaN where a value is missing)
    f0, mu, mus, _ = res[0]
    np.savez_compressed(
        os.path.join(OUT, "c3.npz"),
        theta0=THETA0, theta_true=THETA_TRUE, prior_sd=np.array([2.0]),
        settings=np.array([3, 1675, 48, 1, 80400, 2]),
        input_checksums=input_checksums(data.spec),
        f_obj=np.array([f0]), mu_index=MU_SAMPLE, mu=mu, mu_sum=np.array([mus]),
        grad_step=np.array([STEP]), task_values=vals, neg_f=np.array([vals[0]]), grad=grad,
        seconds=np.array([t_gen, time.perf_counter() - t0]),
        task_seconds=np.array([res[k][3] if k in res else np.nan for k in range(32)]),
        threads=np.array([workers, threads]),
    )
    print(f"c3 golden written: f_obj {f0!r}, {np.isfinite(vals).sum()} of 31 task values, "
          f"{np.isfinite(grad).sum()} gradient coordinates", flush=True)


if __name__ == "__main__":
    main()

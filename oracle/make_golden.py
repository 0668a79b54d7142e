"""Generate golden vectors from the UNMODIFIED reference (stinla) — run in the
development container only (it imports /root/reference/pkg/src, which does
not exist on the GPU box).  Output: tests/golden/*.npz (small, committed).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

Every fixture stores the model INPUTS produced by the reference generators
(designs, observations) next to the reference OUTPUTS, so tests rebuild the
exact same ModelSpec with this package's classes.
"""

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _spec_arrays(prefix, spec):
    out = {
        f"{prefix}dims": np.array(
            [spec.n_processes, spec.n_spatial, spec.n_time, spec.n_fixed], dtype=np.int64
        ),
        f"{prefix}fep": np.array([spec.fixed_effect_precision]),
    }
    for i, (a, y) in enumerate(zip(spec.design, spec.observations)):
        a = a.tocsr()
        out[f"{prefix}A{i}_indptr"] = a.indptr.astype(np.int64)
        out[f"{prefix}A{i}_indices"] = a.indices.astype(np.int64)
        out[f"{prefix}A{i}_data"] = a.data
        out[f"{prefix}A{i}_shape"] = np.array(a.shape, dtype=np.int64)
        out[f"{prefix}y{i}"] = np.asarray(y, dtype=np.float64)
    return out


def main():
    sys.path.insert(0, REF)
    import stinla
    from stinla import bta, bta_dist
    from stinla.inla import FitOptions, ObjectiveEvaluator, ThetaPrior, fd_gradient, fit, minimize
    from stinla.synthetic import SyntheticSettings, generate_synthetic

    os.makedirs(OUT, exist_ok=True)

    # ---- 1. sequential solver: factor, logdet, solve, selected inverse
    cases = [(1, 1, 0), (2, 1, 0), (3, 2, 1), (5, 3, 2), (4, 7, 3), (6, 16, 4), (3, 65, 2),
             (4, 40, 0), (2, 130, 5)]
    g = {}
    for k, (n, b, a) in enumerate(cases):
        rng = np.random.default_rng(900 + k)
        m = bta.random_spd_bta(rng, n, b, a)
        rhs = rng.normal(size=m.dim)
        rhs2 = rng.normal(size=(m.dim, 3))
        g[f"c{k}_shape"] = np.array([n, b, a])
        g[f"c{k}_input"] = m.data.copy()
        g[f"c{k}_rhs"] = rhs
        g[f"c{k}_rhs2"] = rhs2
        f = bta.factorize(m.copy())
        g[f"c{k}_has_arrow"] = np.array([int(f.has_arrow)])
        g[f"c{k}_factor"] = f.matrix.data.copy()
        g[f"c{k}_logdet"] = np.array([bta.logdet(f)])
        g[f"c{k}_solve"] = bta.solve(f, rhs)
        g[f"c{k}_solve2"] = bta.solve(f, rhs2)
        g[f"c{k}_fwd"] = bta.forward_substitute(f, rhs)
        g[f"c{k}_bwd"] = bta.backward_substitute(f, rhs)
        g[f"c{k}_sinv"] = bta.selected_invert(f).data.copy()
    g["ncases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(OUT, "bta_solver.npz"), **g)

    # ---- 2. partitioned solver vs sequential (plans + results)
    d = {}
    plans = [(13, 4, 1.0), (13, 4, 1.6), (24, 4, 1.6), (16, 4, 1.0), (768, 8, 1.6), (96, 2, 1.6)]
    for k, (n, p, lb) in enumerate(plans):
        d[f"plan{k}"] = np.array([n, p, lb])
        d[f"plan{k}_bounds"] = np.array(bta_dist.plan_partitions(n, p, lb).boundaries)
    dist_cases = [(12, 3, 1.6, 3, 2), (17, 4, 1.0, 2, 0), (24, 2, 1.6, 4, 1)]
    for k, (n, p, lb, b, a) in enumerate(dist_cases):
        rng = np.random.default_rng(1300 + k)
        m = bta.random_spd_bta(rng, n, b, a)
        rhs = rng.normal(size=m.dim)
        plan = bta_dist.plan_partitions(n, p, lb)
        f = bta_dist.d_factorize(m.copy(), plan)
        d[f"d{k}_case"] = np.array([n, p, lb, b, a])
        d[f"d{k}_input"] = m.data.copy()
        d[f"d{k}_rhs"] = rhs
        d[f"d{k}_logdet"] = np.array([bta_dist.d_logdet(f)])
        d[f"d{k}_solve"] = bta_dist.d_solve(f, rhs)
        d[f"d{k}_sinv"] = bta_dist.d_selected_invert(f).data.copy()
    d["nplans"] = np.array([len(plans)])
    d["ndist"] = np.array([len(dist_cases)])
    np.savez_compressed(os.path.join(OUT, "bta_dist.npz"), **d)

    # ---- 3. objective values / conditional means / gradients / marginals
    o = {}
    models = [
        ("uni", SyntheticSettings(1, 8, 5, 1, 60), np.array([0.3, 0.2, 0.4, 1.0]), 55,
         [np.array([0.55, -0.15, 0.7, 0.65]), np.zeros(4)]),
        ("tri", SyntheticSettings(3, 6, 4, 1, 40),
         np.concatenate([np.full(6, -0.3), np.full(3, 2.0), np.zeros(3), [0.6, -0.4, 0.3]]), 2,
         [np.concatenate([np.full(6, -0.25), np.full(3, 1.9), np.full(3, 0.05), [0.5, -0.3, 0.2]])]),
        ("biv0", SyntheticSettings(2, 5, 3, 0, 30),
         np.array([0.1, -0.1, 0.2, 0.0, 1.5, 1.2, 0.1, -0.2, 0.4]), 9,
         [np.array([0.15, -0.05, 0.25, 0.05, 1.4, 1.1, 0.0, -0.1, 0.3])]),
    ]
    for name, cfg, theta_true, seed, points in models:
        data = generate_synthetic(cfg, theta_true=theta_true, seed=seed)
        o.update(_spec_arrays(f"{name}_", data.spec))
        ev = ObjectiveEvaluator(data.spec)
        fs, mus, grads = [], [], []
        for p in points:
            f, mu = ev.evaluate(p)
            fs.append(f)
            mus.append(mu)
            grads.append(fd_gradient(ev.objective, p, 1e-3)[1])
        o[f"{name}_points"] = np.array(points)
        o[f"{name}_f"] = np.array(fs)
        o[f"{name}_mu"] = np.array(mus)
        o[f"{name}_grad"] = np.array(grads)
        mu_m, sd_m = ev.latent_marginals(points[0])
        o[f"{name}_sd"] = sd_m
        o[f"{name}_prior_mean"] = ev.prior.mean
        o[f"{name}_prior_sd"] = ev.prior.sd
    np.savez_compressed(os.path.join(OUT, "objective.npz"), **o)

    # ---- 4. end-to-end mode search: bundled univariate.ini and config C1
    e = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        runs = [
            ("ini", SyntheticSettings(1, 20, 10, 2, 300), np.array([0.3, 0.2, 0.5, 1.2]), 1,
             np.zeros(4), 10.0, 1e-3, 1e-12),
            ("c1", SyntheticSettings(1, 300, 12, 2, 3600), np.array([0.3, 0.2, 0.5, 1.2]), 1,
             np.zeros(4), 10.0, 1e-3, 1e-12),
        ]
        for name, cfg, theta_true, seed, theta0, psd, gtol, ftol in runs:
            data = generate_synthetic(cfg, theta_true=theta_true, seed=seed)
            e.update(_spec_arrays(f"{name}_", data.spec))
            ev = ObjectiveEvaluator(data.spec, prior=ThetaPrior.for_dim(4, mean=theta0, sd=psd))
            res = minimize(ev, theta0, gtol=gtol, ftol=ftol, max_iter=100)
            e[f"{name}_theta0"] = theta0
            e[f"{name}_opts"] = np.array([psd, gtol, ftol])
            e[f"{name}_theta"] = res.theta
            e[f"{name}_f"] = np.array([res.f])
            e[f"{name}_iters"] = np.array([res.iterations, res.f_evals])
            e[f"{name}_trace_f"] = np.array([r.f for r in res.trace])
            e[f"{name}_status"] = np.array([res.status])
    np.savez_compressed(os.path.join(OUT, "mode_search.npz"), **e)
    print("golden fixtures written to", os.path.abspath(OUT), "stinla", stinla.__version__)


if __name__ == "__main__":
    main()

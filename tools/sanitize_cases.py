"""Small invocations of every product kernel for compute-sanitizer
(memcheck / racecheck / synccheck): POBTAF (plain, padded stride, partial,
pipelined host upload), POBTAS (all modes, several RHS), POBTASI (plain,
streamed to host, seeded), the assembly / f_obj reductions and the coupling
products of the partitioned solve -- each checked against the numpy oracle so
a sanitizer run also proves the results.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [small|medium]
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import bta_np, inla_np  # noqa: E402
from paper_2507_06938_b200 import bta, bta_dist, inla  # noqa: E402
from paper_2507_06938_b200.synthetic import SyntheticSettings, build_spec  # noqa: E402


def solver_case(n, b, a, rng):
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    f = bta.factorize(bta.BTAMatrix(n, b, a, data))
    assert abs(bta.logdet(f) - bta_np.logdet(ref, n, b, a)) < 1e-9 * abs(bta_np.logdet(ref, n, b, a))
    rhs = rng.normal(size=(n * b + a, 3))
    assert np.allclose(bta.solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs), rtol=1e-9)
    assert np.allclose(bta.forward_substitute(f, rhs[:, 0]),
                       bta_np.forward(ref, n, b, a, has, rhs[:, 0]), rtol=1e-9)
    inv = bta.selected_invert(f).numpy()
    assert np.allclose(inv, bta_np.selected_invert(ref, n, b, a, has), rtol=1e-8, atol=1e-11)
    # pinned host round trip: pipelined upload + streamed inverse
    host = torch.from_numpy(data).pin_memory()
    f2 = bta.factorize(bta.BTAMatrix(n, b, a, host))
    out = torch.empty(data.size, dtype=torch.float64).pin_memory()
    inv2 = bta.selected_invert(f2, out=out)
    assert np.allclose(inv2.numpy(out=out), inv, rtol=1e-12, atol=1e-14)


def dist_case(n, b, a, P, rng):
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy()
    has = bta_np.factorize(ref, n, b, a)
    f = bta_dist.d_factorize(bta.BTAMatrix(n, b, a, data), bta_dist.plan_partitions(n, P))
    rhs = rng.normal(size=(n * b + a, 2))
    assert np.allclose(bta_dist.d_solve(f, rhs), bta_np.solve(ref, n, b, a, has, rhs), rtol=1e-9)
    assert np.allclose(bta_dist.d_selected_invert(f).numpy(),
                       bta_np.selected_invert(ref, n, b, a, has), rtol=1e-8, atol=1e-11)


def objective_case(rng):
    spec = build_spec(SyntheticSettings(2, 6, 4, 1, 30), rng)
    spec.observations = [rng.normal(size=30) for _ in range(2)]
    theta = np.linspace(-0.2, 0.3, inla.HyperParams.dim_for(2))
    for parts in (1, 2):
        ev = inla.ObjectiveEvaluator(spec, partitions=parts)
        f, mu = ev.evaluate(theta)
        fr, mur = inla_np.evaluate(spec, theta, ev.prior.mean, ev.prior.sd)
        assert abs(f - fr) <= 1e-9 * max(1.0, abs(fr)), (f, fr)
        assert np.allclose(mu, mur, rtol=1e-8, atol=1e-10)
        ev.latent_marginals(theta)


def main():
    size = sys.argv[1] if len(sys.argv) > 1 else "small"
    rng = np.random.default_rng(1)
    cases = [(3, 70, 2), (2, 130, 0), (4, 40, 5)]
    if size == "medium":
        cases += [(3, 640, 3), (2, 1300, 6)]
    for n, b, a in cases:
        solver_case(n, b, a, rng)
        print("solver ok", n, b, a, flush=True)
    dist_case(8, 70, 2, 3, rng)
    print("dist ok", flush=True)
    objective_case(rng)
    print("objective ok", flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()

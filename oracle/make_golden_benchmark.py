"""Golden rows of the reference CLI benchmark table (pkg/src/stinla/cli.py:174-229)
from the UNMODIFIED reference, run in the development container only.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_benchmark.py

Writes tests/golden/benchmark_rows.json: every (routine, P, lb, n, b, a, phase,
flop_count) of the default benchmark configuration (n=32, b=4, a=4,
partitions 1-4, lb 1.0 / 1.6, seed 1) -- the seconds column is machine time
and is not part of the fixture.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from stinla import bta, bta_dist
    from stinla.bta import OpCounter

    n, b, a, seed = 32, 4, 4, 1
    rng = np.random.default_rng(seed)
    matrix = bta.random_spd_bta(rng, n, b, a)
    prior_like = matrix.copy()
    prior_like.arrow[...] = 0.0
    prior_like.tip[...] = np.eye(a)
    rhs = rng.normal(size=matrix.dim)
    rows = []
    for lb in (1.0, 1.6):
        for p in (1, 2, 3, 4):
            if p > 1 and n < 2 * p:
                continue
            plan = bta_dist.plan_partitions(n, p, lb if p > 1 else 1.0)

            def record(routine, times, counter):
                for phase in sorted(times):
                    rows.append([routine, p, lb, n, b, a, phase, counter.flops])

            counter, times = OpCounter(), {}
            factor = bta_dist.d_factorize(matrix.copy(), plan, counter=counter, phase_times=times)
            record("factorize", times, counter)
            counter, times = OpCounter(), {}
            bta_dist.d_factorize(prior_like.copy(), plan, counter=counter, phase_times=times)
            record("factorize_bt", times, counter)
            counter, times = OpCounter(), {}
            bta_dist.d_solve(factor, rhs, counter=counter, phase_times=times)
            record("solve", times, counter)
            counter, times = OpCounter(), {}
            bta_dist.d_selected_invert(factor, counter=counter, phase_times=times)
            record("selected_invert", times, counter)
    with open(os.path.join(OUT, "benchmark_rows.json"), "w") as fh:
        json.dump({"config": {"n": n, "b": b, "a": a, "seed": seed}, "rows": rows}, fh, indent=0)
    print(f"{len(rows)} rows")


if __name__ == "__main__":
    main()

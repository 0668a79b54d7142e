"""Reference-compatible solver benchmark table on the device path.

Mirrors the reference CLI's ``benchmark`` command (pkg/src/stinla/cli.py:174-266,
SURVEY.md §8(f) f4): for every load-balance factor and partition count it runs
``d_factorize`` of a random SPD BTA matrix and of its prior-like copy (arrow
zeroed, identity tip), ``d_solve`` and ``d_selected_invert``, and writes
``benchmark.csv`` (plus the evaluation-layer ``task_trace.csv``,
cli.py:243-256) with the reference schema

    routine,P,lb,n,b,a,phase,seconds,flop_count

(one row per (routine, P, lb, phase); ``flop_count`` is the reference's
OpCounter model, floats written with ``repr`` as in dataio.write_table,
dataio.py:33-46).  Inputs come from the reference generator law
(bta.random_spd_bta, same seed and draw order), so the table is comparable
row by row with the reference CLI's output.

    python -m paper_2507_06938_b200.benchmark --out DIR [--n 32 --b 4 --a 4
        --partitions 1,2,3,4 --lb 1.0,1.6 --seed 1]
"""

import argparse
import csv
import os

import numpy as np
import torch

from . import bta, bta_dist, sched
from .bta import OpCounter
from .inla import load_balance_ratio

HEADER = ["routine", "P", "lb", "n", "b", "a", "phase", "seconds", "flop_count"]


def _cell(value):
    if isinstance(value, (float, np.floating)):
        return repr(float(value))
    return value


def write_table(path, header, rows):
    """Plain CSV with one header row, floats via repr (dataio.py:33-46)."""
    with open(path, "w", newline="") as handle:
        writer = csv.writer(handle)
        writer.writerow(header)
        for row in rows:
            writer.writerow([_cell(v) for v in row])


def run_benchmark(n=32, b=4, a=4, partitions=(1, 2, 3, 4), lb_values=(1.0, 1.6), seed=1,
                  out_dir=".", workers=1):
    """Rows of the reference benchmark table (cli.py:186-229) measured on the
    device path; writes ``out_dir/benchmark.csv`` and the evaluation-layer
    ``task_trace.csv`` (cli.py:243-256) and returns the rows."""
    rng = np.random.default_rng(seed)
    matrix = bta.random_spd_bta(rng, n, b, a)
    prior_like = matrix.copy()
    if a > 0:
        prior_like.arrow.zero_()
        prior_like.tip.copy_(torch.eye(a, dtype=prior_like.tip.dtype, device=prior_like.tip.device))
    rhs = rng.normal(size=matrix.dim)

    parts = sorted(set(partitions) | {1})
    rows = []
    for lb in lb_values:
        for p in parts:
            if p > 1 and n < 2 * p:
                continue
            plan = bta_dist.plan_partitions(n, p, lb if p > 1 else 1.0)

            def record(routine, times, counter, p=p, lb=lb):
                for phase, seconds in sorted(times.items()):
                    rows.append({"routine": routine, "P": p, "lb": lb, "n": n, "b": b, "a": a,
                                 "phase": phase, "seconds": seconds,
                                 "flop_count": counter.flops})

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

    os.makedirs(out_dir, exist_ok=True)
    write_table(os.path.join(out_dir, "benchmark.csv"), HEADER,
                [[r[k] for k in HEADER] for r in rows])

    # evaluation-layer trace (cli.py:243-256): one gradient-sized batch of 31
    # factorization tasks dealt over the worker pool, task i -> group i % g1
    small = bta.random_spd_bta(rng, max(2, n // 4), b, a)
    tasks = [(lambda m=small.copy(): bta.logdet(bta.factorize(m))) for _ in range(31)]
    trace = []
    sched.run_tasks(tasks, sched.allocate(workers, dim_theta=15), trace=trace)
    write_table(os.path.join(out_dir, "task_trace.csv"), ["task", "group", "round", "start", "stop"],
                [(r.index, r.group, r.round, r.start, r.stop) for r in trace])
    return rows


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", default=".")
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--a", type=int, default=4)
    ap.add_argument("--partitions", default="1,2,3,4")
    ap.add_argument("--lb", default="1.0,1.6")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--workers", type=int, default=1)
    args = ap.parse_args(argv)
    rows = run_benchmark(args.n, args.b, args.a,
                         tuple(int(v) for v in args.partitions.split(",")),
                         tuple(float(v) for v in args.lb.split(",")), args.seed, args.out,
                         args.workers)
    bta_flops = max(r["flop_count"] for r in rows if r["routine"] == "factorize" and r["P"] == 1)
    bt_flops = max(r["flop_count"] for r in rows if r["routine"] == "factorize_bt" and r["P"] == 1)
    print(f"benchmark: n={args.n} b={args.b} a={args.a}; factorization work ratio "
          f"{bta_flops / bt_flops:.4f} (asymptotic model "
          f"{1 + load_balance_ratio(args.b, args.a):.4f})")
    print(f"outputs: {os.path.join(args.out, 'benchmark.csv')}, "
          f"{os.path.join(args.out, 'task_trace.csv')}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""Reference-compatible benchmark table: the device path's
benchmark.csv has the reference CLI's schema and the same (routine, P, lb,
phase, flop_count) rows as the unmodified reference on the same inputs
(tests/golden/benchmark_rows.json, oracle/make_golden_benchmark.py)."""
import csv
import json
import os

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_benchmark_table_matches_reference_rows(cuda, tmp_path):
    from paper_2507_06938_b200 import benchmark

    gold = json.load(open(os.path.join(HERE, "golden", "benchmark_rows.json")))
    c = gold["config"]
    rows = benchmark.run_benchmark(c["n"], c["b"], c["a"], (1, 2, 3, 4), (1.0, 1.6), c["seed"],
                                   str(tmp_path))
    got = [[r["routine"], r["P"], r["lb"], r["n"], r["b"], r["a"], r["phase"], r["flop_count"]]
           for r in rows]
    assert got == gold["rows"]
    with open(tmp_path / "benchmark.csv") as fh:
        table = list(csv.reader(fh))
    assert table[0] == benchmark.HEADER
    assert len(table) == 1 + len(gold["rows"])
    assert all(float(r[7]) > 0 for r in table[1:])  # seconds
    # evaluation-layer trace (reference cli.py:243-256): 31 tasks dealt i -> i % g1
    rows = benchmark.run_benchmark(c["n"], c["b"], c["a"], (1,), (1.0,), c["seed"],
                                   str(tmp_path), workers=4)
    with open(tmp_path / "task_trace.csv") as fh:
        trace = list(csv.reader(fh))
    assert trace[0] == ["task", "group", "round", "start", "stop"]
    assert [int(r[0]) for r in trace[1:]] == list(range(31))
    assert [int(r[1]) for r in trace[1:]] == [i % 4 for i in range(31)]
    assert [int(r[2]) for r in trace[1:]] == [i // 4 for i in range(31)]

"""Host logic of the time-partitioned solver (S3): partition plans and
separators against the reference's golden plans (tests/test_bta_dist.py:31-38
and oracle/make_golden.py)."""

import warnings

import numpy as np
import pytest

from conftest import golden
from paper_2507_06938_b200 import bta_dist


def test_plans_match_reference_golden():
    g = golden("bta_dist.npz")
    for k in range(int(g["nplans"][0])):
        n, p, lb = g[f"plan{k}"]
        plan = bta_dist.plan_partitions(int(n), int(p), float(lb))
        assert plan.boundaries == tuple(int(x) for x in g[f"plan{k}_bounds"]), (n, p, lb)
        assert sum(plan.sizes) == n and min(plan.sizes) >= 2 - (p == 1)


def test_reference_test_goldens():
    # tests/test_bta_dist.py:31-38 of the reference
    assert bta_dist.plan_partitions(13, 4, 1.6).sizes == (4, 3, 3, 3)
    assert bta_dist.plan_partitions(24, 4, 1.6).sizes == (8, 6, 5, 5)
    assert bta_dist.plan_partitions(768, 8, 1.6).sizes == (142, 90, 90, 90, 89, 89, 89, 89)


def test_plan_errors_and_fallback():
    with pytest.raises(bta_dist.PlanError):
        bta_dist.plan_partitions(5, 3)
    with pytest.raises(bta_dist.PlanError):
        bta_dist.plan_partitions(8, 2, lb=0.5)
    with pytest.raises(bta_dist.PlanError):
        bta_dist.plan_partitions(8, 0)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        plan = bta_dist.plan_partitions_with_fallback(5, 4)
    assert plan.n_partitions == 2 and any("reducing partitions" in str(x.message) for x in w)


def test_separators_and_ranges():
    plan = bta_dist.plan_partitions(12, 3, 1.0)  # (0, 4, 8, 12)
    assert bta_dist._separators(plan) == [3, 4, 7, 8]
    assert bta_dist._partition_ranges(plan) == [(0, 3, None, 3), (5, 7, 4, 7), (9, 12, 8, None)]

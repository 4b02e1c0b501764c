"""Short-trajectory aggregation: the oracle's plain-loop aggregation pinned by
the SPEC examples, and the aggregated-vs-exact property S:332 on the oracle DP.  The device path
(kernel K10 + ragged weighted solve) is checked against these in tests/test_gpu_aggregate.py."""
import numpy as np

import oracle
from inputs import workloads as wl
from oracle.aggregate import aggregate, expand


def test_spec_example_and_identity():
    # [100, 5, 5, 5, 5], threshold 10, bucket 2 -> [100, (5, w2), (5, w2)]
    agg, w, st = aggregate([100, 5, 5, 5, 5.0], 10, 2)
    assert agg == [100, 5, 5] and w == [1, 2, 2] and st == [0, 1, 3, 5]
    # threshold 0 -> identity
    agg, w, st = aggregate([9, 7, 3.0], 0, 4)
    assert agg == [9, 7, 3] and w == [1, 1, 1] and st == [0, 1, 2, 3]
    # all below threshold, bucket = n -> one item of weight n
    agg, w, st = aggregate([3, 2, 1.0], 10, 3)
    assert agg == [3] and w == [3] and st == [0, 3]
    # a threshold equal to a length keeps that trajectory single (">= threshold" is long)
    agg, w, st = aggregate([8, 5, 5, 2, 1.0], 5, 2)
    assert agg == [8, 5, 5, 2] and w == [1, 1, 1, 2]
    assert expand([0, 1, 3], [0, 1, 3, 5]) == [0, 1, 5]


def test_aggregated_not_better_than_exact():
    """aggregated-DP makespan >= exact-DP makespan (a partition of the aggregated items is a
    partition of the trajectories with the same costs), and the expanded partition attains it."""
    prof = wl.float_profile(dtype="f64")
    for s in range(12):
        rng = np.random.default_rng(600 + s)
        L = wl.presort(wl.coding_lengths(rng, 12, 8).astype(np.float64))      # n = 96
        m = int(rng.integers(2, 9))
        thr = float(np.percentile(L, 60))
        agg, w, st = aggregate(list(L), thr, int(rng.integers(2, 6)))
        exact = oracle.solve(oracle.Problem(L, prof.T[:1], prof.F[:1], [0] * m))
        aggd = oracle.solve(oracle.Problem(agg, prof.T[:1], prof.F[:1], [0] * m, w=w))
        assert aggd["opt"] >= exact["opt"]
        full = expand(list(aggd["bounds"]), st)
        p = oracle.Problem(L, prof.T[:1], prof.F[:1], [0] * m)
        worst = max(oracle.group_cost(p, j, int(full[j - 1]), int(full[j])) for j in range(1, m + 1))
        assert worst == aggd["opt"]

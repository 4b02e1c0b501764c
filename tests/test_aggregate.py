"""Short-trajectory aggregation: host bucketing on CPU; the weighted DP
parity on the GPU lives in test_gpu_parity.py."""
import numpy as np

import oracle
from inputs import workloads as wl
from paper_2603_28101_b200.aggregate import aggregate_short, expand_boundaries


def test_spec_example_and_identity():
    # [100, 5, 5, 5, 5], threshold 10, bucket 2 -> [100, (5, w2), (5, w2)]
    agg, w, st = aggregate_short(np.array([100, 5, 5, 5, 5.0]), 10, 2)
    assert list(agg) == [100, 5, 5] and list(w) == [1, 2, 2] and list(st) == [0, 1, 3, 5]
    # threshold 0 -> identity
    agg, w, st = aggregate_short(np.array([9, 7, 3.0]), 0, 4)
    assert list(agg) == [9, 7, 3] and list(w) == [1, 1, 1]
    # all below threshold, bucket = n -> one item of weight n
    agg, w, st = aggregate_short(np.array([3, 2, 1.0]), 10, 3)
    assert list(agg) == [3] and list(w) == [3]
    assert list(expand_boundaries(np.array([0, 1, 3]), np.array([0, 1, 3, 5]))) == [0, 1, 5]


def test_aggregated_not_better_than_exact():
    """aggregated-DP makespan >= exact-DP makespan (a partition of the aggregated items is a
    partition of the trajectories with the same costs), and the expanded partition attains it."""
    prof = wl.float_profile(dtype="f64")
    for s in range(12):
        rng = np.random.default_rng(600 + s)
        L = wl.presort(wl.coding_lengths(rng, 12, 8).astype(np.float64))      # n = 96
        m = int(rng.integers(2, 9))
        thr = float(np.percentile(L, 60))
        agg, w, st = aggregate_short(L, thr, int(rng.integers(2, 6)))
        exact = oracle.solve(oracle.Problem(L, prof.T[:1], prof.F[:1], [0] * m))
        aggd = oracle.solve(oracle.Problem(agg, prof.T[:1], prof.F[:1], [0] * m, w=w))
        assert aggd["opt"] >= exact["opt"]
        full = expand_boundaries(aggd["bounds"], st)
        p = oracle.Problem(L, prof.T[:1], prof.F[:1], [0] * m)
        worst = max(oracle.group_cost(p, j, int(full[j - 1]), int(full[j])) for j in range(1, m + 1))
        assert worst == aggd["opt"]

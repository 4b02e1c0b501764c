"""Short-trajectory aggregation (§5.2) -- the paper's own
speed heuristic: after sorting, consecutive trajectories shorter than a threshold are bucketed
(at most `bucket` per item); each bucket is ONE DP item whose length is the bucket's maximum
(its first element, the list being sorted) and whose weight is its cardinality, so the group
size seen by F is the sum of weights (R5).  The weighted DP runs in the batched kernel
(heddle_place_problem.weights); `expand_boundaries` maps its partition back to trajectories.

Host-side index bookkeeping only (O(n) per problem); the DP arithmetic stays in the kernels.
"""
from __future__ import annotations

import numpy as np


def aggregate_short(lengths_sorted: np.ndarray, threshold: float, bucket: int):
    """lengths_sorted: [n] non-increasing.  Returns (agg_lengths [n'], weights [n'] int32,
    starts [n'+1] int64: item t covers trajectories [starts[t], starts[t+1])).
    threshold <= 0 is the identity."""
    L = np.asarray(lengths_sorted)
    n = L.shape[0]
    if bucket < 1:
        raise ValueError("bucket >= 1")
    long_cnt = int(np.sum(L >= threshold)) if threshold > 0 else n   # sorted: the long ones come first
    starts = list(range(long_cnt))
    starts += list(range(long_cnt, n, bucket))
    starts = np.asarray(starts + [n], dtype=np.int64)
    agg = L[starts[:-1]]
    w = np.diff(starts).astype(np.int32)
    return agg, w, starts


def expand_boundaries(agg_bounds: np.ndarray, starts: np.ndarray) -> np.ndarray:
    """Partition of the aggregated items -> partition of the trajectories (b_j -> starts[b_j])."""
    b = np.asarray(agg_bounds)
    out = np.where(b >= 0, starts[np.clip(b, 0, len(starts) - 1)], -1)
    return out.astype(np.int64)

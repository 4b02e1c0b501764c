"""TEST INFRASTRUCTURE -- short-trajectory aggregation as the paper and SPEC state it, written out
with plain loops (§5.2: "trajectories shorter than a threshold are aggregated
into a single item"; buckets of at most `bucket` consecutive short trajectories of
the sorted order, an item's length is its bucket's maximum and its weight the bucket's size, a
threshold <= 0 is the identity).  Independent of paper_2603_28101_b200 (kernel K10).
Pinned by the SPEC examples S:316-318 (tests/test_aggregate.py)."""
from __future__ import annotations


def aggregate(lengths_sorted, threshold, bucket):
    """lengths_sorted: non-increasing list.  Returns (items, weights, starts) with starts[t] the
    first trajectory of item t and starts[-1] = n."""
    if bucket < 1:
        raise ValueError("bucket >= 1")
    L = list(lengths_sorted)
    n = len(L)
    items, weights, starts = [], [], []
    t = 0
    while t < n:
        if threshold <= 0 or L[t] >= threshold:     # a long trajectory stays one item
            items.append(L[t])
            weights.append(1)
            starts.append(t)
            t += 1
        else:                                        # the short suffix: buckets of <= bucket
            size = min(bucket, n - t)
            items.append(max(L[t:t + size]))
            weights.append(size)
            starts.append(t)
            t += size
    starts.append(n)
    return items, weights, starts


def expand(agg_bounds, starts):
    """Boundaries over items -> boundaries over trajectories."""
    return [starts[b] if b >= 0 else -1 for b in agg_bounds]

"""TEST INFRASTRUCTURE -- plain migration logic from PAPER.md §5.3 and SPEC S:364-381.

retarget_one: walk the group sizes scaled by n*/n (ceiling, R18) and return the group covering the
rank; schedule: greedy, longest trajectory first, endpoint exclusive.  Written independently of
paper_2603_28101_b200/migration.py and its CUDA kernel."""
from __future__ import annotations

import math


def retarget_one(bounds, n_active, rank):
    n = bounds[-1]
    if n_active < 1 or not 0 <= rank < n_active:
        return -1
    sizes = [bounds[i + 1] - bounds[i] for i in range(len(bounds) - 1)]
    total = 0
    for i, s in enumerate(sizes):
        total += math.ceil(s * n_active / n)      # "effective capacity s_i * n*/n"
        if rank < total:
            return i
    return len(sizes) - 1                           # ceil overshoot clamp (SPEC decision)


def schedule(requests, busy=()):
    """requests: (id, src, dst, priority_len, issued_at) tuples."""
    taken, used = [], set(busy)
    order = sorted(requests, key=lambda r: (-r[3], r[4], r[0]))
    for r in order:
        if r[1] == r[2]:
            continue
        if r[1] in used or r[2] in used:
            continue
        taken.append(r[0])
        used.add(r[1])
        used.add(r[2])
    return taken

#!/usr/bin/env python
"""Short-trajectory aggregation: what the heuristic
costs in makespan and saves in DP time, on the paper's call shapes -- configs[1] rollout
(512, 32), the paper's §6.2 size (6400, 16) and configs[4] (65536, 256).

For each threshold (a percentile of the lengths) and the SPEC default bucket 8: aggregate on the
device (K10), solve the ragged weighted batch, and compare with the exact DP of the same problem:
  delta = aggregated makespan / exact makespan - 1   (>= 0 by S:332)
and the device time of each (CUDA events, median of --reps; the aggregated time includes the
aggregation and expansion kernels), for the O(n^2 m) scan -- the DP the paper's heuristic is for --
and for the exact valley solver (HEDDLE_VALLEY).  One instance per call: the aggregated item count
is read back and the items solved as an n'-item problem (a batch would pass ns instead).
    python bench/aggregation.py [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--bucket", type=int, default=8)
    args = ap.parse_args()
    import torch

    import __graft_entry__
    __graft_entry__.build()
    from inputs import workloads as wl
    from paper_2603_28101_b200 import aggregate as agg_mod
    from paper_2603_28101_b200.placer import Placer

    rng = np.random.default_rng(3)
    L6400 = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 800, 8))).astype(np.float32)[None, :]
    cfgs = [("rollout configs[1]", wl.config_rollout()),
            ("paper_6.2", wl.Batch("paper_6.2", 6400, 16, L6400, np.ones((1, 16), np.int32), wl.float_profile())),
            ("large configs[4]", wl.config_large())]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts), out

    for name, b in cfgs:
        L = torch.from_numpy(b.lengths).cuda()
        D = torch.from_numpy(b.degrees.astype(np.int32)).cuda()
        for algo in ("scan", "valley"):
            if algo == "scan" and b.n > 8192:
                continue   # the weighted scan needs one CTA per problem (n' too large here)
            pl = Placer.from_profile(b.profile, max_n=b.n, max_m=b.m, max_batch=1, algo=algo)

            def exact():
                o, _ = pl.solve(L, D)
                return o, pl.backtrack()
            t_exact, (o_ex, _) = timed(exact)
            ex = float(o_ex.cpu()[0])
            for pct in (50, 70, 90):
                thr = float(np.percentile(b.lengths[0], pct))
                a, w, st, na = agg_mod.aggregate(L, thr, args.bucket)
                k = int(na.cpu()[0])

                def aggregated():
                    a, w, st, _ = agg_mod.aggregate(L, thr, args.bucket)
                    o, s = pl.solve(a[:, :k], D, weights=w[:, :k])
                    return o, s, agg_mod.expand(pl.backtrack(), st)
                t_agg, (o_ag, s_ag, full) = timed(aggregated)
                ag = float(o_ag.cpu()[0])
                fb = full.cpu().numpy()[0]
                print(json.dumps({
                    "config": name, "algo": algo, "n": b.n, "m": b.m, "threshold_percentile": pct,
                    "threshold": thr, "bucket": args.bucket, "items": k, "status": int(s_ag.cpu()[0]),
                    "exact_makespan": ex, "aggregated_makespan": ag, "delta": ag / ex - 1.0,
                    "us_exact": round(t_exact, 1), "us_aggregated": round(t_agg, 1),
                    "expanded_boundaries_ok": bool(fb[0] == 0 and fb[-1] == b.n and np.all(np.diff(fb) > 0))}),
                    flush=True)
            pl.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-config timings of the placement DP (BASELINE.json configs + the paper's §6.2 size).

Not the driver's bench line (bench.py is): this records, for DESIGN.md and
profiles/, the device time of solve+backtrack for every configuration on one GPU,
with the kernel path the dispatcher picked, as cells/s and % of the ALU roofline.
    python bench/configs.py [--reps 5] [--only large]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default=None)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--algo", default="scan", help="scan (Eq. 3, every split) / valley (HEDDLE_VALLEY, min-max)")
    ap.add_argument("--dtype", default=None, help="override: f32 / f64 / u32 (integer profile, rounded lengths)")
    ap.add_argument("--semiring", default="minmax")
    ap.add_argument("--objective", action="store_true", help="time the objective-only parametric kernel (N3)")
    args = ap.parse_args()
    import torch

    import __graft_entry__
    __graft_entry__.build()
    from inputs import workloads as wl
    from paper_2603_28101_b200 import _lib
    from paper_2603_28101_b200.placer import Placer

    rng = np.random.default_rng(3)
    L6400 = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 800, 8))).astype(np.float32)[None, :]
    cfgs = {
        "tiny": wl.config_tiny(),
        "rollout": wl.config_rollout(),
        "tp_sweep": wl.config_tp_sweep(),
        "batched": wl.config_batched(),
        "large": wl.config_large(),
        "paper_6.2": wl.Batch("paper_6.2", 6400, 16, L6400, np.ones((1, 16), np.int32), wl.float_profile()),
    }
    peak = 148 * 4 * 32 / 3 * 1965e6
    for name, b in cfgs.items():
        if args.only and name != args.only:
            continue
        if args.dtype == "u32":
            b.profile = wl.int_profile()
            b.lengths = np.minimum(np.rint(b.lengths.astype(np.float64)), wl.MAX_TOKENS).clip(1).astype(np.uint32)
        elif args.dtype == "f64":
            b.profile = wl.float_profile(dtype="f64")
            b.lengths = b.lengths.astype(np.float64)
        pl = Placer.from_profile(b.profile, max_n=b.n, max_m=b.m, max_batch=b.B, kernel=args.kernel,
                                 semiring=args.semiring, algo=args.algo)
        dt = {"u32": torch.uint32, "f32": torch.float32, "f64": torch.float64}[b.profile.dtype]
        L = torch.from_numpy(b.lengths).to(dt).cuda()
        D = torch.from_numpy(b.degrees.astype(np.int32)).cuda()
        if args.objective:
            for _ in range(2):
                pl.objective(L, D)
            torch.cuda.synchronize()
            ts_ = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pl.objective(L, D)
                e1.record()
                torch.cuda.synchronize()
                ts_.append(e0.elapsed_time(e1) / 1e3)
            t = float(np.median(ts_))
            print(json.dumps({"config": name, "n": b.n, "m": b.m, "B": b.B, "kernel": "k7_parametric (objective only)",
                              "ms": 1e3 * t, "solves_per_s": b.B / t,
                              "dp_equivalent_cells_per_s": b.B * _lib.transitions(b.n, b.m) / t}), flush=True)
            pl.close()
            continue
        for _ in range(2):
            pl.solve(L, D)
            pl.backtrack()
        torch.cuda.synchronize()
        times, tsolve = [], []
        l0 = pl.launches
        for _ in range(args.reps):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            pl.solve(L, D)
            e2.record()
            pl.backtrack()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            tsolve.append(e0.elapsed_time(e2) / 1e3)
        t = float(np.median(times))
        ts = float(np.median(tsolve))
        W = b.B * _lib.transitions(b.n, b.m)
        print(json.dumps({"config": name, "n": b.n, "m": b.m, "B": b.B, "dtype": b.profile.dtype,
                          "semiring": args.semiring, "algo": args.algo,
                          "ms": 1e3 * t, "ms_solve": 1e3 * ts, "ms_backtrack": 1e3 * (t - ts), "cells": W, "cells_per_s": W / t, "solves_per_s": b.B / t,
                          "frac_alu_roofline": W / t / peak if args.algo == "scan" else None,
                          "launches_per_solve": (pl.launches - l0) / args.reps}), flush=True)
        pl.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Writes tests/golden/large_f32.npz: the CPU oracle's solution of BASELINE.json configs[4]
(one n = 65536 coding-like instance into m = 256 workers, FP32 costs, Eq. 3 min-max); with
--mode f64 --semiring minplus --out tests/golden/large_f64_minplus.npz the FP64 min-plus solution
of the same instance (the reference for the FP64-accumulated min-plus mode).

Calls only oracle/ (the plain FP64-emulating-FP32 DP of P:592-616, ora_solve_threads: the columns
of each layer shared over OpenMP threads, arithmetic and k order unchanged) and the seeded input
generator inputs/workloads.py.  Nothing here touches the CUDA path.  Stored:

  opt, bounds           the objective dp[m][n] and the canonical boundaries b_0..b_m (R3)
  qj, qi, dp, parent    sampled states: every state on the optimal path, both ends of each layer's
                        computed range [j, n-m+j] (R8) and 48 seeded columns per layer; dp[j][i] and
                        the lowest-index back-pointer parent[j][i] of each
  lengths_sha256        hash of the generated lengths (the test regenerates them and checks it)

Run time: about 17 minutes on 8 cores (5.4e11 transitions).  Usage:
    python tests/golden/make_large_golden.py [--threads N]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from inputs import workloads as wl  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large_f32.npz")
SAMPLES_PER_LAYER = 48
SEED = 0x4C41524745   # "LARGE"


def sample_states(n, m, bounds, seed=SEED):
    rng = np.random.default_rng(seed)
    qj, qi = [], []
    for j in range(1, m + 1):
        lo, hi = (n, n) if j == m else (j, n - m + j)
        cols = {lo, hi, int(bounds[j])}
        cols.update(int(c) for c in rng.integers(lo, hi + 1, size=SAMPLES_PER_LAYER))
        for c in sorted(cols):
            qj.append(j)
            qi.append(c)
    return np.array(qj, dtype=np.int32), np.array(qi, dtype=np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--out", default=OUT)
    ap.add_argument("--mode", default="f32", help="oracle arithmetic: f32 (F32 emulation, the default file), f64")
    ap.add_argument("--semiring", default="minmax", choices=["minmax", "minplus"])
    args = ap.parse_args()
    batch = wl.config_large(n=args.n, m=args.m)
    p = oracle.Problem.from_batch(batch, 0, mode=args.mode,
                                  semiring=oracle.MINMAX if args.semiring == "minmax" else oracle.MINPLUS)
    t = time.time()
    ref = oracle.solve(p, want_tables=True, threads=args.threads)
    dt = time.time() - t
    assert ref["status"] == oracle.OK, ref["status"]
    n, m = batch.n, batch.m
    qj, qi = sample_states(n, m, ref["bounds"])
    np.savez_compressed(
        args.out, opt=np.float64(ref["opt"]), bounds=ref["bounds"].astype(np.int32), qj=qj, qi=qi,
        dp=ref["dp"][qj, qi], parent=ref["parent"][qj, qi].astype(np.int32),
        n=np.int32(n), m=np.int32(m),
        lengths_sha256=np.array(hashlib.sha256(np.ascontiguousarray(batch.lengths).tobytes()).hexdigest()),
        oracle_seconds=np.float64(dt), threads=np.int32(args.threads), mode=np.array(args.mode),
        semiring=np.array(args.semiring))
    print(f"wrote {args.out}: opt {ref['opt']!r}, {qj.size} sampled states, oracle {dt:.0f} s on "
          f"{args.threads} threads")


if __name__ == "__main__":
    main()

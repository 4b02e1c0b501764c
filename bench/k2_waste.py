#!/usr/bin/env python
"""Executed vs algorithmic cells of K2's task geometry: replays the column blocks and
split quarters of dp_batched.cuh for one (n, m) and splits the surplus into its causes.
    python bench/k2_waste.py [--n 1024] [--m 32]
"""
import argparse
import json


def align4(x):
    return (x + 3) & ~3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--m", type=int, default=32)
    a = ap.parse_args()
    n, m = a.n, a.m
    W = 2 * (n - m + 1) + (m - 2) * (n - m + 1) * (n - m + 2) // 2
    ex = rnd = tri = out = 0
    for j in range(2, m):
        imax_layer = n - m + j
        ctop = align4(imax_layer - 63)
        nblk = (ctop + 63 - j) // 64 + 1
        kstart = (j - 1) & ~3
        for t in range(nblk):
            cb = ctop - 64 * t
            imax = min(cb + 63, imax_layer)
            kend = align4(imax)
            Q = 4 * ((kend - kstart + 15) // 16)
            ex += 64 * 4 * Q
            rnd += 64 * (4 * Q - (kend - kstart))
            for c in range(cb, cb + 64):
                if c < j or c > imax_layer:
                    out += kend - kstart
                else:
                    tri += max(0, kend - max(c, kstart))
                    out += max(0, (j - 1) - kstart)
    # the first and last layers run outside the task geometry (one state / one split per column)
    print(json.dumps({"n": n, "m": m, "W": W, "executed_over_W": (ex + 2 * (n - m + 1)) / W,
                      "triangle": tri / W, "rounding_to_16_splits": rnd / W, "outside_columns_and_start": out / W}))


if __name__ == "__main__":
    main()

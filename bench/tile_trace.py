"""Summarise a K5 per-tile timeline written under HEDDLE_PLACE_TILE_TRACE=<file> (diagnostics).

Each record: int64 {ntiles, B, kc, grid, rank, world}; int4 tiles[nentries] = {j, blk | nch << 16, k0, k1};
u64 times[ntiles][6] = %globaltimer (ns) at: start (tile index known), L and G staged (thread 0's share),
row j-1 dependencies met, dp staged, swept, published.
Tile t is entry t // B of problem t % B.

    python bench/tile_trace.py <file> [--record -1]
"""
from __future__ import annotations

import argparse
import json

import numpy as np


def records(path):
    raw = open(path, "rb").read()
    off = 0
    while off < len(raw):
        ntiles, B, kc, grid, rank, world = np.frombuffer(raw, np.int64, 6, off)
        off += 48
        nent = int(ntiles) // int(B)
        tiles = np.frombuffer(raw, np.int32, 4 * nent, off).reshape(nent, 4)
        off += 16 * nent
        t = np.frombuffer(raw, np.uint64, 6 * int(ntiles), off).reshape(int(ntiles), 6).astype(np.int64)
        off += 48 * int(ntiles)
        yield dict(ntiles=int(ntiles), B=int(B), kc=int(kc), grid=int(grid), rank=int(rank), world=int(world),
                   tiles=tiles, t=t)


PHASES = ["stage L,G", "wait row j-1", "stage dp", "sweep", "publish"]


def summarise(r):
    t = r["t"]
    t = t - t[:, 0].min()
    ent = np.repeat(r["tiles"], r["B"], axis=0)
    j = ent[:, 0]
    span = t[:, 5].max()
    slots = r["grid"] * span
    ph = np.diff(t, axis=1)                       # [tiles][5] phase durations
    share = {p: float(ph[:, i].sum() / slots) for i, p in enumerate(PHASES)}
    share["between tiles"] = 1.0 - sum(share.values())
    layers = np.unique(j)
    done = np.array([t[j == k, 5].max() for k in layers])
    dj = np.diff(done)
    return {
        "tiles": r["ntiles"], "B": r["B"], "kc": r["kc"], "grid": r["grid"], "rank": r["rank"], "world": r["world"],
        "span_us": span / 1e3,
        "cta_time_share": share,
        "tile_us_median": {p: float(np.median(ph[:, i]) / 1e3) for i, p in enumerate(PHASES)},
        "tile_us_mean": {p: float(ph[:, i].mean() / 1e3) for i, p in enumerate(PHASES)},
        "layer_done_step_us": {"median": float(np.median(dj) / 1e3), "mean": float(dj.mean() / 1e3),
                               "max": float(dj.max() / 1e3)},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--record", type=int, default=-1)
    args = ap.parse_args()
    recs = list(records(args.path))
    print(json.dumps(summarise(recs[args.record]), indent=1))


if __name__ == "__main__":
    main()

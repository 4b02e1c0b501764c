"""Summarise a K5 per-tile timeline written under HEDDLE_PLACE_TILE_TRACE=<file> (diagnostics).

Each record: int64 {ntiles, B, kc, grid, rank, world}; int4 tiles[nentries] = {j, blk, q, nch};
u64 times[ntiles][4] = %globaltimer (ns) at dequeue, dependencies met, staged, done.
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
        t = np.frombuffer(raw, np.uint64, 4 * int(ntiles), off).reshape(int(ntiles), 4).astype(np.int64)
        off += 32 * int(ntiles)
        yield dict(ntiles=int(ntiles), B=int(B), kc=int(kc), grid=int(grid), rank=int(rank), world=int(world),
                   tiles=tiles, t=t)


def summarise(r):
    t = r["t"]
    t = t - t[:, 0].min()
    ent = np.repeat(r["tiles"], r["B"], axis=0)
    j = ent[:, 0]
    span = t[:, 3].max()
    wait = (t[:, 1] - t[:, 0]).sum()
    stage = (t[:, 2] - t[:, 1]).sum()
    work = (t[:, 3] - t[:, 2]).sum()
    slots = r["grid"] * span
    layers = np.unique(j)
    done = np.array([t[j == k, 3].max() for k in layers])
    first = np.array([t[j == k, 0].min() for k in layers])
    dj = np.diff(done)
    # the tile whose completion ends each layer, and how long it waited / computed
    last = [np.flatnonzero(j == k)[np.argmax(t[j == k, 3])] for k in layers]
    lw = np.array([t[i, 1] - t[i, 0] for i in last])
    ls = np.array([t[i, 2] - t[i, 1] for i in last])
    lc = np.array([t[i, 3] - t[i, 2] for i in last])
    return {
        "tiles": r["ntiles"], "B": r["B"], "kc": r["kc"], "grid": r["grid"], "rank": r["rank"], "world": r["world"],
        "span_us": span / 1e3,
        "cta_time_share": {"waiting": wait / slots, "staging": stage / slots, "sweep+publish": work / slots,
                           "idle (no tile)": 1 - (wait + stage + work) / slots},
        "tile_us_median": {"wait": float(np.median(t[:, 1] - t[:, 0]) / 1e3),
                           "stage": float(np.median(t[:, 2] - t[:, 1]) / 1e3),
                           "sweep+publish": float(np.median(t[:, 3] - t[:, 2]) / 1e3)},
        "layer_done_step_us": {"median": float(np.median(dj) / 1e3), "mean": float(dj.mean() / 1e3),
                               "max": float(dj.max() / 1e3)},
        "layer_last_tile_us_median": {"wait": float(np.median(lw) / 1e3), "stage": float(np.median(ls) / 1e3),
                                      "sweep+publish": float(np.median(lc) / 1e3)},
        "layers_in_flight_median": float(np.median([(first <= x).sum() - (done < x).sum()
                                                    for x in np.linspace(0, span, 200)])),
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

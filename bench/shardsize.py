"""Per-GPU throughput of the batched sweep at the shard sizes bench.py --gpus N gives each rank
(16384 / N problems of configs[3]), on one GPU: how much the last partial wave of K2 costs at
N = 8 (2048 problems = 3.46 waves of 148 SMs x 4 CTAs).  Diagnostics, not a bench line.

    python bench/shardsize.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from inputs import workloads as wl
    from paper_2603_28101_b200.placer import Placer
    full = wl.config_batched()
    dev = torch.device("cuda", 0)
    Lall = torch.from_numpy(full.lengths).to(dev)
    Dall = torch.from_numpy(full.degrees).to(dev)
    pl = Placer.from_profile(full.profile, max_n=full.n, max_m=full.m, max_batch=full.B, device=0)
    for N in (1, 2, 4, 8, 16):
        B = full.B // N
        L, D = Lall[:B].contiguous(), Dall[:B].contiguous()
        for _ in range(3):
            pl.solve(L, D)
            pl.backtrack()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            pl.solve(L, D)
            pl.backtrack()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"gpus_emulated": N, "problems_per_gpu": B, "ms": ms, "us_per_problem": 1e3 * ms / B,
                          "waves_of_592": B / 592}))


if __name__ == "__main__":
    main()

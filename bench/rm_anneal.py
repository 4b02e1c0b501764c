#!/usr/bin/env python
"""Resource-manager simulated annealing (Alg. 2) with batched GPU PresortedDP evaluations.

Paper-sized instance (inferred: 64 GPUs x batch 100 = 6400 trajectories), budget
N = 64 GPUs over MP degrees {1,2,4,8}, alpha = 0.95, eps = 1e-3 T0 (SPEC defaults), P parallel
chains.  The paper's resource manager takes 4.97-5.69 s for one chain on its CPU.
    python bench/rm_anneal.py [--chains 64] [--n 6400]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chains", type=int, default=64)
    ap.add_argument("--n", type=int, default=6400)
    ap.add_argument("--budget", type=int, default=64)
    ap.add_argument("--objective-only", action="store_true", help="makespans by the parametric kernel (N3)")
    ap.add_argument("--algo", default="valley", help="DP solver: valley (N3) or scan (Eq. 3 as written)")
    ap.add_argument("--impl", default="device", choices=["device", "host"],
                    help="device: the whole walk on the GPU (heddle_place_anneal, K9 + ragged solves, CUDA graph); "
                         "host: moves and Metropolis in Python, one solve per distinct worker count")
    args = ap.parse_args()
    import torch

    import __graft_entry__
    __graft_entry__.build()
    from inputs import workloads as wl
    from paper_2603_28101_b200 import allocator as alloc
    rng = wl.rng_for(7)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, args.n // 8, 8)))
    prof = wl.float_profile()
    cfg = alloc.SAConfig(budget=args.budget, m_min=8, m_max=args.budget)
    iu, su = wl.sa_uniforms(11, args.chains, cfg.max_iters)
    rm = alloc.ResourceManager(prof, n_max=args.n, m_max=cfg.m_max, chains=args.chains,
                               objective_only=args.objective_only, algo=args.algo)
    run = rm.anneal if args.impl == "device" else rm.anneal_host
    run(L, alloc.SAConfig(budget=args.budget, m_min=8, m_max=args.budget, max_iters=3), iu, su)  # warm-up
    torch.cuda.synchronize()
    rm.evaluations = 0
    t = time.perf_counter()
    res = run(L, cfg, iu, su)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    homog = {d: rm.makespans(torch.from_numpy(L).cuda(), [tuple([d] * (args.budget // d))])[0][0]
             for d in (1, 2, 4, 8) if args.budget // d >= 8}
    print(json.dumps({"impl": args.impl, "n": args.n, "budget": args.budget, "chains": args.chains,
                      "iterations": res.iterations,
                      "evaluator": "parametric objective (N3)" if args.objective_only else f"DP solve ({args.algo}) + backtrack",
                      "evaluations": res.evaluations, "wall_s": dt, "dp_evals_per_s": res.evaluations / dt,
                      "best_makespan_s": res.best_makespan, "best_degrees": list(res.best_degrees),
                      "homogeneous_makespans_s": homog,
                      "paper_rm_seconds_one_chain": "4.97-5.69 s on the paper's control-plane CPU (P:1088)"}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the presorted-DP placement hot path (Heddle, §5.2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[3], the metric's batched sweep): 16384 independent
placement problems, n = 1024 sorted predicted trajectory lengths into m = 32
workers with random sorted MP degrees over {1,2,4,8}, FP32 costs, Eq. 3 min-max.
A step = one pass of the whole hot path over the batch: validation + cost tables +
every DP layer (heddle_place_solve) and the backtrack (heddle_place_backtrack).
With N GPUs (torchrun, one process per GPU) the 16384 problems are block-sharded
across ranks with no collective (strong scaling: fixed total work).

value = DP cells/s = (problems x W(n, m)) / device time, W = the (state, split)
transitions of Eq. 3 (include/heddle_place.h).  `--impl reference` times the CPU
oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "placement-DP cells/s and solves/s at 1/2/4/8 B200; % of HBM/ALU roofline"
B_TOTAL, N, M = 16384, 1024, 32
WORKLOAD = ("batched sweep (BASELINE configs[3]): 16384 independent N=1024 K=32 placement problems, "
            "coding(Pareto)/search(log-normal) families alternating, predicted FP32 lengths, random sorted "
            "MP degrees over {1,2,4,8}, Eq. 3 min-max")
LARGE_WORKLOAD = ("single large instance (BASELINE configs[4]): N=65536 coding-like predicted lengths into "
                  "K=256 workers, FP32, Eq. 3 min-max")
SM_COUNT = 148
ISSUE_SLOTS_PER_CELL = 3   # ALU cycles per warp-transition: FMNMX (2) + half an FMNMX3 (1); profiles/r01_alu_peaks.jsonl


def transitions(n, m):
    """W(n, m): the (state, split) transitions of Eq. 3 on the computed region (SURVEY §8a,
    DESIGN.md §4) -- 2(n-m+1) + (m-2)(n-m+1)(n-m+2)/2 for m >= 2, 1 for m = 1, 0 for n < m.
    Computed here so the oracle legs never load the CUDA library; the CUDA arm checks it against
    heddle_place_transitions."""
    if n < m or m < 1:
        return 0
    if m == 1:
        return 1
    return 2 * (n - m + 1) + (m - 2) * (n - m + 1) * (n - m + 2) // 2


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def bench_config(workload, world):
    """The `config` object of both arms (identical for the same workload and N)."""
    if workload == "batched":
        return {"workload": WORKLOAD, "problems": B_TOTAL, "n": N, "m": M, "semiring": "minmax",
                "transitions_per_problem": transitions(N, M),
                "parallelism": f"dp{world} (problems block-sharded across ranks, no collective on the data path; "
                               "results all-gathered inside the timed region)",
                "l2": "flushed between timed steps (256 MiB device write, untimed)"}
    return {"workload": LARGE_WORKLOAD, "problems": 1, "n": 65536, "m": 256, "semiring": "minmax",
            "transitions_per_problem": transitions(65536, 256),
            "parallelism": f"split{world} (zigzag 512-column blocks, one dp-row exchange per layer)",
            "l2": "flushed between timed steps (256 MiB device write, untimed)"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(workload):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed ncu summary
    (profiles/*_k2_ncu_summary.json, one `ncu --set full` capture), or None."""
    import glob
    if workload != "batched":
        return None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_k2_ncu_summary.json")))
    if not files:
        return None
    try:
        return json.load(open(files[-1])).get("traffic_bytes")
    except Exception:
        return None


def alu_peak_cells(sm_mhz):
    """ALU-pipe peak of the exhaustive Eq. 3 reduction: per SMSP the ALU pipe takes 2 cycles per
    FMNMX / FMNMX3 warp instruction, and a transition needs one FMNMX (max) and half an FMNMX3
    (min), i.e. 3 ALU cycles per warp-transition: 4 SMSPs x 32 lanes / 3 x 148 SMs x clock
    (profiles/r01_alu_peaks.jsonl)."""
    return SM_COUNT * 4 * 32 / ISSUE_SLOTS_PER_CELL * sm_mhz * 1e6


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def nvlink_kib(dev_index):
    """NVML NVLink data counters of this GPU, summed over its links: (tx KiB, rx KiB), or None.
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX = 138 / 139; scopeId = link, values in KiB.)"""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
        tx = rx = 0
        ok = False
        for link in range(18):
            vals = pynvml.nvmlDeviceGetFieldValues(h, [(138, link), (139, link)])
            if vals[0].nvmlReturn == 0 and vals[1].nvmlReturn == 0:
                tx += vals[0].value.ullVal
                rx += vals[1].value.ullVal
                ok = True
        return (tx, rx) if ok else None
    except Exception:
        return None


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard(B, world, rank):
    lo = rank * B // world
    hi = (rank + 1) * B // world
    return lo, hi


# ------------------------------------------------------------------------------ oracle arm
def run_reference(args):
    """The oracle as it stands (oracle/, plain FP64-emulating-FP32 DP), on the host cores, over a
    bounded sample of the same workload per step.  Never loads the CUDA library."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from inputs import workloads as wl
    oracle.build()
    threads = os.cpu_count() or 1
    sample = args.ref_sample
    if args.workload == "batched":
        batch = wl.config_batched()
        W = transitions(N, M)
    else:
        batch = wl.config_large(n=args.ref_large_n, m=args.ref_large_m)
        W = transitions(batch.n, batch.m)
    times = []
    for step in range(args.warmup + args.steps):
        t = time.perf_counter()
        if args.workload == "batched":
            lo = (step * sample) % batch.B
            idx = np.arange(lo, lo + sample) % batch.B
            rws = np.stack([batch.profile.row_of(batch.degrees[b]) for b in idx])
            _, _, used = oracle.solve_batch(batch.lengths[idx], batch.profile.T, batch.profile.F, rws, mode="f32",
                                            threads=threads)
            units = sample * W
        else:
            oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32"), threads=threads)
            used, units = threads, W
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = units * len(times) / tot
    what = (f"{sample} problems of the batched sweep per step" if args.workload == "batched" else
            f"one n={batch.n}, m={batch.m} prefix-size instance of the configs[4] generator per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.workload, args.gpus),
        "solves_per_s": (sample if args.workload == "batched" else 1) * len(times) / tot,
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": used, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"{what} (FP32-emulating FP64 oracle, plain O(n^2 m) DP with back-pointers, "
                                   f"OpenMP over {'problems' if args.workload == 'batched' else 'columns'}); "
                                   "value = cells of the sample / wall time"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(sample=64):
    """The oracle as it stands, on a bounded sample of the workload, on all host cores."""
    import oracle
    from inputs import workloads as wl
    oracle.build()
    threads = os.cpu_count() or 1
    batch = wl.config_batched(B=sample, seed_problem=1)
    rws = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(sample)])
    t = time.perf_counter()
    _, _, used = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rws, mode="f32", threads=threads)
    dt = time.perf_counter() - t
    return {"value": sample * transitions(N, M) / dt, "unit": "cells/s", "cores": used, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{sample} problems (n={N}, m={M}) of the batched-sweep workload, {dt:.1f} s wall"}


def latency_lines(dev, reps=20):
    """Latency of the paper's own call shapes, solve + backtrack: `us` = CUDA events around each
    call through the Python binding (median of `reps`; includes the host time of the call), and
    `device_us_graph` = the same pair captured as a CUDA graph and replayed back to back (device
    time alone).  configs[1] rollout, configs[2] TP sweep and the paper's §6.2 size (n = 6400,
    m = 16; the paper quotes ~42 ms on its CPU)."""
    import torch
    from inputs import workloads as wl
    from paper_2603_28101_b200.placer import Placer
    rng = np.random.default_rng(3)
    L6400 = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 800, 8))).astype(np.float32)[None, :]
    cfgs = [("rollout configs[1] (512, 32)", wl.config_rollout()),
            ("tp_sweep configs[2] 4 x (4096, 64)", wl.config_tp_sweep()),
            ("paper_6.2 (6400, 16)", wl.Batch("paper_6.2", 6400, 16, L6400, np.ones((1, 16), np.int32),
                                              wl.float_profile()))]
    out = {}
    stream = torch.cuda.current_stream(dev)
    for name, b in cfgs:
        res = {}
        for algo in ("scan", "valley"):
            pl = Placer.from_profile(b.profile, max_n=b.n, max_m=b.m, max_batch=b.B, device=dev.index, algo=algo)
            L = torch.from_numpy(b.lengths).to(dev)
            D = torch.from_numpy(b.degrees.astype(np.int32)).to(dev)
            for _ in range(3):
                pl.solve(L, D)
                pl.backtrack()
            torch.cuda.synchronize()
            ts, tb = [], []
            for _ in range(reps):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(stream)
                pl.solve(L, D)
                e[1].record(stream)
                pl.backtrack()
                e[2].record(stream)
                torch.cuda.synchronize()
                ts.append(e[0].elapsed_time(e[1]) * 1e3)
                tb.append(e[1].elapsed_time(e[2]) * 1e3)
            W = b.B * transitions(b.n, b.m)
            t = statistics.median([a + c for a, c in zip(ts, tb)])
            # device time alone: the solve + backtrack pair captured once as a CUDA graph and replayed
            # back to back (no host work between the kernels)
            dev_us = None
            try:
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(dev)
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    pl.solve(L, D)
                    pl.backtrack()
                    torch.cuda.synchronize()
                    with torch.cuda.graph(g, stream=side):
                        pl.solve(L, D)
                        pl.backtrack()
                torch.cuda.synchronize()
                for _ in range(3):
                    g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                dev_us = e0.elapsed_time(e1) * 1e3 / reps
                del g
            except Exception as ex:   # capture unsupported on this path: report the event time only
                dev_us = f"graph capture failed: {ex}"[:120]
            res[algo] = {"us": round(t, 1), "us_solve": round(statistics.median(ts), 1),
                         "us_backtrack": round(statistics.median(tb), 1), "cells_per_s": W / (t * 1e-6),
                         "device_us_graph": round(dev_us, 1) if isinstance(dev_us, float) else dev_us}
            pl.close()
        out[name] = res
    return out


# ------------------------------------------------------------------------------ CUDA arm
def run_cuda(args):
    import torch
    import torch.distributed as dist

    from inputs import workloads as wl
    from paper_2603_28101_b200 import _lib
    from paper_2603_28101_b200.placer import Placer

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.workload == "batched":
        lo, hi = shard(B_TOTAL, world, rank)
        batch = wl.config_batched()
        n_, m_, b_total = N, M, B_TOTAL
        kernel_name = "k2_dp_batched<F32,MINMAX>"
    else:   # configs[4]: one n=65536, m=256 instance, columns split across ranks (one row exchange per layer)
        batch = wl.config_large()
        lo, hi = 0, 1
        n_, m_, b_total = batch.n, batch.m, 1
        if os.environ.get("HEDDLE_PLACE_EXCHANGE", "") == "nccl":
            exchange = "per-layer NCCL all-gather of the dp row"
            kernel_name = "k3_layer<F32,MINMAX>"
        else:
            exchange = ("fused: the tile finishing a block stores it into every peer's dp row over NVLink peer "
                        "memory")
            kernel_name = "k5_persistent<F32,MINMAX>"
    Bl = hi - lo
    L = torch.from_numpy(np.ascontiguousarray(batch.lengths[lo:hi])).to(dev)
    D = torch.from_numpy(np.ascontiguousarray(batch.degrees[lo:hi].astype(np.int32))).to(dev)
    Lh = torch.from_numpy(np.ascontiguousarray(batch.lengths[lo:hi])).pin_memory()
    Dh = torch.from_numpy(np.ascontiguousarray(batch.degrees[lo:hi].astype(np.int32))).pin_memory()
    if args.workload == "batched":
        placer = Placer.from_profile(batch.profile, max_n=n_, max_m=m_, max_batch=Bl, device=local)
    elif world > 1:
        from paper_2603_28101_b200.dist import split_placer
        placer = split_placer(batch.profile, max_n=n_, max_m=m_, max_batch=1)
    else:
        placer = Placer.from_profile(batch.profile, max_n=n_, max_m=m_, max_batch=1, device=local, kernel="layered")
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    gather = world > 1 and args.workload == "batched"
    if gather:
        from paper_2603_28101_b200.dist import gather_shards

    def step():
        obj, _ = placer.solve(L, D)
        bnd = placer.backtrack()
        if gather:   # the result gather of §8d: every rank ends with all B objectives and boundaries
            gather_shards(obj, B_TOTAL)
            gather_shards(bnd, B_TOTAL)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = placer.launches
    nvl0 = nvlink_kib(local) if world > 1 else None
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))                      # L2 flush between timed iterations (not timed)
            ev[s][0].record(stream)
            obj, _ = placer.solve(L, D)
            ev[s][1].record(stream)
            bnd = placer.backtrack()
            if gather:
                gather_shards(obj, B_TOTAL)
                gather_shards(bnd, B_TOTAL)
            ev[s][2].record(stream)
        torch.cuda.synchronize()
    launches = placer.launches - launches0
    nvl1 = nvlink_kib(local) if nvl0 is not None else None
    nvl = None if (nvl0 is None or nvl1 is None) else [(nvl1[0] - nvl0[0]) * 1024.0 / args.steps,
                                                         (nvl1[1] - nvl0[1]) * 1024.0 / args.steps]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_step = sum(e[0].elapsed_time(e[2]) for e in ev) / 1e3          # seconds, K steps
    t_k2 = sum(e[0].elapsed_time(e[1]) for e in ev) / 1e3            # dominant kernel(s): the solve
    W = transitions(n_, m_)
    assert W == _lib.transitions(n_, m_), "bench.transitions disagrees with heddle_place_transitions"

    # end to end through the public API with host buffers (H2D + solve + backtrack + D2H each step)
    for _ in range(2):
        placer.solve_host(Lh, Dh)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d = d2h = 0
    for s in range(args.steps):
        _, _, _, h2d, d2h = placer.solve_host(Lh, Dh)
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = e0.elapsed_time(e1) / 1e3

    # the same workload by the valley solver (HEDDLE_VALLEY): exact, O(n m log n);
    # reported beside the scan (the metric's kernel), checked identical to it on this rank's problems
    t_valley, same = -1.0, True
    if args.valley and not (args.workload == "large" and world > 1):
        obj_s, _ = placer.solve(L, D)
        bnd_s = placer.backtrack()
        vplacer = Placer.from_profile(batch.profile, max_n=n_, max_m=m_, max_batch=Bl, device=local, algo="valley")
        for _ in range(2):
            vplacer.solve(L, D)
            vplacer.backtrack()
        torch.cuda.synchronize()
        evv = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for s in range(args.steps):
            flush.fill_(float(s))
            evv[s][0].record(stream)
            obj_v, _ = vplacer.solve(L, D)
            bnd_v = vplacer.backtrack()
            evv[s][1].record(stream)
        torch.cuda.synchronize()
        t_valley = sum(e[0].elapsed_time(e[1]) for e in evv) / 1e3
        same = bool(torch.equal(obj_s, obj_v) and torch.equal(bnd_s, bnd_v))
        vplacer.close()

    vals = torch.tensor([t_step, t_k2, t_e2e, float(launches), t_valley, 0.0 if same else 1.0],
                        dtype=torch.float64, device=dev)
    nvl_all = None
    if world > 1:   # NVLink bytes each rank sent / received per step (NVML counters around the timed steps)
        nv = torch.tensor(nvl if nvl is not None else [-1.0, -1.0], dtype=torch.float64, device=dev)
        gathered = [torch.empty_like(nv) for _ in range(world)]
        dist.all_gather(gathered, nv)
        nvl_all = [g.tolist() for g in gathered]
    if world > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        t_step, t_k2, t_e2e = mx[0].item(), mx[1].item(), mx[2].item()
        launches = int(sm[3].item())
        t_valley, same = mx[4].item(), mx[5].item() == 0.0
    cells = b_total * W * args.steps
    if rank == 0:
        value = cells / t_step
        clocks = clk.summary()
        pk = peaks()
        peak_mhz = pk.get("sm_max_mhz", 1965.0)
        # per GPU, the dominant kernel alone (split mode: this rank's share of the cells)
        k2_rate = (Bl * W if args.workload == "batched" else W / world) * args.steps / t_k2
        peak = alu_peak_cells(peak_mhz)
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_step / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(args.workload, world),
            "solves_per_s": b_total * args.steps / t_step,
            "roofline": {"bound": "alu", "achieved": k2_rate / 1e9, "peak": peak / 1e9, "unit": "Gcell/s",
                         "frac": k2_rate / peak,
                         "traffic": args.traffic if args.traffic is not None else ncu_traffic(args.workload),
                         "algorithmic_bytes": (4 * n_ + 4 * m_ + 4 + 4 * (m_ + 1)) * (Bl if args.workload == "batched" else 1),
                         "kernel": kernel_name,
                         "peak_basis": f"148 SMs x 4 SMSP x 32 lanes / 3 ALU-pipe cycles per cell x {peak_mhz:.0f} MHz "
                                       "(measured pipe rates, profiles/r01_alu_peaks.jsonl)",
                         "kernel_share_of_step": t_k2 / t_step},
            "e2e": {"value": cells / t_e2e, "unit": "cells/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": d2h * world},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if t_valley > 0:
            line["valley"] = {
                "what": "same workload and result by the exact valley search (HEDDLE_VALLEY, SURVEY 8f N3), "
                        "solve + backtrack, device-resident; not the metric's kernel",
                "ms_per_step": 1e3 * t_valley / args.steps, "solves_per_s": b_total * args.steps / t_valley,
                "dp_equivalent_cells_per_s": cells / t_valley, "speedup_vs_scan": t_step / t_valley,
                "identical_to_scan": same}
        if args.workload == "large":
            line["exchange"] = exchange
        if nvl_all is not None and min(min(r) for r in nvl_all) < 0:
            line["nvlink"] = {"unavailable": "NVML NVLink throughput counters read N/A on this pool "
                                             "(profiles/r02_nvlink_probe.json); see bench/rank0_ncu.sh"}
        elif nvl_all is not None:
            row_bytes = 4 * (n_ + 1)
            line["nvlink"] = {
                "tx_bytes_per_step_by_rank": [r[0] for r in nvl_all],
                "rx_bytes_per_step_by_rank": [r[1] for r in nvl_all],
                "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX summed over links, around the timed steps "
                          "(includes the end-of-step barriers and, batched, the result gather)",
                "algorithmic_tx_bytes_per_step_per_rank": (
                    (world - 1) * row_bytes * (m_ - 1) / world if args.workload == "large" else None)}
        if not args.no_latency and args.workload == "batched":
            line["latency"] = latency_lines(dev)
        if not args.no_cpu_baseline and world == 1 and args.workload == "batched":
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--workload", default="batched", choices=["batched", "large"],
                    help="batched = configs[3] (the metric's batched sweep, default); large = configs[4] split")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true", help="skip the paper-call-shape latency lines")
    ap.add_argument("--ref-large-n", type=int, default=16384, help="reference arm, --workload large: sample size")
    ap.add_argument("--ref-large-m", type=int, default=64)
    ap.add_argument("--no-valley", dest="valley", action="store_false",
                    help="skip the valley-solver line (HEDDLE_VALLEY) reported beside the scan")
    ap.add_argument("--cpu-sample", type=int, default=2048)
    ap.add_argument("--ref-sample", type=int, default=32)
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per K2 launch (from profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        import __graft_entry__
        __graft_entry__.build()
        run_cuda(args)


if __name__ == "__main__":
    main()

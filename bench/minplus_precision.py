#!/usr/bin/env python
"""Min-plus precision at m = 256: relative error of the objective against FP64 for the
plain FP32 path (F32 sums) and HEDDLE_F32X (F32 costs, FP64 sums), on configs[4] (n = 65536, against
tests/golden/large_f64_minplus.npz) and on n = 4096 (against the live FP64 oracle).
    python bench/minplus_precision.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import __graft_entry__
    __graft_entry__.build()
    import oracle
    from inputs import workloads as wl
    from paper_2603_28101_b200.placer import Placer
    z = np.load(os.path.join(ROOT, "tests", "golden", "large_f64_minplus.npz"))
    for n in (4096, 65536):
        b = wl.config_large(n=n, m=256)
        if n == 65536:
            ref = float(z["opt"])
        else:
            ref = oracle.solve(oracle.Problem.from_batch(b, 0, mode="f64", semiring=oracle.MINPLUS),
                               threads=os.cpu_count() or 1)["opt"]
        for dt in ("f32", "f32x"):
            pl = Placer.from_profile(b.profile, dtype=dt, semiring="minplus", max_n=n, max_m=256, max_batch=1,
                                     kernel="layered")
            obj, st = pl.solve(torch.from_numpy(b.lengths).cuda(), torch.from_numpy(b.degrees).cuda())
            torch.cuda.synchronize()
            got = float(obj.double().cpu()[0])
            print(json.dumps({"n": n, "m": 256, "dtype": dt, "objective": got, "fp64_oracle": ref,
                              "rel_err": abs(got - ref) / ref, "status": int(st.cpu()[0])}), flush=True)
            pl.close()


if __name__ == "__main__":
    main()

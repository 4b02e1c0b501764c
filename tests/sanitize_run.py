"""Small end-to-end exercise of every kernel for compute-sanitizer (not collected by pytest).

    compute-sanitizer --tool memcheck python tests/sanitize_run.py
Runs K1 (init), K2 (batched), K3 (layered: KEEP_PARENTS, kv caps, split emulation),
K5 (persistent) and K4 (warp and CTA backtrack) on small seeded problems and checks
the results against the oracle, so a sanitizer report is tied to a correct run."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from inputs import workloads as wl  # noqa: E402
from tests.parity import assert_exact, run_gpu  # noqa: E402
from paper_2603_28101_b200.placer import Placer  # noqa: E402


def main():
    cases = []
    rng = np.random.default_rng(2)
    n, m = 700, 9
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, (n + 7) // 8, 8)[:n]))
    deg = wl.sorted_degree_vectors(rng, 3, m)
    base = wl.Batch("s", n, m, np.stack([L] * 3).astype(np.float32), deg, wl.float_profile())
    cases.append(("batched", dict(kernel="batched"), base))
    cases.append(("persistent", dict(kernel="layered"), base))
    cases.append(("layered-kp", dict(kernel="layered", keep_parents=True), base))
    kvb = wl.Batch("kv", n, m, base.lengths, deg, base.profile,
                   kv_caps=np.full((3, m), int(L.astype(np.float64).sum() / 5), np.int64))
    cases.append(("layered-kv", dict(kernel="layered"), kvb))
    cases.append(("batched-kv-kp", dict(kernel="batched", keep_parents=True), kvb))
    for name, kw, b in cases:
        g = run_gpu(b, **kw)
        for i in range(b.B):
            ref = oracle.solve(oracle.Problem.from_batch(b, i, mode="f32"), want_tables=True)
            assert_exact(g, i, ref, b, "f32", "minmax", check_parents=kw.get("keep_parents", False), tag=name)
        g["placer"].close()
        print("ok", name, flush=True)
    # min-plus few problems: CTA backtrack
    g = run_gpu(base, semiring="minplus", kernel="layered")
    for i in range(base.B):
        ref = oracle.solve(oracle.Problem.from_batch(base, i, mode="f32", semiring=oracle.MINPLUS))
        assert g["obj"][i] == ref["opt"] and np.array_equal(g["bounds"][i], ref["bounds"])
    print("ok minplus-cta-backtrack", flush=True)
    # split emulation (pack / exchange / unpack)
    L2 = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 263, 8)[:2100]))
    b1 = wl.Batch("split", 2100, 7, L2[None, :].astype(np.float32), np.ones((1, 7), np.int32), wl.float_profile())
    ref = run_gpu(b1, kernel="layered")
    pl = Placer.from_profile(b1.profile, max_n=b1.n, max_m=b1.m, max_batch=1, split=(None, 0, 3))
    got = run_gpu(b1, placer=pl)
    assert np.array_equal(got["bounds"], ref["bounds"]) and np.array_equal(got["obj"], ref["obj"])
    print("ok split-emulation", flush=True)
    torch.cuda.synchronize()
    from paper_2603_28101_b200 import _lib
    v = _lib.lib().heddle_place_debug_violations()
    print(f"bounds violations: {v}")
    assert v in (-1, 0), v
    print("SANITIZE RUN OK")


if __name__ == "__main__":
    main()

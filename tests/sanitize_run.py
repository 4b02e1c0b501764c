"""Small end-to-end exercise of every kernel for compute-sanitizer (not collected by pytest).

    compute-sanitizer --tool memcheck python tests/sanitize_run.py
Runs K1 (init), K2 (batched: F32 / U32, min-max / min-plus), K3 (layered: KEEP_PARENTS, kv caps,
split emulation), K5 (persistent), K8 / K8L (valley, one CTA per problem and per layer), K7
(objective only), K4 (warp and CTA backtrack, state query) and K6 (migration retarget) on small
seeded problems (and the configs[1] rollout problem) and checks the results against the oracle,
so a sanitizer report is tied to a correct run."""
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
    cases.append(("valley-batched", dict(kernel="batched", algo="valley"), base))
    cases.append(("valley-layered", dict(kernel="layered", algo="valley"), base))
    cases.append(("rollout-batched", dict(kernel="batched"), wl.config_rollout()))
    cases.append(("rollout-valley", dict(kernel="batched", algo="valley"), wl.config_rollout()))
    for name, kw, b in cases:
        g = run_gpu(b, **kw)
        for i in range(b.B):
            ref = oracle.solve(oracle.Problem.from_batch(b, i, mode="f32"), want_tables=True)
            assert_exact(g, i, ref, b, "f32", "minmax", check_parents=kw.get("keep_parents", False), tag=name)
        g["placer"].close()
        print("ok", name, flush=True)
    # U32 (bit-exact mode), both semirings, with the state query over the whole region
    from tests.parity import assert_tables_exact
    ub = wl.config_batched(B=4, n=296, m=7, dtype="u32")
    for sr, osr in (("minmax", oracle.MINMAX), ("minplus", oracle.MINPLUS)):
        g = run_gpu(ub, semiring=sr, kernel="batched")
        for i in range(ub.B):
            ref = oracle.solve(oracle.Problem.from_batch(ub, i, mode="u32", semiring=osr), want_tables=True)
            assert_exact(g, i, ref, ub, "u32", sr, tag="u32-" + sr)
            assert_tables_exact(g["placer"], i, ref, ub.n, ub.m, tag="u32-query-" + sr)
        g["placer"].close()
        print("ok u32", sr, flush=True)
    # objective only (K7)
    pl = Placer.from_profile(base.profile, max_n=base.n, max_m=base.m, max_batch=base.B)
    obj, st = pl.objective(torch.from_numpy(base.lengths).cuda(), torch.from_numpy(base.degrees).cuda())
    torch.cuda.synchronize()
    for i in range(base.B):
        assert float(obj[i]) == oracle.solve(oracle.Problem.from_batch(base, i, mode="f32"))["opt"]
    pl.close()
    print("ok objective", flush=True)
    # migration retarget (K6)
    from paper_2603_28101_b200 import migration
    bnd = torch.tensor([[0, 3, 7, 10]], dtype=torch.int32).cuda()
    w = migration.retarget(bnd, torch.tensor([10], dtype=torch.int32).cuda(),
                           torch.zeros(10, dtype=torch.int32).cuda(), torch.arange(10, dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    assert w.cpu().tolist() == [0, 0, 0, 1, 1, 1, 1, 2, 2, 2], w.cpu().tolist()
    print("ok retarget", flush=True)
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

"""GPU: min-plus with FP32 costs and FP64 accumulation (HEDDLE_F32X).

* bit-exact against the oracle's F32X mode (same costs fl32(L*fl32(T*F)), sums in double), on
  tiny random problems (ties, caps, kv caps, mixed degrees) and the rollout config, through the
  batched and the layered kernels; every dp value and back-pointer via heddle_place_query;
* within 1e-6 of the FP64 oracle at m = 256 -- where a plain FP32 sum of 256 terms drifts -- at
  n = 4096 against the live oracle (objective, 1e-6-optimal partition, near-tie boundary walk)
  and at configs[4] (n = 65536) against tests/golden/large_f64_minplus.npz.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from paper_2603_28101_b200.placer import Placer
from tests.parity import (REL_TOL, assert_exact, assert_f64_tolerance, assert_tables_exact, partition_cost_f64,
                          run_gpu, to_dev)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "large_f64_minplus.npz")


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


@pytest.mark.parametrize("kernel", ["batched", "layered"])
def test_f32x_random_tiny_exact(kernel):
    for s in range(120):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, dtype="f32")
        gpu = run_gpu(batch, semiring="minplus", dtype="f32x", kernel=kernel)
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32x", semiring=oracle.MINPLUS),
                           want_tables=True)
        assert_exact(gpu, 0, ref, batch, "f32x", "minplus", tag=f"f32x-{s}")
        if ref["status"] == oracle.OK:
            assert_tables_exact(gpu["placer"], 0, ref, batch.n, batch.m, tag=f"f32x-tables-{s}")
        gpu["placer"].close()


@pytest.mark.parametrize("kernel", ["batched", "layered"])
def test_f32x_rollout_exact(kernel):
    batch = wl.config_rollout()
    gpu = run_gpu(batch, semiring="minplus", dtype="f32x", kernel=kernel)
    ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32x", semiring=oracle.MINPLUS), want_tables=True)
    assert_exact(gpu, 0, ref, batch, "f32x", "minplus", tag="rollout")
    assert_tables_exact(gpu["placer"], 0, ref, batch.n, batch.m, tag="rollout")


def test_f32x_m256_within_1e6_of_f64():
    batch = wl.config_large(n=4096, m=256)
    gpu = run_gpu(batch, semiring="minplus", dtype="f32x", kernel="layered")
    p64 = oracle.Problem.from_batch(batch, 0, mode="f64", semiring=oracle.MINPLUS)
    assert gpu["status"][0] == 0
    assert_f64_tolerance(gpu["obj"][0], gpu["bounds"][0], p64, "minplus", tag="f32x-m256")
    # and bit-exact against the F32X oracle in its own arithmetic
    ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32x", semiring=oracle.MINPLUS),
                       threads=os.cpu_count() or 1)
    assert gpu["obj"][0] == ref["opt"] and np.array_equal(gpu["bounds"][0], ref["bounds"])


@pytest.mark.skipif(not os.path.exists(GOLD), reason="golden file not generated")
def test_f32x_large_config_within_1e6_of_f64_golden():
    z = np.load(GOLD)
    batch = wl.config_large()
    pl = Placer.from_profile(batch.profile, dtype="f32x", semiring="minplus", max_n=batch.n, max_m=batch.m,
                             max_batch=1, kernel="layered")
    obj, st = pl.solve(to_dev(batch.lengths), to_dev(batch.degrees.astype(np.int32)))
    bnd = pl.backtrack()
    torch.cuda.synchronize()
    opt = float(z["opt"])
    got = float(obj.cpu()[0])
    assert int(st.cpu()[0]) == 0
    assert abs(got - opt) <= REL_TOL * opt, (got, opt)
    p64 = oracle.Problem.from_batch(batch, 0, mode="f64", semiring=oracle.MINPLUS)
    cost = partition_cost_f64(p64, bnd.cpu().numpy()[0], "minplus")
    assert cost <= opt * (1 + REL_TOL), (cost, opt)
    pl.close()

"""GPU parity against stored and hand-derived oracle results.

  * configs[4] (n = 65536, m = 256, FP32, Eq. 3 min-max) against tests/golden/large_f32.npz,
    written by tests/golden/make_large_golden.py from oracle/ alone: objective, boundaries and
    every sampled state's dp value and lowest-index back-pointer, bit for bit, for each solve path
    that can run it -- K5 (the layered default), K3 (one launch per layer), K8L (valley);
    split mode over 2+ GPUs is in tests/mgpu_split_check.py.
  * the hand-derived capacity cases of tests/golden/spec_worked_examples.json (R6: a group whose
    token sum or size equals its cap is admissible).
  * U32 (the north_star bit-exact mode) at scale: sampled problems of the full 16384-problem
    configs[3] launch and an n = 8192 layered instance, every dp value and back-pointer of the
    computed region against the oracle's tables; F64 at n = 1024 within 1e-6.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from paper_2603_28101_b200.placer import Placer
from tests.parity import (assert_exact, assert_f64_tolerance, assert_tables_exact, query_gpu, run_gpu, to_dev,
                          TDT)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


# ------------------------------------------------------------------ configs[4] golden
def _large_golden():
    z = np.load(os.path.join(GOLD, "large_f32.npz"))
    batch = wl.config_large()
    assert str(z["lengths_sha256"]) == hashlib.sha256(np.ascontiguousarray(batch.lengths).tobytes()).hexdigest()
    return z, batch


def check_large_against_golden(placer, z, tag):
    bnd = placer.backtrack()
    torch.cuda.synchronize()
    got_b = bnd.cpu().numpy()[0]
    assert np.array_equal(got_b, z["bounds"]), (tag, np.nonzero(got_b != z["bounds"])[0][:5])
    qb = np.zeros(z["qj"].size, dtype=np.int32)
    dp, par = query_gpu(placer, qb, z["qj"], z["qi"])
    bad = np.nonzero((dp != z["dp"]) | (par != z["parent"]))[0]
    assert bad.size == 0, (tag, [(int(z["qj"][t]), int(z["qi"][t]), dp[t], z["dp"][t], int(par[t]),
                                  int(z["parent"][t])) for t in bad[:5]])


@pytest.mark.parametrize("path", ["k5", "k3", "valley"])
def test_large_config_golden(path, monkeypatch):
    z, batch = _large_golden()
    if path == "k3":
        monkeypatch.setenv("HEDDLE_PLACE_NO_PERSISTENT", "1")
    placer = Placer.from_profile(batch.profile, max_n=batch.n, max_m=batch.m, max_batch=1, kernel="layered",
                                 algo="valley" if path == "valley" else "scan")
    L = to_dev(batch.lengths)
    D = to_dev(batch.degrees.astype(np.int32))
    obj, st = placer.solve(L, D)
    torch.cuda.synchronize()
    assert int(st.cpu()[0]) == 0
    assert float(obj.cpu()[0]) == float(z["opt"]), (path, float(obj.cpu()[0]), float(z["opt"]))
    check_large_against_golden(placer, z, path)
    placer.close()


# ------------------------------------------------------------------ capacity golden (R6)
@pytest.mark.parametrize("kernel,algo", [("batched", "scan"), ("layered", "scan"), ("batched", "valley"),
                                         ("layered", "valley")])
def test_capacity_golden_cases(kernel, algo):
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    for case in g["capacity"]:
        if algo == "valley" and case["semiring"] != "minmax":
            continue
        n, m = len(case["L"]), case["m"]
        dt = case["mode"]
        prof = wl.Profile((1,), np.array([case["T"]]), np.array([case["F"]], dtype=np.float64), len(case["F"]), dt)
        ldt = {"u32": np.uint32, "f32": np.float32, "f64": np.float64}[dt]
        batch = wl.Batch("cap", n, m, np.array([case["L"]], dtype=ldt), np.ones((1, m), dtype=np.int32), prof,
                         caps=np.array([case["caps"]], dtype=np.int32) if "caps" in case else None,
                         kv_caps=np.array([case["kv_caps"]], dtype=np.int64) if "kv_caps" in case else None)
        gpu = run_gpu(batch, semiring=case["semiring"], kernel=kernel, algo=algo)
        assert int(gpu["status"][0]) == 0, case["cite"]
        assert gpu["obj"][0] == case["opt"], (gpu["obj"][0], case["cite"])
        assert gpu["bounds"][0].tolist() == case["bounds"], (gpu["bounds"][0].tolist(), case["cite"])
        gpu["placer"].close()


# ------------------------------------------------------------------ U32 / F64 at scale
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
def test_batched_u32_full_launch_tables(semiring):
    """The full configs[3] launch (16384 problems) in U32; 12 sampled problems' complete dp and
    back-pointer tables equal the oracle's."""
    batch = wl.config_batched(dtype="u32")
    gpu = run_gpu(batch, semiring=semiring)
    assert np.all(gpu["status"] == 0)
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    rng = np.random.default_rng(7)
    for b in [0, 1, batch.B - 1] + [int(x) for x in rng.integers(0, batch.B, size=9)]:
        ref = oracle.solve(oracle.Problem.from_batch(batch, b, mode="u32", semiring=sr), want_tables=True)
        assert_exact(gpu, b, ref, batch, "u32", semiring, tag="u32-batched")
        assert_tables_exact(gpu["placer"], b, ref, batch.n, batch.m, tag=f"u32-batched-{semiring}")
    gpu["placer"].close()


@pytest.mark.parametrize("path", ["k5", "k3", "valley"])
def test_layered_u32_n8192_tables(path, monkeypatch):
    batch = wl.config_large(n=8192, m=64, dtype="u32")
    if path == "k3":
        monkeypatch.setenv("HEDDLE_PLACE_NO_PERSISTENT", "1")
    gpu = run_gpu(batch, kernel="layered", algo="valley" if path == "valley" else "scan")
    ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="u32"), want_tables=True,
                       threads=os.cpu_count() or 1)
    assert_exact(gpu, 0, ref, batch, "u32", "minmax", tag=f"u32-8192-{path}")
    assert_tables_exact(gpu["placer"], 0, ref, batch.n, batch.m, tag=f"u32-8192-{path}")
    gpu["placer"].close()


@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
def test_batched_f64_n1024(semiring):
    """F64 at the configs[3] problem size: objective within 1e-6 of the FP64 oracle, partition
    1e-6-optimal, boundaries equal except at oracle near-ties (walked to layer 1)."""
    batch = wl.config_batched(B=296, dtype="f64")
    gpu = run_gpu(batch, semiring=semiring)
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    for b in range(0, batch.B, 37):
        assert gpu["status"][b] == 0
        p = oracle.Problem.from_batch(batch, b, mode="f64", semiring=sr)
        assert_f64_tolerance(gpu["obj"][b], gpu["bounds"][b], p, semiring, tag=f"f64-{b}")
    gpu["placer"].close()

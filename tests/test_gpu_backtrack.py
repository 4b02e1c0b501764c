"""GPU: the backtrack's lowest-argmin search (K4) on instances where the last groups are small
compared with the split range -- slow workers after fast ones, the shape SA proposals produce.

Regression for the 32-ary search that skipped splits after its last probe:
with n = 35 equal lengths, degrees [8, 1], T_8 = 0.01, T_1 = 1, F(s) = 1 + 0.1 (s - 1), the
slow worker must take one trajectory (cost 100 * 1 * F(1) = 100; any larger group costs more,
and the fast worker's 34 trajectories cost 100 * 0.01 * F(34) = 4.3), so the unique optimal
partition is [0, 34, 35] with objective 100 (Eq. 2; Eq. 3).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from tests.parity import assert_exact, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


def slow_fast_profile(s_max=512, dtype="f32"):
    s = np.arange(1, s_max + 1, dtype=np.float64)
    F = np.broadcast_to(1.0 + 0.1 * (s - 1.0), (2, s_max)).copy()
    T = np.array([1.0, 0.01])
    if dtype == "f32":
        T = T.astype(np.float32).astype(np.float64)
        F = F.astype(np.float32).astype(np.float64)
    return wl.Profile((1, 8), T, F, s_max, dtype)


CASES = [("batched", "scan"), ("layered", "scan"), ("batched", "valley"), ("layered", "valley")]


@pytest.mark.parametrize("kernel,algo", CASES)
def test_n35_slow_last_worker(kernel, algo):
    prof = slow_fast_profile()
    L = np.full((1, 35), 100.0, dtype=np.float32)
    batch = wl.Batch("n35", 35, 2, L, np.array([[8, 1]], dtype=np.int32), prof)
    gpu = run_gpu(batch, kernel=kernel, algo=algo)
    assert int(gpu["status"][0]) == 0
    assert gpu["obj"][0] == 100.0
    assert gpu["bounds"][0].tolist() == [0, 34, 35]


@pytest.mark.parametrize("kernel,algo", CASES + [("batched", "scan-minplus"), ("layered", "scan-minplus")])
def test_small_groups_sweep(kernel, algo):
    """Every group size of the slow worker's group from 1 up, over ranges of 33..700 splits:
    random sorted lengths, 2..4 workers with fast workers first; bit-exact against the oracle."""
    semiring = "minplus" if algo.endswith("minplus") else "minmax"
    algo = algo.split("-")[0]
    prof = slow_fast_profile()
    rng = np.random.default_rng(2024)
    probs = []
    for n in list(range(33, 140)) + list(rng.integers(140, 700, size=40)):
        m = int(rng.integers(2, 5))
        L = -np.sort(-rng.integers(1, 400, size=n)).astype(np.float32)
        deg = np.array(sorted(rng.choice([1, 8], size=m), reverse=True), dtype=np.int32)
        probs.append((int(n), m, L, deg))
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    for t, (n, m, L, deg) in enumerate(probs):
        batch = wl.Batch("sweep", n, m, L[None, :], deg[None, :], prof)
        gpu = run_gpu(batch, semiring=semiring, kernel=kernel, algo=algo)
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32", semiring=sr), want_tables=True)
        assert_exact(gpu, 0, ref, batch, "f32", semiring, tag=f"sweep{t} n={n} deg={deg.tolist()}")
        gpu["placer"].close()

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Inputs are the seeded synthetic workloads of inputs/workloads.py, at the
BASELINE.json configs (tiny, rollout, TP sweep, batched sweep) and in the
bench.py launch configuration; see tests/parity.py for the acceptance rule.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from tests.parity import assert_exact, assert_f64_tolerance, run_gpu, to_dev
from tests.parity import run_gpu as _run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


# ------------------------------------------------------------------ configs[0]: tiny, integer, brute force
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
def test_tiny_config_bruteforce(semiring):
    for prob in range(8):
        batch = wl.config_tiny(problem=prob)
        gpu = run_gpu(batch, semiring=semiring, keep_parents=True)
        p = oracle.Problem.from_batch(batch, 0, mode="u32",
                                      semiring=oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS)
        ref = oracle.solve(p, want_tables=True)
        assert_exact(gpu, 0, ref, batch, "u32", semiring, check_parents=True, tag=f"tiny{prob}")
        bf = oracle.brute_contiguous(p)
        assert gpu["obj"][0] == bf["opt"]
        cp = oracle.canonical_parents_bf(p)
        n, m = batch.n, batch.m
        for j in range(2, m):
            got = gpu["parents"][0][j - 1, j:n - m + j + 1]
            assert np.array_equal(got, cp["parent"][j, j:n - m + j + 1]), (prob, j)


KERNELS = ["batched", "layered"]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
@pytest.mark.parametrize("dtype", ["u32", "f32"])
def test_random_tiny_exact(dtype, semiring, kernel):
    """Heavy ties, clamp plateaus, caps, kv caps, heterogeneous degrees: bit-exact."""
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    for s in range(150):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, dtype=dtype)
        kp = (s % 2 == 0) and not (kernel == "layered" and dtype == "u32" and semiring == "minplus")
        gpu = run_gpu(batch, semiring=semiring, keep_parents=kp, kernel=kernel)
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode=dtype, semiring=sr), want_tables=True)
        assert_exact(gpu, 0, ref, batch, dtype, semiring, check_parents=kp, tag=f"{dtype}{s}")
        gpu["placer"].close()


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
def test_random_tiny_f64(semiring, kernel):
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    for s in range(80):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, dtype="f64")
        gpu = run_gpu(batch, semiring=semiring, kernel=kernel)
        p = oracle.Problem.from_batch(batch, 0, mode="f64", semiring=sr)
        ref = oracle.solve(p)
        if ref["status"] != oracle.OK:
            assert gpu["status"][0] == ref["status"]
            continue
        assert gpu["status"][0] == 0
        assert_f64_tolerance(gpu["obj"][0], gpu["bounds"][0], p, semiring, tag=f"f64-{s}")
        gpu["placer"].close()


# ------------------------------------------------------------------ configs[1]: rollout, FP32
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
def test_rollout_config(semiring, kernel):
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    for prob in range(4):
        batch = wl.config_rollout(problem=prob)
        gpu = run_gpu(batch, semiring=semiring, keep_parents=True, kernel=kernel)
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32", semiring=sr), want_tables=True)
        assert_exact(gpu, 0, ref, batch, "f32", semiring, check_parents=True, tag=f"rollout{prob}")
        p64 = oracle.Problem.from_batch(batch, 0, mode="f64", semiring=sr)
        assert_f64_tolerance(gpu["obj"][0], gpu["bounds"][0], p64, semiring, tag=f"rollout{prob}")


@pytest.mark.parametrize("kernel", KERNELS)
def test_rollout_with_caps_and_kv(kernel):
    """Worker batch caps (max_active) and KV token caps on the rollout workload."""
    batch = wl.config_rollout(problem=7)
    rng = np.random.default_rng(11)
    batch.caps = rng.integers(16, 40, size=(1, batch.m)).astype(np.int32)
    total = float(batch.lengths.astype(np.float64).sum())
    batch.kv_caps = rng.integers(int(total / 20), int(total / 8), size=(1, batch.m)).astype(np.int64)
    gpu = run_gpu(batch, keep_parents=True, kernel=kernel)
    ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32"), want_tables=True)
    assert_exact(gpu, 0, ref, batch, "f32", "minmax", check_parents=True, tag="rollout-caps")


# ------------------------------------------------------------------ configs[2]: TP sweep (shared L, stride 0)
@pytest.mark.parametrize("kernel", ["auto", "batched"])
def test_tp_sweep_config(kernel):
    batch = wl.config_tp_sweep()
    gpu = run_gpu(batch, lengths_shared=True, kernel=kernel)
    rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
    opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32")
    for b in range(batch.B):
        assert gpu["status"][b] == 0
        assert gpu["obj"][b] == opt[b], (b, gpu["obj"][b], opt[b])
        assert np.array_equal(gpu["bounds"][b], bounds[b]), b


# ------------------------------------------------------------------ configs[3]: batched sweep
def test_batched_sample_exact():
    batch = wl.config_batched(B=96)
    gpu = run_gpu(batch)
    rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
    opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32")
    assert np.all(gpu["status"] == 0)
    assert np.array_equal(gpu["obj"], opt)
    assert np.array_equal(gpu["bounds"], bounds)


@pytest.mark.parametrize("kernel", KERNELS)
def test_batched_keep_parents(kernel):
    batch = wl.config_batched(B=6, seed_problem=3)
    gpu = run_gpu(batch, keep_parents=True, kernel=kernel)
    for b in range(batch.B):
        ref = oracle.solve(oracle.Problem.from_batch(batch, b, mode="f32"), want_tables=True)
        assert_exact(gpu, b, ref, batch, "f32", "minmax", check_parents=True, tag=f"batched{b}")


def test_batched_full_launch_sampled():
    """The bench.py launch configuration (B=16384, n=1024, m=32), checked on sampled problems."""
    batch = wl.config_batched()
    gpu = run_gpu(batch)
    assert np.all(gpu["status"] == 0)
    idx = np.random.default_rng(5).choice(batch.B, size=24, replace=False)
    idx = np.concatenate([idx, [0, 1, batch.B - 1]])
    rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in idx])
    opt, bounds, _ = oracle.solve_batch(batch.lengths[idx], batch.profile.T, batch.profile.F, rows, mode="f32")
    assert np.array_equal(gpu["obj"][idx], opt)
    assert np.array_equal(gpu["bounds"][idx], bounds)
    # property at every size: boundaries strictly increasing from 0 to n
    bd = gpu["bounds"]
    assert np.all(bd[:, 0] == 0) and np.all(bd[:, -1] == batch.n) and np.all(np.diff(bd, axis=1) > 0)


# ------------------------------------------------------------------ edge cases
def _single(L, deg, dtype="f32", m=None, profile=None, caps=None, semiring="minmax"):
    prof = profile or (wl.float_profile() if dtype != "u32" else wl.int_profile())
    Ln = np.asarray(L)[None, :]
    b = wl.Batch("edge", Ln.shape[1], len(deg), Ln, np.asarray(deg, dtype=np.int32)[None, :], prof,
                 caps=None if caps is None else np.asarray(caps, dtype=np.int32)[None, :])
    return b


@pytest.mark.parametrize("kernel", KERNELS)
def test_edge_cases(kernel):
    f = np.float32
    run_gpu = lambda b: _run(b, kernel=kernel)
    # n = m = 1
    g = run_gpu(_single(np.array([100], f), [1]))
    assert g["status"][0] == 0 and list(g["bounds"][0]) == [0, 1]
    # n = m: singletons
    g = run_gpu(_single(np.array([5, 4, 3], f), [1, 1, 1]))
    assert list(g["bounds"][0]) == [0, 1, 2, 3]
    # n < m: infeasible
    g = run_gpu(_single(np.array([5, 4], f), [1, 1, 1]))
    assert g["status"][0] == 3 and np.all(g["bounds"][0] == -1) and np.isinf(g["obj"][0])
    # unsorted lengths
    g = run_gpu(_single(np.array([1, 5, 3], f), [1, 1]))
    assert g["status"][0] == 2
    # NaN / zero length
    g = run_gpu(_single(np.array([5, np.nan, 3], f), [1, 1]))
    assert g["status"][0] == 4
    g = run_gpu(_single(np.array([5, 3, 0], f), [1, 1]))
    assert g["status"][0] == 4
    # unknown degree / unsorted degrees
    g = run_gpu(_single(np.array([5, 4, 3], f), [3, 1]))
    assert g["status"][0] == 5
    g = run_gpu(_single(np.array([5, 4, 3], f), [1, 2]))
    assert g["status"][0] == 2
    # caps that cannot cover n
    g = run_gpu(_single(np.array([5, 4, 3, 2, 1], f), [1, 1], caps=[2, 2]))
    assert g["status"][0] == 3
    # U32 range guard: a length above the guard is reported, never wrapped
    g = run_gpu(_single(np.array([70000, 3], np.uint32), [1, 1], dtype="u32"))
    assert g["status"][0] == 4


@pytest.mark.parametrize("kernel", KERNELS)
def test_ragged_sizes_and_mixed_batch(kernel):
    """n not a multiple of 4 or of the 128-column warp block; one bad problem in a batch
    does not disturb the others."""
    for n, m in [(129, 3), (130, 7), (257, 2), (383, 31), (1021, 5)]:
        rng = np.random.default_rng(n)
        L = wl.presort_rows(wl.predicted(rng, wl.coding_lengths(rng, (n + 7) // 8, 8)[:n])[None, :])
        L = np.repeat(L, 3, axis=0)
        L[1, 3], L[1, 4] = L[1, 4], L[1, 3] + 1000   # problem 1 unsorted
        deg = wl.sorted_degree_vectors(rng, 3, m)
        batch = wl.Batch("ragged", n, m, L.astype(np.float32), deg, wl.float_profile())
        gpu = run_gpu(batch, keep_parents=True, kernel=kernel)
        assert gpu["status"][1] == 2
        for b in (0, 2):
            ref = oracle.solve(oracle.Problem.from_batch(batch, b, mode="f32"), want_tables=True)
            assert_exact(gpu, b, ref, batch, "f32", "minmax", check_parents=True, tag=f"ragged{n}")


def test_host_e2e_matches_device():
    batch = wl.config_batched(B=32, seed_problem=9)
    gpu = run_gpu(batch)
    pl = gpu["placer"]
    Lh = torch.from_numpy(batch.lengths).pin_memory()
    Dh = torch.from_numpy(batch.degrees.astype(np.int32)).pin_memory()
    obj, bnd, st, h2d, d2h = pl.solve_host(Lh, Dh)
    assert np.array_equal(obj.numpy().astype(np.float64), gpu["obj"])
    assert np.array_equal(bnd.numpy(), gpu["bounds"])
    assert h2d == batch.lengths.nbytes + batch.degrees.astype(np.int32).nbytes
    assert d2h == 4 * batch.B + 4 * batch.B * (batch.m + 1) + 4 * batch.B


@pytest.mark.parametrize("bcast_degrees", [False, True])
def test_host_e2e_chunked_pipeline(bcast_degrees):
    """B large enough that solve_host pipelines its copies in chunks (ragged last chunk, broadcast
    rows copied once): results identical to the device-resident solve of the same problems."""
    from paper_2603_28101_b200.placer import Placer
    batch = wl.config_batched(B=1301, seed_problem=4)
    deg = batch.degrees.astype(np.int32)
    if bcast_degrees:
        deg = deg[:1]
    pl = Placer.from_profile(batch.profile, max_n=batch.n, max_m=batch.m, max_batch=batch.B)
    obj_d, st_d = pl.solve(to_dev(batch.lengths), to_dev(deg))
    bnd_d = pl.backtrack().cpu().numpy()
    obj_d = obj_d.cpu().numpy()
    Lh = torch.from_numpy(batch.lengths).pin_memory()
    Dh = torch.from_numpy(deg).pin_memory()
    obj, bnd, st, h2d, d2h = pl.solve_host(Lh, Dh)
    assert (st.numpy() == 0).all() and (st_d.cpu().numpy() == 0).all()
    assert np.array_equal(obj.numpy(), obj_d)
    assert np.array_equal(bnd.numpy(), bnd_d)
    assert h2d == batch.lengths.nbytes + deg.nbytes
    idx = np.array([0, 591, 592, 650, 1300])      # chunk edges and the ragged tail
    rows = np.stack([batch.profile.row_of(deg[0 if bcast_degrees else b]) for b in idx])
    opt, bounds, _ = oracle.solve_batch(batch.lengths[idx], batch.profile.T, batch.profile.F, rows, mode="f32")
    assert np.array_equal(obj.numpy()[idx], opt)
    assert np.array_equal(bnd.numpy()[idx], bounds)


def test_error_paths():
    from paper_2603_28101_b200 import E_INVALID, E_STATE, HeddleError
    from paper_2603_28101_b200.placer import Placer
    prof = wl.float_profile()
    pl = Placer.from_profile(prof, max_n=64, max_m=8, max_batch=4)
    with pytest.raises(HeddleError) as e:
        pl.backtrack()
    assert e.value.status == E_STATE
    L = to_dev(np.linspace(100, 1, 128, dtype=np.float32)[None, :])
    D = to_dev(np.ones((1, 4), np.int32))
    with pytest.raises(HeddleError) as e:   # n > max_n
        pl.solve(L, D)
    assert e.value.status == E_INVALID
    pl.solve(L[:, :64], D)
    with pytest.raises(HeddleError) as e:   # parents without HEDDLE_KEEP_PARENTS
        pl.backtrack(parents=True)
    assert e.value.status == E_STATE


# ------------------------------------------------------------------ layered kernel at larger n
def test_layered_medium_exact():
    """n = 8192 (beyond nothing for K2 but exercised through K3), m = 16, vs the full oracle."""
    rng = np.random.default_rng(77)
    n, m = 8192, 16
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, n // 8, 8)))
    deg = wl.sorted_degree_vectors(rng, 2, m)
    batch = wl.Batch("medium", n, m, np.stack([L, L]).astype(np.float32), deg, wl.float_profile())
    gpu = run_gpu(batch, kernel="layered")
    rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
    opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32",
                                        threads=2)
    assert np.array_equal(gpu["obj"], opt)
    assert np.array_equal(gpu["bounds"], bounds)


def test_large_config_objective_parametric():
    """configs[4]: n = 65536, m = 256 on one GPU (layered kernel).  The objective is pinned
    exactly by the parametric oracle (P6); the partition must attain it group by group."""
    batch = wl.config_large()
    gpu = run_gpu(batch)
    assert gpu["status"][0] == 0
    p = oracle.Problem.from_batch(batch, 0, mode="f32")
    q = oracle.parametric_opt(p)
    assert gpu["obj"][0] == q["opt"], (gpu["obj"][0], q["opt"])
    bd = gpu["bounds"][0]
    assert bd[0] == 0 and bd[-1] == batch.n and np.all(np.diff(bd) > 0)
    worst = max(oracle.group_cost(p, j, int(bd[j - 1]), int(bd[j])) for j in range(1, batch.m + 1))
    assert worst == q["opt"]


# ------------------------------------------------------------------ split mode (multi-GPU) logic on one GPU
@pytest.mark.parametrize("world", [2, 3, 8])
def test_split_emulation_bit_identical(world):
    """The split-mode ownership / pack / exchange / unpack path, with `world` virtual ranks on
    one GPU (the row is cleared and rebuilt from the exchange buffer every layer), must give
    results bit-identical to the single-GPU solve."""
    from paper_2603_28101_b200.placer import Placer
    rng = np.random.default_rng(5)
    n, m = 8192, 12
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, n // 8, 8)))
    cases = [wl.config_tp_sweep(),
             wl.Batch("split8k", n, m, L[None, :].astype(np.float32), np.ones((1, m), np.int32), wl.float_profile())]
    kvb = wl.Batch("split8k-kv", n, m, L[None, :].astype(np.float32), np.ones((1, m), np.int32),
                   wl.float_profile(), kv_caps=np.full((1, m), int(L.astype(np.float64).sum() / 6), np.int64))
    cases.append(kvb)
    for b in cases:
        ref = run_gpu(b, kernel="layered", lengths_shared=(b.name == "tp_sweep"))
        pl = Placer.from_profile(b.profile, max_n=b.n, max_m=b.m, max_batch=b.B, split=(None, 0, world))
        got = run_gpu(b, placer=pl, lengths_shared=(b.name == "tp_sweep"))
        assert np.array_equal(got["status"], ref["status"]), b.name
        assert np.array_equal(got["obj"], ref["obj"]), b.name
        assert np.array_equal(got["bounds"], ref["bounds"]), b.name


def test_split_multi_gpu_torchrun():
    """Real split mode over NCCL when the box has >= 2 GPUs: torchrun one rank per GPU, the
    n=65536 m=256 instance split by columns, result bit-identical to rank 0's 1-GPU solve."""
    import os
    import subprocess
    import sys
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(ngpu, 8)}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tests", "mgpu_split_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SPLIT OK" in r.stdout


def test_bounds_checked_build():
    """Every kernel path on a debug build whose kernels verify the shared-memory index range of
    each warp task / tile (compute-sanitizer is not available on the pool): zero violations."""
    import os
    import subprocess
    import sys
    import tempfile
    from paper_2603_28101_b200 import _build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(tempfile.mkdtemp(), "libheddle_place_checked.so")
    _build.build_checked(lib)
    env = dict(os.environ, HEDDLE_PLACE_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "sanitize_run.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bounds violations: 0" in r.stdout, r.stdout[-2000:]


# ------------------------------------------------------------------ N1: SA resource manager on the GPU
def test_sa_gpu_matches_oracle_sa():
    """Alg. 2 with batched GPU PresortedDP evaluations follows exactly the oracle's walk
    (same pre-drawn uniforms; FP32 objectives are bit-exact, so every accept decision agrees)."""
    from oracle import sa as osa
    from paper_2603_28101_b200 import allocator as alloc
    rng = np.random.default_rng(21)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 32, 8)))          # n = 256
    prof = wl.float_profile()
    cfg = alloc.SAConfig(budget=48, m_min=2, m_max=40, max_iters=90)
    iu, su = wl.sa_uniforms(3, 6, 90)
    rm = alloc.ResourceManager(prof, n_max=256, m_max=40, chains=6)
    res = rm.anneal_host(L, cfg, iu, su)
    c, N, chains = osa.anneal(L.astype(np.float64), prof.T, prof.F, prof.degrees, 48, iu, su, m_min=2, m_max=40,
                              max_iters=90)
    assert res.best_makespan == c and res.best_degrees == N
    for (cb, nb), (oc, on, otrace), gtrace in zip(res.chain_best, chains, res.trace):
        assert cb == oc and nb == on and gtrace == otrace
    ref = oracle.solve(oracle.Problem(L, prof.T, prof.F, prof.row_of(list(N)), mode="f32"))
    assert np.array_equal(res.best_boundaries, ref["bounds"])
    # the same walk with the exact objective-only (parametric, N3) evaluator
    rm2 = alloc.ResourceManager(prof, n_max=256, m_max=40, chains=6, objective_only=True)
    res2 = rm2.anneal_host(L, cfg, iu, su)
    assert res2.best_makespan == c and res2.best_degrees == N and res2.trace == res.trace
    assert np.array_equal(res2.best_boundaries, ref["bounds"])
    # and with the full scan as the DP solver (the default is the valley search)
    rm3 = alloc.ResourceManager(prof, n_max=256, m_max=40, chains=6, algo="scan")
    res3 = rm3.anneal_host(L, cfg, iu, su)
    assert res3.best_makespan == c and res3.best_degrees == N and res3.trace == res.trace
    assert np.array_equal(res3.best_boundaries, ref["bounds"])


@pytest.mark.parametrize("kernel", ["layered", "batched", "auto"])
def test_context_reuse_across_shapes(kernel):
    """One context, consecutive solves with different (B, n, m) and an invalid problem in between:
    every solve must match the oracle (per-solve state of the persistent kernel is reset)."""
    from paper_2603_28101_b200.placer import Placer
    prof = wl.float_profile()
    pl = Placer.from_profile(prof, max_n=3000, max_m=40, max_batch=5, kernel=kernel)
    rng = np.random.default_rng(17)
    for it, (B, n, m) in enumerate([(1, 2900, 8), (3, 1500, 37), (2, 2999, 12), (5, 700, 3), (1, 2900, 8)]):
        L = wl.presort_rows(wl.predicted(rng, wl.coding_lengths(rng, (n * B + 7) // 8, 8)[: n * B].reshape(B, n)))
        deg = wl.sorted_degree_vectors(rng, B, m)
        if it == 2:
            L[1, 5], L[1, 6] = L[1, 6], L[1, 5] + 100.0     # problem 1 unsorted
        batch = wl.Batch("reuse", n, m, L.astype(np.float32), deg, prof)
        g = run_gpu(batch, placer=pl)
        for b in range(B):
            ref = oracle.solve(oracle.Problem.from_batch(batch, b, mode="f32"))
            if it == 2 and b == 1:
                assert g["status"][b] == 2
                continue
            assert g["status"][b] == 0, (it, b, g["status"])
            assert g["obj"][b] == ref["opt"] and np.array_equal(g["bounds"][b], ref["bounds"]), (it, b)


# ------------------------------------------------------------------ N2: weighted items (aggregation)
@pytest.mark.parametrize("semiring", ["minmax", "minplus"])
@pytest.mark.parametrize("dtype", ["u32", "f32"])
def test_weighted_random_tiny_exact(dtype, semiring):
    """Item weights (group size = sum of weights, R5) with caps / kv caps / ties: bit-exact."""
    sr = oracle.MINMAX if semiring == "minmax" else oracle.MINPLUS
    done = 0
    for s in range(200):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, allow_weights=True,
                               dtype=dtype)
        if batch.weights is None:
            continue
        done += 1
        kp = s % 2 == 0
        gpu = run_gpu(batch, semiring=semiring, keep_parents=kp)
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode=dtype, semiring=sr), want_tables=True)
        assert_exact(gpu, 0, ref, batch, dtype, semiring, check_parents=kp, tag=f"w{dtype}{s}")
        gpu["placer"].close()
    assert done > 50


# ------------------------------------------------------------------ N3: objective-only parametric solver
@pytest.mark.parametrize("dtype", ["u32", "f32", "f64"])
def test_objective_parametric_random_tiny(dtype):
    """The parametric kernel's optimum equals the DP optimum bit for bit (U32 / F32 against the
    oracle in the same arithmetic; F64 against the GPU DP, same Tr<> arithmetic), incl. caps,
    kv caps, ties, infeasible and invalid problems."""
    for s in range(150):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, dtype=dtype)
        g = run_gpu(batch)
        pl = g["placer"]
        L = to_dev(batch.lengths, {"u32": torch.uint32, "f32": torch.float32, "f64": torch.float64}[dtype])
        D = to_dev(batch.degrees.astype(np.int32))
        caps = None if batch.caps is None else to_dev(batch.caps.astype(np.int32))
        kv = None if batch.kv_caps is None else to_dev(batch.kv_caps.astype(np.int64))
        obj, st = pl.objective(L, D, caps=caps, kv_caps=kv)
        torch.cuda.synchronize()
        o = obj.cpu().numpy().astype(np.float64)
        assert int(st.cpu()[0]) == int(g["status"][0]), s
        assert o[0] == g["obj"][0], (s, o[0], g["obj"][0])
        if dtype != "f64":
            ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode=dtype))
            if ref["status"] == oracle.OK:
                assert o[0] == ref["opt"], s
        pl.close()


def test_objective_parametric_batched_and_large():
    """Whole batched launch (16384 problems) and the n = 65536, m = 256 instance: parametric
    objectives identical to the DP's, problem by problem."""
    from paper_2603_28101_b200.placer import Placer
    for batch in (wl.config_batched(), wl.config_large()):
        g = run_gpu(batch)
        L = to_dev(batch.lengths)
        D = to_dev(batch.degrees.astype(np.int32))
        obj, st = g["placer"].objective(L, D)
        torch.cuda.synchronize()
        assert np.all(st.cpu().numpy() == 0)
        assert np.array_equal(obj.cpu().numpy().astype(np.float64), g["obj"])
        g["placer"].close()

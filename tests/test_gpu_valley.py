"""GPU parity of the valley solver (HEDDLE_VALLEY): K8 (one CTA per problem) and
K8L (one launch per layer) against the CPU oracle, bit-exact in objective, boundaries and
back-pointers, over the same seeded workloads as the full-scan kernels; and against the full
scan itself on the launches the oracle cannot finish (16384 problems, n = 65536)."""
import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from tests.parity import assert_exact, assert_f64_tolerance, run_gpu, to_dev

pytestmark = pytest.mark.gpu

VALLEY_KERNELS = ["batched", "layered"]   # K8 / K8L


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


@pytest.fixture(params=["64", "0"], ids=["scan-prefix", "masks"])
def vscan(request, monkeypatch):
    """K8's two descent-prefix paths: scan the few states before the last descent (default), or
    the masks + sparse-table range minimum (HEDDLE_PLACE_VALLEY_SCAN=0)."""
    monkeypatch.setenv("HEDDLE_PLACE_VALLEY_SCAN", request.param)
    return request.param


@pytest.mark.parametrize("kernel", VALLEY_KERNELS)
@pytest.mark.parametrize("dtype", ["u32", "f32"])
def test_valley_random_tiny_exact(dtype, kernel, vscan):
    """Heavy ties, clamp plateaus (flat F), caps, kv caps, heterogeneous degrees, infeasible and
    invalid problems: identical values, lowest-index boundaries and parent tables."""
    for s in range(200):
        batch = wl.tiny_random(s, n_max=24, m_max=7, allow_caps=True, allow_kv=True, dtype=dtype)
        kp = s % 2 == 0
        gpu = run_gpu(batch, keep_parents=kp, kernel=kernel, algo="valley")
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode=dtype), want_tables=True)
        assert_exact(gpu, 0, ref, batch, dtype, "minmax", check_parents=kp, tag=f"valley-{dtype}{s}")
        gpu["placer"].close()


@pytest.mark.parametrize("dtype", ["u32", "f32", "f64"])
def test_valley_cluster_exact(dtype, monkeypatch):
    """The cluster variant of K8 (8 CTAs per problem exchanging each layer's states over
    distributed shared memory; chosen automatically for few problems with > 640 states per
    layer), forced onto tiny problems -- ties, plateaus, caps, kv caps, weights, mixed degrees,
    infeasible and invalid problems, parts of a layer with no state -- and onto the rollout
    config: bit-exact against the oracle (F64: within the tolerance, identical to the scan)."""
    monkeypatch.setenv("HEDDLE_PLACE_K8_CLUSTER", "2")
    done = 0
    for s in range(150):
        batch = wl.tiny_random(s, n_max=24, m_max=7, allow_caps=True, allow_kv=True, allow_weights=s % 3 == 0,
                               dtype=dtype)
        gpu = run_gpu(batch, kernel="batched", algo="valley")
        p = oracle.Problem.from_batch(batch, 0, mode=dtype)
        if dtype == "f64":
            scan = run_gpu(batch, kernel="batched")
            assert gpu["status"][0] == scan["status"][0]
            if int(scan["status"][0]) == 0:
                assert gpu["obj"][0] == scan["obj"][0] and np.array_equal(gpu["bounds"], scan["bounds"]), s
                assert_f64_tolerance(gpu["obj"][0], gpu["bounds"][0], p, "minmax", tag=f"cl-f64-{s}")
            scan["placer"].close()
        else:
            ref = oracle.solve(p, want_tables=True)
            assert_exact(gpu, 0, ref, batch, dtype, "minmax", tag=f"cl-{dtype}{s}")
        gpu["placer"].close()
        done += 1
    if dtype == "f32":
        for prob in range(3):
            batch = wl.config_rollout(problem=prob)
            gpu = run_gpu(batch, kernel="batched", algo="valley")
            ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32"), want_tables=True)
            assert_exact(gpu, 0, ref, batch, "f32", "minmax", tag=f"cl-rollout{prob}")
    assert done == 150


@pytest.mark.parametrize("kernel", VALLEY_KERNELS)
def test_valley_random_tiny_f64(kernel):
    for s in range(100):
        batch = wl.tiny_random(s, n_max=24, m_max=7, allow_caps=True, allow_kv=True, dtype="f64")
        gpu = run_gpu(batch, kernel=kernel, algo="valley")
        scan = run_gpu(batch, kernel=kernel)
        p = oracle.Problem.from_batch(batch, 0, mode="f64")
        ref = oracle.solve(p)
        assert gpu["status"][0] == scan["status"][0]
        if ref["status"] != oracle.OK:
            assert gpu["status"][0] == ref["status"]
            continue
        assert gpu["obj"][0] == scan["obj"][0] and np.array_equal(gpu["bounds"], scan["bounds"]), s
        assert_f64_tolerance(gpu["obj"][0], gpu["bounds"][0], p, "minmax", tag=f"valley-f64-{s}")
        gpu["placer"].close()
        scan["placer"].close()


@pytest.mark.parametrize("dtype", ["u32", "f32"])
def test_valley_weighted_tiny_exact(dtype, vscan):
    done = 0
    for s in range(200):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, allow_weights=True,
                               dtype=dtype)
        if batch.weights is None:
            continue
        done += 1
        kp = s % 2 == 0
        gpu = run_gpu(batch, keep_parents=kp, algo="valley")
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode=dtype), want_tables=True)
        assert_exact(gpu, 0, ref, batch, dtype, "minmax", check_parents=kp, tag=f"valley-w{dtype}{s}")
        gpu["placer"].close()
    assert done > 50


@pytest.mark.parametrize("kernel", VALLEY_KERNELS)
def test_valley_rollout_and_caps(kernel):
    for prob in range(4):
        batch = wl.config_rollout(problem=prob)
        if prob == 3:
            rng = np.random.default_rng(11)
            batch.caps = rng.integers(16, 40, size=(1, batch.m)).astype(np.int32)
            total = float(batch.lengths.astype(np.float64).sum())
            batch.kv_caps = rng.integers(int(total / 20), int(total / 8), size=(1, batch.m)).astype(np.int64)
        gpu = run_gpu(batch, keep_parents=True, kernel=kernel, algo="valley")
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32"), want_tables=True)
        assert_exact(gpu, 0, ref, batch, "f32", "minmax", check_parents=True, tag=f"valley-rollout{prob}")


def test_valley_tp_sweep_and_batched_sample(vscan):
    for batch, shared in ((wl.config_tp_sweep(), True), (wl.config_batched(B=96), False)):
        gpu = run_gpu(batch, lengths_shared=shared, algo="valley")
        rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
        opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32")
        assert np.all(gpu["status"] == 0)
        assert np.array_equal(gpu["obj"], opt), batch.name
        assert np.array_equal(gpu["bounds"], bounds), batch.name


def test_valley_medium_layered_vs_oracle():
    """K8L at n = 4096 (forced layered, several 256-thread blocks per layer) against the oracle."""
    rng = np.random.default_rng(21)
    n, m = 4096, 24
    L = wl.presort(wl.predicted(rng, wl.search_lengths(rng, n // 8, 8)))
    deg = wl.sorted_degree_vectors(rng, 2, m)
    batch = wl.Batch("medium", n, m, np.stack([L, L]).astype(np.float32), deg, wl.float_profile())
    gpu = run_gpu(batch, kernel="layered", algo="valley")
    rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
    opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32",
                                        threads=2)
    assert np.array_equal(gpu["obj"], opt)
    assert np.array_equal(gpu["bounds"], bounds)


def test_valley_layered_batched_mixed_degrees():
    """K8L (forced layered) on 64 bench problems with mixed degrees -- rows whose descents fall
    inside a warp's run and across the 32-element blocks of different CTAs, found by the layer's
    last CTA (row extras fused into the layer launch) -- and on the TP sweep: identical to the
    oracle's objectives and boundaries."""
    for batch, shared in ((wl.config_batched(B=64), False), (wl.config_tp_sweep(), True)):
        gpu = run_gpu(batch, lengths_shared=shared, kernel="layered", algo="valley")
        rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in range(batch.B)])
        opt, bounds, _ = oracle.solve_batch(batch.lengths, batch.profile.T, batch.profile.F, rows, mode="f32",
                                            threads=4)
        assert np.all(gpu["status"] == 0)
        assert np.array_equal(gpu["obj"], opt), batch.name
        assert np.array_equal(gpu["bounds"], bounds), batch.name


def test_valley_layered_cuda_graph_replay():
    """K8L's layer launches carry the programmatic-dependent-launch attribute: captured into a
    CUDA graph (programmatic edges) and replayed, on fresh inputs written into the captured
    buffers, the results equal an eager solve of the same inputs."""
    from paper_2603_28101_b200.placer import Placer
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    n, m = 4096, 24
    deg = wl.sorted_degree_vectors(rng, 2, m)
    mk = lambda: np.stack([wl.presort(wl.predicted(rng, wl.search_lengths(rng, n // 8, 8))) for _ in range(2)]
                          ).astype(np.float32)
    pl = Placer.from_profile(wl.float_profile(), max_n=n, max_m=m, max_batch=2, device=0, kernel="layered",
                             algo="valley")
    L = torch.from_numpy(mk()).to(dev)
    D = torch.from_numpy(deg.astype(np.int32)).to(dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        pl.solve(L, D)
        pl.backtrack()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            obj_g, _ = pl.solve(L, D)
            bnd_g = pl.backtrack()
    torch.cuda.synchronize()
    for _ in range(2):
        L.copy_(torch.from_numpy(mk()))
        g.replay()
        torch.cuda.synchronize()
        got_obj, got_bnd = obj_g.clone(), bnd_g.clone()
        obj, _ = pl.solve(L, D)
        bnd = pl.backtrack()
        torch.cuda.synchronize()
        assert torch.equal(got_obj, obj) and torch.equal(got_bnd, bnd)
    pl.close()


def test_valley_full_launches_equal_scan(vscan):
    """The bench launches: all 16384 batched problems and the n = 65536, m = 256 instance --
    valley objectives and boundaries identical to the full scan's, problem by problem, and
    sampled batched problems identical to the oracle's."""
    for batch in (wl.config_batched(), wl.config_large()):
        scan = run_gpu(batch)
        scan["placer"].close()
        val = run_gpu(batch, algo="valley")
        assert np.all(val["status"] == 0)
        assert np.array_equal(val["obj"], scan["obj"]), batch.name
        assert np.array_equal(val["bounds"], scan["bounds"]), batch.name
        if batch.B > 1:
            idx = np.array([0, 1, 777, batch.B - 1])
            rows = np.stack([batch.profile.row_of(batch.degrees[b]) for b in idx])
            opt, bounds, _ = oracle.solve_batch(batch.lengths[idx], batch.profile.T, batch.profile.F, rows, mode="f32")
            assert np.array_equal(val["obj"][idx], opt)
            assert np.array_equal(val["bounds"][idx], bounds)
        else:   # n = 65536: the parametric oracle pins the objective (P6)
            q = oracle.parametric_opt(oracle.Problem.from_batch(batch, 0, mode="f32"))
            assert val["obj"][0] == q["opt"]
        val["placer"].close()


def test_valley_host_pipeline():
    """solve_host with the valley kernel: the gated pipelined inputs reach K8 too."""
    from paper_2603_28101_b200.placer import Placer
    batch = wl.config_batched(B=1301, seed_problem=6)
    pl = Placer.from_profile(batch.profile, max_n=batch.n, max_m=batch.m, max_batch=batch.B, algo="valley")
    obj_d, _ = pl.solve(to_dev(batch.lengths), to_dev(batch.degrees.astype(np.int32)))
    bnd_d = pl.backtrack().cpu().numpy()
    obj, bnd, st, _, _ = pl.solve_host(torch.from_numpy(batch.lengths).pin_memory(),
                                       torch.from_numpy(batch.degrees.astype(np.int32)).pin_memory())
    assert (st.numpy() == 0).all()
    assert np.array_equal(obj.numpy(), obj_d.cpu().numpy())
    assert np.array_equal(bnd.numpy(), bnd_d)


def test_valley_rejects_minplus_and_split():
    from paper_2603_28101_b200 import E_INVALID, HeddleError
    from paper_2603_28101_b200.placer import Placer
    prof = wl.float_profile()
    with pytest.raises(HeddleError) as e:
        Placer.from_profile(prof, semiring="minplus", max_n=64, max_m=8, max_batch=1, algo="valley")
    assert e.value.status == E_INVALID
    with pytest.raises(HeddleError) as e:
        Placer.from_profile(prof, max_n=64, max_m=8, max_batch=1, algo="valley", split=(None, 0, 2))
    assert e.value.status == E_INVALID

"""GPU: short-trajectory aggregation on the device (K10, heddle_place_aggregate / _expand) and the
ragged weighted solve of the aggregated batch, against oracle/aggregate.py
and the weighted oracle DP, bit for bit; aggregated >= exact."""
import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from oracle.aggregate import aggregate as ora_aggregate, expand as ora_expand
from paper_2603_28101_b200 import aggregate as agg_mod
from paper_2603_28101_b200.placer import Placer
from tests.parity import to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


@pytest.mark.parametrize("dtype", ["f32", "u32", "f64"])
def test_device_aggregate_matches_oracle(dtype):
    rng = np.random.default_rng(9)
    B, n = 24, 400
    rows = []
    for b in range(B):
        L = wl.presort(wl.coding_lengths(rng, n // 8, 8))
        rows.append(L if dtype != "f32" else wl.predicted(rng, L))
    Ls = np.stack([wl.presort(np.asarray(r, dtype=np.float64)) for r in rows])
    npdt = {"f32": np.float32, "u32": np.uint32, "f64": np.float64}[dtype]
    Ls = Ls.astype(npdt)
    tdt = {"f32": torch.float32, "u32": torch.uint32, "f64": torch.float64}[dtype]
    for thr, bucket in ((0.0, 4), (float(np.percentile(Ls, 50)), 8), (1e9, 3), (float(Ls.min()), 1)):
        agg, w, st, na = agg_mod.aggregate(to_dev(Ls, tdt), thr, bucket)
        torch.cuda.synchronize()
        agg = agg.cpu().numpy() if dtype != "u32" else agg.cpu().view(torch.int32).numpy().view(np.uint32)
        w, st, na = w.cpu().numpy(), st.cpu().numpy(), na.cpu().numpy()
        for b in range(B):
            oi, ow, ost = ora_aggregate(list(Ls[b]), thr, bucket)
            k = na[b]
            assert k == len(oi) and list(agg[b, :k]) == oi and list(w[b, :k]) == ow, (thr, bucket, b)
            assert list(st[b, :k]) == ost[:-1] and st[b, n] == n


@pytest.mark.parametrize("algo", ["scan", "valley"])
def test_aggregated_ragged_solve_matches_weighted_oracle(algo):
    """Rollout-shaped problems, aggregated on the device into a ragged batch (different n'),
    solved with weights in one launch, expanded back: equal to the weighted oracle DP on
    oracle/aggregate.py's items, and never better than the exact optimum."""
    prof = wl.float_profile()
    rng = np.random.default_rng(17)
    B, n, m = 12, 512, 32
    Ls = np.stack([wl.presort(wl.predicted(rng, wl.coding_lengths(rng, n // 8, 8))) for _ in range(B)])
    deg = wl.sorted_degree_vectors(rng, B, m).astype(np.int32)
    thr = float(np.percentile(Ls, 70))
    agg, w, st, na = agg_mod.aggregate(to_dev(Ls), thr, 8)
    pl = Placer.from_profile(prof, max_n=n, max_m=m, max_batch=B, algo=algo)
    obj, status = pl.solve(agg, to_dev(deg), weights=w, ns=na)
    bnd = pl.backtrack()
    full = agg_mod.expand(bnd, st)
    torch.cuda.synchronize()
    obj, status, bnd, full = obj.cpu().numpy(), status.cpu().numpy(), bnd.cpu().numpy(), full.cpu().numpy()
    for b in range(B):
        oi, ow, ost = ora_aggregate(list(Ls[b]), thr, 8)
        p = oracle.Problem(np.asarray(oi), prof.T, prof.F, prof.row_of(deg[b]), mode="f32", w=np.asarray(ow))
        ref = oracle.solve(p)
        assert status[b] == 0 and obj[b] == ref["opt"], (b, obj[b], ref["opt"])
        assert np.array_equal(bnd[b], ref["bounds"]), b
        assert list(full[b]) == ora_expand(list(ref["bounds"]), ost), b
        exact = oracle.solve(oracle.Problem(Ls[b], prof.T, prof.F, prof.row_of(deg[b]), mode="f32"))
        assert obj[b] >= exact["opt"]
    pl.close()


@pytest.mark.parametrize("n,m,kernel", [(2000, 12, "layered"), (20000, 8, "auto")])
def test_weighted_layered_valley_matches_oracle(n, m, kernel):
    """Weights on the per-layer valley kernel (K8L): forced at n = 2000, and chosen by the
    dispatcher at n = 20000 (beyond one CTA's shared memory); bit-exact against the weighted
    oracle DP on device-aggregated items, with mixed degrees and a size cap."""
    prof = wl.float_profile()
    rng = np.random.default_rng(23 + n)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, n // 8, 8)))
    agg, w, st, na = agg_mod.aggregate(to_dev(L[None, :]), float(np.percentile(L, 60)), 4)
    k = int(na.cpu()[0])
    A = agg[:, :k].contiguous()
    Wt = w[:, :k].contiguous()
    deg = wl.sorted_degree_vectors(rng, 1, m).astype(np.int32)
    caps = np.full((1, m), -1, np.int32)
    caps[0, -1] = n // 3
    pl = Placer.from_profile(prof, max_n=n, max_m=m, max_batch=1, algo="valley", kernel=kernel)
    obj, stt = pl.solve(A, to_dev(deg), caps=to_dev(caps), weights=Wt)
    bnd = pl.backtrack()
    torch.cuda.synchronize()
    p = oracle.Problem(A.cpu().numpy()[0], prof.T, prof.F, prof.row_of(deg[0]), mode="f32",
                       w=Wt.cpu().numpy()[0], caps=caps[0])
    ref = oracle.solve(p, threads=8)
    assert int(stt.cpu()[0]) == 0 and float(obj.cpu()[0]) == ref["opt"]
    assert np.array_equal(bnd.cpu().numpy()[0], ref["bounds"])
    pl.close()


@pytest.mark.parametrize("keep_parents", [False, True])
def test_weighted_layered_scan_matches_oracle(keep_parents):
    """Weights on the per-layer scan kernel (K3, cost gathered per cell): random tiny weighted
    problems (ties, caps, kv caps, mixed degrees) and a device-aggregated n = 2000 problem, forced
    onto the layered path; bit-exact against the weighted oracle, back-pointers included."""
    from tests.parity import assert_exact, run_gpu
    done = 0
    for s in range(120):
        batch = wl.tiny_random(s, n_max=20, m_max=6, allow_caps=True, allow_kv=True, allow_weights=True,
                               dtype="f32")
        if batch.weights is None:
            continue
        gpu = run_gpu(batch, keep_parents=keep_parents, kernel="layered")
        ref = oracle.solve(oracle.Problem.from_batch(batch, 0, mode="f32"), want_tables=True)
        assert_exact(gpu, 0, ref, batch, "f32", "minmax", check_parents=keep_parents, tag=f"w-layered-{s}")
        gpu["placer"].close()
        done += 1
    assert done > 30
    prof = wl.float_profile()
    rng = np.random.default_rng(41)
    n, m = 2000, 12
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, n // 8, 8)))
    agg, w, st, na = agg_mod.aggregate(to_dev(L[None, :]), float(np.percentile(L, 60)), 4)
    k = int(na.cpu()[0])
    deg = wl.sorted_degree_vectors(rng, 1, m).astype(np.int32)
    b = wl.Batch("agg2000", k, m, agg[:, :k].cpu().numpy(), deg, prof, weights=w[:, :k].cpu().numpy())
    gpu = run_gpu(b, keep_parents=keep_parents, kernel="layered")
    ref = oracle.solve(oracle.Problem.from_batch(b, 0, mode="f32"), want_tables=True, threads=8)
    assert_exact(gpu, 0, ref, b, "f32", "minmax", check_parents=keep_parents, tag="w-layered-2000")

"""GPU: ragged-m batches (heddle_place_problem.ms) and the device-resident annealer (K9,
heddle_place_anneal) for the resource manager of Alg. 2.

* A ragged batch -- problems with different worker counts in one launch, as the SA proposals
  are -- gives, problem by problem, exactly the oracle's objective and canonical boundaries
  (one-CTA kernels: scan K2 and valley K8; objective-only K7), with -1 padding past m_b.
* The device walk equals the oracle's walk (oracle/sa.py, same pre-drawn uniforms) chain by
  chain: every accepted makespan, each chain's best allocation, and the best partition.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import workloads as wl
from paper_2603_28101_b200.placer import Placer
from tests.parity import to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


def ragged_batch(seed, B, n, m_max, dtype="f32"):
    rng = np.random.default_rng(seed)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, (n + 7) // 8, 8)[:n]))
    ms = rng.integers(1, m_max + 1, size=B).astype(np.int32)
    ms[0], ms[-1] = 1, m_max
    deg = np.full((B, m_max), 8, dtype=np.int32)
    for b in range(B):
        deg[b, :ms[b]] = wl.sorted_degree_vectors(rng, 1, int(ms[b]))[0]
    return L.astype(np.float32), deg, ms


@pytest.mark.parametrize("algo", ["scan", "valley"])
def test_ragged_batch_matches_oracle(algo):
    prof = wl.float_profile()
    n, m_max, B = 700, 24, 40
    L, deg, ms = ragged_batch(5, B, n, m_max)
    pl = Placer.from_profile(prof, max_n=n, max_m=m_max, max_batch=B, algo=algo)
    Ld = to_dev(np.broadcast_to(L, (B, n)))
    obj, st = pl.solve(Ld, to_dev(deg), ms=to_dev(ms))
    bnd = pl.backtrack()
    torch.cuda.synchronize()
    obj, st, bnd = obj.cpu().numpy(), st.cpu().numpy(), bnd.cpu().numpy()
    for b in range(B):
        m = int(ms[b])
        ref = oracle.solve(oracle.Problem(L, prof.T, prof.F, prof.row_of(deg[b, :m]), mode="f32"))
        assert st[b] == 0 and obj[b] == ref["opt"], (b, m, obj[b], ref["opt"])
        assert np.array_equal(bnd[b, :m + 1], ref["bounds"]), (b, m)
        assert np.all(bnd[b, m + 1:] == -1), (b, m)
    # objective only (K7) on the same ragged batch
    o2, s2 = pl.objective(Ld, to_dev(deg), ms=to_dev(ms))
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), obj) and np.all(s2.cpu().numpy() == 0)
    # a worker count outside [1, m] is that problem's E_INVALID; the others are unaffected
    bad = ms.copy()
    bad[3] = m_max + 1
    obj3, st3 = pl.solve(Ld, to_dev(deg), ms=to_dev(bad))
    torch.cuda.synchronize()
    st3 = st3.cpu().numpy()
    assert st3[3] == 1 and np.all(np.delete(st3, 3) == 0)
    assert np.array_equal(np.delete(obj3.cpu().numpy(), 3), np.delete(obj, 3))
    pl.close()


@pytest.mark.parametrize("evaluator", ["valley", "scan", "objective"])
def test_device_anneal_matches_oracle_walk(evaluator):
    from oracle import sa as osa
    from paper_2603_28101_b200 import allocator as alloc
    rng = np.random.default_rng(21)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 32, 8)))          # n = 256
    prof = wl.float_profile()
    cfg = alloc.SAConfig(budget=48, m_min=2, m_max=40, max_iters=200)
    iu, su = wl.sa_uniforms(3, 6, 200)
    rm = alloc.ResourceManager(prof, n_max=256, m_max=40, chains=6, objective_only=evaluator == "objective",
                               algo="scan" if evaluator == "scan" else "valley")
    res = rm.anneal(L, cfg, iu, su)
    c, N, chains = osa.anneal(L.astype(np.float64), prof.T, prof.F, prof.degrees, 48, iu, su, m_min=2, m_max=40,
                              max_iters=200)
    assert res.best_makespan == c and res.best_degrees == N
    for (cb, nb), (oc, on, otrace), gtrace in zip(res.chain_best, chains, res.trace):
        assert cb == oc and nb == on and gtrace == otrace
    ref = oracle.solve(oracle.Problem(L, prof.T, prof.F, prof.row_of(list(N)), mode="f32"))
    assert np.array_equal(res.best_boundaries, ref["bounds"])
    host = rm.anneal_host(L, cfg, iu, su)
    assert host.best_makespan == res.best_makespan and host.trace == res.trace and host.iterations == res.iterations

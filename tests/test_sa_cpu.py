"""Resource-manager simulated annealing (Alg. 2): host logic on CPU.

The product's perturbation protocol (paper_2603_28101_b200.allocator) and the oracle's
independent implementation (oracle.sa) must agree move by move; the oracle SA is pinned by
exhaustive enumeration of allocations on small budgets (SPEC S:438 acceptance)."""
import numpy as np
import pytest

from inputs import workloads as wl
from oracle import sa as osa
from paper_2603_28101_b200 import allocator as alloc

D = (1, 2, 4, 8)


def test_move_examples():
    cfg = alloc.SAConfig(budget=8, m_min=1, m_max=8)
    assert alloc._apply_split((8,), cfg, (0.0, 0.0)) == (4, 4)          # split halves a worker
    assert alloc._apply_merge((4, 4), cfg, (0.0, 0.0)) == (8,)          # merge two equal workers
    assert alloc._apply_redistribute((8, 2), cfg, (0.0, 0.0)) is None    # 10 = 8+2 only
    assert alloc._apply_redistribute((4, 4), cfg, (0.0, 0.0)) is None    # 8 = 4+4 only (8+0 not allowed)
    # (4, 4) among (8, 4, 4): 4 + 4 = 8 has no other allowed pair; (8, 4) -> 12 has none either
    assert alloc._apply_redistribute((8, 4, 4), cfg, (0.0, 0.0)) is None
    # (4, 1) -> 5 = 4 + 1 only; (2, 2) -> 4 = 2+2 only; (4, 2) -> 6 = 4 + 2 only
    assert alloc._apply_redistribute((4, 2, 2), cfg, (0.0, 0.0)) is None


@pytest.mark.parametrize("seed", range(40))
def test_product_and_oracle_perturb_agree(seed):
    rng = np.random.default_rng(seed)
    budget = int(rng.choice([8, 16, 24, 32]))
    cfg = alloc.SAConfig(budget=budget, m_min=1, m_max=int(rng.integers(4, 33)))
    iu, su = wl.sa_uniforms(seed, 1, 50)
    s1 = alloc.initial_state(cfg, 1000, iu[0])
    s2 = osa.initial(budget, set(D), cfg.m_min, cfg.m_max, 1000, cfg.init_moves, iu[0])
    assert s1 == s2
    for t in range(50):
        a = alloc.perturb(s1, cfg, su[0, t])
        b = osa.perturb(s2, set(D), cfg.m_min, cfg.m_max, su[0, t])
        assert a == b, (t, s1, a, b)
        assert sum(a) == budget and list(a) == sorted(a, reverse=True)          # budget, sorted mapping
        assert cfg.m_min <= len(a) <= cfg.m_max and set(a) <= set(D)
        s1 = s2 = a


def test_oracle_sa_near_exhaustive_on_small_budgets():
    """SPEC allocator property: on budgets with few sorted compositions, the annealed best is
    within 5 % of the exhaustive optimum on >= 9 of 10 seeds."""
    prof = wl.float_profile()
    rng = np.random.default_rng(4)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 2, 8))).astype(np.float64)   # n = 16
    budget = 16
    best, _ = osa.exhaustive(L, prof.T, prof.F, D, budget, m_min=2, m_max=16)
    good = 0
    for seed in range(10):
        iu, su = wl.sa_uniforms(100 + seed, 2, 200)
        c, N, _ = osa.anneal(L, prof.T, prof.F, D, budget, iu, su, m_min=2, m_max=16)
        assert sum(N) == budget and c >= best
        good += c <= 1.05 * best
    assert good >= 9, good


def test_oracle_sa_best_monotone_and_deterministic():
    prof = wl.float_profile()
    rng = np.random.default_rng(8)
    L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 6, 8))).astype(np.float64)
    iu, su = wl.sa_uniforms(7, 3, 120)
    r1 = osa.anneal(L, prof.T, prof.F, D, 32, iu, su, m_max=24)
    r2 = osa.anneal(L, prof.T, prof.F, D, 32, iu, su, m_max=24)
    assert r1[0] == r2[0] and r1[1] == r2[1]
    for cbest, _, trace in r1[2]:
        assert cbest <= trace[0] and cbest == min(trace)

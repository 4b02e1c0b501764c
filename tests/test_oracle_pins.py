"""Pins for the CPU oracle (oracle/), independent of the oracle's own DP.

Each test checks the oracle against something other than itself:
  * SPEC.md worked examples and a hand-derived counterexample (tests/golden/),
  * brute-force enumeration of contiguous partitions (P1) and of all set
    partitions (Lemma 1, P3), canonical parents from brute-force prefix optima (P2),
  * closed forms (P4), the parametric-search optimum (P6), invariants (P7).
See SURVEY.md §8c for the pin list and DESIGN.md §Oracle for the readings.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from inputs import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")
N_RANDOM = 600


def homog(L, T, F, m, mode="f64", semiring=oracle.MINMAX, **kw):
    return oracle.Problem(L, [T], [F], [0] * m, mode=mode, semiring=semiring, **kw)


# ------------------------------------------------------------------ P5 worked examples
def test_spec_group_cost_examples():
    g = json.load(open(GOLDEN))
    for case in g["group_cost"]:
        p = homog(case["L"], case["T"], case["F"], 1)
        c = oracle.group_cost(p, 1, case["k"], case["i"])
        assert math.isclose(c, case["expected"], rel_tol=1e-15), case["cite"]


def test_spec_dp_examples():
    g = json.load(open(GOLDEN))
    for case in g["dp"]:
        sr = oracle.MINMAX if case["semiring"] == "minmax" else oracle.MINPLUS
        p = homog(case["L"], case["T"], case["F"], case["m"], mode=case["mode"], semiring=sr)
        r = oracle.solve(p, want_tables=True)
        assert r["status"] == oracle.OK
        assert r["opt"] == case["opt"], case["cite"]
        assert list(r["bounds"]) == case["bounds"], case["cite"]
        if "parents" in case:
            for j, row in case["parents"].items():
                for i, k in row.items():
                    assert r["parent"][int(j), int(i)] == k, (j, i)
            for j, row in case["dp"].items():
                for i, v in row.items():
                    assert r["dp"][int(j), int(i)] == v, (j, i)
            bf = oracle.brute_contiguous(p)
            assert bf["opt"] == case["opt"]
            assert list(bf["bounds_lexfirst"]) == case["lexfirst_bounds"]
            assert bf["n_optimal"] == case["n_optimal"]
            cp = oracle.canonical_parents_bf(p)
            for j, row in case["parents"].items():
                for i, k in row.items():
                    assert cp["parent"][int(j), int(i)] == k


def test_capacity_golden_cases():
    """Hand-derived capacity cases (R6): a group whose token sum (or size) EQUALS its worker's cap
    is admissible and is the optimum, so an off-by-one in the cap test fails here."""
    g = json.load(open(GOLDEN))
    for case in g["capacity"]:
        sr = oracle.MINMAX if case["semiring"] == "minmax" else oracle.MINPLUS
        kw = {}
        if "kv_caps" in case:
            kw["kvcaps"] = case["kv_caps"]
        if "caps" in case:
            kw["caps"] = case["caps"]
        p = homog(case["L"], case["T"], case["F"], case["m"], mode=case["mode"], semiring=sr, **kw)
        r = oracle.solve(p)
        assert r["status"] == oracle.OK, case["cite"]
        assert r["opt"] == case["opt"], (r["opt"], case["cite"])
        assert list(r["bounds"]) == case["bounds"], (list(r["bounds"]), case["cite"])
        bf = oracle.brute_contiguous(p)
        assert bf["opt"] == case["opt"], case["cite"]
        if sr == oracle.MINMAX and case["mode"] != "f64":
            assert oracle.parametric_opt(p)["opt"] == case["opt"], case["cite"]


def test_f32x_mode_sums_float32_costs_in_double():
    """F32X: every candidate is the double sum of float32 costs fl32(L*fl32(T*F)); on
    m = n (one item per worker, P4's closed form for the partition) the objective is that sum,
    computed here with numpy's float32 products and a float64 accumulation."""
    rng = np.random.default_rng(12)
    for _ in range(20):
        n = int(rng.integers(2, 40))
        L = np.sort(rng.uniform(1, 5000, size=n).astype(np.float32))[::-1].astype(np.float64)
        T = float(np.float32(rng.uniform(0.01, 0.1)))
        F = [1.0]
        p = oracle.Problem(L, [T], [F], [0] * n, mode="f32x", semiring=oracle.MINPLUS)
        r = oracle.solve(p)
        g = np.float32(T) * np.float32(1.0)
        want = float(np.sum((L.astype(np.float32) * g).astype(np.float64)))
        assert r["status"] == oracle.OK and list(r["bounds"]) == list(range(n + 1))
        assert abs(r["opt"] - want) <= 1e-12 * want, (r["opt"], want)
        f32 = oracle.solve(oracle.Problem(L, [T], [F], [0] * n, mode="f32", semiring=oracle.MINPLUS))
        assert abs(f32["opt"] - want) <= 1e-5 * want       # the float32 chain: same terms, float sums


def test_infeasible_n_less_than_m():
    p = homog([5, 4], 1.0, [1.0], 3)
    assert oracle.solve(p)["status"] == oracle.INFEASIBLE
    assert oracle.brute_contiguous(p)["status"] == oracle.INFEASIBLE


# ------------------------------------------------------------------ P1 / P2 / P6 random tiny
def _random_tiny(seed, **kw):
    b = wl.tiny_random(seed, **kw)
    return b


@pytest.mark.parametrize("semiring", [oracle.MINMAX, oracle.MINPLUS])
@pytest.mark.parametrize("dtype", ["u32", "f64", "f32"])
def test_dp_equals_brute_force(semiring, dtype):
    """P1: DP objective == exhaustive minimum over all C(n-1, m-1) contiguous
    partitions (acceptance 1 S:624); heterogeneous degrees, clamps,
    caps, weights and kv caps included.  The DP's boundaries must attain OPT."""
    for s in range(N_RANDOM // 3):
        b = wl.tiny_random(s, allow_caps=True, allow_weights=True, allow_kv=True, dtype=dtype)
        p = oracle.Problem.from_batch(b, 0, semiring=semiring)
        r = oracle.solve(p)
        bf = oracle.brute_contiguous(p)
        assert r["status"] == bf["status"], s
        assert r["opt"] == bf["opt"], (s, r["opt"], bf["opt"])
        if r["status"] == oracle.OK:
            bd = r["bounds"]
            assert bd[0] == 0 and bd[-1] == p.n and np.all(np.diff(bd) > 0)
            # the returned partition attains OPT (re-evaluated group by group)
            acc = 0.0
            for j in range(1, p.m + 1):
                c = oracle.group_cost(p, j, int(bd[j - 1]), int(bd[j]))
                if semiring == oracle.MINMAX:
                    acc = max(acc, c)
                else:
                    acc = acc + c
            if semiring == oracle.MINMAX or dtype != "f32":
                assert acc == r["opt"], s
            else:
                assert math.isclose(acc, r["opt"], rel_tol=1e-5), s


@pytest.mark.parametrize("semiring", [oracle.MINMAX, oracle.MINPLUS])
def test_parents_equal_canonical_bruteforce(semiring):
    """P2: every back-pointer equals the lowest k whose brute-force prefix optimum
    combined with the group cost reaches the brute-force optimum of the state."""
    for s in range(200):
        b = wl.tiny_random(s, n_max=11, allow_caps=True, allow_weights=True, allow_kv=True)
        p = oracle.Problem.from_batch(b, 0, semiring=semiring)
        r = oracle.solve(p, want_tables=True)
        cp = oracle.canonical_parents_bf(p)
        n, m = p.n, p.m
        for j in range(1, m + 1):
            for i in range(j, n - (m - j) + 1):
                assert r["dp"][j, i] == cp["opt"][j, i], (s, j, i)
                assert r["parent"][j, i] == cp["parent"][j, i], (s, j, i)


def test_parametric_equals_dp_minmax():
    """P6: the exact-m interval feasibility + bisection optimum equals the DP
    optimum bit for bit (MINMAX), at tiny and medium sizes."""
    for s in range(300):
        b = wl.tiny_random(s, allow_caps=True, allow_weights=True, allow_kv=True,
                           dtype=["u32", "f64", "f32"][s % 3])
        p = oracle.Problem.from_batch(b, 0)
        r = oracle.solve(p)
        q = oracle.parametric_opt(p)
        if q["status"] == oracle.INVALID:   # weighted items can make R_j a non-interval: undecided
            assert b.weights is not None, s
            continue
        assert q["status"] == r["status"], s
        assert q["opt"] == r["opt"], (s, q, r["opt"])
    for s in range(6):  # medium: synthetic rollout-shaped problems
        rng = np.random.default_rng(s)
        L = wl.presort(wl.predicted(rng, wl.coding_lengths(rng, 40, 8)).astype(np.float64))
        prof = wl.float_profile()
        deg = wl.sorted_degree_vectors(rng, 1, 16)[0]
        p = oracle.Problem(L, prof.T, prof.F, prof.row_of(deg), mode="f32")
        assert oracle.parametric_opt(p)["opt"] == oracle.solve(p)["opt"]


# ------------------------------------------------------------------ P3 Lemma 1
def test_lemma1_setpartition_equals_contiguous():
    """Lemma 1 (acceptance 2 S:625): with homogeneous workers,
    size-only monotone F and unit weights, the optimum over ALL set partitions
    equals the optimum over contiguous partitions of the descending-sorted list."""
    checked = 0
    for s in range(400):
        rng = np.random.default_rng(9000 + s)
        n = int(rng.integers(1, 9))
        m = int(rng.integers(1, min(n, 3) + 1))
        L = wl.presort(rng.choice([1.0, 2.0, 3.0, 5.0, 8.0], size=n))
        smax = int(rng.integers(1, 6))
        steps = rng.choice([0.0, 0.5, 1.0], size=smax)
        F = 1.0 + np.cumsum(steps) - steps[0]
        cap = [int(rng.integers(1, n + 1))] * m if rng.random() < 0.3 else None
        p = homog(L, float(rng.uniform(0.5, 2)), F, m, caps=cap)
        sp = oracle.brute_setpartition(p)
        bf = oracle.brute_contiguous(p)
        assert sp["status"] == bf["status"]
        assert sp["opt"] == bf["opt"], (s, sp, bf)
        checked += 1
    assert checked == 400


# ------------------------------------------------------------------ P4 closed forms
def test_closed_forms():
    for s in range(200):
        rng = np.random.default_rng(500 + s)
        n = int(rng.integers(1, 17))
        L = wl.presort(rng.integers(1, 50, size=n).astype(np.float64))
        T = float(rng.integers(1, 4))
        smax = int(rng.integers(1, 20))
        steps = rng.integers(0, 3, size=smax).astype(np.float64)
        F = 1.0 + np.cumsum(steps) - steps[0]
        Fc = lambda size: F[min(size, smax) - 1]
        # m = 1: dp[n][1] = L(tau_1) T F(n)
        r = oracle.solve(homog(L, T, F, 1))
        assert r["opt"] == L[0] * T * Fc(n) and list(r["bounds"]) == [0, n]
        # m = n: singletons, OPT = L[0] T F(1), bounds 0..n
        r = oracle.solve(homog(L, T, F, n))
        assert r["opt"] == L[0] * T * Fc(1) and list(r["bounds"]) == list(range(n + 1))
        # F == 1 (MINMAX): every candidate ties at L[0] T => lowest k = j-1 everywhere
        m = int(rng.integers(1, n + 1))
        r = oracle.solve(homog(L, T, [1.0], m))
        assert r["opt"] == L[0] * T
        assert list(r["bounds"]) == list(range(m)) + [n]
        # F == 1 (MINPLUS): OPT = T (L[0] + sum of the m-1 smallest lengths)
        r = oracle.solve(homog(L, T, [1.0], m, semiring=oracle.MINPLUS))
        expect = L[0] * T + sum(L[t] * T for t in range(n - m + 1, n))
        assert math.isclose(r["opt"], expect, rel_tol=1e-12), (r["opt"], expect)
        # all lengths equal c, F strictly increasing: OPT = c T F(ceil(n/m))
        c = float(rng.integers(1, 9))
        Fs = 1.0 + np.arange(n + 1, dtype=np.float64)
        r = oracle.solve(homog([c] * n, T, Fs, m))
        assert r["opt"] == c * T * Fs[math.ceil(n / m) - 1]
        # MINPLUS, equal lengths, linear F: every partition costs c T (m + a (n - m))
        a = 0.5
        Fl = 1.0 + a * np.arange(n + 1, dtype=np.float64)
        r = oracle.solve(homog([c] * n, T, Fl, m, semiring=oracle.MINPLUS))
        assert math.isclose(r["opt"], c * T * (m + a * (n - m)), rel_tol=1e-12)


# ------------------------------------------------------------------ P7 invariants
def test_invariants_homogeneous_minmax():
    """dp[j][.] non-decreasing in i; OPT non-increasing in m (S:333 'adding a worker
    never increases the DP makespan'); OPT >= L[0] T F(1); each candidate row
    v(k) = max(dp[j-1][k], cost_j(k, i)) is a valley (quasi-convex)."""
    for s in range(60):
        rng = np.random.default_rng(1234 + s)
        L = wl.presort(wl.coding_lengths(rng, 5, 8).astype(np.float64))
        n = L.size
        prof = wl.float_profile(dtype="f64")
        prev = math.inf
        for m in (1, 2, 3, 5, 8, 13):
            p = oracle.Problem(L, prof.T[:1], prof.F[:1], [0] * m)
            r = oracle.solve(p, want_tables=True)
            assert r["opt"] <= prev
            prev = r["opt"]
            assert r["opt"] >= L[0] * prof.T[0] * prof.F[0, 0]
            dp = r["dp"]
            for j in range(1, m + 1):
                row = dp[j, j:n - (m - j) + 1]
                assert np.all(np.diff(row) >= 0), (s, m, j)
            if m == 5:
                j, i = 3, n - 2
                v = [max(dp[j - 1, k], oracle.group_cost(p, j, k, i)) for k in range(j - 1, i)]
                v = np.array(v)
                kmin = int(np.argmin(v))
                assert np.all(np.diff(v[:kmin + 1]) <= 0) and np.all(np.diff(v[kmin:]) >= 0)


def test_f32_emulation_within_tolerance_of_f64():
    """F32EMU (the library's float32 arithmetic) objective within 1e-6 relative of FP64."""
    for s in range(20):
        b = wl.config_rollout(problem=s)
        p64 = oracle.Problem.from_batch(b, 0, mode="f64")
        p32 = oracle.Problem.from_batch(b, 0, mode="f32")
        o64 = oracle.solve(p64)["opt"]
        o32 = oracle.solve(p32)["opt"]
        assert abs(o32 - o64) <= 1e-6 * o64


def test_u32_profile_range_guard_fits():
    """The synthetic integer profile keeps max L * max G below 2^32 - 65536."""
    prof = wl.int_profile()
    G = prof.T[:, None] * prof.F
    assert wl.MAX_TOKENS * G.max() < 2 ** 32 - 65536


def test_generators_long_tail():
    """Workload shape checks (P:243 max > 4x median; S:140 P95/P50 >= 3 for coding)."""
    rng = wl.rng_for(9)
    L = wl.coding_lengths(rng, 512, 8)
    assert L.max() / np.median(L) > 4
    assert np.percentile(L, 95) / np.percentile(L, 50) >= 3
    S = wl.search_lengths(rng, 512, 8)
    assert S.max() / np.median(S) > 4
    b = wl.config_batched(B=8)
    assert np.all(np.diff(b.lengths.astype(np.float64), axis=1) <= 0)
    assert np.all(np.diff(b.degrees, axis=1) <= 0)


# ------------------------------------------------------------------ P8: the valley characterisation
@pytest.mark.parametrize("mode", ["u32", "f32", "f64"])
def test_valley_characterisation_on_oracle_tables(mode):
    """P8 (the premise of the HEDDLE_VALLEY kernels), on the oracle's own tables.
    With L non-increasing and F non-decreasing:
      * c_i(k) (cost of items [k, i) on worker j) is non-increasing in k and non-decreasing in i;
      * with sm_i(k) = min(dp[j-1][k..i-1]) (non-decreasing in k) and k* = the first split with
        sm_i(k) >= c_i(k):  dp[j][i] = min(sm_i(k*), c_i(k*-1)), and k* is non-decreasing in i;
      * the lowest argmin is the first e >= kappa with dp[j-1][e] <= dp[j][i], kappa = the first
        k with c_i(k) <= dp[j][i];
      * with one MP degree for all workers every computed dp row is non-decreasing in i (the
        suffix minimum is then the row itself); with mixed degrees it need not be -- a case
        below must show a descent, so the suffix minimum is really needed.
    Ties, clamp plateaus, caps, kv caps and weights included (tiny_random)."""
    checked = descents = 0
    for s in range(150):
        batch = wl.tiny_random(s, n_max=18, m_max=6, allow_caps=True, allow_kv=True, allow_weights=(s % 3 == 0),
                               dtype=mode)
        p = oracle.Problem.from_batch(batch, 0, mode=mode)
        r = oracle.solve(p, want_tables=True)
        if r["status"] not in (oracle.OK, oracle.INFEASIBLE) or batch.n < batch.m:
            continue
        dp, par = r["dp"], r["parent"]
        n, m = batch.n, batch.m
        homogeneous = len(set(batch.degrees[0].tolist())) == 1
        for j in range(1, m + 1):
            row = [dp[j][i] for i in range(j, n - m + j + 1)]
            mono = all(a <= b for a, b in zip(row, row[1:]))
            assert mono or not homogeneous, (s, j)
            descents += not mono
        for j in range(2, m + 1):
            last_t = -1
            for i in (range(j, n - m + j + 1) if j < m else [n]):
                ks = list(range(j - 1, i))
                c = [oracle.group_cost(p, j, k, i) for k in ks]
                assert all(a >= b for a, b in zip(c, c[1:])), (s, j, i)
                if i > j:
                    assert all(oracle.group_cost(p, j, k, i - 1) <= ck for k, ck in zip(ks[:-1], c)), (s, j, i)
                prev = [dp[j - 1][k] for k in ks]
                sm = [min(prev[q:]) for q in range(len(ks))]
                t = next((q for q in range(len(ks)) if sm[q] >= c[q]), len(ks))
                kst = ks[t] if t < len(ks) else i      # (i = none crossed)
                assert kst >= last_t, (s, j, i)
                last_t = kst
                v = sm[t] if t < len(ks) else math.inf
                if t > 0:
                    v = min(v, c[t - 1])
                assert v == dp[j][i], (s, j, i, v, dp[j][i])
                if v != math.inf:
                    kappa = next(q for q in range(len(ks)) if c[q] <= v)
                    arg = next(q for q in range(kappa, len(ks)) if prev[q] <= v)
                    assert par[j][i] == ks[arg], (s, j, i)
                checked += 1
    assert checked > 1000 and descents > 0

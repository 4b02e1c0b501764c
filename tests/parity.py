"""Shared helpers for the GPU-vs-oracle parity tests (acceptance rule: SURVEY §8c).

  * integer (U32) and float32-emulated oracle: objective, boundaries and every
    back-pointer equal BIT FOR BIT;
  * FP64 oracle: |OPT_gpu - OPT_ora| <= 1e-6 OPT_ora, the GPU's partition costs
    at most OPT_ora (1 + 1e-6) under FP64 arithmetic, and its boundaries equal
    the oracle's except where the oracle's own candidate gap at the first
    differing layer is below 1e-6 relative (north_star near-tie rule).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2603_28101_b200.placer import Placer

REL_TOL = 1e-6  # north_star: "objective within 1e-6 relative" for FP32/FP64 costs
SR = {"minmax": oracle.MINMAX, "minplus": oracle.MINPLUS}
TDT = {"u32": torch.uint32, "f32": torch.float32, "f64": torch.float64, "f32x": torch.float32}


def to_dev(a, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dt is not None:
        t = t.to(dt)
    return t.cuda()


def run_gpu(batch, semiring="minmax", keep_parents=False, dtype=None, placer=None, lengths_shared=False,
            kernel="auto", algo="scan"):
    dtype = dtype or batch.profile.dtype
    if placer is None:
        # weighted items: group sizes reach the total weight, which must fit the cost table (max_n)
        max_n = batch.n if batch.weights is None else max(batch.n, int(batch.weights.sum(axis=1).max()))
        placer = Placer(batch.profile.degrees, batch.profile.T, batch.profile.F, dtype=dtype, semiring=semiring,
                        max_n=max_n, max_m=batch.m, max_batch=batch.B, keep_parents=keep_parents, kernel=kernel,
                        algo=algo)
    L = to_dev(batch.lengths[:1] if lengths_shared else batch.lengths, TDT[dtype])
    if lengths_shared:
        L = L[0]
        L = L.expand(batch.B, batch.n)
    D = to_dev(batch.degrees.astype(np.int32))
    caps = None if batch.caps is None else to_dev(batch.caps.astype(np.int32))
    kv = None if batch.kv_caps is None else to_dev(batch.kv_caps.astype(np.int64))
    w = None if batch.weights is None else to_dev(batch.weights.astype(np.int32))
    obj, st = placer.solve(L, D, caps=caps, kv_caps=kv, weights=w)
    if keep_parents:
        bnd, par = placer.backtrack(parents=True)
    else:
        bnd, par = placer.backtrack(), None
    torch.cuda.synchronize()
    out = dict(obj=obj.cpu().numpy().astype(np.float64) if obj.dtype != torch.uint64 else
               obj.cpu().view(torch.int64).numpy().astype(np.uint64).astype(np.float64),
               status=st.cpu().numpy(), bounds=bnd.cpu().numpy(),
               parents=None if par is None else par.cpu().numpy(), placer=placer)
    return out


def gpu_inf(dtype, semiring):
    if dtype == "u32":
        return float(2 ** 64 - 1) if semiring == "minplus" else float(2 ** 32 - 1)
    return float("inf")


def assert_exact(gpu, b, ref, batch, dtype, semiring, check_parents=False, tag=""):
    """Bit-exact parity of problem b against an oracle result in the same arithmetic."""
    st = int(gpu["status"][b])
    if ref["status"] == oracle.INFEASIBLE:
        assert st == 3, (tag, b, st)
        assert gpu["obj"][b] == gpu_inf(dtype, semiring), (tag, b)
        assert np.all(gpu["bounds"][b] == -1), (tag, b)
        return
    assert st == 0, (tag, b, st)
    assert gpu["obj"][b] == ref["opt"], (tag, b, gpu["obj"][b], ref["opt"])
    assert np.array_equal(gpu["bounds"][b], ref["bounds"]), (tag, b, gpu["bounds"][b], ref["bounds"])
    if check_parents:
        n, m = batch.n, batch.m
        par = gpu["parents"][b]            # [m, n+1], row j-1 = layer j
        for j in range(1, m + 1):
            lo, hi = (n, n) if (j == m and m > 1) else (j, n - m + j)
            want = ref["parent"][j, lo:hi + 1]
            got = par[j - 1, lo:hi + 1]
            assert np.array_equal(got, want), (tag, b, j, np.nonzero(got != want)[0][:5])


def partition_cost_f64(p, bounds, semiring):
    acc = 0.0
    for j in range(1, len(bounds)):
        c = oracle.group_cost(p, j, int(bounds[j - 1]), int(bounds[j]))
        acc = max(acc, c) if semiring == "minmax" else acc + c
    return acc


def assert_f64_tolerance(gpu_obj, gpu_bounds, p64, semiring, tag=""):
    """FP64-oracle acceptance: objective within 1e-6 relative, GPU partition 1e-6-optimal
    under FP64 costs, boundaries equal except at oracle near-ties (<1e-6 gap)."""
    ref = oracle.solve(p64, want_tables=True)
    opt = ref["opt"]
    assert abs(gpu_obj - opt) <= REL_TOL * opt, (tag, gpu_obj, opt)
    cost = partition_cost_f64(p64, gpu_bounds, semiring)
    assert cost <= opt * (1 + REL_TOL), (tag, cost, opt)
    # near-tie walk: follow the GPU's own backtrack from layer m down to layer 1; at
    # every layer where its split differs from the oracle's back-pointer of the SAME state, the
    # oracle's candidate values of the two splits must tie within 1e-6 relative
    dp = ref["dp"]
    m = len(ref["bounds"]) - 1
    assert gpu_bounds[m] == p64.n and gpu_bounds[0] == 0, (tag, gpu_bounds)
    for j in range(m, 1, -1):
        i = int(gpu_bounds[j])
        kg = int(gpu_bounds[j - 1])
        ko = int(ref["parent"][j, i])
        if kg == ko:
            continue

        def v(k):
            c = oracle.group_cost(p64, j, k, i)
            return max(dp[j - 1, k], c) if semiring == "minmax" else dp[j - 1, k] + c
        assert ko >= 0 and abs(v(kg) - v(ko)) <= REL_TOL * v(ko), (tag, j, kg, ko, v(kg), v(ko))


def region_states(n, m, b=0):
    """All states (b, j, i) of the computed region (R8): i in [j, n-m+j] for j < m, i = n for j = m."""
    qj, qi = [], []
    for j in range(1, m + 1):
        lo, hi = (n, n) if (j == m and m > 1) else (j, n - m + j)
        qj.append(np.full(hi - lo + 1, j, dtype=np.int32))
        qi.append(np.arange(lo, hi + 1, dtype=np.int32))
    qj, qi = np.concatenate(qj), np.concatenate(qi)
    return np.full(qj.size, b, dtype=np.int32), qj, qi


def query_gpu(placer, qb, qj, qi):
    """dp values (float64, +inf for the dtype's infinity) and back-pointers of sampled states of the
    placer's last solve, through heddle_place_query."""
    dp, par = placer.query(to_dev(qb), to_dev(qj), to_dev(qi))
    torch.cuda.synchronize()
    if dp.dtype == torch.uint64:
        v = dp.cpu().view(torch.int64).numpy().astype(np.uint64)
        out = v.astype(np.float64)
        out[v == np.uint64(2 ** 64 - 1)] = np.inf
    elif dp.dtype == torch.uint32:
        v = dp.cpu().numpy().astype(np.uint64)
        out = v.astype(np.float64)
        out[v == np.uint64(2 ** 32 - 1)] = np.inf
    else:
        out = dp.cpu().numpy().astype(np.float64)
    return out, par.cpu().numpy()


def assert_tables_exact(placer, b, ref, n, m, tag=""):
    """Every dp value and back-pointer of problem b's computed region, read back through
    heddle_place_query, equal to the oracle's tables bit for bit (U32 / F32-emulation modes)."""
    qb, qj, qi = region_states(n, m, b)
    dp, par = query_gpu(placer, qb, qj, qi)
    want_dp = ref["dp"][qj, qi]
    want_par = ref["parent"][qj, qi]
    bad = np.nonzero((dp != want_dp) | (par != want_par))[0]
    assert bad.size == 0, (tag, b, [(int(qj[t]), int(qi[t]), dp[t], want_dp[t], int(par[t]), int(want_par[t]))
                                    for t in bad[:5]])

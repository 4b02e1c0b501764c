"""TEST INFRASTRUCTURE -- plain CPU Sort-Initialized Simulated Annealing (§6.2, Alg. 2,
P:739-765) with oracle.solve as PresortedDP.  Written from the paper and the readings R13-R16
of DESIGN.md, independently of paper_2603_28101_b200/allocator.py; both consume the same
pre-drawn uniforms (inputs.workloads.sa_uniforms) through the same documented protocol:

  per iteration, per chain: u = (u_kind, u_first, u_second, u_accept)
  kind order starts at floor(3 u_kind) in (split, merge, redistribute) and falls through to the
  next kind when a move is inapplicable; candidates are listed in the documented order and
  picked by floor(u * count); an inapplicable step leaves the state unchanged.
"""
from __future__ import annotations

import math

import numpy as np

from . import Problem, solve


def makespan(L, T, F, degrees_all, state, mode="f32"):
    """Alg. 2 line 3 / 8: PresortedDP of the sorted allocation (worker j -> j-th degree)."""
    rows = [list(degrees_all).index(d) for d in state]
    r = solve(Problem(L, T, F, rows, mode=mode))
    return r["opt"], r["bounds"]


def moves_split(state, D, m_max):
    """Degrees d (descending, distinct) that can split into two d/2."""
    if len(state) >= m_max:
        return []
    return sorted({d for d in state if d % 2 == 0 and (d // 2) in D}, reverse=True)


def moves_merge(state, D, m_min):
    if len(state) <= m_min:
        return []
    return sorted({d for d in state if state.count(d) >= 2 and (2 * d) in D}, reverse=True)


def moves_redistribute(state, D):
    """[((v, w), [(x, y), ...])] over distinct value pairs v >= w present in the state."""
    out = []
    vals = sorted(set(state), reverse=True)
    Dd = sorted(D, reverse=True)
    for a in range(len(vals)):
        for b in range(a, len(vals)):
            v, w = vals[a], vals[b]
            if v == w and state.count(v) < 2:
                continue
            alt = [(x, y) for x in Dd for y in Dd if x >= y and x + y == v + w and (x, y) != (v, w)]
            if alt:
                out.append(((v, w), alt))
    return out


def pick(seq, u):
    return seq[min(int(u * len(seq)), len(seq) - 1)]


def perturb(state, D, m_min, m_max, u):
    kind0 = min(int(u[0] * 3), 2)
    for t in range(3):
        kind = (kind0 + t) % 3
        s = list(state)
        if kind == 0:
            c = moves_split(state, D, m_max)
            if c:
                d = pick(c, u[1])
                s.remove(d)
                s += [d // 2, d // 2]
                return tuple(sorted(s, reverse=True))
        elif kind == 1:
            c = moves_merge(state, D, m_min)
            if c:
                d = pick(c, u[1])
                s.remove(d)
                s.remove(d)
                s.append(2 * d)
                return tuple(sorted(s, reverse=True))
        else:
            c = moves_redistribute(state, D)
            if c:
                (v, w), alt = pick(c, u[1])
                x, y = pick(alt, u[2])
                s.remove(v)
                s.remove(w)
                s += [x, y]
                return tuple(sorted(s, reverse=True))
    return tuple(state)


def initial(budget, D, m_min, m_max, n, init_moves, u):
    feas = [d for d in sorted(D, reverse=True) if budget % d == 0 and m_min <= budget // d <= min(m_max, n)]
    d = pick(feas, u[0])
    s = tuple([d] * (budget // d))
    for t in range(init_moves):
        s2 = perturb(s, D, m_min, m_max, u[1 + 3 * t: 4 + 3 * t])
        if len(s2) <= n:
            s = s2
    return s


def anneal(L, T, F, degrees_all, budget, init_u, step_u, cooling=0.95, eps_frac=1e-3, max_iters=2000,
           m_min=1, m_max=64, init_moves=8, mode="f32"):
    """Independent chains of Alg. 2.  Returns (best makespan, best degrees, per-chain traces)."""
    D = set(degrees_all)
    n = len(L)
    res = []
    for c in range(init_u.shape[0]):
        N = initial(budget, D, m_min, m_max, n, init_moves, init_u[c])            # lines 1-2
        C, _ = makespan(L, T, F, degrees_all, N, mode)                             # line 3
        Tm, Cbest, Nbest = C, C, N                                                 # line 4
        eps = eps_frac * C
        trace = [C]
        it = 0
        while Tm > eps and it < min(max_iters, step_u.shape[1]):                   # line 5
            Np = perturb(N, D, m_min, m_max, step_u[c, it])                        # lines 6-7
            if len(Np) > n:
                Np = N
            Cp, _ = makespan(L, T, F, degrees_all, Np, mode)                       # line 8
            dlt = Cp - C                                                           # line 9
            if dlt < 0 or step_u[c, it, 3] < math.exp(-dlt / Tm):                  # lines 10-11
                N, C = Np, Cp
                trace.append(C)
            if C < Cbest:                                                          # lines 13-14
                Cbest, Nbest = C, N
            Tm = cooling * Tm                                                      # line 16
            it += 1
        res.append((Cbest, Nbest, trace))
    b = min(range(len(res)), key=lambda i: (res[i][0], i))
    return res[b][0], res[b][1], res


def exhaustive(L, T, F, degrees_all, budget, m_min=1, m_max=64, mode="f32"):
    """Minimum over every sorted allocation (multiset of allowed degrees summing to the budget)."""
    D = sorted(set(degrees_all), reverse=True)
    best = (math.inf, None)

    def rec(prefix, rem, maxd):
        nonlocal best
        if rem == 0:
            if m_min <= len(prefix) <= min(m_max, len(L)):
                c, _ = makespan(L, T, F, degrees_all, tuple(prefix), mode)
                if c < best[0]:
                    best = (c, tuple(prefix))
            return
        if len(prefix) >= min(m_max, len(L)):
            return
        for d in D:
            if d <= maxd and d <= rem:
                rec(prefix + [d], rem - d, d)
    rec([], budget, max(D))
    return best


__all__ = ["anneal", "exhaustive", "perturb", "initial", "makespan"]
_ = np

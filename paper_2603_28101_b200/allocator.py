"""Sort-initialised simulated annealing over per-worker MP degrees (§6.2, Alg. 2),
with every PresortedDP evaluation running on the GPU.

Alg. 2 is one sequential chain; the GPU turns the "~120 DPs of ~42 ms each" of the paper's resource
manager (Table) into P independent chains walked together.
`ResourceManager.anneal` runs the whole walk on the device (heddle_place_anneal, kernel K9): per
iteration a perturb kernel, ONE ragged solve of all P proposals (their worker counts differ) and a
Metropolis kernel, captured once as a CUDA graph -- the host only draws the start states and reads
the results.  `ResourceManager.anneal_host` is the same walk with the moves and the acceptance in
Python (one solve per distinct worker count per iteration), kept as a reference.

Readings (R13-R16; the paper names the moves but does not define them):
  * state: the sorted (descending) multiset of degrees {N_i}, sum N_i = N (budget);
  * split: a worker of degree d with d/2 allowed -> two workers of d/2;
    merge: two workers of equal degree d with 2d allowed -> one worker of 2d;
    redistribute: two workers (v, w) -> another pair (x, y) of allowed degrees with x + y = v + w;
    the worker count m changes with split / merge and stays in [m_min, m_max] (and <= n);
  * T0 = the initial state's makespan, T <- alpha T each iteration, stop
    when T <= eps_frac * T0 or after max_iters; accept if dC < 0 or u < exp(-dC / T).
  * randomness is an INPUT (inputs.workloads.sa_uniforms): per chain, init uniforms and 4
    uniforms per iteration (move kind, first choice, second choice, acceptance), consumed by
    the fixed protocol below, so the walk is reproducible and checkable step by step.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from .placer import Placer


@dataclasses.dataclass
class SAConfig:
    budget: int                      # total GPUs N
    degrees: tuple = (1, 2, 4, 8)    # allowed MP degrees D
    cooling: float = 0.95            # alpha
    eps_frac: float = 1e-3           # epsilon = eps_frac * T0
    max_iters: int = 2000
    m_min: int = 1
    m_max: int = 64
    init_moves: int = 8              # random moves applied to the homogeneous start


# ----------------------------------------------------------------------------- moves
def _apply_split(state, cfg, u):
    D = set(cfg.degrees)
    if len(state) + 1 > cfg.m_max:
        return None
    cand = sorted({d for d in state if d % 2 == 0 and d // 2 in D}, reverse=True)
    if not cand:
        return None
    d = cand[min(int(u[0] * len(cand)), len(cand) - 1)]
    s = list(state)
    s.remove(d)
    s += [d // 2, d // 2]
    return tuple(sorted(s, reverse=True))


def _apply_merge(state, cfg, u):
    D = set(cfg.degrees)
    if len(state) - 1 < cfg.m_min:
        return None
    cand = sorted({d for d in state if state.count(d) >= 2 and 2 * d in D}, reverse=True)
    if not cand:
        return None
    d = cand[min(int(u[0] * len(cand)), len(cand) - 1)]
    s = list(state)
    s.remove(d)
    s.remove(d)
    s.append(2 * d)
    return tuple(sorted(s, reverse=True))


def _apply_redistribute(state, cfg, u):
    Ds = sorted(cfg.degrees, reverse=True)
    vals = sorted(set(state), reverse=True)
    pairs = []
    for i, v in enumerate(vals):
        for w in vals[i:]:
            if v == w and state.count(v) < 2:
                continue
            alts = [(x, y) for x in Ds for y in Ds if x >= y and x + y == v + w and (x, y) != (v, w)]
            if alts:
                pairs.append(((v, w), alts))
    if not pairs:
        return None
    (v, w), alts = pairs[min(int(u[0] * len(pairs)), len(pairs) - 1)]
    x, y = alts[min(int(u[1] * len(alts)), len(alts) - 1)]
    s = list(state)
    s.remove(v)
    s.remove(w)
    s += [x, y]
    return tuple(sorted(s, reverse=True))


MOVES = (_apply_split, _apply_merge, _apply_redistribute)


def perturb(state, cfg, u4):
    """Alg. 2 Perturb under the fixed protocol: kind = floor(3 u0), then the next kinds
    in order if inapplicable; u1, u2 pick inside the move; unchanged if nothing applies."""
    first = min(int(u4[0] * 3), 2)
    for t in range(3):
        nxt = MOVES[(first + t) % 3](state, cfg, (u4[1], u4[2]))
        if nxt is not None:
            return nxt
    return state


def initial_state(cfg, n, u_init):
    """Homogeneous start with the degree picked by u_init[0] among those that give an allowed
    worker count, then cfg.init_moves random moves (u_init[1:] in groups of 3), sorted."""
    feas = [d for d in sorted(cfg.degrees, reverse=True)
            if cfg.budget % d == 0 and cfg.m_min <= cfg.budget // d <= min(cfg.m_max, n)]
    if not feas:
        raise ValueError("no homogeneous allocation fits the budget and worker bounds")
    d = feas[min(int(u_init[0] * len(feas)), len(feas) - 1)]
    s = tuple([d] * (cfg.budget // d))
    for t in range(cfg.init_moves):
        s2 = perturb(s, cfg, u_init[1 + 3 * t: 4 + 3 * t])
        if len(s2) <= n:
            s = s2
    return s


# ----------------------------------------------------------------------------- driver
@dataclasses.dataclass
class SAResult:
    best_degrees: tuple
    best_makespan: float
    best_boundaries: np.ndarray
    iterations: int
    evaluations: int
    chain_best: list
    trace: list          # per chain: accepted makespans (for tests)


class ResourceManager:
    """Batched-GPU evaluator for the SA walk.  One Placer (max_batch = chains)."""

    def __init__(self, profile, n_max, m_max, chains, device=None, objective_only=False, algo="valley"):
        """objective_only: evaluate makespans with the exact parametric kernel (heddle_place_objective,
        N3) instead of the full DP; the best allocation's partition is solved by the DP at the end.
        algo: the DP's solver, "valley" (N3, exact, O(n m log n)) or "scan" (every split of Eq. 3);
        both give identical makespans and partitions."""
        self.placer = Placer.from_profile(profile, max_n=n_max, max_m=m_max, max_batch=chains, device=device,
                                          algo=algo)
        self.dev = self.placer.device
        self.evaluations = 0
        self.objective_only = objective_only

    def makespans(self, L, states):
        """PresortedDP makespan of each degree multiset (sorted mapping); one batched
        solve per distinct worker count.  L: device tensor [n], sorted descending."""
        out = [None] * len(states)
        by_m = {}
        for idx, s in enumerate(states):
            by_m.setdefault(len(s), []).append(idx)
        n = L.shape[-1]
        for m, idxs in sorted(by_m.items()):
            if m > n:
                for i in idxs:
                    out[i] = (math.inf, None)
                continue
            deg = torch.tensor([states[i] for i in idxs], dtype=torch.int32, device=self.dev)
            Lb = L.reshape(1, n).expand(len(idxs), n)
            if self.objective_only:
                obj, st = self.placer.objective(Lb, deg)
                bnds = [None] * len(idxs)
            else:
                obj, st = self.placer.solve(Lb, deg)
                bnds = self.placer.backtrack().cpu().numpy()
            objs = obj.double().cpu().numpy()
            self.evaluations += len(idxs)
            for r, i in enumerate(idxs):
                out[i] = (float(objs[r]), bnds[r])
        return out

    def anneal(self, lengths, cfg: SAConfig, init_uniforms, step_uniforms) -> SAResult:
        """P chains of Alg. 2 on the device (heddle_place_anneal); same inputs and result as
        anneal_host.  init_uniforms [P, 1 + 3 cfg.init_moves], step_uniforms [P, iters, 4]."""
        import ctypes
        from . import _lib as C
        if set(cfg.degrees) != set(int(d) for d in self.placer._deg):
            raise ValueError("SAConfig.degrees must be the profile's degrees")
        L = lengths if isinstance(lengths, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(lengths))
        L = L.to(self.dev).reshape(-1).contiguous()
        n = L.shape[0]
        P = init_uniforms.shape[0]
        M = cfg.m_max
        iters = min(cfg.max_iters, step_uniforms.shape[1])
        starts = [initial_state(cfg, n, init_uniforms[c]) for c in range(P)]
        rows = np.full((P, M), max(cfg.degrees), dtype=np.int32)
        for c, st in enumerate(starts):
            rows[c, :len(st)] = st
        init_deg = torch.from_numpy(rows).to(self.dev)
        init_m = torch.tensor([len(st) for st in starts], dtype=torch.int32, device=self.dev)
        u = torch.from_numpy(np.ascontiguousarray(step_uniforms[:, :iters, :], dtype=np.float64)).to(self.dev)
        best = torch.empty(P, dtype=torch.float64, device=self.dev)
        best_deg = torch.empty((P, M), dtype=torch.int32, device=self.dev)
        best_m = torch.empty(P, dtype=torch.int32, device=self.dev)
        trace = torch.empty((P, iters + 1), dtype=torch.float64, device=self.dev)
        accepted = torch.empty((P, max(iters, 1)), dtype=torch.int32, device=self.dev)
        nit = ctypes.c_int32(0)
        p = lambda t: ctypes.c_void_p(t.data_ptr())
        args = C.AnnealArgs(n, p(L), P, cfg.m_min, M, p(init_deg), p(init_m), p(u), iters, cfg.cooling,
                            cfg.eps_frac, 1 if self.objective_only else 0)
        out = C.AnnealOut(p(best), p(best_deg), p(best_m), p(trace), p(accepted),
                          ctypes.cast(ctypes.byref(nit), ctypes.c_void_p))
        s = torch.cuda.current_stream(self.dev).cuda_stream
        C.check(C.lib().heddle_place_anneal(self.placer._h, ctypes.byref(args), ctypes.byref(out),
                                            ctypes.c_void_p(s)), "heddle_place_anneal")
        it = nit.value
        self.evaluations += P * (1 + it)
        best_h, bdeg_h, bm_h = best.cpu().numpy(), best_deg.cpu().numpy(), best_m.cpu().numpy()
        tr_h, acc_h = trace.cpu().numpy(), accepted.cpu().numpy()
        chain_best = [(float(best_h[c]), tuple(int(d) for d in bdeg_h[c, :bm_h[c]])) for c in range(P)]
        traces = [[float(tr_h[c, 0])] + [float(tr_h[c, t + 1]) for t in range(it) if acc_h[c, t]] for c in range(P)]
        b = min(range(P), key=lambda c: (chain_best[c][0], c))
        bounds = None
        if math.isfinite(chain_best[b][0]):   # the best allocation's partition: one DP + backtrack
            saved, self.objective_only = self.objective_only, False
            bounds = self.makespans(L, [chain_best[b][1]])[0][1]
            self.evaluations -= 1
            self.objective_only = saved
        return SAResult(chain_best[b][1], chain_best[b][0], bounds, it, self.evaluations, chain_best, traces)

    def anneal_host(self, lengths, cfg: SAConfig, init_uniforms, step_uniforms) -> SAResult:
        """P chains of Alg. 2 with the moves and the Metropolis step on the host (reference for
        anneal); init_uniforms [P, 1 + 3 cfg.init_moves], step_uniforms [P, iters, 4]."""
        L = lengths if isinstance(lengths, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(lengths))
        L = L.to(self.dev).reshape(-1)
        n = L.shape[0]
        P = init_uniforms.shape[0]
        cur = [initial_state(cfg, n, init_uniforms[c]) for c in range(P)]
        ev = self.makespans(L, cur)
        C = [e[0] for e in ev]
        best = [(C[c], cur[c], ev[c][1]) for c in range(P)]
        T = list(C)
        eps = [cfg.eps_frac * t for t in C]
        trace = [[c0] for c0 in C]
        it = 0
        iters = min(cfg.max_iters, step_uniforms.shape[1])
        while it < iters:
            live = [c for c in range(P) if T[c] > eps[c]]
            if not live:
                break
            props = {c: perturb(cur[c], cfg, step_uniforms[c, it]) for c in live}
            for c in live:                              # proposals beyond n workers are infeasible
                if len(props[c]) > n:
                    props[c] = cur[c]
            res = self.makespans(L, [props[c] for c in live])
            for (c, (Cn, bd)) in zip(live, res):
                d = Cn - C[c]
                if d < 0 or step_uniforms[c, it, 3] < math.exp(-d / T[c]):
                    cur[c], C[c] = props[c], Cn
                    trace[c].append(Cn)
                    if Cn < best[c][0]:
                        best[c] = (Cn, props[c], bd)
                T[c] *= cfg.cooling
            it += 1
        b = min(range(P), key=lambda c: (best[c][0], c))
        bounds = best[b][2]
        if bounds is None and math.isfinite(best[b][0]):   # objective-only walk: one DP for the partition
            saved, self.objective_only = self.objective_only, False
            bounds = self.makespans(L, [best[b][1]])[0][1]
            self.evaluations -= 1
            self.objective_only = saved
        return SAResult(best[b][1], best[b][0], bounds, it, self.evaluations,
                        [(x[0], x[1]) for x in best], trace)

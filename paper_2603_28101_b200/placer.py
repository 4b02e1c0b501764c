"""Thin torch-facing wrapper over the C ABI (argument marshalling only).

    placer = Placer(profile, dtype="f32", max_n=1024, max_m=32, max_batch=16384)
    obj, status = placer.solve(lengths, degrees)       # device tensors, async on the current stream
    bounds = placer.backtrack()                          # [B, m+1] int32 boundaries b_0=0 < ... < b_m=n

PAPER.md §5.2: presorted DP; see include/heddle_place.h for the
exact semantics of each argument.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as C

_TORCH_DT = {C.U32: torch.uint32, C.F32: torch.float32, C.F64: torch.float64, C.F32X: torch.float32}
_NP_DT = {C.U32: np.uint32, C.F32: np.float32, C.F64: np.float64, C.F32X: np.float32}


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _rows(t, B, width, name):
    """(tensor, stride) for a [B, width] or broadcast [width] device tensor."""
    if t is None:
        return None, 0
    if t.dim() == 1:
        if t.shape[0] != width:
            raise ValueError(f"{name}: expected {width} entries, got {t.shape[0]}")
        return t.contiguous(), 0
    if t.shape[-1] != width or t.shape[0] not in (1, B):
        raise ValueError(f"{name}: expected [{B}, {width}], got {tuple(t.shape)}")
    if t.shape[0] == 1:
        return t[0].contiguous(), 0
    if t.stride(-1) != 1:
        t = t.contiguous()
    return t, t.stride(0)


class Placer:
    """One heddle_place context: a profile (MP degrees, T, F) and workspace limits."""

    def __init__(self, degrees, T, F, *, dtype="f32", semiring="minmax", max_n, max_m, max_batch,
                 device=None, keep_parents=False, kernel="auto", algo="scan", split=None):
        """split=(unique_id_bytes or None, rank, world): multi-GPU split mode (collective solves);
        unique_id None with rank 0 runs the single-device emulation of `world` ranks.
        algo: "scan" evaluates every split of Eq. 3; "valley" (min-max only) finds the same
        values and argmins by the valley search (HEDDLE_VALLEY, O(n m log n))."""
        self.dtype = C.DTYPES[dtype] if isinstance(dtype, str) else dtype
        self.semiring = C.SEMIRINGS[semiring] if isinstance(semiring, str) else semiring
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        npdt = _NP_DT[self.dtype]
        self._deg = np.ascontiguousarray(np.asarray(degrees, dtype=np.int32))
        self._T = np.ascontiguousarray(np.asarray(T).astype(npdt))
        F = np.asarray(F)
        if F.ndim == 1:
            F = F[None, :]
        self._F = np.ascontiguousarray(F.astype(npdt))
        cfg = C.Config(self.device.index, self.dtype, self.semiring, max_n, max_m, max_batch, self._deg.size,
                       self._deg.ctypes.data, self._T.ctypes.data, self._F.ctypes.data, self._F.shape[1],
                       (C.KEEP_PARENTS if keep_parents else 0) | C.KERNELS[kernel] | C.ALGOS[algo])
        h = ctypes.c_void_p()
        if split is None:
            C.check(C.lib().heddle_place_init(ctypes.byref(cfg), ctypes.byref(h)), "heddle_place_init")
        else:
            uid, rank, world = split
            idbuf = None if uid is None else ctypes.create_string_buffer(bytes(uid), len(uid))
            C.check(C.lib().heddle_place_init_split(ctypes.byref(cfg), idbuf, rank, world, ctypes.byref(h)),
                    "heddle_place_init_split")
        self._h = h
        self.keep_parents = keep_parents
        self.algo = algo
        self.max_n, self.max_m, self.max_batch = max_n, max_m, max_batch
        self._last = None

    @classmethod
    def from_profile(cls, profile, **kw):
        """From an inputs.workloads.Profile-like object (degrees, T, F, dtype)."""
        kw.setdefault("dtype", profile.dtype)
        return cls(profile.degrees, profile.T, profile.F, **kw)

    def close(self):
        if getattr(self, "_h", None):
            C.lib().heddle_place_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def objective_dtype(self):
        if self.dtype == C.U32 and self.semiring == C.MINPLUS:
            return torch.uint64
        if self.dtype == C.F32X:
            return torch.float64
        return _TORCH_DT[self.dtype]

    @property
    def launches(self) -> int:
        return int(C.lib().heddle_place_launch_count(self._h))

    def _problem(self, lengths, degrees, caps, kv_caps, weights=None, ms=None, ns=None):
        if lengths.dim() == 1:
            lengths = lengths[None, :]
        B, n = lengths.shape
        if degrees.dim() == 1:
            m = degrees.shape[0]
        else:
            m = degrees.shape[-1]
        if lengths.dtype != _TORCH_DT[self.dtype]:
            raise TypeError(f"lengths must be {_TORCH_DT[self.dtype]}, got {lengths.dtype}")
        for t, nm in ((lengths, "lengths"), (degrees, "degrees"), (caps, "caps"), (kv_caps, "kv_caps"),
                      (weights, "weights")):
            if t is not None and t.device != self.device:
                raise ValueError(f"{nm} must live on {self.device}")
        L, ls = _rows(lengths, B, n, "lengths")
        D, ds = _rows(degrees.to(torch.int32), B, m, "degrees")
        Cp, cs = _rows(None if caps is None else caps.to(torch.int32), B, m, "caps")
        K, ks = _rows(None if kv_caps is None else kv_caps.to(torch.int64), B, m, "kv_caps")
        Wt, wts = _rows(None if weights is None else weights.to(torch.int32), B, n, "weights")
        def counts(t, nm):
            if t is None:
                return None
            if t.device != self.device:
                raise ValueError(f"{nm} must live on {self.device}")
            t = t.to(torch.int32).contiguous()
            if t.shape != (B,):
                raise ValueError(f"{nm}: expected [{B}], got {tuple(t.shape)}")
            return t
        Ms, Ns = counts(ms, "ms"), counts(ns, "ns")
        keep = (L, D, Cp, K, Wt, Ms, Ns)
        p = C.Problem(n, m, B, L.data_ptr(), ls, D.data_ptr(), ds, Cp.data_ptr() if Cp is not None else None, cs,
                      K.data_ptr() if K is not None else None, ks, Wt.data_ptr() if Wt is not None else None, wts,
                      Ms.data_ptr() if Ms is not None else None, Ns.data_ptr() if Ns is not None else None)
        return p, keep, B, n, m

    def solve(self, lengths, degrees, caps=None, kv_caps=None, stream=None, weights=None, ms=None, ns=None):
        """Enqueue the DP on `stream` (default: torch's current stream).  Returns
        (objective[B], status[B]) device tensors.  `weights` ([B, n] int >= 1): aggregated items
        (short-trajectory aggregation); group size = sum of weights.  `ms` ([B] int):
        per-problem worker counts of a ragged batch (degrees padded to [B, max m]); `ns` ([B] int):
        per-problem item counts (lengths / weights padded to [B, max n])."""
        p, keep, B, n, m = self._problem(lengths, degrees, caps, kv_caps, weights, ms, ns)
        obj = torch.empty(B, dtype=self.objective_dtype, device=self.device)
        st = torch.empty(B, dtype=torch.int32, device=self.device)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        C.check(C.lib().heddle_place_solve(self._h, ctypes.byref(p), _ptr(obj), _ptr(st), ctypes.c_void_p(s)),
                "heddle_place_solve")
        self._last = (keep, B, n, m)  # keep inputs alive until backtrack
        return obj, st

    def objective(self, lengths, degrees, caps=None, kv_caps=None, stream=None, ms=None, ns=None):
        """Exact min-max optimum only (no partition), by the parametric search kernel (N3):
        bit-identical to solve()'s objective at O(m log n) probes per bisection step."""
        p, keep, B, n, m = self._problem(lengths, degrees, caps, kv_caps, None, ms, ns)
        obj = torch.empty(B, dtype=self.objective_dtype, device=self.device)
        st = torch.empty(B, dtype=torch.int32, device=self.device)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        C.check(C.lib().heddle_place_objective(self._h, ctypes.byref(p), _ptr(obj), _ptr(st), ctypes.c_void_p(s)),
                "heddle_place_objective")
        self._keep_obj = keep
        return obj, st

    def backtrack(self, parents=False, stream=None):
        """Boundaries [B, m+1] (and parents [B, m, n+1] when requested) of the last solve."""
        if self._last is None:
            C.check(C.E_STATE, "heddle_place_backtrack")
        _, B, n, m = self._last
        bnd = torch.empty((B, m + 1), dtype=torch.int32, device=self.device)
        par = torch.empty((B, m, n + 1), dtype=torch.int32, device=self.device) if parents else None
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        C.check(C.lib().heddle_place_backtrack(self._h, _ptr(bnd), _ptr(par), ctypes.c_void_p(s)),
                "heddle_place_backtrack")
        return (bnd, par) if parents else bnd

    def query(self, qb, qj, qi, stream=None):
        """dp[j][i] and the lowest-index back-pointer parent[j][i] of sampled states (b, j, i) of the
        last solve (heddle_place_query).  qb, qj, qi: int32 device tensors of equal length.
        Returns (dp[nq] in the objective dtype, parent[nq] int32)."""
        if self._last is None:
            C.check(C.E_STATE, "heddle_place_query")
        qb, qj, qi = (t.to(device=self.device, dtype=torch.int32).contiguous() for t in (qb, qj, qi))
        nq = qb.numel()
        dp = torch.empty(nq, dtype=self.objective_dtype, device=self.device)
        par = torch.empty(nq, dtype=torch.int32, device=self.device)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        C.check(C.lib().heddle_place_query(self._h, nq, _ptr(qb), _ptr(qj), _ptr(qi), _ptr(dp), _ptr(par),
                                           ctypes.c_void_p(s)), "heddle_place_query")
        self._keep_q = (qb, qj, qi)
        return dp, par

    def solve_host(self, lengths, degrees, caps=None, kv_caps=None, stream=None, weights=None):
        """End to end with host (numpy / pinned torch CPU) buffers: H2D, solve, backtrack, D2H.
        Returns (objective, boundaries, status, bytes_h2d, bytes_d2h) as host arrays."""
        def host(a, dt):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                return a if a.dtype == dt else a.to(dt)
            return torch.from_numpy(np.ascontiguousarray(a)).to(dt)
        Lh = host(lengths, _TORCH_DT[self.dtype])
        if Lh.dim() == 1:
            Lh = Lh[None, :]
        Dh = host(degrees, torch.int32)
        Ch = host(caps, torch.int32)
        Kh = host(kv_caps, torch.int64)
        Wh = host(weights, torch.int32)
        B, n = Lh.shape
        m = Dh.shape[-1]
        L, ls = _rows(Lh, B, n, "lengths")
        D, ds = _rows(Dh, B, m, "degrees")
        Cp, cs = _rows(Ch, B, m, "caps")
        K, ks = _rows(Kh, B, m, "kv_caps")
        Wt, wts = _rows(Wh, B, n, "weights")
        p = C.Problem(n, m, B, L.data_ptr(), ls, D.data_ptr(), ds, Cp.data_ptr() if Cp is not None else None, cs,
                      K.data_ptr() if K is not None else None, ks, Wt.data_ptr() if Wt is not None else None, wts)
        obj = torch.empty(B, dtype=self.objective_dtype).pin_memory()
        bnd = torch.empty((B, m + 1), dtype=torch.int32).pin_memory()
        st = torch.empty(B, dtype=torch.int32).pin_memory()
        h2d, d2h = ctypes.c_int64(0), ctypes.c_int64(0)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        C.check(C.lib().heddle_place_solve_host(self._h, ctypes.byref(p), _ptr(obj), _ptr(bnd), _ptr(st),
                                                ctypes.c_void_p(s), ctypes.byref(h2d), ctypes.byref(d2h)),
                "heddle_place_solve_host")
        return obj, bnd, st, h2d.value, d2h.value

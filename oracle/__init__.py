"""TEST INFRASTRUCTURE -- the CPU FP64 oracle for Heddle's presorted DP.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2603_28101_b200) never imports it and shares no code with it.

A thin ctypes wrapper around oracle/heddle_oracle.c (plain C, FP64, see that
file's header for the paper citations and the readings R1..R8).
Parity status per function:
  solve                 -- pinned: SPEC worked examples, brute force (P1, P2),
                           closed forms (P4), parametric search (P6), invariants (P7)
  brute_contiguous      -- pinned: closed forms, SPEC worked examples
  canonical_parents_bf  -- pinned: hand-derived counterexample parents (P5)
  brute_setpartition    -- pinned: closed forms (equal lengths), Lemma 1 agreement
  parametric_opt        -- pinned: brute force (P1)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "heddle_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

F64, F32EMU, U32, F32X = 0, 1, 2, 3
MINMAX, MINPLUS = 0, 1
OK, INVALID, INFEASIBLE, TOO_LARGE = 0, 1, 3, 9
MODE_OF = {"f64": F64, "f32": F32EMU, "u32": U32, "f32x": F32X}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
                               "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("semiring", ctypes.c_int32),
                ("L", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("num_degrees", ctypes.c_int32),
                ("T", ctypes.c_void_p), ("F", ctypes.c_void_p),
                ("s_max", ctypes.c_int32),
                ("layer_deg", ctypes.c_void_p),
                ("caps", ctypes.c_void_p), ("kvcaps", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER(_Problem)
        vp = ctypes.c_void_p
        _lib.ora_solve.argtypes = [P, vp, vp, vp, vp]
        _lib.ora_solve_threads.argtypes = [P, vp, vp, vp, vp, ctypes.c_int32]
        _lib.ora_group_cost.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        _lib.ora_group_cost.restype = ctypes.c_double
        _lib.ora_brute_contiguous.argtypes = [P, vp, vp, vp]
        _lib.ora_canonical_parents_bf.argtypes = [P, vp, vp]
        _lib.ora_brute_setpartition.argtypes = [P, vp]
        _lib.ora_parametric_opt.argtypes = [P, vp]
        _lib.ora_feasible.argtypes = [P, ctypes.c_double]
        _lib.ora_solve_batch.argtypes = [P, ctypes.c_int32, vp, vp, vp, vp, ctypes.c_int32]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Problem:
    """One placement problem in oracle form.  `layer_rows` indexes profile rows
    (worker j uses profile row layer_rows[j-1]).  Arrays are kept alive here."""

    def __init__(self, L, T, F, layer_rows, mode="f64", semiring=MINMAX,
                 caps=None, kvcaps=None, w=None):
        self.L = np.ascontiguousarray(np.asarray(L, dtype=np.float64).reshape(-1))
        self.T = np.ascontiguousarray(np.asarray(T, dtype=np.float64).reshape(-1))
        F = np.asarray(F, dtype=np.float64)
        if F.ndim == 1:
            F = F[None, :]
        self.F = np.ascontiguousarray(F)
        self.rows = np.ascontiguousarray(np.asarray(layer_rows, dtype=np.int32).reshape(-1))
        self.caps = None if caps is None else np.ascontiguousarray(np.asarray(caps, dtype=np.int64).reshape(-1))
        self.kvcaps = None if kvcaps is None else np.ascontiguousarray(np.asarray(kvcaps, dtype=np.float64).reshape(-1))
        self.w = None if w is None else np.ascontiguousarray(np.asarray(w, dtype=np.int32).reshape(-1))
        self.n, self.m = self.L.size, self.rows.size
        self.mode = MODE_OF.get(mode, mode)
        self.semiring = semiring
        self.s = _Problem(self.n, self.m, self.mode, semiring, _ptr(self.L).value, _ptr(self.w) and _ptr(self.w).value,
                          self.T.size, _ptr(self.T).value, _ptr(self.F).value, self.F.shape[1],
                          _ptr(self.rows).value, _ptr(self.caps) and _ptr(self.caps).value,
                          _ptr(self.kvcaps) and _ptr(self.kvcaps).value)

    @classmethod
    def from_batch(cls, batch, b=0, mode=None, semiring=MINMAX):
        prof = batch.profile
        mode = mode or prof.dtype
        caps = None if batch.caps is None else batch.caps[b]
        kv = None if batch.kv_caps is None else batch.kv_caps[b]
        w = None if batch.weights is None else batch.weights[b]
        return cls(batch.lengths[b], prof.T, prof.F, prof.row_of(batch.degrees[b]), mode=mode,
                   semiring=semiring, caps=caps, kvcaps=kv, w=w)


def solve(p: Problem, want_tables=False, threads=1):
    """The DP (ora_solve).  threads > 1 shares each layer's columns over OpenMP threads
    (ora_solve_threads); the result is identical."""
    n, m = p.n, p.m
    dp = np.empty((m + 1, n + 1), dtype=np.float64) if want_tables else None
    par = np.empty((m + 1, n + 1), dtype=np.int32) if want_tables else None
    b = np.empty(m + 1, dtype=np.int32)
    opt = np.zeros(1, dtype=np.float64)
    if threads == 1:
        st = lib().ora_solve(ctypes.byref(p.s), _ptr(dp), _ptr(par), _ptr(b), _ptr(opt))
    else:
        st = lib().ora_solve_threads(ctypes.byref(p.s), _ptr(dp), _ptr(par), _ptr(b), _ptr(opt), threads)
    return dict(status=st, opt=float(opt[0]), bounds=b, dp=dp, parent=par)


def group_cost(p: Problem, j: int, k: int, i: int) -> float:
    """Cost of items [k, i) as group j (1-based), Eq. 2 group term."""
    return lib().ora_group_cost(ctypes.byref(p.s), j, k, i)


def brute_contiguous(p: Problem):
    b = np.empty(p.m + 1, dtype=np.int32)
    opt = np.zeros(1)
    cnt = np.zeros(1, dtype=np.int64)
    st = lib().ora_brute_contiguous(ctypes.byref(p.s), _ptr(opt), _ptr(b), _ptr(cnt))
    return dict(status=st, opt=float(opt[0]), bounds_lexfirst=b, n_optimal=int(cnt[0]))


def canonical_parents_bf(p: Problem):
    o = np.empty((p.m + 1, p.n + 1))
    par = np.empty((p.m + 1, p.n + 1), dtype=np.int32)
    st = lib().ora_canonical_parents_bf(ctypes.byref(p.s), _ptr(o), _ptr(par))
    return dict(status=st, opt=o, parent=par)


def brute_setpartition(p: Problem):
    opt = np.zeros(1)
    st = lib().ora_brute_setpartition(ctypes.byref(p.s), _ptr(opt))
    return dict(status=st, opt=float(opt[0]))


def parametric_opt(p: Problem):
    opt = np.zeros(1)
    st = lib().ora_parametric_opt(ctypes.byref(p.s), _ptr(opt))
    return dict(status=st, opt=float(opt[0]))


def solve_batch(lengths, T, F, layer_rows, mode="f64", semiring=MINMAX, threads=0):
    """B problems with shared n, m, profile (no caps/weights); OpenMP over problems.
    Returns (opt[B], bounds[B, m+1], threads_used)."""
    lengths = np.ascontiguousarray(np.asarray(lengths, dtype=np.float64))
    rows = np.ascontiguousarray(np.asarray(layer_rows, dtype=np.int32))
    B, n = lengths.shape
    m = rows.shape[1]
    proto = Problem(lengths[0], T, F, rows[0], mode=mode, semiring=semiring)
    opt = np.empty(B)
    bounds = np.empty((B, m + 1), dtype=np.int32)
    used = lib().ora_solve_batch(ctypes.byref(proto.s), B, _ptr(lengths), _ptr(rows), _ptr(opt),
                                 _ptr(bounds), threads)
    return opt, bounds, used

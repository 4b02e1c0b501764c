"""CPU-side checks of the C-ABI library: it loads, exports every symbol the header
declares, its host-only entry points behave, and no call aborts without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "heddle_place.h")


@pytest.fixture(scope="module")
def C():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_28101_b200 import _lib
    return _lib


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(heddle_place_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(C):
    syms = declared_symbols()
    assert "heddle_place_init" in syms and "heddle_place_solve" in syms and "heddle_place_backtrack" in syms
    lib = C.lib()
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/heddle_place.h but not exported"
    assert set(C.SYMBOLS) == set(syms)


def test_exports_are_c_abi(C):
    out = os.popen(f"nm -D --defined-only {C.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), f"{s} not an unmangled text symbol"


def test_transitions_formula_matches_loop_count(C):
    """W(n, m) == the number of (state, split) pairs on the computed region
    i in [j, n-m+j], k in [j-1, i-1] (layer m: only i = n)."""
    def count(n, m):
        if n < m:
            return 0
        w = 0
        for j in range(1, m + 1):
            lo, hi = (n, n) if j == m else (j, n - m + j)
            for i in range(lo, hi + 1):
                w += (i - j + 1) if j > 1 else 1
        return w
    for n, m in [(16, 4), (512, 32), (10, 2), (10, 10), (7, 1), (64, 63), (100, 2), (3, 5)]:
        assert C.transitions(n, m) == count(n, m), (n, m)
    assert C.transitions(1024, 32) == 14807616
    assert C.transitions(65536, 256) == 2 * 65281 + 254 * 65281 * 65282 // 2


def test_strerror(C):
    for s in range(10):
        assert isinstance(C.strerror(s), str) and C.strerror(s)
    assert C.strerror(C.E_UNSORTED).startswith("lengths")


def test_init_without_gpu_returns_status(C):
    """No GPU here: init must return a status (never abort) -- E_CUDA -- and argument
    errors must be reported before touching the device."""
    lib = C.lib()
    deg = np.array([1, 2], dtype=np.int32)
    T = np.array([1.0, 0.5], dtype=np.float32)
    F = np.ones((2, 4), dtype=np.float32)
    cfg = C.Config(0, C.F32, C.MINMAX, 16, 4, 1, 2, deg.ctypes.data, T.ctypes.data, F.ctypes.data, 4, 0)
    h = ctypes.c_void_p()
    st = lib.heddle_place_init(ctypes.byref(cfg), ctypes.byref(h))
    assert st in (C.E_CUDA, C.OK)
    if st == C.OK:
        lib.heddle_place_destroy(h)
    assert h.value is None or st == C.OK
    bad = C.Config(0, C.F32, C.MINMAX, 0, 4, 1, 2, deg.ctypes.data, T.ctypes.data, F.ctypes.data, 4, 0)
    assert lib.heddle_place_init(ctypes.byref(bad), ctypes.byref(h)) == C.E_INVALID
    Fdec = F.copy()
    Fdec[0, 2] = 0.5   # F decreasing: violates the monotone premise
    cfg2 = C.Config(0, C.F32, C.MINMAX, 16, 4, 1, 2, deg.ctypes.data, T.ctypes.data, Fdec.ctypes.data, 4, 0)
    assert lib.heddle_place_init(ctypes.byref(cfg2), ctypes.byref(h)) == C.E_RANGE
    Ti = np.array([70000, 1], dtype=np.uint32)
    Fi = np.full((2, 4), 70000, dtype=np.uint32)   # T*F >= 2^32 - 65536: U32 range guard
    cfg3 = C.Config(0, C.U32, C.MINMAX, 16, 4, 1, 2, deg.ctypes.data, Ti.ctypes.data, Fi.ctypes.data, 4, 0)
    assert lib.heddle_place_init(ctypes.byref(cfg3), ctypes.byref(h)) == C.E_RANGE
    assert lib.heddle_place_solve(None, None, None, None, None) == C.E_INVALID
    assert lib.heddle_place_backtrack(None, None, None, None) == C.E_INVALID
    lib.heddle_place_destroy(None)
    assert lib.heddle_place_launch_count(None) == -1


def test_product_path_has_no_oracle_import():
    """The product package must never import or link oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2603_28101_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "heddle_oracle" not in src and "liboracle" not in src, f


def test_split_block_ownership(C):
    """Zigzag ownership: every column block owned by exactly one rank, and the triangular
    work (block b costs ~ b + 1/2 column-blocks of splits) is balanced across ranks."""
    for ncb in (1, 3, 16, 128, 129, 255):
        for world in (1, 2, 3, 4, 8):
            owned = [C.split_blocks(ncb, world, r) for r in range(world)]
            allb = sorted(b for o in owned for b in o)
            assert allb == list(range(ncb)), (ncb, world)
            if ncb % (2 * world) == 0:
                work = [sum(b + 0.5 for b in o) for o in owned]
                assert max(work) == min(work), (ncb, world, work)
    with pytest.raises(ValueError):
        C.split_blocks(4, 2, 2)

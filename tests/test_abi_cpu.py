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


def test_round2_entry_points_reject_bad_arguments_without_a_gpu(C):
    """The round-2 entry points validate their host-side arguments before touching the device:
    null pointers / sizes / contexts give HEDDLE_E_INVALID (1) and never abort."""
    L = C.lib()
    vp = ctypes.c_void_p
    E_INVALID = 1
    # state query without a context or with a negative count
    assert L.heddle_place_query(None, 1, None, None, None, None, None, None) == E_INVALID
    # aggregation: null buffers, bad sizes / bucket, NaN threshold, unknown dtype
    buf = (ctypes.c_int32 * 64)()
    p = ctypes.cast(buf, vp)
    assert L.heddle_place_aggregate(1, None, 0, 8, 1, 1.0, 2, p, p, p, p, None) == E_INVALID
    assert L.heddle_place_aggregate(1, p, 0, 0, 1, 1.0, 2, p, p, p, p, None) == E_INVALID
    assert L.heddle_place_aggregate(1, p, 0, 8, 1, 1.0, 0, p, p, p, p, None) == E_INVALID
    assert L.heddle_place_aggregate(1, p, 0, 8, 1, float("nan"), 2, p, p, p, p, None) == E_INVALID
    assert L.heddle_place_aggregate(7, p, 0, 8, 1, 1.0, 2, p, p, p, p, None) == E_INVALID
    assert L.heddle_place_aggregate(1, p, -1, 8, 1, 1.0, 2, p, p, p, p, None) == E_INVALID
    # expansion: null buffers, m < 1
    assert L.heddle_place_expand(None, 2, 1, p, 8, p, None) == E_INVALID
    assert L.heddle_place_expand(p, 0, 1, p, 8, p, None) == E_INVALID
    # annealer: null context / arguments
    args, out = C.AnnealArgs(), C.AnnealOut()
    assert L.heddle_place_anneal(None, ctypes.byref(args), ctypes.byref(out), None) == E_INVALID
    # split plan: bad arguments
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    assert L.heddle_place_split_plan(8, 16, 2, 0, ctypes.byref(a), ctypes.byref(b)) == -1   # n < m
    assert L.heddle_place_split_plan(16, 8, 2, 2, ctypes.byref(a), ctypes.byref(b)) == -1   # rank >= world
    assert L.heddle_place_split_plan(16, 8, 2, 0, None, ctypes.byref(b)) == -1


def test_problem_struct_layout_matches_header(C):
    """The ctypes mirrors of the ABI structs carry every field the header declares, in order."""
    src = open(HEADER).read()
    def fields_of(body):
        out = []
        for names in re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\*?\s+\*?\s*([A-Za-z_]+(?:\s*,\s*[A-Za-z_]+)*);",
                                body, re.M):
            out += [x.strip() for x in names.split(",")]
        return out
    body = src[src.index("typedef struct {\n  int32_t n;                    /* trajectories per problem"):]
    body = body[:body.index("} heddle_place_problem;")]
    fields = fields_of(body)
    assert [f[0] for f in C.Problem._fields_] == fields, (fields, C.Problem._fields_)
    body = src[src.index("} heddle_place_anneal_args;") - 1600:src.index("} heddle_place_anneal_args;")]
    body = body[body.index("typedef struct {"):]
    fields = fields_of(body)
    assert [f[0] for f in C.AnnealArgs._fields_] == fields, (fields, C.AnnealArgs._fields_)
    body = src[src.index("} heddle_place_anneal_out;") - 1200:src.index("} heddle_place_anneal_out;")]
    body = body[body.index("typedef struct {"):]
    assert [f[0] for f in C.AnnealOut._fields_] == fields_of(body)

"""ctypes binding of include/heddle_place.h -- argument marshalling only.

Every step of the placement DP runs in the CUDA kernels of libheddle_place.so;
this module only turns torch tensors into device pointers and streams.  There
is no CPU fallback: importing it without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEDDLE_PLACE_LIB") or os.path.join(_HERE, "libheddle_place.so")

OK, E_INVALID, E_UNSORTED, E_INFEASIBLE, E_RANGE, E_UNKNOWN_DEGREE, E_STATE, E_CUDA, E_NCCL, E_NOMEM = range(10)
U32, F32, F64, F32X = 0, 1, 2, 3
MINMAX, MINPLUS = 0, 1
KEEP_PARENTS = 0x1
FORCE_BATCHED = 0x2
FORCE_LAYERED = 0x4
VALLEY = 0x8
KERNELS = {"auto": 0, "batched": FORCE_BATCHED, "layered": FORCE_LAYERED}
ALGOS = {"scan": 0, "valley": VALLEY}   # full scan of the splits (Eq. 3) / valley search (min-max, N3)

DTYPES = {"u32": U32, "f32": F32, "f64": F64, "f32x": F32X}   # f32x: F32 costs, FP64 min-plus sums
SEMIRINGS = {"minmax": MINMAX, "minplus": MINPLUS}

# exported symbols declared in include/heddle_place.h (tests check the .so exports all of them)
SYMBOLS = ("heddle_place_init", "heddle_place_solve", "heddle_place_backtrack", "heddle_place_query",
           "heddle_place_solve_host",
           "heddle_place_launch_count", "heddle_place_transitions", "heddle_place_destroy",
           "heddle_place_strerror", "heddle_place_nccl_unique_id", "heddle_place_init_split",
           "heddle_place_split_blocks", "heddle_place_split_plan", "heddle_place_debug_violations", "heddle_place_retarget",
           "heddle_place_objective", "heddle_place_anneal", "heddle_place_aggregate", "heddle_place_expand")


class Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("dtype", ctypes.c_int32), ("semiring", ctypes.c_int32),
                ("max_n", ctypes.c_int32), ("max_m", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("num_degrees", ctypes.c_int32), ("degrees", ctypes.c_void_p),
                ("T", ctypes.c_void_p), ("F", ctypes.c_void_p), ("s_max", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("B", ctypes.c_int32),
                ("lengths", ctypes.c_void_p), ("lengths_stride", ctypes.c_int64),
                ("degrees", ctypes.c_void_p), ("degrees_stride", ctypes.c_int64),
                ("caps", ctypes.c_void_p), ("caps_stride", ctypes.c_int64),
                ("kv_caps", ctypes.c_void_p), ("kv_caps_stride", ctypes.c_int64),
                ("weights", ctypes.c_void_p), ("weights_stride", ctypes.c_int64),
                ("ms", ctypes.c_void_p), ("ns", ctypes.c_void_p)]


class AnnealArgs(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("lengths", ctypes.c_void_p), ("chains", ctypes.c_int32),
                ("m_min", ctypes.c_int32), ("m_max", ctypes.c_int32), ("init_degrees", ctypes.c_void_p),
                ("init_m", ctypes.c_void_p), ("uniforms", ctypes.c_void_p), ("iters", ctypes.c_int32),
                ("cooling", ctypes.c_double), ("eps_frac", ctypes.c_double), ("objective_only", ctypes.c_int32)]


class AnnealOut(ctypes.Structure):
    _fields_ = [("best_makespan", ctypes.c_void_p), ("best_degrees", ctypes.c_void_p), ("best_m", ctypes.c_void_p),
                ("trace", ctypes.c_void_p), ("accepted", ctypes.c_void_p), ("iterations", ctypes.c_void_p)]


class HeddleError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} ({status})")


_lib = None


def lib() -> ctypes.CDLL:
    """Load libheddle_place.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.heddle_place_init.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(vp)]
        L.heddle_place_init.restype = ctypes.c_int
        L.heddle_place_solve.argtypes = [vp, ctypes.POINTER(Problem), vp, vp, vp]
        L.heddle_place_solve.restype = ctypes.c_int
        L.heddle_place_backtrack.argtypes = [vp, vp, vp, vp]
        L.heddle_place_backtrack.restype = ctypes.c_int
        L.heddle_place_query.argtypes = [vp, ctypes.c_int32, vp, vp, vp, vp, vp, vp]
        L.heddle_place_anneal.argtypes = [vp, ctypes.POINTER(AnnealArgs), ctypes.POINTER(AnnealOut), vp]
        L.heddle_place_anneal.restype = ctypes.c_int
        L.heddle_place_aggregate.argtypes = [ctypes.c_int32, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_double, ctypes.c_int32, vp, vp, vp, vp, vp]
        L.heddle_place_aggregate.restype = ctypes.c_int
        L.heddle_place_expand.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, ctypes.c_int32, vp, vp]
        L.heddle_place_expand.restype = ctypes.c_int
        L.heddle_place_query.restype = ctypes.c_int
        L.heddle_place_solve_host.argtypes = [vp, ctypes.POINTER(Problem), vp, vp, vp, vp,
                                              ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.heddle_place_solve_host.restype = ctypes.c_int
        L.heddle_place_launch_count.argtypes = [vp]
        L.heddle_place_launch_count.restype = ctypes.c_int64
        L.heddle_place_transitions.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.heddle_place_transitions.restype = ctypes.c_int64
        L.heddle_place_destroy.argtypes = [vp]
        L.heddle_place_destroy.restype = None
        L.heddle_place_nccl_unique_id.argtypes = [vp, ctypes.c_int32]
        L.heddle_place_nccl_unique_id.restype = ctypes.c_int
        L.heddle_place_init_split.argtypes = [ctypes.POINTER(Config), vp, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.POINTER(vp)]
        L.heddle_place_init_split.restype = ctypes.c_int
        L.heddle_place_split_blocks.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, ctypes.c_int32]
        L.heddle_place_split_plan.argtypes = [ctypes.c_int32] * 4 + [vp, vp]
        L.heddle_place_split_plan.restype = ctypes.c_int32
        L.heddle_place_split_blocks.restype = ctypes.c_int32
        L.heddle_place_objective.argtypes = [vp, ctypes.POINTER(Problem), vp, vp, vp]
        L.heddle_place_objective.restype = ctypes.c_int
        L.heddle_place_retarget.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, ctypes.c_int32, vp, vp]
        L.heddle_place_retarget.restype = ctypes.c_int
        L.heddle_place_debug_violations.argtypes = []
        L.heddle_place_debug_violations.restype = ctypes.c_int64
        L.heddle_place_strerror.argtypes = [ctypes.c_int]
        L.heddle_place_strerror.restype = ctypes.c_char_p
        _lib = L
    return _lib


def strerror(status: int) -> str:
    return lib().heddle_place_strerror(status).decode()


def transitions(n: int, m: int) -> int:
    """W(n, m): algorithmic transitions of one problem (the DP-cell unit of the metric)."""
    return int(lib().heddle_place_transitions(n, m))


def check(status: int, what: str):
    if status != OK:
        raise HeddleError(status, what)


def split_blocks(ncb: int, world: int, rank: int) -> list[int]:
    """Column blocks (512 columns each) that `rank` computes in split mode (zigzag ownership)."""
    cnt = lib().heddle_place_split_blocks(ncb, world, rank, None, 0)
    if cnt < 0:
        raise ValueError("bad split arguments")
    buf = (ctypes.c_int32 * max(cnt, 1))()
    lib().heddle_place_split_blocks(ncb, world, rank, buf, cnt)
    return list(buf[:cnt])


def split_plan(n: int, m: int, world: int, rank: int) -> tuple[int, int]:
    """(pieces this rank publishes to each peer, pieces it receives) per problem in split mode."""
    pub, arr = ctypes.c_int64(0), ctypes.c_int64(0)
    if lib().heddle_place_split_plan(n, m, world, rank, ctypes.byref(pub), ctypes.byref(arr)) != 0:
        raise ValueError("heddle_place_split_plan: bad arguments")
    return pub.value, arr.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().heddle_place_nccl_unique_id(buf, 128), "heddle_place_nccl_unique_id")
    return buf.raw

"""B200-native presorted-DP trajectory placement (Heddle, arxiv 2603.28101, §5.2).

Product path: include/heddle_place.h (C ABI) -> libheddle_place.so (sm_100a CUDA
kernels, csrc/) -> this thin binding.  No CPU fallback: the binding raises when
the library is missing.
"""
from ._lib import (E_CUDA, E_INFEASIBLE, E_INVALID, E_NCCL, E_NOMEM, E_RANGE, E_STATE, E_UNKNOWN_DEGREE,
                   E_UNSORTED, F32, F64, KEEP_PARENTS, MINMAX, MINPLUS, OK, U32, HeddleError, strerror,
                   transitions)

__all__ = ["Placer", "transitions", "strerror", "HeddleError", "OK", "E_INVALID", "E_UNSORTED", "E_INFEASIBLE",
           "E_RANGE", "E_UNKNOWN_DEGREE", "E_STATE", "E_CUDA", "E_NCCL", "E_NOMEM", "U32", "F32", "F64",
           "MINMAX", "MINPLUS", "KEEP_PARENTS"]


def __getattr__(name):
    if name == "Placer":  # torch-facing wrapper, imported lazily (torch import is slow)
        from .placer import Placer
        return Placer
    raise AttributeError(name)

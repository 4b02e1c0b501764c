"""Short-trajectory aggregation (§5.2) -- the paper's own
speed heuristic, on the device (kernel K10, heddle_place_aggregate / heddle_place_expand).

After the presort, trajectories shorter than a threshold are bucketed (at most `bucket` per item);
each bucket is ONE DP item whose length is the bucket's maximum (its first element, the rows being
sorted) and whose weight is its cardinality, so the group size seen by F is the sum of weights
(R5).  The aggregated batch is ragged (n' differs per problem): solve it with
`Placer.solve(agg, degrees, weights=w, ns=n_agg)`, then `expand` maps the boundaries back.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib as C

_DT = {torch.float32: C.F32, torch.float64: C.F64, torch.uint32: C.U32}


def aggregate(lengths: torch.Tensor, threshold: float, bucket: int, stream=None):
    """lengths: device [B, n] (or [n]) rows non-increasing.  Returns device tensors
    (agg_lengths [B, n], weights [B, n] int32, starts [B, n+1] int32, n_agg [B] int32); rows are
    valid up to n_agg[b]."""
    L = lengths if lengths.dim() == 2 else lengths[None, :]
    if L.stride(-1) != 1:
        L = L.contiguous()
    B, n = L.shape
    agg = torch.empty((B, n), dtype=L.dtype, device=L.device)
    w = torch.empty((B, n), dtype=torch.int32, device=L.device)
    starts = torch.empty((B, n + 1), dtype=torch.int32, device=L.device)
    nagg = torch.empty(B, dtype=torch.int32, device=L.device)
    s = (stream or torch.cuda.current_stream(L.device)).cuda_stream
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    C.check(C.lib().heddle_place_aggregate(_DT[L.dtype], p(L), L.stride(0) if B > 1 else 0, n, B, float(threshold),
                                           int(bucket), p(agg), p(w), p(starts), p(nagg), ctypes.c_void_p(s)),
            "heddle_place_aggregate")
    return agg, w, starts, nagg


def expand(agg_boundaries: torch.Tensor, starts: torch.Tensor, stream=None) -> torch.Tensor:
    """Boundaries [B, m+1] of the aggregated solve -> trajectory boundaries [B, m+1] (-1 kept)."""
    bd = agg_boundaries.to(torch.int32).contiguous()
    st = starts.to(torch.int32).contiguous()
    B, m1 = bd.shape
    out = torch.empty_like(bd)
    s = (stream or torch.cuda.current_stream(bd.device)).cuda_stream
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    C.check(C.lib().heddle_place_expand(p(bd), m1 - 1, B, p(st), st.shape[1] - 1, p(out), ctypes.c_void_p(s)),
            "heddle_place_expand")
    return out

"""Trajectory migration (§5.3): retarget on the GPU, transmission scheduling
on the host.

* `retarget` -- batched rank -> worker lookup with capacities ceil(s_i n*/n),
  one CUDA thread per query (heddle_place_retarget).
* `schedule_transfers` -- the trajectory-aware transmission scheduler: take
  pending KV-migration requests longest trajectory first, skip any that shares a source or
  destination worker with a selected or running transfer; returns one conflict-free batch.
  It is an O(R log R) greedy over a handful of requests per epoch, i.e. control-plane host logic.
"""
from __future__ import annotations

import ctypes
import dataclasses

import torch

from . import _lib as C


def retarget(boundaries: torch.Tensor, n_active: torch.Tensor, query_problem: torch.Tensor,
             query_rank: torch.Tensor, stream=None) -> torch.Tensor:
    """boundaries [B, m+1] int32 (device), n_active [B], query_problem / query_rank [Q] (0-based rank
    among active trajectories, longest first) -> worker [Q] int32 (-1 for invalid queries)."""
    bd = boundaries.to(torch.int32).contiguous()
    B, m1 = bd.shape
    na = n_active.to(device=bd.device, dtype=torch.int32).contiguous()
    qp = query_problem.to(device=bd.device, dtype=torch.int32).contiguous()
    qr = query_rank.to(device=bd.device, dtype=torch.int32).contiguous()
    out = torch.empty(qp.shape[0], dtype=torch.int32, device=bd.device)
    s = (stream or torch.cuda.current_stream(bd.device)).cuda_stream
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    C.check(C.lib().heddle_place_retarget(p(bd), m1 - 1, B, p(na), p(qp), p(qr), qp.shape[0], p(out),
                                          ctypes.c_void_p(s)), "heddle_place_retarget")
    return out


@dataclasses.dataclass(frozen=True)
class MigrationRequest:
    trajectory_id: int
    src: int
    dst: int
    priority_len: float     # predicted total tokens of the trajectory
    issued_at: float = 0.0


def schedule_transfers(pending, busy_endpoints=()):
    """One conflict-free batch: longest trajectory first (ties: earliest issued, then id); a request
    is taken iff neither endpoint is busy or already claimed in this batch."""
    claimed = set(busy_endpoints)
    batch = []
    for r in sorted(pending, key=lambda r: (-r.priority_len, r.issued_at, r.trajectory_id)):
        if r.src == r.dst or r.src in claimed or r.dst in claimed:
            continue
        batch.append(r)
        claimed.update((r.src, r.dst))
    return batch

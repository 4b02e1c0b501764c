"""Multi-GPU drivers (one process per GPU, torch.distributed for the plumbing).

* Independent problems -- batched sweeps, TP/config sweeps, SA candidate batches
  (SURVEY §8e): the B problems are block-sharded across ranks; each rank solves and
  backtracks its shard on its own GPU with no collective on the data path.  The
  optional result gather at the end is one all_gather per output.
* Split mode (one large instance): see `split_placer` -- the columns of every DP
  layer are dealt to the ranks in zigzag 512-column blocks.  Inside libheddle_place.so
  the tile that finishes a block stores it into every peer's dp row over NVLink peer
  memory (CUDA IPC) and bumps the peers' arrival counters (fused exchange);
  HEDDLE_PLACE_EXCHANGE=nccl selects one NCCL all-gather of the row per layer instead.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block partition of B problems: rank r gets [r*B//P, (r+1)*B//P)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * B // world, (rank + 1) * B // world


def gather_shards(local: torch.Tensor, B: int, group=None) -> torch.Tensor:
    """All-gather per-rank shards (first dim = the rank's problems) back into [B, ...]
    in problem order.  Shards may differ in size by one (block partition)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(B, world, r)[1] - shard_range(B, world, r)[0] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(out, sizes)], dim=0)


def solve_sharded(placer, lengths, degrees, caps=None, kv_caps=None, gather=True, group=None):
    """Solve the rank's shard of a [B, n] batch and (optionally) gather objective,
    boundaries and status of all B problems on every rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = lengths.shape[0]
    lo, hi = shard_range(B, world, rank)

    def sl(t):
        return None if t is None else (t[lo:hi] if t.dim() == 2 and t.shape[0] == B else t)
    obj, st = placer.solve(lengths[lo:hi], sl(degrees), caps=sl(caps), kv_caps=sl(kv_caps))
    bnd = placer.backtrack()
    if not gather or world == 1:
        return obj, bnd, st
    return gather_shards(obj, B, group), gather_shards(bnd, B, group), gather_shards(st, B, group)


def split_placer(profile, *, max_n, max_m, max_batch=1, group=None, **kw):
    """Create a split-mode Placer on this rank's GPU: rank 0 draws the NCCL unique id and
    broadcasts it over the torch.distributed group; every rank then joins the library's
    NCCL communicator.  Solves on the returned placer are collective."""
    from . import _lib as C
    from .placer import Placer
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [C.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Placer.from_profile(profile, max_n=max_n, max_m=max_m, max_batch=max_batch,
                               split=(obj[0], rank, world), **kw)

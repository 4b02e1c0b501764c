"""Host logic of the multi-GPU path on CPU: world_size-2 gloo process groups.

The CUDA solve itself needs a GPU; here the sharding and result gathering are
exercised with per-rank stand-in results (problem ids), and must reassemble the
batch in problem order exactly once.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28101_b200.dist import gather_shards, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partition():
    for B in (1, 2, 7, 16384, 16385):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(B, world, r)
                assert 0 <= lo <= hi <= B
                assert hi - lo in (B // world, B // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(B))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(B, world, rank)
    ids = torch.arange(lo, hi, dtype=torch.int64)
    obj = ids.to(torch.float32) * 0.5                    # stand-in objective of each problem
    bnd = torch.stack([ids * 10 + j for j in range(5)], dim=1).to(torch.int32)
    st = (ids % 3).to(torch.int32)
    g_obj = gather_shards(obj, B)
    g_bnd = gather_shards(bnd, B)
    g_st = gather_shards(st, B)
    allids = torch.arange(B, dtype=torch.int64)
    ok = (torch.equal(g_obj, allids.to(torch.float32) * 0.5)
          and torch.equal(g_bnd, torch.stack([allids * 10 + j for j in range(5)], dim=1).to(torch.int32))
          and torch.equal(g_st, (allids % 3).to(torch.int32)))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 64, 1025])
def test_gather_shards_gloo_world2(B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res


# ------------------------------------------------------------------ split mode host logic (world 2, 3)
def _split_worker(rank, world, port, q):
    """One rank of the split-mode control plane: the unique-id broadcast of dist.split_placer, the
    zigzag column ownership (heddle_place_split_blocks) and the fused exchange's per-rank publish /
    arrival counts (heddle_place_split_plan), checked across ranks over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_28101_b200 import _lib as C
    ok = True
    obj = [C.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, obj[0])
    ok &= len(obj[0]) == 128 and all(i == ids[0] for i in ids)
    for n, m in ((65536, 256), (8192, 12), (4096, 64), (2100, 7), (600, 300)):
        ncb = (n - m + 3) // 512 + 1
        mine = C.split_blocks(ncb, world, rank)
        owners = [None] * world
        dist.all_gather_object(owners, mine)
        allb = sorted(b for o in owners for b in o)
        ok &= allb == list(range(ncb))                     # every block owned exactly once
        # zigzag balance: the triangular work (splits below each column, summed) per rank
        work = sum(sum(min(c, n) for c in range(512 * b, 512 * b + 512)) for b in mine)
        works = [None] * world
        dist.all_gather_object(works, work)
        if ncb >= 4 * world:
            ok &= max(works) / (sum(works) / world) < 1.0 + 2.0 * world / ncb
        pub, arr = C.split_plan(n, m, world, rank)
        plans = [None] * world
        dist.all_gather_object(plans, (pub, arr))
        total = sum(p for p, _ in plans)
        ok &= arr == total - pub                          # every peer's publications arrive here
        ok &= sum(a for _, a in plans) == (world - 1) * total
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_host_logic_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)], res

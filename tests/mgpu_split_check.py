"""torchrun helper (not collected by pytest): split-mode solve of configs[4] over all ranks,
compared bit for bit with a single-GPU solve on rank 0 and, at the configs[4] size, on every rank
with the oracle's stored solution (tests/golden/large_f32.npz: objective, boundaries and the
sampled states' dp values and lowest-index back-pointers).  Prints SPLIT OK on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    dist.barrier()
    from inputs import workloads as wl
    from paper_2603_28101_b200.dist import split_placer
    from paper_2603_28101_b200.placer import Placer
    n = int(os.environ.get("SPLIT_N", 65536))
    m = int(os.environ.get("SPLIT_M", 256))
    batch = wl.config_large(n=n, m=m)
    L = torch.from_numpy(batch.lengths).cuda()
    D = torch.from_numpy(batch.degrees).cuda()
    pl = split_placer(batch.profile, max_n=n, max_m=m)
    obj, st = pl.solve(L, D)
    bnd = pl.backtrack()
    torch.cuda.synchronize()
    res = torch.cat([obj.view(torch.int32).to(torch.int64), st.to(torch.int64), bnd.to(torch.int64).view(-1)])
    allres = [torch.empty_like(res) for _ in range(world)]
    dist.all_gather(allres, res)
    ok = all(torch.equal(a, res) for a in allres)
    gold = os.path.join(ROOT, "tests", "golden", "large_f32.npz")
    if n == 65536 and m == 256 and os.path.exists(gold):
        z = np.load(gold)
        qd = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()
        dp, par = pl.query(qd(np.zeros(z["qj"].size)), qd(z["qj"]), qd(z["qi"]))
        torch.cuda.synchronize()
        g_ok = (float(obj[0]) == float(z["opt"]) and np.array_equal(bnd.cpu().numpy()[0], z["bounds"])
                and np.array_equal(dp.cpu().numpy().astype(np.float64), z["dp"])
                and np.array_equal(par.cpu().numpy(), z["parent"]))
        print(f"rank {rank}: oracle golden (objective, boundaries, {z['qj'].size} sampled dp values and "
              f"back-pointers) identical={g_ok}", flush=True)
        flag = torch.tensor([0 if g_ok else 1], device="cuda")
        dist.all_reduce(flag)
        ok = ok and int(flag.item()) == 0
    if rank == 0:
        ref = Placer.from_profile(batch.profile, max_n=n, max_m=m, max_batch=1, kernel="layered")
        o1, s1 = ref.solve(L, D)
        b1 = ref.backtrack()
        torch.cuda.synchronize()
        ok = ok and torch.equal(o1, obj) and torch.equal(b1, bnd) and int(s1[0]) == 0
        print(f"objective {float(obj[0]):.6f} world {world} identical_across_ranks_and_1gpu={ok}")
        print("SPLIT OK" if ok else "SPLIT MISMATCH", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

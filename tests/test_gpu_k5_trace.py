"""K5 dataflow schedule, checked from its own per-tile timeline (HEDDLE_PLACE_TILE_TRACE).

The persistent kernel lets a tile of layer j start as soon as the row j-1 blocks covering its
split range are final.  From the recorded %globaltimer stamps this test checks that no tile read
row j-1 (stamp 2, "dependencies met") before every chunk of every block it depends on had finished
its sweep (stamp 4), that every block got all its chunks, and that the chunks of a block tile its
split range exactly.  The solve's result is compared with the batched kernel's.
"""
import os

import numpy as np
import pytest
import torch

from inputs import workloads as wl

pytestmark = pytest.mark.gpu


def _solve(batch, kernel, trace=None):
    from paper_2603_28101_b200.placer import Placer
    if trace:
        os.environ["HEDDLE_PLACE_TILE_TRACE"] = trace
    try:
        pl = Placer.from_profile(batch.profile, max_n=batch.n, max_m=batch.m, max_batch=batch.B, device=0,
                                 kernel=kernel)
        obj, st = pl.solve(torch.from_numpy(batch.lengths).cuda(), torch.from_numpy(batch.degrees).cuda())
        bnd = pl.backtrack()
        torch.cuda.synchronize()
    finally:
        os.environ.pop("HEDDLE_PLACE_TILE_TRACE", None)
    return obj.cpu(), st.cpu(), bnd.cpu()


@pytest.mark.parametrize("kd", [None, "128"])
def test_k5_schedule_respects_dependencies(tmp_path, kd):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench"))
    import tile_trace as tt
    batch = wl.config_tp_sweep()               # 4 problems, n=4096, m=64: 63 dependent layers
    if kd:
        os.environ["HEDDLE_PLACE_K5_KD"] = kd
    try:
        path = str(tmp_path / "k5.bin")
        o5, s5, b5 = _solve(batch, "layered", trace=path)
    finally:
        os.environ.pop("HEDDLE_PLACE_K5_KD", None)
    o2, s2, b2 = _solve(batch, "batched")
    assert torch.equal(o5, o2) and torch.equal(s5, s2) and torch.equal(b5, b2)

    rec = list(tt.records(path))[-1]
    B, n, m = rec["B"], batch.n, batch.m
    t = rec["t"]
    assert (t > 0).all(), "every tile stamped"
    assert (np.diff(t, axis=1) >= 0).all(), "stamps in phase order"
    ent = np.repeat(rec["tiles"], B, axis=0)
    prob = np.tile(np.arange(B), len(rec["tiles"]))
    j, blk, nch, k0, k1 = ent[:, 0], ent[:, 1] & 0xFFFF, ent[:, 1] >> 16, ent[:, 2], ent[:, 3]
    swept = {}
    chunks = {}
    for i in range(len(t)):
        key = (int(j[i]), int(prob[i]), int(blk[i]))
        swept[key] = max(swept.get(key, 0), int(t[i, 4]))
        chunks.setdefault(key, []).append((int(k0[i]), int(k1[i]), int(nch[i])))
    for (jj, b, bb), ch in chunks.items():
        ch.sort()
        assert len(ch) == ch[0][2], "a block gets exactly its chunk count"
        assert ch[0][0] == (jj - 1) & ~3, "chunks start at the layer's first split"
        assert all(ch[q][1] == ch[q + 1][0] for q in range(len(ch) - 1)), "chunks tile the split range"
    for i in range(len(t)):
        jj, b = int(j[i]), int(prob[i])
        if jj < 3:
            continue                                  # row 1 comes from the prologue
        pc = (jj - 1) & ~3
        lo, hi = max(int(k0[i]), jj - 1), min(int(k1[i]) - 1, n - m + jj - 1)
        for bb in range((lo - pc) // 512, (hi - pc) // 512 + 1):
            assert t[i, 2] >= swept[(jj - 1, b, bb)], (jj, b, bb)

"""N4: migration retarget and transmission scheduler.  CPU tests pin the
oracle to SPEC's worked examples and check the host scheduler against it; the GPU retarget kernel
is checked against the oracle on random plans."""
import numpy as np
import pytest

from oracle import migration as om
from paper_2603_28101_b200.migration import MigrationRequest, schedule_transfers


def test_retarget_spec_examples():
    # n=8, sizes [2, 6], n*=4 -> scaled [1, 3]; rank 0 (longest) -> worker 0, ranks 1..3 -> worker 1
    b = [0, 2, 8]
    assert [om.retarget_one(b, 4, r) for r in range(4)] == [0, 1, 1, 1]
    # n* = n and unchanged rank -> the original group
    for r in range(8):
        assert om.retarget_one(b, 8, r) == (0 if r < 2 else 1)
    # ceil overshoot clamps to the last worker; invalid rank -> -1
    assert om.retarget_one([0, 1, 2, 3], 2, 1) == 1          # caps ceil(2/3) = 1 each
    assert om.retarget_one(b, 4, 4) == -1


def test_schedule_spec_examples_and_agreement():
    A = (1, 1, 2, 100.0, 0.0)
    Bq = (2, 2, 3, 90.0, 0.0)
    Cq = (3, 4, 5, 80.0, 0.0)
    assert om.schedule([A, Bq, Cq]) == [1, 3]                       # batch {A, C}
    assert om.schedule([(7, 1, 2, 5.0, 0.0)]) == [7]                 # single request
    assert om.schedule([(1, 1, 2, 3.0, 0), (2, 1, 3, 9.0, 0), (3, 1, 4, 1.0, 0)]) == [2]   # shared src
    rng = np.random.default_rng(0)
    for _ in range(200):
        R = int(rng.integers(1, 12))
        reqs = [(i, int(rng.integers(0, 6)), int(rng.integers(0, 6)), float(rng.integers(1, 50)),
                 float(rng.integers(0, 3))) for i in range(R)]
        busy = set(rng.choice(6, size=int(rng.integers(0, 3)), replace=False).tolist())
        want = om.schedule(reqs, busy)
        got = [r.trajectory_id for r in schedule_transfers(
            [MigrationRequest(i, s, d, p, t) for (i, s, d, p, t) in reqs], busy)]
        assert got == want
        ends = [e for r in got for e in (reqs[r][1], reqs[r][2])]
        assert len(ends) == len(set(ends)) and not (set(ends) & busy)   # batch exclusivity


@pytest.mark.gpu
def test_retarget_gpu_matches_oracle():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_28101_b200.migration import retarget
    rng = np.random.default_rng(3)
    B, m = 64, 16
    bounds = np.zeros((B, m + 1), np.int32)
    for b in range(B):
        n = int(rng.integers(m, 3000))
        cuts = np.sort(rng.choice(np.arange(1, n), size=m - 1, replace=False))
        bounds[b] = np.concatenate([[0], cuts, [n]])
    na = np.array([int(rng.integers(1, bounds[b, -1] + 1)) for b in range(B)], np.int32)
    qp = rng.integers(0, B, size=5000).astype(np.int32)
    qr = np.array([int(rng.integers(-1, na[p] + 1)) for p in qp], np.int32)
    got = retarget(torch.from_numpy(bounds).cuda(), torch.from_numpy(na), torch.from_numpy(qp),
                   torch.from_numpy(qr)).cpu().numpy()
    want = np.array([om.retarget_one(list(bounds[p]), int(na[p]), int(r)) for p, r in zip(qp, qr)])
    assert np.array_equal(got, want)

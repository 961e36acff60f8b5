"""World-size-2 gloo test of the multi-GPU protocol (CPU): candidate sharding and the
16-byte winner exchange reproduce the single-process first-minimum, ties included."""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _lexmin(rows):
    best = None
    for v, i in rows:
        if best is None or v < best[0] or (v == best[0] and i < best[1]):
            best = (v, i)
    return best


def _worker(rank, world, port, makespans, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_06790_b200.batch import exchange_winners, shard

    lo, hi = shard(len(makespans), rank, world)
    local = makespans[lo:hi]
    j = int(np.argmin(local))  # first minimum, like K5 on the device
    rec = torch.empty(2, dtype=torch.float64)
    rec[0] = float(local[j])
    rec[1:2] = torch.tensor([lo + j], dtype=torch.int64).view(torch.float64)
    rows = exchange_winners(rec)
    got = [(float(r[0]), int(r[1:2].view(torch.int64).item())) for r in rows]
    q.put((rank, (lo, hi), _lexmin(got)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_winner_exchange():
    rng = np.random.default_rng(1)
    makespans = np.round(rng.uniform(100, 200, size=1001), 1)
    makespans[[17, 600, 900]] = 50.0        # tie across both ranks: first index wins
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 500
    procs = [ctx.Process(target=_worker, args=(r, 2, port, makespans, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == (0, 500) and res[1][1] == (500, 1001)
    want = (float(makespans.min()), int(np.argmin(makespans)))
    assert res[0][2] == res[1][2] == want == (50.0, 17)

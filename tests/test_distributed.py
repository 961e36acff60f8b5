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


def _sharded_worker(rank, world, port, makespans, fail_at, q):
    """One rank of sweep_sharded's protocol with the device steps replaced by numpy:
    index bases, the winner exchange (gloo all-gather), gather_all and failure agreement."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_06790_b200.batch import SweepResult, exchange_winners
    from paper_2002_06790_b200.errors import UnknownOpError
    from paper_2002_06790_b200.sharded import _sweep_distributed

    seen = {}

    def local(cfgs, gof, base):
        ms = np.asarray([makespans[c] for c in cfgs], np.float64)
        seen["base"], seen["n"] = base, len(cfgs)
        res = SweepResult(ms, ms / 2, -1, float("nan"))
        rec = torch.empty(2, dtype=torch.float64)
        j = int(np.argmin(ms)) if len(ms) else 0
        rec[0] = float(ms[j]) if len(ms) else float("inf")
        rec[1:2] = torch.tensor([base + j if len(ms) else 2 ** 63 - 1], dtype=torch.int64).view(torch.float64)
        bad = [k for k, c in enumerate(cfgs) if c in fail_at]
        failure = (bad[0], UnknownOpError({f"n{cfgs[bad[0]]}": "Op"})) if bad else None
        return res, rec, failure

    def best(rec, group):
        rows = exchange_winners(rec, group)
        got = [(float(r[0]), int(r[1:2].view(torch.int64).item())) for r in rows]
        v, i = _lexmin(got)
        out = torch.empty(2, dtype=torch.float64)
        out[0] = v
        out[1:2] = torch.tensor([i], dtype=torch.int64).view(torch.float64)
        return out

    cfgs = list(range(len(makespans)))
    try:
        out = _sweep_distributed(None, None, cfgs, [0] * len(cfgs), None, False, True, 1, None, True, rank, world,
                                 _local=local, _best=best)
        q.put((rank, seen, ("ok", out.best_index, out.best_makespan, out.makespan.tolist(), out.cp_len.tolist())))
    except UnknownOpError as e:
        q.put((rank, seen, ("err", sorted(e.nodes))))
    dist.barrier()
    dist.destroy_process_group()


def _run_sharded(world, makespans, fail_at=()):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29950 + os.getpid() % 40 + world
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, makespans, set(fail_at), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_sweep_sharded_protocol_two_and_three_ranks():
    rng = np.random.default_rng(4)
    makespans = np.round(rng.uniform(100, 200, size=1003), 1)
    makespans[[501, 502, 999]] = 42.0  # tie straddling the 2-rank boundary (501 on rank 1)
    want_i = int(np.argmin(makespans))
    for world in (2, 3):
        res = _run_sharded(world, makespans)
        for rank, seen, (kind, bi, bv, ms, cp) in res:
            assert kind == "ok"
            assert (seen["base"], seen["base"] + seen["n"]) == (1003 * rank // world, 1003 * (rank + 1) // world)
            assert (bi, bv) == (want_i, 42.0)
            assert ms == makespans.tolist() and cp == (makespans / 2).tolist()


def test_sweep_sharded_first_failure_wins_on_every_rank():
    makespans = np.arange(10, 0, -1, dtype=np.float64)
    res = _run_sharded(2, makespans, fail_at=(8, 3, 7))
    assert [r[2] for r in res] == [("err", ["n3"]), ("err", ["n3"])]

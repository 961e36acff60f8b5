"""GPU (>= 2 devices): sweep_sharded == sweep_variants on one GPU, bit for bit.

Run with ``gpurun --gpus 2`` (skipped on one GPU).  Covers both modes of sharded.py:
several devices from one process (P2P winner reduction) and one rank per GPU under
torchrun (NCCL all-gather of the 16-byte winners + k_argmin_records), including a tie
for the best makespan that straddles the shard boundary (the first index must win).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _need_two():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")


def resnet_grid(n=2048):
    """The first ``n`` C2 candidates (bench.py's resnet50-dp8 grid)."""
    sys.path.insert(0, str(ROOT))
    import bench

    graphs, db, configs, graph_of = bench.build_workload(0, n, "resnet50-dp8")
    return graphs, db, configs, graph_of


def tie_list(configs, best):
    """``configs`` with the best candidate's config copied into both shards of a 2-way split
    (index 5 and just past the middle): the best makespan is tied across the boundary."""
    others = [c for k, c in enumerate(configs) if k != best]
    L = len(others) + 2
    tied = others[:5] + [configs[best]] + others[5:]
    tied.insert(L // 2 + 3, configs[best])
    return tied


def test_sharded_devices_equal_single_gpu():
    _need_two()
    import paper_2002_06790_b200 as fw

    graphs, db, configs, graph_of = resnet_grid()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = fw.sweep_variants(graphs, db, configs, graph_of)
        tied = tie_list(configs, ref.best_index)
        one = fw.sweep_variants(graphs, db, tied, [0] * len(tied), device=0)
        two = fw.sweep_sharded(graphs, db, tied, devices=[0, 1], keep_schedules=True)
    half = len(tied) // 2
    assert one.makespan[:half].min() == one.makespan[half:].min() == one.best_makespan  # tie across shards
    assert two.best_index == one.best_index <= 5 and two.best_makespan == one.best_makespan
    assert np.array_equal(one.makespan, two.makespan) and np.array_equal(one.cp_len, two.cp_len)
    # schedules of candidates from either shard rebuild like the single-GPU ones
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        one_k = fw.sweep_variants(graphs, db, tied, [0] * len(tied), device=0, keep_schedules=True)
    for i in (0, len(tied) - 1):
        assert two.schedule(i).to_json() == one_k.schedule(i).to_json()


def test_sharded_devices_multiclass_vgg():
    _need_two()
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2002_06790_b200 as fw

    graphs, db, configs, graph_of = bench.build_workload(0, 10032, "vgg16-sweep")
    configs, graph_of = configs[::7], graph_of[::7]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        one = fw.sweep_variants(graphs, db, configs, graph_of, device=0)
        two = fw.sweep_sharded(graphs, db, configs, graph_of, devices=[0, 1])
    assert np.array_equal(one.makespan, two.makespan) and np.array_equal(one.cp_len, two.cp_len)
    assert (one.best_index, one.best_makespan) == (two.best_index, two.best_makespan)


_RANK_SCRIPT = r"""
import json, os, sys, warnings
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch, torch.distributed as dist
rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{{local}}"))
import paper_2002_06790_b200 as fw
from test_gpu_sharded import resnet_grid
graphs, db, configs, graph_of = resnet_grid()
from test_gpu_sharded import tie_list
configs = tie_list(configs, {best})
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    r = fw.sweep_sharded(graphs, db, configs)
json.dump(dict(best=r.best_index, best_ms=r.best_makespan, ms=r.makespan.tolist(), cp=r.cp_len.tolist()),
          open(os.path.join({out!r}, f"rank{{rank}}.json"), "w"))
dist.barrier()
dist.destroy_process_group()
"""


def test_sharded_torchrun_nccl(tmp_path):
    _need_two()
    import paper_2002_06790_b200 as fw

    graphs, db, configs, graph_of = resnet_grid()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = fw.sweep_variants(graphs, db, configs, graph_of, device=0)
        tied = tie_list(configs, ref.best_index)
        one = fw.sweep_variants(graphs, db, tied, [0] * len(tied), device=0)
    script = tmp_path / "rank.py"
    script.write_text(_RANK_SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"), best=ref.best_index,
                                          out=str(tmp_path)))
    port = 29500 + os.getpid() % 400
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(script)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for rank in range(2):
        got = json.loads((tmp_path / f"rank{rank}.json").read_text())
        assert got["best"] == one.best_index and got["best_ms"] == one.best_makespan
        assert got["ms"] == one.makespan.tolist() and got["cp"] == one.cp_len.tolist()

"""CPU: bench.py's reference arm runs the unmodified reference (baseline/_ref) on the bench
workloads, and it agrees with the oracle port the GPU results are checked against.

baseline/_ref is the reference pip-installed from /root/reference (git-ignored; it travels
to the GPU box with the snapshot).  Skipped where it is not installed.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

pytestmark = pytest.mark.skipif(not bench.reference_available(), reason="baseline/_ref not installed")


@pytest.mark.parametrize("workload, picks", [("resnet50-dp8", (0, 3)), ("bert-large-ps-ar", (1, 2)),
                                             ("vgg16-sweep", (5,))])
def test_reference_candidates_equal_oracle(workload, picks):
    bench._CPU_STATE.clear()
    bench._CPU_STATE["w"] = bench.build_workload(0, 64 if workload != "vgg16-sweep" else 10032, workload)
    graphs, db, cfgs, graph_of = bench._CPU_STATE["w"]
    for i in picks:
        j = (i * 7919) % len(cfgs)
        assert bench._ref_candidate(i) == bench._run_candidate_ps_aware(graphs[graph_of[j]], db, cfgs[j])


def test_reference_arm_line_shape(capsys):
    import argparse

    args = argparse.Namespace(workload="vgg16-sweep", steps=1, warmup=0, sims=None, cpu_sample=4, no_cpu=True)
    bench.run_reference(args)
    import json

    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"] == bench.bench_config(args, 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0

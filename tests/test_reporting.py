"""CPU: the C++ Chrome-trace writer (dfsim_trace_write, reporting.py:43-74) is byte-identical
to the reference's to_trace on every golden schedule, and to the oracle's restatement on
adversarial strings (escapes, non-ASCII, astral code points, half-way rounding)."""

from __future__ import annotations

import hashlib

import pytest

from oracle import dfsim_oracle as O
from paper_2002_06790_b200 import reporting as RP
from paper_2002_06790_b200.model import Schedule, ScheduledNode


def _schedule(doc):
    return Schedule(entries=[ScheduledNode(*e) for e in doc["entries"]], makespan_us=doc["makespan_us"],
                    per_device_busy_us=doc["per_device_busy_us"])


def test_trace_writer_matches_reference_golden(engine_cases, pipeline_cases):
    n = 0
    for case in list(engine_cases) + list(pipeline_cases):
        exp = case["expect"]
        if "schedule" not in exp:
            continue
        text = RP.to_trace(_schedule(exp["schedule"]))
        if "trace" in exp:
            assert text == exp["trace"], case["name"]
        assert len(text.encode()) == exp["trace_bytes"], case["name"]
        assert hashlib.sha256(text.encode()).hexdigest() == exp["trace_sha256"], case["name"]
        n += 1
    assert n > 200


@pytest.mark.parametrize("seed", range(3))
def test_trace_writer_adversarial_strings(seed):
    import random

    rng = random.Random(seed)
    alphabet = ['"', "\\", "\n", "\t", "\x00", "\x1f", "\x7f", "a", "Z", " ", "é", "中", "\U0001F600", "\ud800", "/"]
    entries = []
    devices = {}
    for i in range(60):
        nid = "".join(rng.choice(alphabet) for _ in range(rng.randint(1, 6))) + f"#{i}"
        dev = rng.choice(["gpu0", "gpu1", "link:é", "fab\"ric"])
        op = rng.choice(["", "Conv2D", "Mat\\Mul", "x\U0001F600"])
        s = rng.choice([0.5, 1.5, 2.5, 1e15 + 0.5, 3.4999999999, rng.uniform(0, 1e6)])
        f = s + rng.choice([0.0, 0.5, 1.5, rng.uniform(0, 10)])
        src = rng.choice(["Override", "ExactRecord", "FittedModel", "CommFormula", "Customé"])
        entries.append(ScheduledNode(nid, dev, s, f, src, op))
        devices[dev] = 0.0
    if seed == 1:
        devices.pop("gpu1", None)  # entries on a device outside the busy dict -> tid = len(devices)
    sched = Schedule(entries=entries, makespan_us=0.0, per_device_busy_us=devices)
    want = O.to_trace([(e.node_id, e.device, e.start_us, e.finish_us) for e in entries],
                      {e.node_id: e.op_type for e in entries}, {e.node_id: e.source for e in entries}, devices)
    assert RP.to_trace(sched) == want


def test_trace_writer_empty():
    assert RP.to_trace(Schedule(entries=[], makespan_us=0.0, per_device_busy_us={})) == "[]\n"

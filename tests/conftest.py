"""Shared test plumbing: markers, fixture loading, sys.path."""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def load_cases(name: str) -> list[dict]:
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt") as fh:
        return json.load(fh)


def case_graph(case):
    from paper_2002_06790_b200.model import parse_graph
    return parse_graph(case["graph"])


def case_table(case):
    from paper_2002_06790_b200.model import DurationEntry, DurationTable
    return DurationTable(entries={k: DurationEntry(v, s) for k, (v, s) in case["durations"].items()})


@pytest.fixture(scope="session")
def engine_cases():
    return load_cases("engine_cases")


@pytest.fixture(scope="session")
def pipeline_cases():
    return load_cases("pipeline_cases")

"""CPU-only checks: the C-ABI library and its exports, host lowering, generators."""

from __future__ import annotations

import ctypes
import re
import warnings
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, case_graph

HEADER = ROOT / "include" / "dfsim_b200.h"


def _header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:const\s+)?\w+\s*\*?\s*(dfsim_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2002_06790_b200 import build, native

    build.build()
    lib = ctypes.CDLL(str(native.LIB_PATH))
    names = _header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(native.EXPORTED)
    assert native.load_library().dfsim_abi_version() == 1


def test_library_is_sm100a():
    from paper_2002_06790_b200 import native
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(tmp_path):
    from paper_2002_06790_b200 import native
    from paper_2002_06790_b200.errors import NativeError

    with pytest.raises(NativeError):
        native.load_library(tmp_path / "nope.so")


def test_host_csr_matches_oracle_lowering(engine_cases):
    from oracle import native_oracle as NO
    from paper_2002_06790_b200.lowering import host_csr

    for case in engine_cases[:60]:
        g = case_graph(case)
        h, o = host_csr(g), NO.Csr(g)
        assert h["ids"] == o.ids
        assert np.array_equal(h["succ_off"], o.off) and np.array_equal(h["succ_idx"], o.idx)
        assert np.array_equal(h["indeg"], o.indeg)
        assert [h["devices"][d] for d in h["device"]] == [o.devices[d] for d in o.dev]


def test_generators_match_reference(engine_cases, pipeline_cases):
    """workloads.py generators reproduce the reference's synth.py output exactly."""
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import load_profiles, parse_graph, serialize_graph

    by_name = {c["name"]: c for c in engine_cases}
    for seed in range(0, 100, 7):
        nodes = 20 + (seed * 13) % 181
        g = W.random_dag(nodes, 0.02 + (seed % 5) * 0.03, seed=seed, num_devices=1 + seed % 4)
        assert serialize_graph(g) == by_name[f"c1_{seed}"]["graph"]
    pc = {c["name"]: c for c in pipeline_cases}
    assert serialize_graph(W.layered_cnn(16)) == pc["c7_r1"]["graph"]
    assert serialize_graph(W.chain(3)) == pc["chain_demo"]["graph"]
    from paper_2002_06790_b200.model import save_profiles
    assert save_profiles(W.planted_profiles(W.CNN_LAWS)).replace('"provenance": "synthetic laws"', "") == \
        pc["c7_r1"]["profiles"].replace('"provenance": "synthetic laws for LayeredCNN"', "")
    rng = W.SplitMix64(0)
    assert [rng.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_fit_matches_reference_coefficients(pipeline_cases):
    """Host fit (same numpy lstsq) -> the reference's fitted durations are reproduced by
    the Python oracle's predict; pins the coefficient pipeline without a GPU."""
    from paper_2002_06790_b200.lowering import fit_for_grid
    from paper_2002_06790_b200.model import load_profiles
    from oracle import dfsim_oracle as O

    case = next(c for c in pipeline_cases if c["name"] == "two_feature_fit")
    db = load_profiles(case["profiles"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        m = fit_for_grid(db, "MatMul", "test-hw")
        assert (m.feature_names, m.coefficients, m.intercept) == O._fit(
            [db.op_records[("MatMul", "test-hw")][k] for k in sorted(db.op_records[("MatMul", "test-hw")])])

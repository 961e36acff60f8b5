"""GPU: the bounds-checked build (libdfsim_b200_checked.so, -DDFSIM_CHECKED).

compute-sanitizer is closed on this GPU pool (profiles/r2_sanitizer.txt).  In its place the
library is built a second time with device-side checks on every index the kernels derive
from table data (engine successor / counter / ring entries, K4 v2 / v3 slot, stage, spill and
record indices, K3 large successors, K1 edge slots; csrc/internal.cuh DFSIM_CHECK).
* profiles/sanitize_run.py -- every kernel, 10/16/32-lane groups, forced ring overflows, K4
  v2 and v3, PS and multi-class streams, K3 large + K4 wide, formulas -- must run clean.
* A deliberately corrupted K4 v3 record must trip its check (the checker itself works).
Each case runs in a fresh process: the library is chosen at import (DFSIM_LIB=checked)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2002_06790_b200" / "libdfsim_b200_checked.so"


def _run(code_or_file, timeout=600):
    env = {**os.environ, "DFSIM_LIB": "checked"}
    args = [sys.executable, str(code_or_file)] if str(code_or_file).endswith(".py") else [sys.executable, "-c",
                                                                                            code_or_file]
    return subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module", autouse=True)
def checked_lib():
    if not CHECKED.exists():
        from paper_2002_06790_b200 import build

        build.build(checked=True)


def test_checked_build_runs_every_kernel_clean():
    r = _run(ROOT / "profiles" / "sanitize_run.py")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize run done" in r.stdout
    assert "libdfsim_b200_checked.so" in r.stdout  # the checked library was the one loaded


CORRUPT = r'''
import warnings, numpy as np, torch
from paper_2002_06790_b200 import native, prepare, workloads as W
from paper_2002_06790_b200.batch import TopologyClass
from paper_2002_06790_b200.errors import NativeError
from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig
assert native.LIB_PATH.name == "libdfsim_b200_checked.so"
prepare.LANE_MIN_SIMS = 1
torch.cuda.set_device(0)
warnings.simplefilter("ignore")
g = W.layered_cnn(6); db = W.planted_profiles(W.CNN_LAWS)
cfgs = [StrategyConfig(replicas=4, device_map=tuple(f"gpu{i}" for i in range(4)), gradient_markers=("grad_conv_*",),
                       hardware="synth-hw", op_gap_us=0.25 * k) for k in range(40)]
tc = TopologyClass(g, db, cfgs, 0)
assert tc.fused and tc.tables.lane is not None
o = tc.run()
torch.cuda.synchronize()
blocks = tc.tables.t["l_blocks"]
ns = tc.tables.lane["n_slots"]
rec = blocks[0:4].clone()
blocks[0] = (rec[0].item() & ~0xfff) | (1 << 12) | ns  # record 0: the first row past the slot rows (in bounds: a spill stage)
try:
    tc.run()
    torch.cuda.synchronize()
except NativeError as e:
    print("CAUGHT", e)
'''


def test_corrupted_record_trips_the_check():
    r = _run(CORRUPT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "CAUGHT" in r.stdout and "device bounds check failed" in r.stdout, r.stdout[-2000:]

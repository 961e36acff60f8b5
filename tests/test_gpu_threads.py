"""GPU: the drop-in under the reference's concurrency model.

The reference lets any number of independent simulations run concurrently
and its CLI sweep fans configs over a ThreadPoolExecutor (cli.py:133-137).  ctypes drops
the GIL during every C call, so 8 threads here call ``simulate`` / ``critical_path`` /
``estimate_all`` / ``sweep`` at once on one device (one shared context, the threads'
own streams or the default stream); every result must equal the serial run's.
"""

from __future__ import annotations

import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _workload():
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200 import workloads as W

    g = W.layered_cnn(8)
    db = W.planted_profiles(W.CNN_LAWS)
    cfgs = []
    for k in range(16):
        R = 1 + k % 4
        cfgs.append(fw.StrategyConfig(replicas=R, device_map=tuple(f"gpu{i}" for i in range(R)),
                                      gradient_markers=("grad_conv_*",), hardware="synth-hw",
                                      op_gap_us=0.25 * (k // 4)))
    return fw, g, db, cfgs


def _one(fw, g, db, cfg, use_stream):
    import torch

    def body():
        gx = fw.expand_data_parallel(g, cfg).graph
        table = fw.estimate_all(gx, db, cfg)
        s = fw.simulate(gx, table)
        cp = fw.critical_path(gx, {e.node_id: e.finish_us - e.start_us for e in s.entries})
        res = fw.sweep(g, db, [cfg, fw.StrategyConfig(**{**cfg.__dict__, "op_gap_us": cfg.op_gap_us + 1.0})])
        return s.to_json(), cp, list(res.makespan), list(res.cp_len), res.best_index

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if use_stream:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out = body()
            st.synchronize()
            return out
        return body()


@pytest.mark.parametrize("use_stream", [False, True])
def test_eight_threads_equal_serial(use_stream):
    fw, g, db, cfgs = _workload()
    serial = [_one(fw, g, db, c, use_stream) for c in cfgs]
    for _ in range(3):  # several rounds: interleavings differ from run to run
        with ThreadPoolExecutor(max_workers=8) as pool:
            got = list(pool.map(lambda c: _one(fw, g, db, c, use_stream), cfgs))
        assert got == serial


def test_threads_sweep_multiclass():
    """Concurrent multi-class sweeps (each launching on its own side streams)."""
    fw, g, db, cfgs = _workload()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        want = fw.sweep(g, db, cfgs)

        def run(_):
            r = fw.sweep(g, db, cfgs)
            return r.makespan.copy(), r.cp_len.copy(), r.best_index

        with ThreadPoolExecutor(max_workers=8) as pool:
            for ms, cp, best in pool.map(run, range(16)):
                assert np.array_equal(ms, want.makespan) and np.array_equal(cp, want.cp_len)
                assert best == want.best_index

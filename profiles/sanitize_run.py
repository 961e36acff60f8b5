"""Small workload touching every kernel of libdfsim_b200.so, for compute-sanitizer -- or, on a
pool without it, for the bounds-checked build:

    DFSIM_LIB=checked python profiles/sanitize_run.py      (tests/test_gpu_checked.py)
    compute-sanitizer --tool racecheck python profiles/sanitize_run.py   (memcheck, synccheck alike)

Covers: K1 expand (+ re-expansion), K2 estimate, K2a resolve, K3 v1 exact engine, K3 v2 fused
engine with 10-, 16- and 32-lane candidate groups and a forced FIFO-ring overflow (exact
re-run, then K4 v3 over just the re-run candidates), K3 large (a graph beyond shared
memory), K4 v1 / v2 (levels) / v3 (lanes) / wide, K5 argmin (+ records), K6 summarize, the
formula kernels, and PS / multi-class sweeps on several streams.  Prints one line per part.
"""

from __future__ import annotations

import os
import sys
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.batch import TopologyClass
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig
    from paper_2002_06790_b200.prepare import ClassTables

    warnings.simplefilter("ignore")
    torch.cuda.set_device(0)
    from paper_2002_06790_b200 import native

    print(f"library: {native.LIB_PATH.name}", flush=True)
    from paper_2002_06790_b200 import prepare

    prepare.LANE_MIN_SIMS = 1  # K4 v3 on these small classes too
    cnn = W.layered_cnn(6)
    cdb = W.planted_profiles(W.CNN_LAWS)

    def cfgs(R, n, path="PCIeSwitch", sync="allreduce", algo="RingAnalytic"):
        return [StrategyConfig(replicas=R, device_map=tuple(f"gpu{i}" for i in range(R)),
                               collective=CollectiveConfig(algo, path), gradient_markers=("grad_conv_*",),
                               hardware="synth-hw", op_gap_us=0.25 * k, sync=sync,
                               overrides={"conv_01@r0": 1.5} if k % 3 == 1 else {}) for k in range(n)]

    # K3 v2 with 10-lane (R=4: 5 devices), 16-lane (R=12) and 32-lane (R=20) groups; K4 v3 / v2
    for R in (4, 12, 20):
        for kernel in ("lanes", "levels"):
            os.environ["DFSIM_CP_KERNEL"] = kernel
            tc = TopologyClass(cnn, cdb, cfgs(R, 40), 0)
            tc.expand()
            o = tc.run(schedules=True)
            torch.cuda.synchronize()
            assert tc.fused, "the sanitizer run must reach the fused kernels"
            print(f"fused R={R} {kernel}: fused={tc.fused} k4v3={tc.tables.lane is not None if tc.tables else None} "
                  f"best={int(tc.best(o)[1:2].view(torch.int64))}", flush=True)
    os.environ["DFSIM_CP_KERNEL"] = "lanes"
    # forced ring overflow -> exact re-run (and K4 v3 / v2 over the schedules)
    for kernel in ("lanes", "levels"):
        os.environ["DFSIM_CP_KERNEL"] = kernel
        ClassTables.QCAP = 2
        tc = TopologyClass(cnn, cdb, cfgs(4, 33), 0)
        o = tc.run(schedules=True)
        torch.cuda.synchronize()
        assert o.get("fallback_rows"), "QCAP=2 must overflow"
        print(f"overflow {kernel}: re-run {len(o.get('fallback_rows', []))}", flush=True)
        ClassTables.QCAP = 16
    os.environ["DFSIM_CP_KERNEL"] = "lanes"
    # unfused K2 -> K3 v1 -> K4 v1 (+ path walk), summaries (K6) and drop-in calls
    res = fw.sweep(cnn, cdb, cfgs(3, 12), fused=False, keep_schedules=True)
    rep = res.summaries(range(4))
    g = cnn
    cfg = cfgs(2, 1)[0]
    gx = fw.expand_data_parallel(g, cfg).graph
    s = fw.simulate(gx, fw.estimate_all(gx, cdb, cfg))
    fw.critical_path(gx, {e.node_id: e.finish_us - e.start_us for e in s.entries})
    print(f"unfused + summaries: {len(rep)} reports, makespan {s.makespan_us:.3f}", flush=True)
    # PS and multi-class sweeps on several streams
    ps = [StrategyConfig(**{**c.__dict__, "overrides": {"aggregate_*": 2.0}})  # no PSAggregate records here
          for c in cfgs(4, 4, sync="parameter_server")]
    mix = cfgs(2, 4) + ps + cfgs(3, 4, algo="MeasuredThroughput")
    r2 = fw.sweep(cnn, cdb, mix)
    print(f"multi-class sweep: best {r2.best_index}", flush=True)
    # K3 large + K4 wide: a graph beyond the shared-memory engines
    big = W.layered_dag(70_000, 350, devices=4)
    from paper_2002_06790_b200.lowering import LoweredGraph
    from paper_2002_06790_b200.simulator import critical_path_arrays, simulate_arrays

    lg = LoweredGraph(big, 0)
    rng = np.random.default_rng(1)
    d = torch.tensor(rng.uniform(0.5, 3, (2, lg.n)), device="cuda:0")
    ob = simulate_arrays(lg, d)
    cp = critical_path_arrays(lg, ob["start"], ob["finish"])
    torch.cuda.synchronize()
    print(f"large engine + wide CP: {cp['cp_len'].cpu().numpy().round(3).tolist()}", flush=True)
    # formula kernels
    m = fw.LinearCostModel("Op", "hw", ("a", "b"), (1.5, -2.0), 3.0, None)
    print(f"formulas: predict {fw.predict(m, [2.0, 1.0])}, ring "
          f"{fw.allreduce_time(2 ** 20, 4, fw.ProfileDB(), algo='RingAnalytic', fallback_link=fw.DeviceSpec('l', 'Link', '', 1000.0, 1.0))}",
          flush=True)
    torch.cuda.synchronize()
    print("sanitize run done")


if __name__ == "__main__":
    main()

"""Benchmark: batched strategy simulation of a ResNet-50 DP8 training graph on B200.

Workload (BASELINE.json configs[1]): ResNet-50 training graph (564 nodes/replica),
data-parallel over 8 workers, one ring allreduce per parameter gradient over the
(synthetic) NVLink link model.  Candidates = hardware tag (8 planted profile sets)
x op_gap_us grid, all in one topology class.  One step = the hot path over one
batch: K1 expand (device) -> K2 estimate -> K3 simulate (full schedules) ->
K4 critical path -> K5 argmin (+ NCCL all-gather of winners when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sims S] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Multi-GPU: launched by torch.distributed.run,
one rank per GPU, each rank simulates its own S candidates (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "strategy simulations/sec (graph-nodes/s) at 1/2/4/8 B200 vs CPU ref; % HBM"
WORKLOADS = {  # name -> (BASELINE.json config, default candidates per GPU)
    "resnet50-dp8": ("ResNet-50 training graph, data-parallel 8 workers, ring allreduce over NVLink link model", 65536),
    "bert-large-dp8": ("BERT-large graph, allreduce per layer gradient, 8 workers over NVLink", 16384),
    "dag1m": ("synthetic 1M-node DAG x 4096 candidate strategies sharded across 8 GPUs with NCCL argmin", 512),
}
WORKLOAD = "resnet50-dp8"
N_HW = 8
HW_TAGS = tuple(f"B200-profile-{i}" for i in range(N_HW))
_GRAPHS = {}


def build_workload(rank: int, sims: int, workload: str = WORKLOAD):
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    if workload not in _GRAPHS:
        if workload == "dag1m":
            g = W.layered_dag(1_000_000, 1000, devices=8)
            _GRAPHS[workload] = (g, W.dag_profiles(HW_TAGS))
        else:
            g = W.resnet50_training(batch=32) if workload == "resnet50-dp8" else W.bert_large_training()
            _GRAPHS[workload] = (g, W.model_profiles(g, HW_TAGS))
    g, db = _GRAPHS[workload]
    dmap = tuple(f"gpu{i}" for i in range(8))
    coll = CollectiveConfig("RingAnalytic", "NVLink")
    configs = []
    for i in range(sims):
        gi = rank * sims + i  # global candidate index
        hw, gap = HW_TAGS[gi % N_HW], 1e-3 * (gi // N_HW)
        if workload == "dag1m":
            configs.append(StrategyConfig(hardware=hw, op_gap_us=gap))
        else:
            configs.append(StrategyConfig(replicas=8, device_map=dmap, collective=coll, gradient_markers=("wgrad_*",),
                                          hardware=hw, op_gap_us=gap))
    return g, db, configs


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU baseline (oracle port)


_CPU_STATE = {}


def _cpu_worker(i):
    from oracle import dfsim_oracle as O

    g, db, cfgs = _CPU_STATE["w"]
    ms, cp, *_ = O.run_candidate(g, db, cfgs[i % len(cfgs)])
    return ms


def cpu_baseline_dag(workers: int, target_s: float):
    """C5 CPU baseline: the oracle's estimate (Python, once per hardware tag) feeding the
    C restatement of simulate + critical path (oracle/engine_oracle.c) on all cores."""
    import numpy as np

    from oracle import dfsim_oracle as O
    from oracle import native_oracle as NO

    g, db, cfgs = build_workload(0, 2 * N_HW, "dag1m")
    csr = NO.Csr(g)
    t0 = time.perf_counter()
    base = {}
    rows = []
    for cfg in cfgs[: N_HW]:
        tab = O.estimate(g, db, cfg)
        base[cfg.hardware] = np.array([tab[nid][0] for nid in csr.ids])
    est_s = (time.perf_counter() - t0) / N_HW
    for i in range(workers):
        cfg = cfgs[i % len(cfgs)]
        rows.append(base[cfg.hardware])  # op_gap of the first 8 candidates is 0
    dur = np.stack(rows)
    t0 = time.perf_counter()
    rc, ms, cp = NO.simulate_batch(csr, dur, threads=workers)
    sim_s = time.perf_counter() - t0
    per_cand = est_s + sim_s * workers / len(rows)  # core-seconds per candidate
    return {"value": workers / per_cand, "unit": "sims/s", "cores": workers, "kind": "port",
            "sample": f"{len(rows)} candidates of dag1m: oracle Python estimate ({est_s:.1f} s/candidate, "
                      f"once per hardware tag) + C engine oracle simulate+critical path ({sim_s:.1f} s wall "
                      f"for {len(rows)} on {workers} threads); value = cores / core-seconds per candidate"}


def cpu_baseline(sample: int | None = None, workers: int | None = None, target_s: float = 15.0,
                 workload: str = WORKLOAD):
    """The oracle's restatement of the reference per-candidate path
    (expand -> estimate -> simulate -> critical path, cli.py:83-87), in Python like
    the reference, over a process pool of all host cores."""
    import multiprocessing as mp

    workers = workers or len(os.sched_getaffinity(0))
    if workload == "dag1m":
        return cpu_baseline_dag(workers, target_s)
    g, db, cfgs = build_workload(0, 64, workload)
    _CPU_STATE["w"] = (g, db, cfgs)
    t0 = time.perf_counter()
    _cpu_worker(0)
    one = time.perf_counter() - t0
    n = sample or max(workers, int(target_s * workers / max(one, 1e-3)))
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        list(pool.imap_unordered(_cpu_worker, range(n), chunksize=1))
    wall = time.perf_counter() - t0
    return {"value": n / wall, "unit": "sims/s", "cores": workers, "kind": "port",
            "sample": f"{n} candidates of {workload} through oracle/dfsim_oracle.run_candidate "
                      f"(Python restatement of the reference path) on {workers} processes; "
                      f"single-candidate latency {one:.3f} s"}


# ----------------------------------------------------------------------------- GPU arm


def b_table_bytes(lp) -> int:
    keys = ("soff", "sname", "sval", "ek", "em", "mk", "moff", "mname", "mcoef", "micpt", "nk", "nt", "uok", "uthr",
            "ulat")
    return int(sum(lp.tensors[k].numel() * lp.tensors[k].element_size() for k in keys))


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2002_06790_b200 import native
    from paper_2002_06790_b200.batch import TopologyClass, gather_best

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    S = args.sims or WORKLOADS[args.workload][1]
    g, db, configs = build_workload(rank, S, args.workload)
    t_setup = time.perf_counter()
    tc = TopologyClass(g, db, configs, local)
    setup_s = time.perf_counter() - t_setup
    lg, lp = tc.lg, tc.lp
    N, E, D = lg.n, lg.n_edges, lg.n_devices
    ctx = native.Context.get(local)
    dev = f"cuda:{local}"
    out = {}
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    rec = torch.empty(2, dtype=torch.float64, device=dev)

    def step(events=None):
        tc.expand()
        o = tc.run(schedules=True, out=out, events=events)
        r = tc.best(o, index_base=rank * S, record=rec)
        if world > 1:
            r = gather_best(r)
        return r

    clocks = ClockSampler(local).__enter__()  # sampled through warm-up, timed steps and e2e
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stages = ("estimate", "simulate", "critical_path")
    ev_steps = []
    step_ms = []
    launches0 = ctx.launches()
    if True:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush (256 MiB write) outside the timed events
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            evs = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in stages}
            e0.record()
            best = step(evs)
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            ev_steps.append({k: a.elapsed_time(b) for k, (a, b) in evs.items()})
    launches = ctx.launches() - launches0
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    sims_per_s = S * world / (ms_per_step / 1e3)
    best_v = float(best[0].item())
    best_i = int(best[1:2].view(torch.int64).item())

    # ---- roofline of the dominant kernel (k_simulate): algorithmic bytes per launch / avg launch time
    b_table = b_table_bytes(lp)
    b_sim = 40 * N + 4 * E + 20 + b_table
    sim_ms = statistics.mean(s["simulate"] for s in ev_steps)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = S * b_sim / (sim_ms / 1e3) / 1e9
    kernel_name = "k_simulate_fused" if tc.fused else "k_simulate"
    traffic = None  # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
    prof = ROOT / "profiles" / "r1_ncu_full.json"
    if prof.exists() and args.workload == "resnet50-dp8" and S == 65536:
        for k in json.loads(prof.read_text()):
            if kernel_name in k.get("Kernel Name", ""):
                traffic = k["dram_bytes_per_launch"]

    # ---- e2e through the public C-ABI path with host buffers: H2D candidate arrays, D2H results
    strat = lp.t_strat
    host_in = {k: v.cpu().pin_memory() for k, v in strat.items()}
    host_ms = torch.empty(S, dtype=torch.float64).pin_memory()
    host_cp = torch.empty(S, dtype=torch.float64).pin_memory()
    host_rec = torch.empty(2, dtype=torch.float64).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host_in.values())
    d2h = host_ms.numel() * 8 + host_cp.numel() * 8 + 16
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, v in host_in.items():
            strat[k].copy_(v, non_blocking=True)
        r = step()
        host_ms.copy_(out["makespan"], non_blocking=True)
        host_cp.copy_(out["cp_len"], non_blocking=True)
        host_rec.copy_(r, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    clocks.__exit__()
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = S * world / (e2e_total / args.steps / 1e3)

    if rank == 0:
        line = {
            "metric": METRIC, "value": sims_per_s, "unit": "sims/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "baseline_config": WORKLOADS[args.workload][0], "nodes_per_sim": N, "edges_per_sim": E, "devices_per_sim": D,
                       "sims_per_gpu": S, "hardware_tags": N_HW, "collective": "RingAnalytic/NVLink (synthetic row)",
                       "outputs": "full schedules (start+finish per node), makespan, busy, CP length, argmin",
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "setup_s_host_lowering": round(setup_s, 3)},
            "graph_nodes_per_s": sims_per_s * N,
            "best": {"makespan_us": best_v, "index": best_i},
            "stage_ms": {k: statistics.mean(s[k] for s in ev_steps) for k in stages},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": kernel_name,
                         "traffic_source": "profiles/r1_ncu_full.json (ncu --set full, same config)" if traffic else None,
                         "b_sim_bytes": b_sim, "b_table_bytes": b_table,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
            "e2e": {"value": e2e_value, "unit": "sims/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample, workload=args.workload)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    per_step = max(2.0, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(args.cpu_sample, target_s=per_step, workload=args.workload)
    vals, base, walls = [], None, []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        base = cpu_baseline(args.cpu_sample, target_s=per_step, workload=args.workload)
        walls.append(time.perf_counter() - t0)
        vals.append(base["value"])
    v = statistics.mean(vals)
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "sims/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": args.workload, "baseline_config": WORKLOADS[args.workload][0]},
        "cpu_baseline": {**base, "value": v},
        "e2e": {"value": v, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sims", type=int, default=None, help="candidates per GPU (default per workload)")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default=WORKLOAD)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

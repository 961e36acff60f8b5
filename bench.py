"""Benchmark: batched strategy simulation on B200 (hot path of arXiv 2002.06790's dfsim).

Default workload (BASELINE.json configs[1], `--workload resnet50-dp8`): ResNet-50
training graph (564 nodes/replica), data-parallel over 8 workers, one ring allreduce
per parameter gradient over the (synthetic) NVLink link model.  Candidates =
hardware tag (8 planted profile sets) x op_gap_us grid, one topology class.
Other workloads: `bert-large-ps-ar` (configs[3]: BERT-large, {PS, allreduce} x {2, 4, 8}
workers x {PCIe, NVLink, RDMA}, 18 topology classes), `vgg16-sweep` (configs[2]: 209 batch
sizes x 8 worker counts x PS/allreduce x PCIe/NVLink/RDMA = 10,032 candidates in 45
topology classes), `dag1m` (configs[4]: 1M-node DAG).

One step = the hot path over one batch, per topology class: K1 expand (device) ->
K2a resolve -> K3 simulate (full schedules) -> K4 critical path, then K5 argmin
(+ NCCL all-gather of per-GPU winners when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sims S] [--workload W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Multi-GPU: launched by torch.distributed.run, one
rank per GPU; each rank simulates its own candidates (weak scaling).
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
    "vgg16-sweep": ("VGG-16 strategy sweep: 10k candidates over batch size x worker count x PS/allreduce x "
                    "PCIe/NVLink/RDMA", 10032),
    "bert-large-ps-ar": ("BERT-large graph, parameter-server vs allreduce with per-layer gradient comm overlap",
                         16384),
    "dag1m": ("synthetic 1M-node DAG x 4096 candidate strategies sharded across 8 GPUs with NCCL argmin", 512),
}
WORKLOAD = "resnet50-dp8"
N_HW = 8
HW_TAGS = tuple(f"B200-profile-{i}" for i in range(N_HW))
VGG_BATCHES = tuple(8 * i for i in range(1, 210))
VGG_PATHS = ("PCIeSwitch", "NVLink", "RDMA")
_CACHE = {}


def _vgg_grid():
    """The 10,032 (batch, workers, sync, path) candidates of config C3, in a fixed order."""
    out = []
    for b in range(len(VGG_BATCHES)):
        for R in range(1, 9):
            for sync in ("allreduce", "parameter_server"):
                for path in VGG_PATHS:
                    out.append((b, R, sync, path))
    return out


def build_workload(rank: int, sims: int, workload: str = WORKLOAD):
    """Returns (graphs, db, configs, graph_of) for this rank's candidates."""
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    if workload not in _CACHE:
        if workload == "dag1m":
            g = W.layered_dag(1_000_000, 1000, devices=8)
            _CACHE[workload] = ([g], W.dag_profiles(HW_TAGS))
        elif workload == "vgg16-sweep":
            graphs = [W.vgg16_training(batch=b) for b in VGG_BATCHES]
            _CACHE[workload] = (graphs, W.model_profiles(graphs[0], HW_TAGS[:1]))
        else:
            g = W.resnet50_training(batch=32) if workload == "resnet50-dp8" else W.bert_large_training()  # C2 / C4
            _CACHE[workload] = ([g], W.model_profiles(g, HW_TAGS))
    graphs, db = _CACHE[workload]
    configs, graph_of = [], []
    if workload == "vgg16-sweep":
        grid = _vgg_grid()
        world = max(1, int(os.environ.get("WORLD_SIZE", 1)))
        lo, hi = len(grid) * rank // world, len(grid) * (rank + 1) // world
        for b, R, sync, path in grid[lo:hi][:sims]:
            dmap = tuple(f"gpu{i}" for i in range(R))
            sync = sync if R > 1 else "allreduce"  # one worker: no gradient exchange either way
            configs.append(StrategyConfig(replicas=R, device_map=dmap,
                                          collective=CollectiveConfig("MeasuredThroughput", path),
                                          gradient_markers=("wgrad_*",), hardware=HW_TAGS[0], sync=sync))
            graph_of.append(b)
        return graphs, db, configs, graph_of
    if workload == "bert-large-ps-ar":
        # C4: {allreduce, parameter server} x workers {2, 4, 8} x links, one gradient exchange per
        # layer parameter (the wgrad_* nodes) so communication overlaps the rest of the backward pass
        grid = [(R, sync, path) for R in (2, 4, 8) for sync in ("allreduce", "parameter_server")
                for path in VGG_PATHS]
        only = tuple(os.environ["DFSIM_C4_ONLY"].split(",")) if os.environ.get("DFSIM_C4_ONLY") else None
        for i in range(sims):
            gi = rank * sims + i
            R, sync, path = grid[gi % len(grid)]
            k = gi // len(grid)
            if only and (str(R), sync) != only:  # measurement knob: one (workers, sync) group only
                continue
            configs.append(StrategyConfig(replicas=R, device_map=tuple(f"gpu{j}" for j in range(R)),
                                          collective=CollectiveConfig("RingAnalytic", path),
                                          gradient_markers=("wgrad_*",), hardware=HW_TAGS[k % N_HW],
                                          op_gap_us=1e-3 * (k // N_HW), sync=sync))
            graph_of.append(0)
        return graphs, db, configs, graph_of
    dmap = tuple(f"gpu{i}" for i in range(8))
    coll = CollectiveConfig("RingAnalytic", "NVLink")
    # measurement knob (not the headline): every K-th C2 candidate carries manual overrides
    ov_every = int(os.environ.get("DFSIM_BENCH_OVERRIDES", 0))
    for i in range(sims):
        gi = rank * sims + i  # global candidate index
        hw, gap = HW_TAGS[gi % N_HW], 1e-3 * (gi // N_HW)
        if workload == "dag1m":
            configs.append(StrategyConfig(hardware=hw, op_gap_us=gap))
        else:
            ov = ({"l2_b0_conv1@r*": 50.0 + gi % 7, "fc@r0": 20.0} if ov_every and gi % ov_every == 0 else {})
            configs.append(StrategyConfig(replicas=8, device_map=dmap, collective=coll, gradient_markers=("wgrad_*",),
                                          hardware=hw, op_gap_us=gap, overrides=ov))
        graph_of.append(0)
    return graphs, db, configs, graph_of


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clocks and throttle reasons sampled (every ~5 ms via NVML, else nvidia-smi) while the
    benchmark runs; summary() reports the median SM clock under load and every reason seen."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = "nvml"

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), int(rs)))
                self._stop.wait(0.005)
            return
        except Exception:
            self.source = "nvidia-smi"
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                r = [x.strip() for x in out.stdout.strip().split(",")]
                bits = sum(v for k, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                              "sw_power_cap"), (0x8, 0x40, 0x20, 0x4))
                           if r[2 + list(self.REASONS).index(k)] == "Active")
                self.rows.append((float(r[0]), float(r[1]), bits))
            except Exception:
                pass
            self._stop.wait(0.2)

    def start(self):
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max((r[1] for r in self.rows),
                                                                                   default=None),
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


# ----------------------------------------------------------------------------- CPU baselines

REF_DIR = ROOT / "baseline" / "_ref"  # the unmodified reference, pip-installed
_CPU_STATE = {}


def reference_available() -> bool:
    return (REF_DIR / "dfsim" / "engine.py").exists()


def _ref():
    """The installed reference package (baseline/_ref/dfsim), imported on first use."""
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import dfsim  # noqa: F401
    from dfsim import costmodel, engine, graph, profiledb, strategy

    return graph, profiledb, strategy, costmodel, engine


def _ref_objects(gi: int, j: int):
    """Reference-typed (graph, db, config, pre-expanded) of candidate j, cached per worker.
    Our synthetic workloads are converted through the reference's own JSON formats
    (serialize_graph / save_profiles write the documents parse_graph / load_profiles read)."""
    from paper_2002_06790_b200.model import save_profiles, serialize_graph

    rg, rdb, rst, _, _ = _ref()
    graphs, db, cfgs, graph_of = _CPU_STATE["w"]
    cache = _CPU_STATE.setdefault("ref_cache", {})
    if "db" not in cache:
        cache["db"] = rdb.load_profiles(save_profiles(db))
    c = cfgs[j]
    rc = rst.StrategyConfig(replicas=c.replicas, device_map=tuple(c.device_map),
                            collective=rst.CollectiveConfig(c.collective.algo, c.collective.path),
                            gradient_markers=tuple(c.gradient_markers), hardware=c.hardware,
                            op_gap_us=c.op_gap_us, overrides=dict(c.overrides))
    if getattr(c, "sync", "allreduce") == "parameter_server":
        # the reference has no parameter server: its graph comes from this repo's
        # PS expansion (built here, outside the timed call); estimate + simulate + CP are the reference's
        key = ("ps", gi, c.replicas, c.collective.path)
        if key not in cache:
            from paper_2002_06790_b200.ps import expand_parameter_server

            cache[key] = rg.parse_graph(serialize_graph(expand_parameter_server(graphs[gi], c, db).graph))
        return cache[key], cache["db"], rc, True
    if ("g", gi) not in cache:
        cache[("g", gi)] = rg.parse_graph(serialize_graph(graphs[gi]))
    return cache[("g", gi)], cache["db"], rc, False


def _ref_candidate(i: int) -> float:
    """The reference's per-candidate path, cli.py:71-116 without file I/O: expand (when asked,
    cli.py:83) -> estimate_all -> simulate -> critical_path on finish - start (reporting.py:128)."""
    graphs, db, cfgs, graph_of = _CPU_STATE["w"]
    j = (i * 7919) % len(cfgs)  # spread the sample over the whole grid
    g, rdb, cfg, pre = _ref_objects(graph_of[j], j)
    rg, _, rst, rcost, reng = _ref()
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if not pre and (cfg.replicas > 1 or cfg.device_map):
            g = rst.expand_data_parallel(g, cfg).graph
        table = rcost.estimate_all(g, rdb, cfg)
        s = reng.simulate(g, table)
        rg.critical_path(g, {e.node_id: e.finish_us - e.start_us for e in s.entries})
    return s.makespan_us


def _run_candidate_ps_aware(g, db, cfg):
    """Oracle per-candidate path; PS candidates use this repo's PS expansion (no reference exists)."""
    from oracle import dfsim_oracle as O

    if getattr(cfg, "sync", "allreduce") == "parameter_server":
        from paper_2002_06790_b200.ps import expand_parameter_server

        gx = expand_parameter_server(g, cfg, db).graph
        table = O.estimate(gx, db, cfg)
        entries, ms, _ = O.simulate(gx, {k: v[0] for k, v in table.items()})
        O.critical_path(gx, {nid: f - s for nid, _, s, f in entries})
        return ms
    return O.run_candidate(g, db, cfg)[0]


def _port_candidate(i: int) -> float:
    graphs, db, cfgs, graph_of = _CPU_STATE["w"]
    j = (i * 7919) % len(cfgs)
    return _run_candidate_ps_aware(graphs[graph_of[j]], db, cfgs[j])


def _warm(fn):
    """Pool initializer job: one candidate per worker so conversions/caches are built untimed."""
    return fn(0)


def cpu_baseline_dag(workers: int, target_s: float, kind: str):
    """C5: estimate once per hardware tag, then simulate + critical path per candidate on all
    cores.  kind "reference": the installed reference (estimate_all, simulate, critical_path);
    "port": the oracle's Python estimate + the C restatement of the engine."""
    import numpy as np

    graphs, db, cfgs, graph_of = build_workload(0, 2 * N_HW, "dag1m")
    _CPU_STATE["w"] = (graphs, db, cfgs, graph_of)
    g = graphs[0]
    if kind == "reference":
        import multiprocessing as mp

        rg, _, _, rcost, reng = _ref()
        t0 = time.perf_counter()
        gr, rdb, rc, _ = _ref_objects(0, 0)
        conv_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        table = rcost.estimate_all(gr, rdb, rc)
        est_s = time.perf_counter() - t0
        _CPU_STATE["dag_ref"] = (rg, reng, gr, table)

        def one(_):
            rg_, reng_, gr_, table_ = _CPU_STATE["dag_ref"]
            sch = reng_.simulate(gr_, table_)
            rg_.critical_path(gr_, {e.node_id: e.finish_us - e.start_us for e in sch.entries})
            return sch.makespan_us

        _CPU_STATE["dag_one"] = one
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(workers) as pool:
            list(pool.map(_dag_ref_job, range(workers), chunksize=1))
        sim_s = time.perf_counter() - t0  # one candidate per core, all in parallel
        per_cand = est_s + sim_s  # core-seconds per candidate
        return {"value": workers / per_cand, "unit": "sims/s", "cores": workers, "kind": "reference",
                "sample": f"{workers} candidates of dag1m through the installed reference (baseline/_ref): "
                          f"estimate_all {est_s:.1f} s (once per hardware tag), simulate + critical_path "
                          f"{sim_s:.1f} s wall for one candidate per core; graph conversion {conv_s:.1f} s "
                          f"untimed; value = cores / core-seconds per candidate"}
    from oracle import dfsim_oracle as O
    from oracle import native_oracle as NO

    csr = NO.Csr(g)
    t0 = time.perf_counter()
    base = {}
    for cfg in cfgs[: N_HW]:
        tab = O.estimate(g, db, cfg)
        base[cfg.hardware] = np.array([tab[nid][0] for nid in csr.ids])
    est_s = (time.perf_counter() - t0) / N_HW
    dur = np.stack([base[cfgs[i % len(cfgs)].hardware] for i in range(workers)])  # op_gap of these is 0
    t0 = time.perf_counter()
    NO.simulate_batch(csr, dur, threads=workers)
    sim_s = time.perf_counter() - t0
    per_cand = est_s + sim_s * workers / len(dur)  # core-seconds per candidate
    return {"value": workers / per_cand, "unit": "sims/s", "cores": workers, "kind": "port",
            "sample": f"{len(dur)} candidates of dag1m: oracle Python estimate ({est_s:.1f} s/candidate, "
                      f"once per hardware tag) + C engine oracle simulate+critical path ({sim_s:.1f} s wall "
                      f"for {len(dur)} on {workers} threads); value = cores / core-seconds per candidate"}


def _dag_ref_job(i):
    return _CPU_STATE["dag_one"](i)


def cpu_baseline(sample: int | None = None, workers: int | None = None, target_s: float = 15.0,
                 workload: str = WORKLOAD, kind: str | None = None):
    """The reference's per-candidate CPU path on all host cores (a process pool: the reference's
    own --jobs thread pool is GIL-bound).  kind "reference" (default when
    baseline/_ref is installed): the unmodified reference (_ref_candidate); "port": the oracle's
    Python restatement (oracle/dfsim_oracle.run_candidate).  Candidates are spread over the
    whole grid; each worker converts its inputs once, untimed (one warm-up candidate)."""
    import multiprocessing as mp

    workers = workers or len(os.sched_getaffinity(0))
    kind = kind or ("reference" if reference_available() else "port")
    if workload == "dag1m":
        return cpu_baseline_dag(workers, target_s, kind)
    _CPU_STATE["w"] = build_workload(0, WORKLOADS[workload][1], workload)
    worker = _ref_candidate if kind == "reference" else _port_candidate
    t0 = time.perf_counter()
    worker(0)  # conversion + one candidate in this process
    t1 = time.perf_counter()
    worker(1)
    one = time.perf_counter() - t1
    n = sample or max(workers, int(target_s * workers / max(one, 1e-3)))
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        list(pool.map(worker, range(2, 2 + workers), chunksize=1))  # per-worker caches, untimed
        t0 = time.perf_counter()
        list(pool.imap_unordered(worker, range(2 + workers, 2 + workers + n), chunksize=1))
        wall = time.perf_counter() - t0
    what = ("the installed reference (baseline/_ref dfsim: expand_data_parallel -> estimate_all -> simulate -> "
            "critical_path, cli.py:71-116 without I/O)" if kind == "reference"
            else "oracle/dfsim_oracle.run_candidate (Python restatement of the reference path)")
    ps = " PS candidates: graph from this repo's PS expansion (the reference has none), built untimed." \
        if workload in ("vgg16-sweep", "bert-large-ps-ar") else ""
    return {"value": n / wall, "unit": "sims/s", "cores": workers, "kind": kind,
            "sample": f"{n} candidates of {workload} spread over the {len(_CPU_STATE['w'][2])}-candidate grid "
                      f"through {what} on {workers} processes; single-candidate latency {one:.3f} s.{ps}"}


# ----------------------------------------------------------------------------- GPU arm


def b_table_bytes(lp) -> int:
    """B_table of one candidate: the staged (op, hw) models, exact records and
    link rows, plus the feature vectors of ONE graph variant (a class holding GV graph variants,
    e.g. one per batch size in C3, stores GV variants' vectors; a candidate reads its own)."""
    nb = lambda k: lp.tensors[k].numel() * lp.tensors[k].element_size()  # noqa: E731
    shared = sum(nb(k) for k in ("ek", "em", "mk", "moff", "mname", "mcoef", "micpt", "nk", "nt", "uok", "uthr", "ulat"))
    per_variant = sum(nb(k) for k in ("soff", "sname", "sval")) / max(1, lp.n_gvariants)
    return int(shared + per_variant)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2002_06790_b200 import native
    from paper_2002_06790_b200.batch import TopologyClass, gather_best, group_classes

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but {world} rank(s) were launched")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    S = args.sims or WORKLOADS[args.workload][1]
    graphs, db, configs, graph_of = build_workload(rank, S, args.workload)
    S = len(configs)
    index_base = rank * S if args.workload != "vgg16-sweep" else len(_vgg_grid()) * rank // world
    t_setup = time.perf_counter()
    classes = []
    for idx in group_classes(graphs, configs, graph_of, db):  # the library's topology classes
        tc = TopologyClass(graphs[graph_of[idx[0]]], db, [configs[i] for i in idx], local, graphs=graphs,
                           graph_of=[graph_of[i] for i in idx])
        classes.append((tc, idx, {}))
    if os.environ.get("DFSIM_LPT", "1") == "1":  # most work first (as sweep_variants): no long-CTA tail
        classes.sort(key=lambda c: -c[0].lg.n * len(c[1]))
    setup_s = time.perf_counter() - t_setup
    ctx = native.Context.get(local)
    dev = f"cuda:{local}"
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    makespan = torch.empty(S, dtype=torch.float64, device=dev)
    cp_len = torch.empty(S, dtype=torch.float64, device=dev)
    rec = torch.empty(2, dtype=torch.float64, device=dev)
    t_idx = [torch.as_tensor(idx, dtype=torch.int64, device=dev) for _, idx, _ in classes]
    single = len(classes) == 1

    # several topology classes: each class's launches go to one of --streams streams so that small
    # classes (a few chunks each) share the GPU instead of running one after another; every
    # stream has its own device scratch inside the context (csrc/ctx.cu).  The whole multi-class
    # launch sequence is captured once into a CUDA graph and replayed per step (it is launch-
    # bound otherwise); ring-overflow flags of all classes share one buffer, so a step needs a
    # single device->host check before the (rare) exact re-runs.
    streams = [torch.cuda.Stream(local) for _ in range(min(len(classes), args.streams))] if not single else []
    flags_all = torch.zeros(S, dtype=torch.int32, device=dev)
    off = 0
    for tc, idx, o in classes:
        o["flags"] = flags_all[off:off + len(idx)]
        off += len(idx)

    def launch_all(events=None):
        if streams:
            cur = torch.cuda.current_stream(local)
            for st in streams:
                st.wait_stream(cur)
            for k, (tc, _, o) in enumerate(classes):
                with torch.cuda.stream(streams[k % len(streams)]):
                    tc.expand()
                    tc.run(schedules=True, out=o, defer_fallback=True,
                           events=class_evs[k] if events is not None else None)
            for st in streams:
                cur.wait_stream(st)
        for tc, _, o in (classes if not streams else ()):
            tc.expand()
            tc.run(schedules=True, out=o, events=events if single else None, defer_fallback=True)
        if single:
            o = classes[0][2]
            ms_all, cp_all = o["makespan"], o["cp_len"]
        else:
            for (tc, _, o), ti in zip(classes, t_idx):
                makespan.index_copy_(0, ti, o["makespan"])
                cp_len.index_copy_(0, ti, o["cp_len"])
            ms_all, cp_all = makespan, cp_len
        ctx.call("dfsim_argmin", S, native.ptr(ms_all), index_base, native.ptr(rec))
        return ms_all, cp_all

    graph = None
    replays = [0, 0]  # [our kernel launches per replay, replays so far]

    def step(events=None):
        nonlocal graph
        if graph is not None:
            graph.replay()
            replays[1] += 1
            ms_all, cp_all = (makespan, cp_len)
        else:
            ms_all, cp_all = launch_all(events)
        if bool(flags_all.any()):  # exact re-run of ring overflows, then their critical paths
            for tc, _, o in classes:
                if tc.fallback_if_needed(o):
                    tc.critical_path_only(o)
            if not single:
                for (tc, _, o), ti in zip(classes, t_idx):
                    makespan.index_copy_(0, ti, o["makespan"])
                    cp_len.index_copy_(0, ti, o["cp_len"])
            ctx.call("dfsim_argmin", S, native.ptr(ms_all), index_base, native.ptr(rec))
        r = gather_best(rec) if world > 1 else rec
        return r, ms_all, cp_all

    stages = ("estimate", "simulate", "critical_path")
    # stage events of the single-class step live inside the graph as external event-record
    # nodes, so each replay times its own kernels (the roofline reads them)
    graph_evs = {k: (torch.cuda.Event(enable_timing=True, external=True),
                     torch.cuda.Event(enable_timing=True, external=True)) for k in stages}
    # several classes: each class's engine launch is bracketed by its own events on its own
    # stream inside the real (concurrent) step; the engine span is first start -> last end
    class_evs = [{"simulate": (torch.cuda.Event(enable_timing=True, external=True),
                               torch.cuda.Event(enable_timing=True, external=True))} for _ in classes]

    cap_stream = torch.cuda.Stream(local)

    def capture():
        nonlocal graph
        # per-stream device scratch: size it on the capture stream first (no allocation may
        # happen while a stream is capturing)
        cap_stream.wait_stream(torch.cuda.current_stream(local))
        with torch.cuda.stream(cap_stream):
            launch_all()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = ctx.launches()
        with torch.cuda.graph(g, stream=cap_stream):
            launch_all(graph_evs)
        torch.cuda.synchronize()
        replays[0] = ctx.launches() - n0
        graph = g

    clocks = ClockSampler(local).start()  # sampled through warm-up, timed steps and e2e
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if not args.no_graph:
        capture()
        step()  # one replay before timing
        torch.cuda.synchronize()

    ev_steps, step_ms = [], []
    launches0 = ctx.launches()
    replays0 = replays[1]
    for _ in range(args.steps):
        flush.zero_()  # L2 flush (256 MiB write) outside the timed events
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in stages}
        e0.record()
        best, _, _ = step(evs)
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        if single:
            src = graph_evs if graph is not None else evs
            ev_steps.append({k: a.elapsed_time(b) for k, (a, b) in src.items()})
        elif graph is not None:  # engine span of the concurrent class launches in this step
            starts = [e0.elapsed_time(c["simulate"][0]) for c in class_evs]
            ends = [e0.elapsed_time(c["simulate"][1]) for c in class_evs]
            ev_steps.append({"simulate": max(ends) - min(starts)})
    launches = ctx.launches() - launches0 + (replays[1] - replays0) * replays[0]  # graph replays count too
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    S_total = S  # candidates of all ranks (vgg16-sweep splits one fixed grid: strong scaling)
    if world > 1:
        t = torch.tensor([S], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        S_total = int(t.item())
    sims_per_s = S_total / (ms_per_step / 1e3)
    best_v = float(best[0].item())
    best_i = int(best[1:2].view(torch.int64).item())
    n_nodes = [tc.lg.n for tc, _, _ in classes]
    mean_n = sum(n * len(idx) for n, (_, idx, _) in zip(n_nodes, classes)) / S

    # ---- roofline of the dominant kernel: algorithmic bytes per launch / its launch time
    tc0 = classes[0][0]
    kernel_name = "k_simulate_fused" if tc0.fused else "k_simulate"
    b_sim_total = sum(len(idx) * (40 * tc.lg.n + 4 * tc.lg.n_edges + 20 + b_table_bytes(tc.lp))
                      for tc, idx, _ in classes)
    roofline = None
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    if ev_steps:
        sim_ms = statistics.mean(s["simulate"] for s in ev_steps)
    else:  # (eager multi-class steps) time the engine launches alone, each class once
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        outs = [o for _, _, o in classes]
        a.record()
        for (tc, _, _), o in zip(classes, outs):
            if tc.fused:
                ctx.call("dfsim_simulate_fused", native.ctypes.byref(tc.tables.sim_struct),
                         native.ctypes.byref(tc.fused_strat), native.ptr(o["sched"]),
                         native.ptr(o["makespan"]), native.ptr(o["busy"]), native.ptr(o["n_placed"]),
                         native.ptr(o["flags"]))
        b.record()
        torch.cuda.synchronize()
        sim_ms = a.elapsed_time(b)
    achieved = b_sim_total / (sim_ms / 1e3) / 1e9
    traffic = None  # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
    profs = sorted((ROOT / "profiles").glob("r*_ncu_full.json"))  # the latest round's capture
    prof = profs[-1] if profs else ROOT / "profiles" / "r1_ncu_full.json"
    if prof.exists() and args.workload == "resnet50-dp8" and S == 65536:
        for k in json.loads(prof.read_text()):
            if kernel_name in k.get("Kernel Name", ""):
                traffic = k["dram_bytes_per_launch"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kernel_name,
                "traffic_source": f"profiles/{prof.name} (ncu --set full, same config)" if traffic else None,
                "b_sim_bytes_mean": b_sim_total / S,
                # the whole step against the same contract bytes (north star: >= 50% of the HBM roofline)
                "step_achieved": b_sim_total / (ms_per_step / 1e3) / 1e9,
                "step_frac": b_sim_total / (ms_per_step / 1e3) / 1e9 / peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                "kernel_ms": sim_ms, "launches_timed": len(classes),
                "kernel_ms_source": ("CUDA events around the engine launch of the timed steps" if single else
                                     "span from the first class's engine start to the last class's engine end "
                                     "inside the timed (concurrent) steps") if ev_steps else "serialised re-run"}

    # ---- e2e through the public C-ABI path with host buffers: H2D candidate arrays, D2H results.
    # A class's candidate arrays (hw, op_gap, algo, path, override set, graph variant) sit back to
    # back in its one device table buffer (lowering.upload), so each class takes ONE copy of that
    # byte range from a pinned host mirror
    def strat_region(tc):
        ts = list(tc.lp.t_strat.values())
        lo = min(t.data_ptr() for t in ts)
        hi = max(t.data_ptr() + t.numel() * t.element_size() for t in ts)
        base = ts[0]
        st = base.untyped_storage()
        dev_view = torch.empty(0, dtype=torch.uint8, device=base.device).set_(st, lo - st.data_ptr(), (hi - lo,))
        return dev_view, dev_view.cpu().pin_memory()

    host_in = [strat_region(tc) for tc, _, _ in classes]
    host_ms = torch.empty(S, dtype=torch.float64).pin_memory()
    host_cp = torch.empty(S, dtype=torch.float64).pin_memory()
    host_rec = torch.empty(2, dtype=torch.float64).pin_memory()
    h2d = sum(hv.numel() for _, hv in host_in)
    d2h = host_ms.numel() * 8 + host_cp.numel() * 8 + 16
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for dv, hv in host_in:
            dv.copy_(hv, non_blocking=True)
        r, ms_all, cp_all = step()
        host_ms.copy_(ms_all, non_blocking=True)
        host_cp.copy_(cp_all, non_blocking=True)
        host_rec.copy_(r, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    clocks.stop()
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = S_total / (e2e_total / args.steps / 1e3)
    cold = None if args.no_cold else measure_cold(args, graphs, db, configs, graph_of, rank, world, dev, S_total)

    if rank == 0:
        tcf = classes[0][0]
        line = {
            "metric": METRIC, "value": sims_per_s, "unit": "sims/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.workload == "vgg16-sweep" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "shape": {"nodes_per_sim": n_nodes[0] if single else round(mean_n, 1),
                      "edges_per_sim": tcf.lg.n_edges if single else None,
                      "devices_per_sim": tcf.lg.n_devices if single else None,
                      "topology_classes": len(classes)},
            "setup_s_host_lowering": round(setup_s, 3),
            "graph_nodes_per_s": sims_per_s * mean_n,
            "best": {"makespan_us": best_v, "index": best_i},
            "stage_ms": {k: statistics.mean(s[k] for s in ev_steps) for k in stages} if single else None,
            "roofline": roofline,
            "e2e": {"value": e2e_value, "unit": "sims/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "e2e_cold": cold,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if single and not args.no_reports:
            line["reports"] = measure_reports(classes[0][0], classes[0][2], args.report_rows)
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample, workload=args.workload)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure_cold(args, graphs, db, configs, graph_of, rank, world, dev, S_total, runs: int = 3):
    """One-shot sweeps through the public API, from host objects to host results: the wall time
    of sweep_variants (one GPU) / sweep_sharded (one rank per GPU) including class construction
    (expansion, lowering, tables, fits), the hot path and the D2H of makespans, critical paths
    and the best index.  Graph-object caches are dropped before every run; median of ``runs``,
    max over ranks."""
    import warnings

    import torch
    import torch.distributed as dist

    from paper_2002_06790_b200 import sweep_sharded, sweep_variants

    if world > 1:  # the global candidate list; sweep_sharded gives each rank the slice it ran above
        if args.workload == "vgg16-sweep":
            all_cfg, all_gof = build_workload_all(args, world)
        else:
            all_cfg, all_gof = [], []
            for r in range(world):
                _, _, c, gof = build_workload(r, len(configs), args.workload)
                all_cfg += c
                all_gof += gof
    walls, setups = [], []
    for _ in range(runs):
        for g in graphs:
            for attr in ("_dfsim_b200_lowered", "_dfsim_base_rows", "_dfsim_base_arr", "_dfsim_grad_keys"):
                try:
                    object.__delattr__(g, attr)
                except AttributeError:
                    pass
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if world > 1:
                res = sweep_sharded(graphs, db, all_cfg, all_gof, gather_all=False)
            else:
                res = sweep_variants(graphs, db, configs, graph_of)
        walls.append(time.perf_counter() - t0)
        assert res.best_index >= 0
    wall = statistics.median(walls)
    if world > 1:
        t = torch.tensor([wall], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    return {"value": S_total / wall, "unit": "sims/s", "wall_s": wall, "runs": runs,
            "what": "median wall time of a one-shot sweep_variants / sweep_sharded call from host objects to host "
                    "makespans + critical paths + best index, class construction included, graph caches dropped"}


def build_workload_all(args, world):
    """The whole C3 grid (build_workload splits it by WORLD_SIZE)."""
    saved = os.environ.get("WORLD_SIZE")
    os.environ["WORLD_SIZE"] = "1"
    try:
        _, _, cfg, gof = build_workload(0, len(_vgg_grid()), "vgg16-sweep")
    finally:
        if saved is None:
            os.environ.pop("WORLD_SIZE", None)
        else:
            os.environ["WORLD_SIZE"] = saved
    return cfg, gof


def measure_reports(tc, o, rows: int, cpu_rows: int = 8):
    """SURVEY.md §8f consumers of the schedules left in HBM: K6 summaries (+ K4 critical
    paths) for ``rows`` candidates timed on the device, and the Chrome trace of one
    schedule through the C++ writer; beside them the oracle's Python summarize/to_trace
    on the same schedules (1 core) as the CPU reference for these rows."""
    import numpy as np
    import torch

    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200.reporting import TraceTables, run_summary
    from paper_2002_06790_b200.simulator import critical_path_arrays

    rows = min(rows, tc.lp.n_sims)
    tables = tc.summary_tables()
    ctx = tc.ctx

    def device_pass():
        st, fi = tc.rows_by_rank_batch(o, range(rows))
        out = run_summary(ctx, tables, st, fi)
        critical_path_arrays(tc.lg, st, fi, paths=True)
        return st, fi, out

    device_pass()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st, fi, (order, _, _, _) = device_pass()
    b.record()
    torch.cuda.synchronize()
    dev_ms = a.elapsed_time(b)
    # CPU reference on the same schedules (entries rebuilt from the device result)
    g, lg = tc.graph, tc.lg
    ids = tc.ids
    dev_of = lg.device_of_rank()
    op = {nid: n.op_type for nid, n in g.nodes.items()}
    kinds = {d: spec.kind for d, spec in g.devices.items()}
    sh, fh, oh = st[:cpu_rows].cpu().numpy(), fi[:cpu_rows].cpu().numpy(), order[:cpu_rows].cpu().numpy()
    t0 = time.perf_counter()
    for j in range(min(cpu_rows, rows)):
        entries = [(ids[v], lg.devices[dev_of[v]], float(sh[j, v]), float(fh[j, v])) for v in oh[j, : lg.n].tolist()]
        busy = {}
        for nid, d, s_, f_ in entries:
            busy[d] = busy.get(d, 0.0) + (f_ - s_)
        cp = O.critical_path(g, {nid: f_ - s_ for nid, _, s_, f_ in entries})
        O.summarize(entries, op, kinds, busy, max(e[3] for e in entries), cp)
    cpu_s = (time.perf_counter() - t0) / min(cpu_rows, rows)
    # trace of one schedule: C++ writer vs the oracle's Python writer
    tracks = sorted(set(g.devices) | set(lg.devices))
    tid = {d: k for k, d in enumerate(tracks)}
    tt = TraceTables(ids, [g.nodes[nid].op_type or nid for nid in ids], np.zeros(lg.n, np.uint8),
                     [tid[lg.devices[d]] for d in dev_of], tracks)
    tt.write(oh[0, : lg.n], sh[0], fh[0])  # warm: first call sizes the reusable output buffer
    t0 = time.perf_counter()
    text = tt.write(oh[0, : lg.n], sh[0], fh[0])
    cpp_ms = (time.perf_counter() - t0) * 1e3
    entries = [(ids[v], lg.devices[dev_of[v]], float(sh[0, v]), float(fh[0, v])) for v in oh[0, : lg.n].tolist()]
    t0 = time.perf_counter()
    ref_text = O.to_trace(entries, op, {nid: "Override" for nid in ids}, {d: 0.0 for d in tracks})
    py_ms = (time.perf_counter() - t0) * 1e3
    return {"summaries": rows, "device_ms": dev_ms, "summaries_per_s": rows / (dev_ms / 1e3),
            "cpu_summaries_per_s": 1.0 / cpu_s, "cpu_kind": "port (oracle summarize + critical_path, 1 core)",
            "trace_bytes": len(text), "trace_ms_cpp": cpp_ms, "trace_ms_python_oracle": py_ms,
            "trace_identical": text == ref_text}


def bench_config(args, world: int) -> dict:
    """The workload description both arms print (the driver compares them)."""
    S = args.sims or WORKLOADS[args.workload][1]
    if args.workload == "vgg16-sweep":  # one fixed grid split over the ranks (strong scaling)
        S = min(S, len(_vgg_grid())) // world
    return {"workload": args.workload, "baseline_config": WORKLOADS[args.workload][0], "sims_per_gpu": S,
            "outputs": "full schedules (start+finish per node), makespan, busy, CP length, argmin",
            "l2": "flushed between steps (256 MiB write outside the timed events)"}


def run_reference(args):
    """The reference arm: the unmodified reference's CPU path (baseline/_ref, else the oracle
    port) on every host core, rank 0 only; each step one bounded sample of the workload's grid."""
    import multiprocessing as mp

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return
    kind = "reference" if reference_available() else "port"
    workers = len(os.sched_getaffinity(0))
    vals, walls, base = [], [], None
    if args.workload == "dag1m":  # ~a minute per candidate per core: one round per step
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            base = cpu_baseline(workers=workers, workload=args.workload, kind=kind)
            walls.append(time.perf_counter() - t0)
            vals.append(base["value"])
    else:
        _CPU_STATE["w"] = build_workload(0, WORKLOADS[args.workload][1], args.workload)
        worker = _ref_candidate if kind == "reference" else _port_candidate
        worker(0)
        t1 = time.perf_counter()
        worker(1)
        one = time.perf_counter() - t1
        per_step = max(2.0, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
        n = args.cpu_sample or max(workers, int(per_step * workers / max(one, 1e-3)))
        nxt = 2
        with mp.get_context("fork").Pool(workers) as pool:
            list(pool.map(worker, range(nxt, nxt + workers), chunksize=1))  # per-worker conversion, untimed
            nxt += workers
            for k in range(args.warmup + max(1, args.steps)):
                t0 = time.perf_counter()
                list(pool.imap_unordered(worker, range(nxt, nxt + n), chunksize=1))
                wall = time.perf_counter() - t0
                nxt += n
                if k >= args.warmup:
                    walls.append(wall)
                    vals.append(n / wall)
        what = ("the installed reference (baseline/_ref dfsim: expand_data_parallel -> estimate_all -> simulate -> "
                "critical_path, cli.py:71-116 without I/O)" if kind == "reference"
                else "oracle/dfsim_oracle.run_candidate (Python restatement of the reference path)")
        base = {"unit": "sims/s", "cores": workers, "kind": kind,
                "sample": f"per step {n} candidates of {args.workload} spread over the "
                          f"{len(_CPU_STATE['w'][2])}-candidate grid through {what} on {workers} processes; "
                          f"single-candidate latency {one:.3f} s"}
    v = statistics.mean(vals)
    line = {
        "metric": METRIC, "value": v, "unit": "sims/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True, "scaling": "strong" if args.workload == "vgg16-sweep" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": bench_config(args, world),
        "cpu_baseline": {**base, "value": v},
        "e2e": {"value": v, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference" and not args.no_cpu:  # the oracle port beside it, one short sample
        line["port_baseline"] = cpu_baseline(workers=workers, target_s=5.0, workload=args.workload, kind="port")
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--no-cold", action="store_true", help="skip the one-shot (cold) end-to-end sweeps")
    ap.add_argument("--no-reports", action="store_true", help="skip the summary/trace measurement")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--report-rows", type=int, default=1024, help="schedules summarised in the reports line")
    ap.add_argument("--streams", type=int, default=32, help="multi-class workloads: concurrent class streams (= CUDA_DEVICE_MAX_CONNECTIONS)")
    args = ap.parse_args()
    # concurrent topology classes need more hardware work queues than the default 8
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` on its own: one process per GPU through torch.distributed.run
        # (the same launch the driver uses), NCCL's init log on so the N ranks are visible
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
                   NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd, env=env))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

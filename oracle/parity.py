"""TEST INFRASTRUCTURE ONLY -- whole-grid oracle answers for the full-size parity tests.

Never imported by the package.  For a candidate grid (one graph or one graph per
candidate, a list of StrategyConfigs) this builds every candidate's duration row with the
oracle's restatement of estimate_all (dfsim_oracle.estimate, costmodel.py:282-331) and runs
the C restatement of simulate + critical_path (engine_oracle.c, engine.py:96-146,
graph.py:424-485) on all host cores.

Sharing work across candidates is exact, not an approximation:
* candidates of one topology class (same expanded graph, cli.py:83) share the expansion;
* within a class, estimate_all depends on the config only through the hardware tag, the
  collective (algo, path), the overrides and op_gap_us, and op_gap_us enters as ONE IEEE
  add on Compute nodes resolved from an exact record or a fitted model
  (costmodel.py:305-320: ``rec.mean + gap`` / ``predict(...) + gap``).  So the row of a
  candidate = the gap-0 row of its (hardware, algo, path) + gap on those nodes, which is the
  same double the reference computes.  Candidates with overrides are estimated one by one.
Parameter-server candidates use the product's PS expansion (ps.py; the reference has none)
and the oracle for everything after it, like bench.py's CPU leg.
"""

from __future__ import annotations

import dataclasses
import multiprocessing as mp
import os
import warnings

import numpy as np

from . import dfsim_oracle as O
from . import native_oracle as NO

_STATE: dict = {}


def expanded(g, cfg, db):
    """The graph a candidate simulates (cli.py:83: expand when replicas > 1 or a device_map)."""
    if getattr(cfg, "sync", "allreduce") == "parameter_server":
        from paper_2002_06790_b200.ps import expand_parameter_server

        return expand_parameter_server(g, cfg, db).graph
    if cfg.replicas > 1 or cfg.device_map:
        return O.expand(g, cfg)[0]
    return g


def class_key(cfg, gi):
    if getattr(cfg, "sync", "allreduce") == "parameter_server":
        return ("ps", gi, cfg.replicas, tuple(cfg.device_map), tuple(cfg.gradient_markers), cfg.collective.path,
                getattr(cfg, "ps_device", None))
    if not (cfg.replicas > 1 or cfg.device_map):
        return ("plain", gi)
    return ("dp", gi, cfg.replicas, tuple(cfg.device_map), tuple(cfg.gradient_markers), cfg.collective.path)


def _estimate_job(job):
    """(class position, variant key) -> (base row by rank, gap-eligible mask)."""
    k, vkey = job
    gx, csr, cfg = _STATE["classes"][k]
    hw, algo, path = vkey
    c = dataclasses.replace(cfg, hardware=hw, op_gap_us=0.0, overrides={},
                            collective=dataclasses.replace(cfg.collective, algo=algo, path=path))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tab = O.estimate(gx, _STATE["db"], c)
    base = np.array([tab[nid][0] for nid in csr.ids], np.float64)
    elig = np.array([gx.nodes[nid].kind == O.COMPUTE and tab[nid][1] in ("ExactRecord", "FittedModel")
                     for nid in csr.ids])
    return k, vkey, base, elig


def _override_job(job):
    k, i = job
    gx, csr, _ = _STATE["classes"][k]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tab = O.estimate(gx, _STATE["db"], _STATE["configs"][i])
    return i, np.array([tab[nid][0] for nid in csr.ids], np.float64)


def _class_job(job):
    """Expansion + rank CSR of one class (first candidate's config)."""
    k, gi, i = job
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gx = expanded(_STATE["graphs"][gi], _STATE["configs"][i], _STATE["db"])
    return k, gx, NO.Csr(gx)


def oracle_grid(graphs, db, configs, graph_of=None, workers: int | None = None, on_rows=None, chunk: int = 2048):
    """Oracle answers for every candidate.

    Returns dict(makespan[S], cp_len[S], cp_src_id[S], busy[S] {device: us},
    classes=[(csr, candidate indices)]).  ``on_rows(k, idx, start, finish)`` (optional) is
    called for every chunk of class k with the oracle schedules [len(idx), N] by node rank.
    """
    graph_of = list(graph_of) if graph_of is not None else [0] * len(configs)
    workers = workers or len(os.sched_getaffinity(0))
    keys, members = {}, []
    for i, cfg in enumerate(configs):
        key = class_key(cfg, graph_of[i])
        if key not in keys:
            keys[key] = len(members)
            members.append([])
        members[keys[key]].append(i)
    _STATE.update(graphs=graphs, db=db, configs=configs)
    ctx = mp.get_context("fork")
    # plain classes simulate the graph itself (nothing to expand; the caller's graph object may
    # also carry device state that does not pickle): lowered here, the others in workers
    classes = [None] * len(members)
    expand_jobs = []
    for k, m in enumerate(members):
        c = configs[m[0]]
        if class_key(c, graph_of[m[0]])[0] == "plain":
            classes[k] = (graphs[graph_of[m[0]]], NO.Csr(graphs[graph_of[m[0]]]), c)
        else:
            expand_jobs.append((k, graph_of[m[0]], m[0]))
    if expand_jobs:
        with ctx.Pool(workers) as pool:
            for k, gx, csr in pool.map(_class_job, expand_jobs, chunksize=1):
                classes[k] = (gx, csr, configs[members[k][0]])
    _STATE["classes"] = classes
    with ctx.Pool(workers) as pool:  # forked again: the workers see the classes
        jobs, ov_jobs = set(), []
        for k, m in enumerate(members):
            for i in m:
                c = configs[i]
                if c.overrides:
                    ov_jobs.append((k, i))
                else:
                    jobs.add((k, (c.hardware, c.collective.algo, c.collective.path)))
        rows = {(k, v): (b, e) for k, v, b, e in pool.map(_estimate_job, sorted(jobs), chunksize=1)}
        ov_rows = dict(pool.map(_override_job, ov_jobs, chunksize=1)) if ov_jobs else {}
    S = len(configs)
    out = dict(makespan=np.zeros(S), cp_len=np.zeros(S), cp_src_id=[None] * S, busy=[None] * S, classes=[])
    for k, m in enumerate(members):
        _, csr, _ = _STATE["classes"][k]
        out["classes"].append((csr, m))
        for a in range(0, len(m), chunk):
            idx = m[a:a + chunk]
            d = []
            for i in idx:
                c = configs[i]
                if c.overrides:
                    d.append(ov_rows[i])
                    continue
                b, e = rows[(k, (c.hardware, c.collective.algo, c.collective.path))]
                d.append(np.where(e, b + float(c.op_gap_us), b))
            rc, ms, cp, st, fi, busy, src = NO.simulate_batch_full(csr, np.stack(d), threads=workers)
            assert rc == 0, "oracle: some candidate has a cycle"
            for j, i in enumerate(idx):
                out["makespan"][i], out["cp_len"][i] = ms[j], cp[j]
                out["cp_src_id"][i] = csr.ids[src[j]] if src[j] >= 0 else None
                out["busy"][i] = {csr.devices[dv]: busy[j, dv] for dv in range(csr.n_dev)}
            if on_rows is not None:
                on_rows(k, idx, st, fi)
    return out


def first_minimum(makespan) -> int:
    """Best strategy: the first index among the minimum makespans (min(range(S), key=...))."""
    ms = np.asarray(makespan)
    return int(np.argmin(ms)) if ms.size else -1


# ----------------------------------------------------------------------------- isolated runs
#
# The GPU tests hold a CUDA context (and its threads): forking a worker pool from such a
# process can deadlock in the child.  oracle_grid_isolated runs the whole oracle grid in a
# fresh interpreter (no CUDA) and hands the answers back through files.


def _cli(argv=None):
    import argparse
    import pickle
    import sys
    from pathlib import Path

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True)
    ap.add_argument("--sims", type=int, default=None)
    ap.add_argument("--select", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--schedules", action="store_true")
    a = ap.parse_args(argv)
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import bench

    graphs, db, configs, graph_of = bench.build_workload(0, a.sims or bench.WORKLOADS[a.workload][1], a.workload)
    if a.select:
        pick = [int(x) for x in a.select.split(",")]
        configs, graph_of = [configs[i] for i in pick], [graph_of[i] for i in pick]
    out = Path(a.out)
    files = {}

    def on_rows(k, idx, st, fi):
        if k not in files:
            n = st.shape[1]
            files[k] = (np.lib.format.open_memmap(out / f"start_{k}.npy", "w+", np.float64, (len(configs), n)),
                        np.lib.format.open_memmap(out / f"finish_{k}.npy", "w+", np.float64, (len(configs), n)))
        files[k][0][idx] = st
        files[k][1][idx] = fi

    res = oracle_grid(graphs, db, configs, graph_of, on_rows=on_rows if a.schedules else None)
    for s_, f_ in files.values():
        s_.flush()
        f_.flush()
    res["classes"] = [(list(csr.ids), list(csr.devices), m) for csr, m in res["classes"]]
    with open(out / "grid.pkl", "wb") as fh:
        pickle.dump(res, fh)


def oracle_grid_isolated(workload: str, sims: int | None = None, select=None, schedules: bool = False,
                         tmpdir=None, timeout: float = 1200):
    """``oracle_grid`` over bench.build_workload(0, sims, workload) (optionally the candidates
    ``select``) in a fresh process.  Returns the same dict; with ``schedules`` also
    ``start(k)`` / ``finish(k)``: memory-mapped [S, N] oracle schedules by rank of class k
    (rows of candidates outside class k are unset)."""
    import pickle
    import subprocess
    import sys
    import tempfile
    from pathlib import Path

    d = Path(tmpdir or tempfile.mkdtemp(prefix="dfsim_oracle_"))
    cmd = [sys.executable, "-m", "oracle.parity", "--workload", workload, "--out", str(d)]
    if sims:
        cmd += ["--sims", str(sims)]
    if select:
        cmd += ["--select", ",".join(str(int(i)) for i in select)]
    if schedules:
        cmd.append("--schedules")
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run(cmd, cwd=str(root), capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"oracle grid failed: {r.stderr[-3000:]}")
    with open(d / "grid.pkl", "rb") as fh:
        res = pickle.load(fh)
    res["start"] = lambda k: np.load(d / f"start_{k}.npy", mmap_mode="r")
    res["finish"] = lambda k: np.load(d / f"finish_{k}.npy", mmap_mode="r")
    res["dir"] = d
    return res


if __name__ == "__main__":
    _cli()

"""TEST INFRASTRUCTURE ONLY -- ctypes front of oracle/build/libdfsim_oracle.so.

Lowers a graph to rank-ordered CSR with its own code (independent of the
product's lowering), then calls the C restatement of engine.py:96-146 and
graph.py:446-485.  Used by tests for large instances and by bench.py's CPU
baseline.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libdfsim_oracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.oracle_simulate.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P, P, P, P, P]
        L.oracle_critical_path.argtypes = [ctypes.c_int32, P, P, P, P, P, P, P]
        L.oracle_simulate_batch.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, P, ctypes.c_int64, P, P, P,
                                            ctypes.c_int32]
        L.oracle_simulate_batch_full.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, P, ctypes.c_int64, P, P,
                                                 P, P, P, P, P, ctypes.c_int32]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Csr:
    """Rank-ordered CSR of a graph (graph.py:122-135 semantics)."""

    def __init__(self, g):
        self.ids = sorted(g.nodes)
        rank = {nid: i for i, nid in enumerate(self.ids)}
        self.devices = sorted(set(g.devices) | {n.device for n in g.nodes.values()})
        drank = {d: i for i, d in enumerate(self.devices)}
        n = len(self.ids)
        succ = [[] for _ in range(n)]
        for nid, node in g.nodes.items():
            for pid, _ in node.inputs:
                if pid in rank:
                    succ[rank[pid]].append(rank[nid])
        self.off = np.zeros(n + 1, dtype=np.int32)
        self.off[1:] = np.cumsum([len(s) for s in succ]) if n else []
        self.idx = np.array([m for s in succ for m in sorted(s)], dtype=np.int32)
        self.indeg = np.array([len(g.nodes[nid].inputs) for nid in self.ids], dtype=np.int32)
        self.dev = np.array([drank[g.nodes[nid].device] for nid in self.ids], dtype=np.int32)
        self.n, self.n_dev = n, len(self.devices)


def simulate(csr: Csr, dur: np.ndarray):
    """Returns (status, start, finish, busy[n_dev], makespan, entry_order)."""
    n = csr.n
    dur = np.ascontiguousarray(dur, dtype=np.float64)
    start = np.empty(max(n, 1)); finish = np.empty(max(n, 1)); busy = np.zeros(max(csr.n_dev, 1))
    ms = np.zeros(1); order = np.empty(max(n, 1), dtype=np.int32); placed = np.zeros(1, dtype=np.int32)
    rc = lib().oracle_simulate(n, csr.n_dev, _p(csr.off), _p(csr.idx), _p(csr.indeg), _p(csr.dev), _p(dur),
                               _p(start), _p(finish), _p(busy), _p(ms), _p(order), _p(placed))
    return rc, start[:n], finish[:n], busy[:csr.n_dev], float(ms[0]), order[:n]


def critical_path(csr: Csr, d: np.ndarray):
    d = np.ascontiguousarray(d, dtype=np.float64)
    length = np.zeros(1); path = np.empty(max(csr.n, 1), dtype=np.int32); plen = np.zeros(1, dtype=np.int32)
    rc = lib().oracle_critical_path(csr.n, _p(csr.off), _p(csr.idx), _p(csr.indeg), _p(d), _p(length), _p(path),
                                    _p(plen))
    return rc, float(length[0]), path[: int(plen[0])]


def simulate_batch(csr: Csr, dur: np.ndarray, threads: int | None = None):
    """S independent (simulate, critical_path) runs; dur is [S, N]. Returns (status, makespan, cp_len)."""
    dur = np.ascontiguousarray(dur, dtype=np.float64)
    S = dur.shape[0]
    ms = np.zeros(S); cp = np.zeros(S)
    threads = threads or len(os.sched_getaffinity(0))
    rc = lib().oracle_simulate_batch(csr.n, csr.n_dev, _p(csr.off), _p(csr.idx), _p(csr.indeg), _p(csr.dev), S,
                                     _p(dur), _p(ms), _p(cp), threads)
    return rc, ms, cp


def simulate_batch_full(csr: Csr, dur: np.ndarray, threads: int | None = None):
    """Like simulate_batch, plus every schedule: returns (status, makespan, cp_len, start, finish,
    busy, cp_src) with start/finish [S, N] by rank, busy [S, n_dev] and cp_src [S] (path head rank)."""
    dur = np.ascontiguousarray(dur, dtype=np.float64)
    S, n = dur.shape[0], csr.n
    ms, cp = np.zeros(S), np.zeros(S)
    st, fi = np.empty((S, max(n, 1))), np.empty((S, max(n, 1)))
    busy = np.zeros((S, max(csr.n_dev, 1)))
    src = np.full(S, -1, np.int32)
    threads = threads or len(os.sched_getaffinity(0))
    rc = lib().oracle_simulate_batch_full(n, csr.n_dev, _p(csr.off), _p(csr.idx), _p(csr.indeg), _p(csr.dev), S,
                                          _p(dur), _p(ms), _p(cp), _p(st), _p(fi), _p(busy), _p(src), threads)
    return rc, ms, cp, st[:, :n], fi[:, :n], busy[:, : csr.n_dev], src

"""Large graph documents through the C++ loader.

``load_graph(text)`` is ``parse_graph`` (graph.py:192-293) for documents where Python's
json.loads and per-node object construction dominate setup (tens of seconds at 10^6
nodes).  csrc/document.cpp parses the document once and hands back, in node-rank order,
everything the device path needs: the CSR of ``lowering.host_csr`` and the per-node
op / kind / feature-signature / communication rows of ``lowering.node_rows``.  The
returned :class:`DocumentGraph` is duck-compatible with ``DataflowGraph``: its ``nodes``
mapping materialises an ``OpNode`` from the document's own text only when one is looked
at, so a sweep over a plain (unexpanded) class never builds per-node Python objects.

Documents outside the well-formed subset the loader accepts (anything the reference
warns about or rejects) are parsed by ``model.parse_graph``, so warnings and errors are
exactly the reference's.  Host code; the kernels are unchanged.
"""

from __future__ import annotations

import ctypes
import json
from collections.abc import Mapping

import numpy as np

from . import native
from .model import DataflowGraph, OpNode, TensorShape, parse_graph

KINDS = ("Compute", "Transfer", "Collective")


def _strings(blob_ptr, off_ptr, n: int) -> list[str]:
    if n <= 0:
        return []
    off = np.ctypeslib.as_array(ctypes.cast(off_ptr, ctypes.POINTER(ctypes.c_int64)), shape=(n + 1,)).copy()
    raw = ctypes.string_at(blob_ptr, int(off[-1])) if off[-1] else b""
    return [raw[off[k]:off[k + 1]].decode("utf-8") for k in range(n)]


def _array(ptr, n: int, ctype, dtype):
    if n <= 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), shape=(n,)).astype(dtype, copy=True)


class _LazyNodes(Mapping):
    """``nodes`` of a DocumentGraph: document order, OpNodes built on first access."""

    def __init__(self, doc: "DocumentGraph"):
        self._doc = doc
        self._cache: dict = {}

    def __len__(self):
        return self._doc.n

    def __iter__(self):
        ids = self._doc.ids
        return (ids[r] for r in self._doc.doc_order)

    def __contains__(self, nid):
        return nid in self._doc.rank

    def __getitem__(self, nid):
        node = self._cache.get(nid)
        if node is None:
            r = self._doc.rank[nid]  # KeyError for unknown ids, like a dict
            node = self._cache[nid] = self._doc.materialize(r)
        return node


class DocumentGraph:
    """A graph document loaded by csrc/document.cpp (see the module docstring)."""

    def __init__(self, data: bytes, handle):
        v = native.load_library().dfsim_document_view(handle).contents
        self._data = data
        self.n = int(v.n_nodes)
        self.ids = _strings(v.id_blob, v.id_off, self.n)
        self.rank = {nid: i for i, nid in enumerate(self.ids)}
        self.op_names = _strings(v.op_blob, v.op_off, int(v.n_ops))
        self.dev_names = _strings(v.dev_blob, v.dev_off, int(v.n_devices))
        fnames = _strings(v.fname_blob, v.fname_off, int(v.n_fnames))
        n, E = self.n, int(v.n_edges)
        i32, i64, u8, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8, ctypes.c_double
        self.op_of = _array(v.op_of, n, i32, np.int32)
        self.kind_of = _array(v.kind_of, n, u8, np.uint8)
        self.csr = dict(ids=self.ids, rank=self.rank, devices=self.dev_names,
                        indeg=_array(v.indeg, n, i32, np.int32), device=_array(v.dev_of, n, i32, np.int32),
                        succ_off=_array(v.succ_off, n + 1, i32, np.int32),
                        succ_idx=_array(v.succ_idx, E, i32, np.int32),
                        sources=_array(v.sources, int(v.n_sources), i32, np.int32),
                        queue_off=_array(v.queue_off, len(self.dev_names) + 1, i32, np.int32),
                        max_indeg=int(v.max_indeg))
        if n == 0:
            self.csr["succ_off"] = np.zeros(1, np.int32)
        self.sig_of = _array(v.sig_of, n, i32, np.int32)
        ns = int(v.n_sigs)
        soff = _array(v.sig_off, ns + 1, i64, np.int64)
        sfn = _array(v.sig_fname, int(soff[-1]) if ns else 0, i32, np.int32)
        sfv = _array(v.sig_fval, int(soff[-1]) if ns else 0, f64, np.float64)
        self.signatures = [tuple((fnames[sfn[j]], float(sfv[j])) for j in range(soff[k], soff[k + 1]))
                           for k in range(ns)]
        self.comm = dict(ok=_array(v.comm_ok, n, u8, np.uint8), bytes=_array(v.comm_bytes, n, i64, np.int64),
                         group=_array(v.group_size, n, i32, np.int32), thr=_array(v.link_thr, n, f64, np.float64),
                         lat=_array(v.link_lat, n, f64, np.float64))
        self._lo = _array(v.node_lo, n, i64, np.int64)
        self._hi = _array(v.node_hi, n, i64, np.int64)
        self.doc_order = np.argsort(self._lo, kind="stable")
        meta = json.loads(data[v.meta_lo:v.meta_hi]) if v.meta_lo >= 0 else {}
        devs = data[v.decl_lo:v.decl_hi].decode("utf-8") if v.decl_lo >= 0 else "[]"
        self.devices = parse_graph('{"format_version": 1, "devices": ' + devs + "}").devices
        self.metadata = dict(meta)
        self.nodes = _LazyNodes(self)

    def materialize(self, r: int) -> OpNode:
        """OpNode of rank r from its own JSON object (parse_graph's conversions)."""
        nd = json.loads(self._data[self._lo[r]:self._hi[r]])
        refs = []
        for ref in nd.get("inputs", []):
            pid, _, slot = ref.rpartition(":")
            refs.append((pid, int(slot)))
        shapes = tuple(TensorShape(tuple(s["dims"]), s.get("dtype_bytes", 4)) for s in nd.get("output_shapes", []))
        return OpNode(nd["id"], nd["op"], nd["device"], nd["kind"], dict(nd.get("attrs", {})), tuple(refs), shapes)

    def in_degree(self) -> dict:
        return dict(zip(self.ids, self.csr["indeg"].tolist()))

    def to_graph(self) -> DataflowGraph:
        """A plain DataflowGraph (every node materialised, document order)."""
        return DataflowGraph(nodes={nid: self.nodes[nid] for nid in self.nodes}, devices=dict(self.devices),
                             metadata=dict(self.metadata))


def load_graph(text) -> "DocumentGraph | DataflowGraph":
    """parse_graph for large documents: the C++ loader, else the reference semantics."""
    data = text.encode("utf-8", "surrogatepass") if isinstance(text, str) else bytes(text)
    lib = native.load_library()
    handle = native.P()
    why = ctypes.create_string_buffer(256)
    rc = lib.dfsim_document_parse(data, len(data), ctypes.byref(handle), why, 256)
    if rc != 0:  # outside the loader's subset: warnings / errors exactly as parse_graph gives them
        return parse_graph(data.decode("utf-8", "surrogatepass"))
    try:
        return DocumentGraph(data, handle)
    finally:
        lib.dfsim_document_free(handle)

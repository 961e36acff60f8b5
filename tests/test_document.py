"""CPU: the C++ graph-document loader (csrc/document.cpp, document.load_graph) against
parse_graph + host_csr + node_rows on every golden graph, the model generators and
adversarial documents; documents outside its subset fall back to parse_graph's exact
warnings and errors."""

from __future__ import annotations

import json
import warnings

import numpy as np
import pytest

from paper_2002_06790_b200 import workloads as W
from paper_2002_06790_b200.document import DocumentGraph, load_graph
from paper_2002_06790_b200.errors import GraphFormatError, GraphFormatWarning
from paper_2002_06790_b200.lowering import host_csr, node_rows
from paper_2002_06790_b200.model import parse_graph, serialize_graph


def _same(text: str):
    ref = parse_graph(text)
    doc = load_graph(text)
    assert isinstance(doc, DocumentGraph)
    h_ref, h_doc = host_csr(ref), host_csr(doc)
    for k in ("ids", "devices", "sources", "max_indeg"):
        assert (list(h_ref[k]) if k != "max_indeg" else h_ref[k]) == (list(h_doc[k]) if k != "max_indeg" else h_doc[k]), k
    for k in ("indeg", "device", "succ_off", "succ_idx", "queue_off"):
        assert np.array_equal(np.asarray(h_ref[k]), np.asarray(h_doc[k])), k
    rows = node_rows(ref, h_ref["ids"])
    for i, (feats, ok, b, gs, thr, lat) in enumerate(rows):
        assert doc.signatures[doc.sig_of[i]] == feats, (i, feats)
        assert (int(doc.comm["ok"][i]), int(doc.comm["bytes"][i]), int(doc.comm["group"][i]),
                float(doc.comm["thr"][i]), float(doc.comm["lat"][i])) == (ok, b, gs, thr, lat), i
    for i, nid in enumerate(h_ref["ids"]):
        n = ref.nodes[nid]
        assert doc.op_names[doc.op_of[i]] == n.op_type and ("Compute", "Transfer", "Collective")[doc.kind_of[i]] == n.kind
        assert doc.nodes[nid] == n
    assert list(doc.nodes) == list(ref.nodes)
    assert doc.devices == ref.devices and doc.metadata == ref.metadata
    # first-appearance order of ops and signatures, as LoweredProfiles interns them
    seen_ops, seen_sigs = {}, {}
    for i, nid in enumerate(h_ref["ids"]):
        seen_ops.setdefault(ref.nodes[nid].op_type, len(seen_ops))
        seen_sigs.setdefault(rows[i][0], len(seen_sigs))
    assert list(seen_ops) == doc.op_names and list(seen_sigs) == doc.signatures


def test_loader_matches_parse_graph_on_golden_graphs(engine_cases, pipeline_cases):
    n = 0
    for case in list(engine_cases) + list(pipeline_cases):
        texts = [case["graph"]] + ([case["expect"]["expanded"]] if "expanded" in case.get("expect", {}) else [])
        for text in texts:
            with warnings.catch_warnings():
                warnings.simplefilter("error")  # golden documents are well-formed: no fallback
                try:
                    parse_graph(text)
                except Exception:
                    continue
            _same(text)
            n += 1
    assert n > 200


@pytest.mark.parametrize("make", [lambda: W.resnet50_training(batch=8), lambda: W.bert_large_training(layers=2),
                                  lambda: W.layered_dag(5000, 100, devices=8), lambda: W.vgg16_training(batch=4)])
def test_loader_matches_parse_graph_on_model_graphs(make):
    _same(serialize_graph(make()))


def test_loader_adversarial_but_valid_document():
    doc = {"format_version": "1.3", "metadata": {"k": [1, {"x": None}]},
           "devices": [{"id": "gpu0", "kind": "Compute"},
                       {"id": "lénk", "kind": "Link", "hardware": "h", "throughput_mbps": 10, "latency_us": 0.5},
                       {"id": "fab", "kind": "CollectiveResource", "throughput_mbps": 1.0}],
           "nodes": [
               {"id": "bé", "op": "Op", "kind": "Compute", "device": "gpu0",
                "attrs": {"a": -0.0, "z": 12345678901234567, "flag": True, "s": "x", "n": None, "lst": [1]},
                "output_shapes": [{"dims": [2, 3]}, {"dims": [], "dtype_bytes": 2}]},
               {"id": "a\U0001F600", "op": "", "kind": "Transfer", "device": "lénk",
                "attrs": {"bytes": 1048576}, "inputs": ["bé:0", "bé:1", "bé:0"]},
               {"id": "c", "op": "AllReduce", "kind": "Collective", "device": "fab",
                "attrs": {"bytes": 64, "group": ["gpu0", "gpu1"], "in1_dim0x": 3.5}, "inputs": ["a\U0001F600:0"]},
               {"id": "d", "op": "Op", "kind": "Compute", "device": "gpu0", "attrs": {"a": 0.0},
                "output_shapes": [{"dims": [2, 3]}, {"dims": [], "dtype_bytes": 2}]},
           ]}
    _same(json.dumps(doc))
    _same(json.dumps(doc, ensure_ascii=False, indent=3))


@pytest.mark.parametrize("mutate, expect", [
    (lambda d: d.update(extra=1), GraphFormatWarning),                       # unknown top field: warns
    (lambda d: d["nodes"][0].update(bogus=1), GraphFormatWarning),           # unknown node field: warns
    (lambda d: d["nodes"].append(dict(d["nodes"][0])), GraphFormatError),    # duplicate id
    (lambda d: d["nodes"][1].update(inputs=["nope:0"]), GraphFormatError),   # dangling producer
    (lambda d: d["nodes"][1].update(inputs=["x:7"]), GraphFormatError),      # bad slot
    (lambda d: d["nodes"][0].update(kind="Weird"), GraphFormatError),        # bad kind
    (lambda d: d.update(format_version=2), GraphFormatError),
])
def test_loader_falls_back_to_reference_semantics(mutate, expect):
    d = {"format_version": 1, "devices": [{"id": "gpu0", "kind": "Compute"}],
         "nodes": [{"id": "x", "op": "Op", "kind": "Compute", "device": "gpu0", "output_shapes": [{"dims": [1]}]},
                   {"id": "y", "op": "Op", "kind": "Compute", "device": "gpu0", "inputs": ["x:0"]}]}
    mutate(d)
    text = json.dumps(d)
    if expect is GraphFormatWarning:
        with pytest.warns(GraphFormatWarning):
            g = load_graph(text)
        assert not isinstance(g, DocumentGraph)
    else:
        with pytest.raises(expect):
            load_graph(text)


def test_loader_rejects_what_python_would_parse_differently():
    """Forms the reference reads with Python conversions fall back instead of being guessed."""
    base = {"format_version": 1, "nodes": [{"id": "x", "op": "Op", "kind": "Compute", "device": "g",
                                            "attrs": {"v": 1}}]}
    for attrs in ({"v": float("nan")}, {"bytes": True}, {"v": 10 ** 30}):
        d = json.loads(json.dumps(base))
        d["nodes"][0]["attrs"] = attrs
        g = load_graph(json.dumps(d))
        assert not isinstance(g, DocumentGraph)
        assert g.nodes["x"].attrs == parse_graph(json.dumps(d)).nodes["x"].attrs or attrs.get("v") != attrs.get("v")


@pytest.mark.parametrize("seed", range(150))
def test_loader_random_documents(seed):
    """Random well-formed documents (ids with escapes and non-ASCII, numeric / boolean / string /
    nested attrs, multi-output shapes, duplicate references, link and collective devices) load
    identically; random corruptions fall back to parse_graph's exact behaviour."""
    import random

    rng = random.Random(seed)
    alphabet = "abcxyz_0189-./é漢\"\\ \t"
    n = rng.randint(1, 60)
    ids = set()
    while len(ids) < n:
        ids.add("".join(rng.choice(alphabet) for _ in range(rng.randint(1, 8))).replace(":", "") or "n")
    ids = list(ids)
    devs = [{"id": f"gpu{k}", "kind": "Compute"} for k in range(rng.randint(1, 4))]
    devs.append({"id": "lnk", "kind": "Link", "throughput_mbps": rng.choice([10, 2.5e3]), "latency_us": rng.random()})
    devs.append({"id": "fab", "kind": "CollectiveResource", "throughput_mbps": 1.0})
    nodes = []
    n_out = [rng.randint(0, 2) for _ in ids]
    for i, nid in enumerate(ids):
        kind = rng.choice(["Compute", "Compute", "Transfer", "Collective"])
        dev = {"Compute": rng.choice(devs[:-2])["id"], "Transfer": "lnk", "Collective": "fab"}[kind]
        attrs = {}
        for k in range(rng.randint(0, 5)):
            attrs[rng.choice(["a", "b", "flops", "k", "n", "bytes", "group", "z9", "é"])] = rng.choice(
                [rng.randint(-5, 10 ** 6), rng.random() * 100, rng.randint(1, 9), 7, None, "s", [1, 2], {"x": 1},
                 -0.0, True])
        nd = {"id": nid, "op": rng.choice(["MatMul", "Add", "", "Send", "AllReduce"]), "kind": kind, "device": dev,
              "attrs": attrs,
              "inputs": [f"{ids[j]}:{rng.randint(0, max(1, n_out[j]) - 1) if rng.random() < 0.97 else 5}"
                         for j in rng.sample(range(i), min(i, rng.randint(0, 3)))] if i else [],
              "output_shapes": [{"dims": [rng.randint(0, 9) for _ in range(rng.randint(0, 3))],
                                 "dtype_bytes": rng.choice([1, 2, 4])} for _ in range(n_out[i])]}
        if nd["inputs"] and rng.random() < 0.2:
            nd["inputs"].append(nd["inputs"][0])  # duplicate reference
        nodes.append(nd)
    doc = {"format_version": rng.choice([1, "1", "1.7"]), "metadata": {"seed": seed}, "devices": devs, "nodes": nodes}
    text = json.dumps(doc, ensure_ascii=rng.random() < 0.5, indent=rng.choice([None, 1, 2]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            ref = parse_graph(text)
        except Exception as exc:  # e.g. a slot beyond a producer's outputs, a feature-name collision
            with pytest.raises(type(exc)):
                load_graph(text)
            return
        try:
            rows = node_rows(ref, host_csr(ref)["ids"])
        except ValueError:
            rows = None  # attr/feature collisions are rejected by estimate, not by parse_graph
        got = load_graph(text)
    if rows is None or isinstance(got, type(ref)):
        assert list(got.nodes) == list(ref.nodes)
        return
    _same(text)

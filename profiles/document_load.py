"""Setup cost of a large graph document: parse_graph + host_csr (Python, the reference's
path) against the C++ loader (document.load_graph).  Host-only; run in the build container.

    python profiles/document_load.py [nodes] > profiles/r1_document_load.txt
"""
import json
import platform
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2002_06790_b200 import workloads as W  # noqa: E402
from paper_2002_06790_b200.document import load_graph  # noqa: E402
from paper_2002_06790_b200.lowering import host_csr  # noqa: E402
from paper_2002_06790_b200.model import parse_graph, serialize_graph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
g = W.layered_dag(n, 1000, devices=8)
text = serialize_graph(g)
t = time.perf_counter()
d = load_graph(text)
h = host_csr(d)
t_cpp = time.perf_counter() - t
t = time.perf_counter()
p = parse_graph(text)
hp = host_csr(p)
t_py = time.perf_counter() - t
assert list(h["ids"]) == list(hp["ids"]) and (h["succ_idx"] == hp["succ_idx"]).all()
print(json.dumps({"nodes": n, "edges": int(h["succ_off"][-1]), "document_mb": round(len(text) / 1e6, 1),
                  "cpp_loader_s": round(t_cpp, 2), "python_parse_graph_plus_host_csr_s": round(t_py, 2),
                  "speedup": round(t_py / t_cpp, 1), "host": platform.processor() or platform.machine(),
                  "note": "single thread; same CSR checked equal"}))

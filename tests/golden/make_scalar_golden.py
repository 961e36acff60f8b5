"""Golden vectors for the scalar drop-in functions, produced by the REAL reference here.

    python tests/golden/make_scalar_golden.py     (only where /root/reference exists)

Writes ``scalar_cases.json.gz``: predict (costmodel.py:158-165) on seeded models and feature
vectors (1-5 features, mixed magnitudes so CPython's compensated sum matters), transfer_time /
allreduce_time (costmodel.py:176-223) over the reference's own Table-1 sample DB
(pkg/samples/v100_table1.profdb) and synthetic NVLink rows, their argument errors, and
topological_order (graph.py:424-443) of seeded random DAGs (the reference's generator,
synth.py RandomDAG) including a cycle.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
if not REF.exists():
    sys.exit("reference not present; fixtures are generated only in the build container")
sys.path.insert(0, str(REF / "src"))
from dfsim.costmodel import LinearCostModel, allreduce_time, predict, transfer_time  # noqa: E402
from dfsim.errors import CycleError, DfsimError  # noqa: E402
from dfsim.graph import DeviceSpec, OpNode, TensorShape, make_graph, serialize_graph, topological_order  # noqa: E402
from dfsim.profiledb import load_profiles, save_profiles  # noqa: E402


def _err(fn):
    try:
        return {"value": fn()}
    except (ValueError, DfsimError) as e:
        return {"error": type(e).__name__, "message": str(e)}


def main():
    rng = random.Random(2002_06790)
    predicts = []
    for k in range(400):
        nf = 1 + k % 5
        coefs = [rng.choice([1, -1]) * 10 ** rng.uniform(-6, 6) for _ in range(nf)]
        icpt = rng.uniform(-1e3, 1e3)
        feats = [rng.choice([0.0, 1.0, 3.0, 10 ** rng.uniform(-3, 7)]) for _ in range(nf)]
        m = LinearCostModel("Op", "hw", tuple(f"f{i}" for i in range(nf)), tuple(coefs), icpt, None)
        predicts.append({"coefs": coefs, "intercept": icpt, "features": feats, "expect": predict(m, feats)})
    db = load_profiles((REF / "samples" / "v100_table1.profdb").read_text())
    comms = []
    for (scen, path, n), rec in sorted(db.link_records.items()):
        link = DeviceSpec(id="l", kind="Link", throughput_mbps=rec.throughput_mbps, latency_us=rec.latency_us)
        for b in (1, 4096, 2 ** 20, 100 * 2 ** 20, 3 * 10 ** 9, 0, -5):
            comms.append({"fn": "transfer_time", "bytes": b, "thr": rec.throughput_mbps, "lat": rec.latency_us,
                          "expect": _err(lambda: transfer_time(b, link))})
    fallback = DeviceSpec(id="f", kind="Link", throughput_mbps=858306.0, latency_us=1.25)
    for path in ("QPI", "PCIeSwitch", "RootComplex", "NVLink"):
        for n in (1, 2, 3, 4, 8):
            for algo in ("MeasuredThroughput", "RingAnalytic", "Bogus"):
                for fb in (None, fallback):
                    for b in (2 ** 20, 100 * 2 ** 20, 12345677, 0):
                        comms.append({"fn": "allreduce_time", "bytes": b, "n": n, "algo": algo, "path": path,
                                      "fallback": None if fb is None else [fb.throughput_mbps, fb.latency_us],
                                      "expect": _err(lambda: allreduce_time(b, n, db, algo=algo, path=path,
                                                                            fallback_link=fb))})
    topo = []
    for seed in range(12):
        r = random.Random(seed)
        n = r.randint(1, 300)
        nodes = []
        names = [f"{r.choice('abcxyz')}{r.randint(0, 999)}_{i}" for i in range(n)]
        for i in range(n):
            ins = sorted({names[r.randrange(i)] for _ in range(r.randint(0, 3))}) if i else []
            nodes.append(OpNode(names[i], "Op", "gpu0", inputs=tuple((p, 0) for p in ins),
                                output_shapes=(TensorShape((2,), 4),)))
        if seed == 11:  # a cycle: the first node also consumes the last
            nodes[0] = OpNode(names[0], "Op", "gpu0", inputs=((names[-1], 0),), output_shapes=(TensorShape((2,), 4),))
        g = make_graph(nodes, [DeviceSpec("gpu0", "Compute")])
        topo.append({"graph": json.loads(serialize_graph(g)), "expect": _err(lambda: topological_order(g))})
    doc = {"predict": predicts, "comm": comms, "profiles": json.loads(save_profiles(db)), "topo": topo}
    with gzip.open(OUT / "scalar_cases.json.gz", "wt") as f:
        json.dump(doc, f)
    print(f"{len(predicts)} predict, {len(comms)} comm, {len(topo)} topo cases")


if __name__ == "__main__":
    main()

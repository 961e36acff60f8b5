"""GPU: the parameter-server expansion emitted by K1 on the device (expand.cu, PS mode) equals
the host construction (ps.expand_parameter_server followed by the rank CSR of graph.py:122-135)
for every PS topology class of the C3 / C4 bench grids: ids, devices, successor CSR with
multiplicity, in-degrees, device ranks and sources -- and re-expansion reproduces it."""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _ps_classes(workload, limit=None):
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2002_06790_b200.batch import class_key

    graphs, db, configs, graph_of = bench.build_workload(0, bench.WORKLOADS[workload][1], workload)
    seen, out = set(), []
    for cfg, gi in zip(configs, graph_of):
        if getattr(cfg, "sync", "") != "parameter_server":
            continue
        k = (class_key(cfg), cfg.collective.path, gi if workload != "vgg16-sweep" else gi % 7)
        if k in seen:
            continue
        seen.add(k)
        out.append((graphs[gi], cfg))
    return db, out[:limit]


@pytest.mark.parametrize("workload, limit", [("bert-large-ps-ar", None), ("vgg16-sweep", 24)])
def test_device_ps_expansion_equals_host(workload, limit):
    from paper_2002_06790_b200.expansion import ExpansionPlan
    from paper_2002_06790_b200.lowering import host_csr
    from paper_2002_06790_b200.ps import expand_parameter_server

    db, classes = _ps_classes(workload, limit)
    assert classes
    for g, cfg in classes:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            plan = ExpansionPlan(g, cfg, 0, build_objects=False, db=db)
            gx = expand_parameter_server(g, cfg, db, cfg.ps_device).graph
        host = host_csr(gx)
        lg = plan.lowered
        N = lg.n
        assert plan.ids == host["ids"] and N == len(host["ids"])
        assert plan.devices == sorted(set(gx.devices) | {n.device for n in gx.nodes.values()})
        assert np.array_equal(lg.t_succ_off[: N + 1].cpu().numpy(), host["succ_off"])
        assert np.array_equal(lg.t_succ_idx[: lg.n_edges].cpu().numpy(), host["succ_idx"])
        assert np.array_equal(lg.t_indeg[:N].cpu().numpy(), host["indeg"])
        dev_names = [plan.devices[d] for d in lg.t_dev[:N].cpu().numpy().tolist()]
        assert dev_names == [gx.nodes[i].device for i in plan.ids]
        assert np.array_equal(lg.t_sources[: lg.n_sources].cpu().numpy(), host["sources"])
        plan.reexpand(topo=True, check=True)
        # the lazily built objects are the host expansion's
        assert sorted(plan.graph.nodes) == plan.ids


@pytest.mark.parametrize("workload, limit", [("resnet50-dp8", 1), ("bert-large-ps-ar", None), ("vgg16-sweep", 12)])
def test_single_launch_k1_equals_multi_kernel_k1(workload, limit, monkeypatch):
    """K1 for small classes runs as one CTA (k_expand_small: block radix sort of 32-bit keys);
    its CSR, in-degrees, devices, sources, and queue offsets must equal the
    multi-kernel path's (cub device radix sort / scan / select) array for array."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2002_06790_b200.batch import class_key
    from paper_2002_06790_b200.expansion import ExpansionPlan

    graphs, db, configs, graph_of = bench.build_workload(0, bench.WORKLOADS[workload][1], workload)
    seen, classes = set(), []
    for cfg, gi in zip(configs, graph_of):
        k = (class_key(cfg), cfg.collective.path, gi if workload != "vgg16-sweep" else gi % 5)
        if k not in seen:
            seen.add(k)
            classes.append((graphs[gi], cfg))
    for g, cfg in classes[:limit]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            plan = ExpansionPlan(g, cfg, 0, build_objects=False, db=db)
        lg = plan.lowered
        N = lg.n
        arrays = lambda: [lg.t_succ_off[: N + 1].cpu(), lg.t_succ_idx[: lg.n_edges].cpu(), lg.t_indeg[:N].cpu(),  # noqa: E731
                          lg.t_dev[:N].cpu(), lg.t_sources[: lg.n_sources].cpu(),
                          lg.t_queue_off[: lg.n_devices + 1].cpu()]
        small = arrays()
        monkeypatch.setenv("DFSIM_K1_MULTI", "1")
        plan.reexpand(topo=True, check=True)
        multi = arrays()
        monkeypatch.delenv("DFSIM_K1_MULTI")
        plan.reexpand(topo=True, check=True)
        again = arrays()
        for a, b, c in zip(small, multi, again):
            assert np.array_equal(a.numpy(), b.numpy()) and np.array_equal(a.numpy(), c.numpy())

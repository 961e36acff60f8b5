"""Topology-class grouping (batch.group_classes, expansion.path_roles) is sound: every config of
one class expands -- on the host, through the oracle's data-parallel expansion
(strategy.py:170-282) or the PS construction -- to the same ids, successor CSR, in-degrees and
device ranks, so one device-side structure (K1's CSR, the fused engine's tables) serves the
whole class.  Paths share a class when only the added devices' names differ; a base device
that an expansion's added device would collide with under one path splits that path off; a
PS path without its link record is a class of its own whose expansion raises."""

from __future__ import annotations

import dataclasses
import warnings

import numpy as np
import pytest

PATHS = ("PCIeSwitch", "NVLink", "RDMA", "QPI")  # QPI: no gpu-gpu-uni row (PS expansion fails)


def _graphs():
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import DEVICE_LINK, TRANSFER, DeviceSpec, OpNode

    g0, g1, g2 = W.layered_cnn(4), W.layered_cnn(4, batch=64), W.layered_cnn(6)
    first = sorted(g0.nodes)[0]

    def with_link(name):  # g0 plus a transfer on a link device called ``name``
        g = dataclasses.replace(g0, nodes=dict(g0.nodes), devices=dict(g0.devices))
        g.nodes["xfer_in"] = OpNode("xfer_in", "Copy", name, kind=TRANSFER, inputs=((first, 0),),
                                    attrs={"src_device": "gpu0", "dst_device": "host0", "bytes": 4096})
        g.devices[name] = DeviceSpec(name, DEVICE_LINK, "", 1000.0, 1.0)
        return g

    # named like: the NVLink allreduce fabric of gpu0+gpu1 (g3), the NVLink PS up-link of gpu0
    # (g4), the PS device (g5) -- an expansion replaces the spec of each
    return [g0, g1, g2, with_link("collective:NVLink:gpu0+gpu1"), with_link("link:NVLink:gpu0->ps0"),
            with_link("ps0")]


def _configs():
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    out = [(StrategyConfig(hardware="synth-hw"), 0)]
    for gi in range(6):
        for R in (2, 3):
            for sync in ("allreduce", "parameter_server"):
                for path in PATHS:
                    cfg = StrategyConfig(replicas=R, device_map=tuple(f"gpu{i}" for i in range(R)),
                                         collective=CollectiveConfig("RingAnalytic", path),
                                         gradient_markers=("grad_conv_*",), hardware="synth-hw", sync=sync,
                                         # the planted profiles hold no PSAggregate records
                                         overrides={"aggregate_*": 2.0} if sync == "parameter_server" else {})
                    out.append((cfg, gi))
    return out


def _expand(g, cfg, db):
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200.ps import expand_parameter_server

    if cfg.sync == "parameter_server":
        return expand_parameter_server(g, cfg, db, cfg.ps_device).graph
    return O.expand(g, cfg)[0]


def _structure(g, cfg, db):
    from paper_2002_06790_b200.errors import DfsimError
    from paper_2002_06790_b200.lowering import host_csr

    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            h = host_csr(_expand(g, cfg, db))
    except DfsimError as e:
        return ("raises", type(e).__name__)
    return (tuple(h["ids"]), h["succ_off"].tobytes(), h["succ_idx"].tobytes(), h["indeg"].tobytes(),
            h["device"].tobytes(), len(h["devices"]))


@pytest.fixture(scope="module")
def grouped():
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.batch import group_classes

    db = W.planted_profiles(W.CNN_LAWS, links=W.SYNTH_LINKS + W.SYNTH_FABRIC_LINKS)
    graphs, pairs = _graphs(), _configs()
    configs, graph_of = [c for c, _ in pairs], [gi for _, gi in pairs]
    return db, graphs, configs, graph_of, group_classes(graphs, configs, graph_of, db)


def test_classes_partition_the_configs(grouped):
    _, _, configs, _, classes = grouped
    flat = sorted(i for c in classes for i in c)
    assert flat == list(range(len(configs)))
    assert all(list(c) == sorted(c) for c in classes)  # config order kept inside a class


def test_every_class_expands_to_one_structure(grouped):
    db, graphs, configs, graph_of, classes = grouped
    for members in classes:
        shapes = {_structure(graphs[graph_of[i]], configs[i], db) for i in members}
        assert len(shapes) == 1, [(configs[i].collective.path, configs[i].sync, graph_of[i]) for i in members]


def test_paths_merge_unless_roles_differ(grouped):
    db, graphs, configs, graph_of, classes = grouped
    cls_of = {i: k for k, c in enumerate(classes) for i in c}

    def cls(gi, R, sync, path):
        (i,) = [i for i, c in enumerate(configs) if graph_of[i] == gi and c.replicas == R and c.sync == sync
                and c.collective.path == path]
        return cls_of[i]

    for R in (2, 3):
        # allreduce: every path one class; the same-structure graph variant g1 shares it
        assert len({cls(gi, R, "allreduce", p) for gi in (0, 1) for p in PATHS}) == 1
        assert cls(2, R, "allreduce", "NVLink") != cls(0, R, "allreduce", "NVLink")  # other structure
        # PS: paths with a link record merge; QPI (no record) stays apart and raises
        ps = {p: cls(0, R, "parameter_server", p) for p in PATHS}
        assert ps["PCIeSwitch"] == ps["NVLink"] == ps["RDMA"] != ps["QPI"]
        assert _structure(graphs[0], configs[classes[ps["QPI"]][0]], db)[0] == "raises"
    # g3's link is the NVLink allreduce device of gpu0+gpu1: R=2 NVLink expands to one device
    # fewer, so it is split from the other paths; at R=3 the names differ and all paths merge
    g3 = {p: cls(3, 2, "allreduce", p) for p in PATHS}
    assert g3["PCIeSwitch"] == g3["RDMA"] == g3["QPI"] != g3["NVLink"]
    assert len({cls(3, 3, "allreduce", p) for p in PATHS}) == 1
    s_nv = _structure(graphs[3], configs[classes[g3["NVLink"]][0]], db)
    s_pc = _structure(graphs[3], configs[classes[g3["PCIeSwitch"]][0]], db)
    assert s_nv[5] == s_pc[5] - 1
    # g4's link is the NVLink PS up-link of gpu0: PS NVLink is split off at R = 2 and 3 alike
    for R in (2, 3):
        g4 = {p: cls(4, R, "parameter_server", p) for p in PATHS}
        assert g4["PCIeSwitch"] == g4["RDMA"] != g4["NVLink"] != g4["QPI"]
        assert len({cls(4, R, "allreduce", p) for p in PATHS}) == 1
        # g5's link is the PS device: every path expands alike (the device keeps its name)
        assert cls(5, R, "parameter_server", "PCIeSwitch") == cls(5, R, "parameter_server", "NVLink")


def test_per_candidate_objects_group_by_value():
    """Sweeps often build a fresh device_map / marker tuple per candidate: grouping keys on
    the values, not on object identity."""
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.batch import group_classes
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    db = W.planted_profiles(W.CNN_LAWS)
    g = W.layered_cnn(4)
    cfgs = [StrategyConfig(replicas=2, device_map=tuple(["gpu0", "gpu1"][:]), op_gap_us=0.1 * k,
                           collective=CollectiveConfig("RingAnalytic", "PCIeSwitch"),
                           gradient_markers=tuple(["grad_conv_*"]), hardware="synth-hw") for k in range(50)]
    cfgs += [dataclasses.replace(c, device_map=("gpu1", "gpu0")) for c in cfgs[:7]]
    classes = group_classes([g], cfgs, [0] * len(cfgs), db)
    assert [list(c) for c in classes] == [list(range(50)), list(range(50, 57))]
    assert np.all([c.device_map == ("gpu1", "gpu0") for c in cfgs[50:]])


def test_configs_without_ps_fields():
    """The reference's own StrategyConfig has no ``sync`` / ``ps_device`` (PS is an extension):
    such configs group as allreduce / plain, on the column path."""
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.batch import group_classes
    from paper_2002_06790_b200.model import CollectiveConfig

    @dataclasses.dataclass(frozen=True)
    class RefConfig:  # the reference's strategy.py:31-58 fields only
        replicas: int = 1
        device_map: tuple = ()
        collective: CollectiveConfig = CollectiveConfig()
        gradient_markers: tuple = ()
        hardware: str = "synth-hw"
        op_gap_us: float = 0.0
        overrides: dict = dataclasses.field(default_factory=dict)

    db = W.planted_profiles(W.CNN_LAWS)
    g = W.layered_cnn(3)
    dp = dict(replicas=2, device_map=("gpu0", "gpu1"), gradient_markers=("grad_conv_*",))
    cfgs = [RefConfig(**dp, collective=CollectiveConfig("RingAnalytic", p)) for p in ("PCIeSwitch", "NVLink")]
    cfgs += [RefConfig(), RefConfig(op_gap_us=1.0), RefConfig(**dp)]
    classes = group_classes([g], cfgs, [0] * len(cfgs), db)
    assert [list(c) for c in classes] == [[0, 1, 4], [2, 3]]
    same = [RefConfig(**dp, op_gap_us=0.1 * k) for k in range(5)]
    assert [list(c) for c in group_classes([g], same, [0] * 5, db)] == [list(range(5))]

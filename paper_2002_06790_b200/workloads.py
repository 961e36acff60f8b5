"""Synthetic workloads: graphs, profile DBs and strategy grids for configs C1-C5.

The reference-compatible generators (SplitMix64, Chain, LayeredCNN, RandomDAG,
planted-law profiles) reproduce pkg/src/dfsim/synth.py:33-407 bit-for-bit (pinned
by tests/test_workloads.py against fixtures made by the reference).  They are
fixture/input generators, not part of the simulated hot path.
"""

from __future__ import annotations

from .model import (
    DEVICE_COMPUTE,
    DeviceSpec,
    LinkRecord,
    OpNode,
    OpSignature,
    ProfileDB,
    ProfileRecord,
    TensorShape,
    db_insert,
    make_graph,
)

MASK64 = (1 << 64) - 1


class SplitMix64:
    """Portable PRNG of synth.py:33-71 (golden-gamma step, 30/27/31 mix)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def randint(self, lo: int, hi: int) -> int:
        if hi < lo:
            raise ValueError(f"empty range [{lo}, {hi}]")
        return lo + self.next_u64() % (hi - lo + 1)


def _gpus(n: int, hw: str = "synth-hw"):
    return [DeviceSpec(f"gpu{i}", DEVICE_COMPUTE, hw) for i in range(n)]


# (feature, slope, intercept) planted laws -- synth.py:123-161
CNN_LAWS = {
    "Input": (None, 0.0, 5.0),
    "Conv2D": ("in_channels", 12.5, 40.0),
    "Relu": ("in0_dim3", 0.05, 8.0),
    "MatMul": ("k", 0.02, 30.0),
    "SoftmaxLoss": ("in0_dim1", 0.0, 15.0),
    "MatMulGrad": ("k", 0.03, 35.0),
    "Conv2DBackpropFilter": ("in_channels", 14.0, 50.0),
    "Conv2DBackpropInput": ("in_channels", 13.0, 45.0),
    "ApplyGradientDescent": ("in0_dim2", 0.5, 10.0),
}
CHAIN_OPS = ("MatMul", "Relu", "Add")
RANDOM_OPS = ("MatMul", "Relu", "Add", "Mul")
SYNTH_LINKS = (
    LinkRecord("gpu-gpu-uni", "PCIeSwitch", 2, 12000.0),
    LinkRecord("host-to-gpu", "PCIeSwitch", 1, 11000.0),
    LinkRecord("gpu-to-host", "PCIeSwitch", 1, 13000.0),
    LinkRecord("nccl-allreduce", "PCIeSwitch", 2, 10000.0),
    LinkRecord("nccl-allreduce", "PCIeSwitch", 4, 8000.0),
    LinkRecord("nccl-allreduce", "PCIeSwitch", 8, 6000.0),
)
DEFAULT_GRID = tuple(float(2 ** i) for i in range(16))


def chain(n: int = 3):
    shape = TensorShape((32, 64), 4)
    nodes = [OpNode(f"node_{i:03d}", CHAIN_OPS[i % 3], "gpu0", attrs={"cost_hint": (i % 16) + 1},
                    inputs=((f"node_{i - 1:03d}", 0),) if i else (), output_shapes=(shape,)) for i in range(n)]
    return make_graph(nodes, _gpus(1), {"model": f"chain-{n}", "batch": 32})


def layered_cnn(layers: int = 4, batch: int = 32):
    """LayeredCNN of synth.py:224-342 (forward conv/relu, backward filter/input, apply)."""
    hw, kernel = 16, 3
    ch = [8 * (1 + (i % 8)) for i in range(layers)]
    cin = [3] + ch[:-1]
    act = lambda c: TensorShape((batch, hw, hw, c), 4)  # noqa: E731
    nodes = [OpNode("input", "Input", "gpu0", output_shapes=(act(3),))]
    prev = "input"
    for i in range(layers):
        nodes.append(OpNode(f"conv_{i:02d}", "Conv2D", "gpu0",
                            attrs={"batch": batch, "in_channels": cin[i], "out_channels": ch[i], "kernel": kernel,
                                   "stride": 1}, inputs=((prev, 0),), output_shapes=(act(ch[i]),)))
        nodes.append(OpNode(f"relu_{i:02d}", "Relu", "gpu0", inputs=((f"conv_{i:02d}", 0),),
                            output_shapes=(act(ch[i]),)))
        prev = f"relu_{i:02d}"
    k_dim = hw * hw * ch[-1]
    nodes.append(OpNode("fc", "MatMul", "gpu0", attrs={"m": batch, "k": k_dim, "n": 10}, inputs=((prev, 0),),
                        output_shapes=(TensorShape((batch, 10), 4),)))
    nodes.append(OpNode("loss", "SoftmaxLoss", "gpu0", inputs=(("fc", 0),), output_shapes=(TensorShape((1,), 4),)))
    nodes.append(OpNode("dfc", "MatMulGrad", "gpu0", attrs={"m": batch, "k": k_dim, "n": 10},
                        inputs=(("loss", 0),), output_shapes=(act(ch[-1]),)))
    up = "dfc"
    for i in reversed(range(layers)):
        wshape = TensorShape((kernel, kernel, cin[i], ch[i]), 4)
        ga = {"in_channels": cin[i], "out_channels": ch[i], "kernel": kernel}
        nodes.append(OpNode(f"grad_conv_{i:02d}", "Conv2DBackpropFilter", "gpu0", attrs=dict(ga),
                            inputs=((up, 0),), output_shapes=(wshape,)))
        nodes.append(OpNode(f"bwd_{i:02d}", "Conv2DBackpropInput", "gpu0", attrs=dict(ga), inputs=((up, 0),),
                            output_shapes=(act(cin[i]),)))
        nodes.append(OpNode(f"apply_conv_{i:02d}", "ApplyGradientDescent", "gpu0",
                            inputs=((f"grad_conv_{i:02d}", 0),), output_shapes=(wshape,)))
        up = f"bwd_{i:02d}"
    return make_graph(nodes, _gpus(1), {"model": f"layered-cnn-{layers}", "batch": batch})


def random_dag(nodes: int, density: float, seed: int = 0, num_devices: int = 1):
    """RandomDAG of synth.py:345-367 (O(N^2) RNG draws; fixtures only)."""
    rng = SplitMix64(seed)
    shape = TensorShape((16, 16), 4)
    width = max(4, len(str(nodes - 1)))
    ids = [f"node_{i:0{width}d}" for i in range(nodes)]
    out = []
    for j in range(nodes):
        ins = tuple((ids[i], 0) for i in range(j) if rng.uniform() < density)
        dev = f"gpu{rng.randint(0, num_devices - 1)}"
        out.append(OpNode(ids[j], RANDOM_OPS[j % 4], dev, attrs={"cost_hint": rng.randint(1, 16)}, inputs=ins,
                          output_shapes=(shape,)))
    return make_graph(out, _gpus(num_devices), {"model": f"random-dag-{nodes}", "seed": seed})


def planted_profiles(laws: dict, hardware: str = "synth-hw", grid=DEFAULT_GRID, links=SYNTH_LINKS) -> ProfileDB:
    """gen_profiles of synth.py:373-407: one record per grid point of each law."""
    db = ProfileDB(hardware_tags=[hardware], provenance="synthetic laws")
    for link in links:
        db_insert(db, link)
    for op in sorted(laws):
        feat, slope, icpt = laws[op]
        pts = [((), icpt)] if feat is None else [(((feat, x),), slope * x + icpt) for x in grid]
        for feats, mean in pts:
            db_insert(db, ProfileRecord(OpSignature(op, hardware, feats), mean, 0.0, 1000))
    return db


def chain_laws():
    return {op: ("cost_hint", 10.0, 5.0) for op in CHAIN_OPS}


def random_laws():
    return {op: ("cost_hint", 10.0, 5.0) for op in RANDOM_OPS}

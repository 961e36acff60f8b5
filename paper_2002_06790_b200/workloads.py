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


# ----------------------------------------------------------------------------- model graphs
#
# Training graphs in the LayeredCNN style (forward ops, backward data/weight
# gradients, one ApplyGradientDescent per parameter tensor; every parameter
# gradient is named grad_* so `gradient_markers=("dgrad_*",)` selects them).
# Shapes are NHWC activations; each compute node carries an `mflops` attribute
# that the planted cost laws key on, so durations scale with batch size.

NVLINK5_UNI_MBPS = 900e9 / 2 ** 20      # 900 GB/s per direction, read as MiB (costmodel.py:34)
SYNTH_FABRIC_LINKS = (
    # synthetic rows (not measurements): NVLink 5 / NVSwitch and 400 Gb/s RDMA
    LinkRecord("gpu-gpu-uni", "NVLink", 2, NVLINK5_UNI_MBPS, 1.5),
    LinkRecord("nccl-allreduce", "NVLink", 8, 0.8 * NVLINK5_UNI_MBPS, 0.0),
    LinkRecord("gpu-gpu-uni", "RDMA", 2, 50e9 / 2 ** 20, 5.0),
    LinkRecord("nccl-allreduce", "RDMA", 8, 0.7 * 50e9 / 2 ** 20, 0.0),
)


class _Builder:
    def __init__(self, batch: int, device: str = "gpu0"):
        self.batch, self.device = batch, device
        self.nodes: list[OpNode] = []
        self.shape: dict[str, TensorShape] = {}
        self.params: list[tuple[str, str, TensorShape]] = []  # (grad node, apply node, shape)

    def add(self, nid, op, inputs, shape, mflops, **attrs):
        attrs = dict(attrs)
        attrs["mflops"] = round(float(mflops), 6)
        self.nodes.append(OpNode(nid, op, self.device, attrs=attrs, inputs=tuple((p, 0) for p in inputs),
                                 output_shapes=(shape,)))
        self.shape[nid] = shape
        return nid

    def act(self, h, w, c):
        return TensorShape((self.batch, h, w, c), 4)


def resnet50_training(batch: int = 32, image: int = 224, classes: int = 1000):
    """ResNet-50 v1.5 training step: 176 forward, ~230 backward, 107 update nodes."""
    b = _Builder(batch)
    B = batch
    fwd = []  # (kind, node, meta) in forward order for the backward pass

    def conv(nid, x, cin, cout, k, stride, h):
        ho = (h + stride - 1) // stride
        fl = 2.0 * B * ho * ho * cout * cin * k * k / 1e6
        b.add(nid, "Conv2D", [x], b.act(ho, ho, cout), fl, batch=B, in_channels=cin, out_channels=cout,
              kernel=k, stride=stride)
        fwd.append(("conv", nid, (x, cin, cout, k, stride, h, ho)))
        return nid, ho

    def bn(nid, x, c, h):
        b.add(nid, "FusedBatchNorm", [x], b.act(h, h, c), 8.0 * B * h * h * c / 1e6, channels=c)
        fwd.append(("bn", nid, (x, c, h)))
        return nid

    def relu(nid, x, c, h):
        b.add(nid, "Relu", [x], b.act(h, h, c), 1.0 * B * h * h * c / 1e6)
        fwd.append(("relu", nid, (x, c, h)))
        return nid

    x = b.add("input", "Input", [], b.act(image, image, 3), 0.0)
    x, h = conv("conv1", x, 3, 64, 7, 2, image)
    x = relu("conv1_relu", bn("conv1_bn", x, 64, h), 64, h)
    h2 = (h + 1) // 2
    fwd.append(("pool", "pool1", (x, 64, h)))
    x = b.add("pool1", "MaxPool", [x], b.act(h2, h2, 64), 9.0 * B * h2 * h2 * 64 / 1e6, kernel=3, stride=2)
    h, cin = h2, 64
    for s, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for blk in range(blocks):
            p = f"l{s + 1}_b{blk}"
            stride = 2 if (blk == 0 and s > 0) else 1
            block_in, hin = x, h
            y, h1 = conv(f"{p}_conv1", x, cin, width, 1, 1, h)
            y = relu(f"{p}_relu1", bn(f"{p}_bn1", y, width, h1), width, h1)
            y, h2 = conv(f"{p}_conv2", y, width, width, 3, stride, h1)
            y = relu(f"{p}_relu2", bn(f"{p}_bn2", y, width, h2), width, h2)
            y, h3 = conv(f"{p}_conv3", y, width, 4 * width, 1, 1, h2)
            y = bn(f"{p}_bn3", y, 4 * width, h3)
            sc = block_in
            if blk == 0:
                sc, _ = conv(f"{p}_down", block_in, cin, 4 * width, 1, stride, hin)
                sc = bn(f"{p}_down_bn", sc, 4 * width, h3)
            add = b.add(f"{p}_add", "Add", [y, sc], b.act(h3, h3, 4 * width), 1.0 * B * h3 * h3 * 4 * width / 1e6)
            fwd.append(("add", add, (y, sc, block_in)))
            x = relu(f"{p}_out", add, 4 * width, h3)
            h, cin = h3, 4 * width
    pool = b.add("avgpool", "AvgPool", [x], TensorShape((B, cin), 4), 1.0 * B * h * h * cin / 1e6)
    fc = b.add("fc", "MatMul", [pool], TensorShape((B, classes), 4), 2.0 * B * cin * classes / 1e6,
               m=B, k=cin, n=classes)
    loss = b.add("loss", "SoftmaxLoss", [fc], TensorShape((1,), 4), 5.0 * B * classes / 1e6)
    _backward(b, fwd, pool, fc, loss, cin, classes)
    return make_graph(b.nodes, _gpus(1), {"model": "resnet50", "batch": batch})


def _backward(b: _Builder, fwd, pool, fc, loss, feat, classes):
    """Reverse-mode graph: data grads flow backwards; weight grads feed their updates."""
    B = b.batch
    dl = b.add("dgrad_loss_in", "SoftmaxLossGrad", [loss, fc], b.shape[fc], 5.0 * B * classes / 1e6)
    gw = b.add("wgrad_fc", "MatMulGradFilter", [dl, pool], TensorShape((feat, classes), 4),
               2.0 * B * feat * classes / 1e6, m=B, k=feat, n=classes)
    b.params.append((gw, "apply_fc", b.shape[gw]))
    dx = b.add("dgrad_fc_in", "MatMulGradInput", [dl], b.shape[pool], 2.0 * B * feat * classes / 1e6,
               m=B, k=feat, n=classes)
    last = fwd[-1][1]
    hh = b.shape[last].dims[1]
    grad_of = {last: b.add("dgrad_avgpool", "AvgPoolGrad", [dx], b.shape[last], 1.0 * B * hh * hh * feat / 1e6)}
    pending: dict[str, list[str]] = {}   # activation -> gradient contributions (summed by AddN)

    def contribute(act, g):
        pending.setdefault(act, []).append(g)

    def grad_for(node):
        if node in grad_of:
            return grad_of[node]
        parts = pending.pop(node)
        if len(parts) == 1:
            grad_of[node] = parts[0]
        else:
            s = b.shape[node]
            grad_of[node] = b.add(f"dgrad_{node}_sum", "AddN", parts, s, float(len(parts)) * s.num_elements() / 1e6)
        return grad_of[node]

    for kind, nid, meta in reversed(fwd):
        if nid not in grad_of and nid not in pending:
            continue  # output not on the gradient path
        g = grad_for(nid)
        if kind == "relu":
            x, c, h = meta
            contribute(x, b.add(f"dgrad_{nid}_in", "ReluGrad", [g, nid], b.shape[x], 1.0 * B * h * h * c / 1e6))
        elif kind == "bn":
            x, c, h = meta
            gp = b.add(f"wgrad_{nid}", "FusedBatchNormGradParams", [g, x], TensorShape((2, c), 4),
                       4.0 * B * h * h * c / 1e6, channels=c)
            b.params.append((gp, f"apply_{nid}", b.shape[gp]))
            contribute(x, b.add(f"dgrad_{nid}_in", "FusedBatchNormGrad", [g, x, gp], b.shape[x],
                                8.0 * B * h * h * c / 1e6, channels=c))
        elif kind == "conv":
            x, cin, cout, k, stride, h, ho = meta
            fl = 2.0 * B * ho * ho * cout * cin * k * k / 1e6
            gw = b.add(f"wgrad_{nid}", "Conv2DBackpropFilter", [g, x], TensorShape((k, k, cin, cout), 4), fl,
                       batch=B, in_channels=cin, out_channels=cout, kernel=k, stride=stride)
            b.params.append((gw, f"apply_{nid}", b.shape[gw]))
            if x != "input":
                contribute(x, b.add(f"dgrad_{nid}_in", "Conv2DBackpropInput", [g], b.shape[x], fl, batch=B,
                                    in_channels=cin, out_channels=cout, kernel=k, stride=stride))
        elif kind == "pool":
            x, c, h = meta
            contribute(x, b.add(f"dgrad_{nid}_in", "MaxPoolGrad", [g, x], b.shape[x], 9.0 * B * h * h * c / 1e6))
        elif kind == "add":
            y, sc, _ = meta
            contribute(y, g)
            contribute(sc, g)
    for gnode, apply_id, shape in b.params:
        b.add(apply_id, "ApplyGradientDescent", [gnode], shape, 3.0 * shape.num_elements() / 1e6)


def vgg16_training(batch: int = 32, image: int = 224, classes: int = 1000):
    """VGG-16 training step (13 conv + 3 fc layers; 16 weight gradients)."""
    b = _Builder(batch)
    B = batch
    fwd = []
    x = b.add("input", "Input", [], b.act(image, image, 3), 0.0)
    h, cin = image, 3
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    li = 0
    for item in cfg:
        if item == "M":
            ho = h // 2
            nid = b.add(f"pool{li}", "MaxPool", [x], b.act(ho, ho, cin), 4.0 * B * ho * ho * cin / 1e6,
                        kernel=2, stride=2)
            fwd.append(("pool", nid, (x, cin, h)))
            x, h = nid, ho
            continue
        li += 1
        fl = 2.0 * B * h * h * item * cin * 9 / 1e6
        c = b.add(f"conv{li}", "Conv2D", [x], b.act(h, h, item), fl, batch=B, in_channels=cin, out_channels=item,
                  kernel=3, stride=1)
        fwd.append(("conv", c, (x, cin, item, 3, 1, h, h)))
        r = b.add(f"conv{li}_relu", "Relu", [c], b.act(h, h, item), 1.0 * B * h * h * item / 1e6)
        fwd.append(("relu", r, (c, item, h)))
        x, cin = r, item
    flat = b.add("flatten", "Reshape", [x], TensorShape((B, h * h * cin), 4), 0.01)
    fwd.append(("flat", flat, (x,)))
    feat, x = h * h * cin, flat
    for i, n_out in enumerate((4096, 4096)):
        f = b.add(f"fc{i + 1}", "MatMul", [x], TensorShape((B, n_out), 4), 2.0 * B * feat * n_out / 1e6,
                  m=B, k=feat, n=n_out)
        fwd.append(("fc", f, (x, feat, n_out)))
        r = b.add(f"fc{i + 1}_relu", "Relu", [f], TensorShape((B, n_out), 4), 1.0 * B * n_out / 1e6)
        fwd.append(("relu", r, (f, n_out, 1)))
        x, feat = r, n_out
    fc = b.add("fc3", "MatMul", [x], TensorShape((B, classes), 4), 2.0 * B * feat * classes / 1e6,
               m=B, k=feat, n=classes)
    loss = b.add("loss", "SoftmaxLoss", [fc], TensorShape((1,), 4), 5.0 * B * classes / 1e6)
    # backward
    dl = b.add("dgrad_loss_in", "SoftmaxLossGrad", [loss, fc], b.shape[fc], 5.0 * B * classes / 1e6)
    gw = b.add("wgrad_fc3", "MatMulGradFilter", [dl, x], TensorShape((feat, classes), 4),
               2.0 * B * feat * classes / 1e6, m=B, k=feat, n=classes)
    b.params.append((gw, "apply_fc3", b.shape[gw]))
    g = b.add("dgrad_fc3_in", "MatMulGradInput", [dl], b.shape[x], 2.0 * B * feat * classes / 1e6,
              m=B, k=feat, n=classes)
    for kind, nid, meta in reversed(fwd):
        if kind == "relu":
            src, c, hh = meta
            g = b.add(f"dgrad_{nid}_in", "ReluGrad", [g, nid], b.shape[src], 1.0 * B * hh * hh * c / 1e6)
        elif kind == "fc":
            src, fin, fout = meta
            fl = 2.0 * B * fin * fout / 1e6
            gw = b.add(f"wgrad_{nid}", "MatMulGradFilter", [g, src], TensorShape((fin, fout), 4), fl,
                       m=B, k=fin, n=fout)
            b.params.append((gw, f"apply_{nid}", b.shape[gw]))
            g = b.add(f"dgrad_{nid}_in", "MatMulGradInput", [g], b.shape[src], fl, m=B, k=fin, n=fout)
        elif kind == "flat":
            g = b.add("dgrad_flatten_in", "Reshape", [g], b.shape[meta[0]], 0.01)
        elif kind == "pool":
            src, c, hh = meta
            g = b.add(f"dgrad_{nid}_in", "MaxPoolGrad", [g, src], b.shape[src], 4.0 * B * hh * hh * c / 1e6)
        elif kind == "conv":
            src, ci, co, k, st, hh, ho = meta
            fl = 2.0 * B * ho * ho * co * ci * k * k / 1e6
            gw = b.add(f"wgrad_{nid}", "Conv2DBackpropFilter", [g, src], TensorShape((k, k, ci, co), 4), fl,
                       batch=B, in_channels=ci, out_channels=co, kernel=k, stride=st)
            b.params.append((gw, f"apply_{nid}", b.shape[gw]))
            if src != "input":
                g = b.add(f"dgrad_{nid}_in", "Conv2DBackpropInput", [g], b.shape[src], fl, batch=B,
                          in_channels=ci, out_channels=co, kernel=k, stride=st)
    for gnode, apply_id, shape in b.params:
        b.add(apply_id, "ApplyGradientDescent", [gnode], shape, 3.0 * shape.num_elements() / 1e6)
    return make_graph(b.nodes, _gpus(1), {"model": "vgg16", "batch": batch})


def bert_large_training(batch: int = 8, seq: int = 512, layers: int = 24, hidden: int = 1024, heads: int = 16,
                        vocab: int = 30522):
    """BERT-large training step from a per-layer template (8 weight matrices + 2 LayerNorms per layer)."""
    b = _Builder(batch)
    B, T, Hd = batch, seq, hidden
    act = TensorShape((B, T, Hd), 4)
    mm = lambda m, k, n: 2.0 * m * k * n / 1e6  # noqa: E731
    x = b.add("input", "Input", [], TensorShape((B, T), 4), 0.0)
    x = b.add("embed", "Gather", [x], act, B * T * Hd / 1e6, vocab=vocab, hidden=Hd)
    saved = []
    for l in range(layers):
        p = f"layer{l:02d}"
        q = b.add(f"{p}_qkv", "MatMul", [x], TensorShape((B, T, 3 * Hd), 4), mm(B * T, Hd, 3 * Hd), m=B * T, k=Hd,
                  n=3 * Hd)
        s = b.add(f"{p}_scores", "BatchMatMul", [q], TensorShape((B, heads, T, T), 4), mm(B * heads * T, Hd // heads, T),
                  m=B * heads * T, k=Hd // heads, n=T)
        sm = b.add(f"{p}_softmax", "Softmax", [s], b.shape[s], 5.0 * B * heads * T * T / 1e6)
        ctxv = b.add(f"{p}_context", "BatchMatMul", [sm, q], act, mm(B * heads * T, T, Hd // heads),
                     m=B * heads * T, k=T, n=Hd // heads)
        o = b.add(f"{p}_attn_out", "MatMul", [ctxv], act, mm(B * T, Hd, Hd), m=B * T, k=Hd, n=Hd)
        a1 = b.add(f"{p}_add1", "Add", [o, x], act, B * T * Hd / 1e6)
        n1 = b.add(f"{p}_ln1", "LayerNorm", [a1], act, 8.0 * B * T * Hd / 1e6, hidden=Hd)
        f1 = b.add(f"{p}_ffn1", "MatMul", [n1], TensorShape((B, T, 4 * Hd), 4), mm(B * T, Hd, 4 * Hd), m=B * T,
                   k=Hd, n=4 * Hd)
        ge = b.add(f"{p}_gelu", "Gelu", [f1], b.shape[f1], 8.0 * B * T * 4 * Hd / 1e6)
        f2 = b.add(f"{p}_ffn2", "MatMul", [ge], act, mm(B * T, 4 * Hd, Hd), m=B * T, k=4 * Hd, n=Hd)
        a2 = b.add(f"{p}_add2", "Add", [f2, n1], act, B * T * Hd / 1e6)
        x = b.add(f"{p}_ln2", "LayerNorm", [a2], act, 8.0 * B * T * Hd / 1e6, hidden=Hd)
        saved.append((p, q, sm, ctxv, n1, ge, f1))
    pooled = b.add("pooler", "MatMul", [x], TensorShape((B, Hd), 4), mm(B, Hd, Hd), m=B, k=Hd, n=Hd)
    loss = b.add("loss", "SoftmaxLoss", [pooled], TensorShape((1,), 4), 5.0 * B * Hd / 1e6)
    g = b.add("dgrad_loss_in", "SoftmaxLossGrad", [loss], b.shape[pooled], 5.0 * B * Hd / 1e6)
    gw = b.add("wgrad_pooler", "MatMulGradFilter", [g, x], TensorShape((Hd, Hd), 4), mm(B, Hd, Hd), m=B, k=Hd, n=Hd)
    b.params.append((gw, "apply_pooler", b.shape[gw]))
    g = b.add("dgrad_pooler_in", "MatMulGradInput", [g], act, mm(B, Hd, Hd), m=B, k=Hd, n=Hd)
    prev_out = x
    for p, q, sm, ctxv, n1, ge, f1 in reversed(saved):
        gl2 = b.add(f"wgrad_{p}_ln2", "LayerNormGradParams", [g, prev_out], TensorShape((2, Hd), 4),
                    4.0 * B * T * Hd / 1e6, hidden=Hd)
        b.params.append((gl2, f"apply_{p}_ln2", b.shape[gl2]))
        g2 = b.add(f"dgrad_{p}_ln2_in", "LayerNormGrad", [g, gl2], act, 8.0 * B * T * Hd / 1e6, hidden=Hd)
        for name, src, k_, n_ in (("ffn2", ge, 4 * Hd, Hd),):
            gw = b.add(f"wgrad_{p}_{name}", "MatMulGradFilter", [g2, src], TensorShape((k_, n_), 4),
                       mm(B * T, k_, n_), m=B * T, k=k_, n=n_)
            b.params.append((gw, f"apply_{p}_{name}", b.shape[gw]))
        gge = b.add(f"dgrad_{p}_ffn2_in", "MatMulGradInput", [g2], b.shape[ge], mm(B * T, 4 * Hd, Hd), m=B * T,
                    k=4 * Hd, n=Hd)
        gf1 = b.add(f"dgrad_{p}_gelu_in", "GeluGrad", [gge, f1], b.shape[f1], 8.0 * B * T * 4 * Hd / 1e6)
        gw = b.add(f"wgrad_{p}_ffn1", "MatMulGradFilter", [gf1, n1], TensorShape((Hd, 4 * Hd), 4),
                   mm(B * T, Hd, 4 * Hd), m=B * T, k=Hd, n=4 * Hd)
        b.params.append((gw, f"apply_{p}_ffn1", b.shape[gw]))
        gn1 = b.add(f"dgrad_{p}_ffn1_in", "MatMulGradInput", [gf1], act, mm(B * T, Hd, 4 * Hd), m=B * T, k=Hd,
                    n=4 * Hd)
        s1 = b.add(f"dgrad_{p}_n1_sum", "AddN", [gn1, g2], act, 2.0 * B * T * Hd / 1e6)
        gl1 = b.add(f"wgrad_{p}_ln1", "LayerNormGradParams", [s1, n1], TensorShape((2, Hd), 4),
                    4.0 * B * T * Hd / 1e6, hidden=Hd)
        b.params.append((gl1, f"apply_{p}_ln1", b.shape[gl1]))
        ga1 = b.add(f"dgrad_{p}_ln1_in", "LayerNormGrad", [s1, gl1], act, 8.0 * B * T * Hd / 1e6, hidden=Hd)
        gw = b.add(f"wgrad_{p}_attn_out", "MatMulGradFilter", [ga1, ctxv], TensorShape((Hd, Hd), 4),
                   mm(B * T, Hd, Hd), m=B * T, k=Hd, n=Hd)
        b.params.append((gw, f"apply_{p}_attn_out", b.shape[gw]))
        gc = b.add(f"dgrad_{p}_attn_out_in", "MatMulGradInput", [ga1], act, mm(B * T, Hd, Hd), m=B * T, k=Hd, n=Hd)
        gsm = b.add(f"dgrad_{p}_context_in", "BatchMatMulGrad", [gc, q], b.shape[sm], mm(B * heads * T, T, Hd // heads),
                    m=B * heads * T, k=T, n=Hd // heads)
        gs = b.add(f"dgrad_{p}_softmax_in", "SoftmaxGrad", [gsm, sm], b.shape[sm], 5.0 * B * heads * T * T / 1e6)
        gq = b.add(f"dgrad_{p}_scores_in", "BatchMatMulGrad", [gs, q], b.shape[q],
                   mm(B * heads * T, Hd // heads, T), m=B * heads * T, k=Hd // heads, n=T)
        gw = b.add(f"wgrad_{p}_qkv", "MatMulGradFilter", [gq], TensorShape((Hd, 3 * Hd), 4), mm(B * T, Hd, 3 * Hd),
                   m=B * T, k=Hd, n=3 * Hd)
        b.params.append((gw, f"apply_{p}_qkv", b.shape[gw]))
        gx = b.add(f"dgrad_{p}_qkv_in", "MatMulGradInput", [gq], act, mm(B * T, Hd, 3 * Hd), m=B * T, k=Hd, n=3 * Hd)
        g = b.add(f"dgrad_{p}_in_sum", "AddN", [gx, ga1], act, 2.0 * B * T * Hd / 1e6)
        prev_out = n1
    gw = b.add("wgrad_embed", "GatherGrad", [g], TensorShape((vocab, Hd), 4), B * T * Hd / 1e6, vocab=vocab,
               hidden=Hd)
    b.params.append((gw, "apply_embed", b.shape[gw]))
    for gnode, apply_id, shape in b.params:
        b.add(apply_id, "ApplyGradientDescent", [gnode], shape, 3.0 * shape.num_elements() / 1e6)
    return make_graph(b.nodes, _gpus(1), {"model": "bert-large", "batch": batch, "seq": seq})


def model_profiles(graph, hardware_tags, seed: int = 1, grid_points: int = 16, links=SYNTH_FABRIC_LINKS + SYNTH_LINKS):
    """Planted offline-profiling DB for every op type of ``graph`` on every hardware tag.

    Each (op, hw) gets a 16-point grid over `mflops` with a planted linear law
    (hw-specific throughput and launch overhead, small deterministic noise so the
    OLS coefficients are non-trivial doubles); ops without `mflops` get one
    zero-feature exact record.  MatMul additionally gets a 2-feature (k, m) grid
    of 24 points so predict's multi-term compensated sum is exercised.
    """
    rng = SplitMix64(seed)
    db = ProfileDB(hardware_tags=list(hardware_tags), provenance="synthetic planted laws (not measurements)")
    for link in links:
        db_insert(db, link)
    ops = sorted({n.op_type for n in graph.nodes.values()} | {"PSAggregate"})  # PS aggregation (ps.py)
    for h, hw in enumerate(hardware_tags):
        speed = 1.0 + 0.37 * h            # tflops-ish scale per hardware generation
        for op in ops:
            icpt = 3.0 + 7.0 * rng.uniform() + 0.25 * h
            slope = (0.0008 + 0.004 * rng.uniform()) / speed
            lo, hi = 0.01, 2.0e5
            for i in range(grid_points):
                x = lo * (hi / lo) ** (i / (grid_points - 1))
                x = float(f"{x:.6g}")
                noise = 1.0 + 0.002 * (rng.uniform() - 0.5)
                db_insert(db, ProfileRecord(OpSignature(op, hw, (("mflops", x),)), (slope * x + icpt) * noise))
            if op == "MatMul":
                for i in range(24):
                    k, m = float(rng.randint(64, 8192)), float(rng.randint(1, 4096))
                    mean = (2e-6 * k * m * 0.5 / speed + 0.01 * k / speed + 0.002 * m + icpt)
                    db_insert(db, ProfileRecord(OpSignature(op, hw, (("k", k), ("m", m))), mean))
        db_insert(db, ProfileRecord(OpSignature("Input", hw, (("mflops", 0.0),)), 4.0 + h))
    return db


def layered_dag(nodes: int = 1_000_000, width: int = 1000, devices: int = 8, seed: int = 5, max_fanin: int = 3):
    """O(E) layered DAG for config C5: ``nodes / width`` layers; each node of layer l > 0 reads
    1..max_fanin distinct producers of layer l-1 (SplitMix64-seeded); node j of a layer runs on
    gpu (j % devices).  Ids are zero-padded so rank order == creation order."""
    rng = SplitMix64(seed)
    shape = TensorShape((16, 16), 4)
    digits = len(str(nodes - 1))
    ids = [f"n{i:0{digits}d}" for i in range(nodes)]
    out = []
    for i in range(nodes):
        layer, j = divmod(i, width)
        ins = ()
        if layer:
            base = (layer - 1) * width
            k = 1 + rng.next_u64() % max_fanin
            picks = sorted({base + (rng.next_u64() % width) for _ in range(k)})
            ins = tuple((ids[p], 0) for p in picks)
        out.append(OpNode(ids[i], RANDOM_OPS[i % 4], f"gpu{j % devices}",
                          attrs={"cost_hint": 1 + rng.next_u64() % 16}, inputs=ins, output_shapes=(shape,)))
    return make_graph(out, _gpus(devices), {"model": f"layered-dag-{nodes}", "seed": seed})


def dag_profiles(hardware_tags, seed: int = 3):
    """Planted cost_hint laws per (op, hardware tag): each tag its own slope/intercept set."""
    rng = SplitMix64(seed)
    db = ProfileDB(hardware_tags=list(hardware_tags), provenance="synthetic planted laws (not measurements)")
    for hw in hardware_tags:
        for op in RANDOM_OPS:
            slope, icpt = 2.0 + 10.0 * rng.uniform(), 1.0 + 5.0 * rng.uniform()
            for x in DEFAULT_GRID:
                db_insert(db, ProfileRecord(OpSignature(op, hw, (("cost_hint", x),)), slope * x + icpt))
    return db

"""Drop-in ``estimate_all`` (costmodel.py:282-331) and its batched form.

The host lowers the profile DB once (lowering.LoweredProfiles: feature-vector
interning, exact-record keys, numpy-fitted models, link rows, resolved
overrides); the per-(strategy, node) fallback chain runs in the sm_100a kernel
``dfsim_estimate_batch`` (csrc/estimate.cu).
"""

from __future__ import annotations

import numpy as np

from . import native
from .errors import UnknownOpError
from .lowering import LoweredProfiles
from .model import SOURCE_TAGS, DurationEntry, DurationTable

SRC_BAD_BYTES, SRC_NEGATIVE, SRC_UNKNOWN = 253, 254, 255


def estimate_batch(lp: LoweredProfiles, n_nodes: int, out=None) -> dict:
    """K2 over every strategy of ``lp``: dur [S, N] f64, src [S, N] u8, bad [S] i32 (device)."""
    import torch

    dev = f"cuda:{lp.device}"
    S = lp.n_sims
    o = out if out is not None else {}
    o.setdefault("dur", torch.empty((S, max(n_nodes, 1)), dtype=torch.float64, device=dev))
    o.setdefault("src", torch.empty((S, max(n_nodes, 1)), dtype=torch.uint8, device=dev))
    o.setdefault("bad", torch.empty(S, dtype=torch.int32, device=dev))
    ctx = native.Context.get(lp.device)
    ctx.call("dfsim_estimate_batch", n_nodes, native.ctypes.byref(lp.struct), native.ctypes.byref(lp.strategies),
             native.ptr(o["dur"]), native.ptr(o["src"]), native.ptr(o["bad"]))
    return o


def raise_for_row(g, ids, dur_row: np.ndarray, src_row: np.ndarray):
    """The reference's error for one strategy: the first ValueError in id order
    (transfer_time bytes check, costmodel.py:180-181; DurationEntry, 78-80),
    else UnknownOpError over every unresolved node (costmodel.py:327-330)."""
    bad = np.nonzero(src_row >= SRC_BAD_BYTES)[0]
    values = np.nonzero((src_row == SRC_BAD_BYTES) | (src_row == SRC_NEGATIVE))[0]
    if len(values):
        i = int(values[0])
        nid = ids[i]
        if src_row[i] == SRC_BAD_BYTES:
            raise ValueError(f"bytes must be > 0, got {g.nodes[nid].attrs.get('bytes')}")
        raise ValueError(f"durations are nonnegative microseconds, got {float(dur_row[i])}")
    if len(bad):
        raise UnknownOpError({ids[i]: g.nodes[ids[i]].op_type for i in bad.tolist()})


def estimate_all(g, db, cfg, device: int | None = None) -> DurationTable:
    """Resolve a duration for every node or raise UnknownOpError (costmodel.py:282-331)."""
    ctx = native.Context.get(device)
    ids = sorted(g.nodes)
    lp = LoweredProfiles(g, ids, db, [cfg], ctx.device)
    if not ids:
        return DurationTable(entries={})
    o = estimate_batch(lp, len(ids))
    dur = o["dur"][0].cpu().numpy()
    src = o["src"][0].cpu().numpy()
    if int(o["bad"][0].item()):
        raise_for_row(g, ids, dur, src)
    return DurationTable(entries={nid: DurationEntry(float(dur[i]), SOURCE_TAGS[src[i]])
                                  for i, nid in enumerate(ids)})

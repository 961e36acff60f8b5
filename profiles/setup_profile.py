"""Host setup (class construction) profile of the bench workloads: the one-shot
``sweep_variants`` call with the graphs' caches dropped (as bench.py's e2e_cold), after two
warm-up calls (library, context and the CUDA caching allocator warm); wall time per workload,
then the top cProfile entries by own time.  python profiles/setup_profile.py [workload ...]"""

from __future__ import annotations

import cProfile
import io
import pstats
import sys
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CACHES = ("_dfsim_b200_lowered", "_dfsim_base_rows", "_dfsim_base_arr", "_dfsim_grad_keys")


def _drop(graphs):
    for g in graphs:
        for k in CACHES:
            g.__dict__.pop(k, None)


def main(names):
    import torch

    import bench
    from paper_2002_06790_b200 import sweep_variants

    torch.cuda.init()
    for wl in names:
        graphs, db, configs, graph_of = bench.build_workload(0, bench.WORKLOADS[wl][1], wl)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            walls = []
            for _ in range(3):
                _drop(graphs)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = sweep_variants(graphs, db, configs, graph_of)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            _drop(graphs)
            pr = cProfile.Profile()
            pr.enable()
            sweep_variants(graphs, db, configs, graph_of)
            torch.cuda.synchronize()
            pr.disable()
        out = io.StringIO()
        pstats.Stats(pr, stream=out).sort_stats("tottime").print_stats(30)
        print(f"== {wl}: one-shot sweep_variants {[round(w, 3) for w in walls]} s for {len(configs)} candidates "
              f"({len(res.classes)} classes, best {res.best_index})")
        print(out.getvalue())


if __name__ == "__main__":
    main(sys.argv[1:] or ["resnet50-dp8", "bert-large-ps-ar", "vgg16-sweep"])

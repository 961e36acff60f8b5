"""Host setup (class construction) profile of the bench workloads: wall time per workload and
the top cProfile entries.  python profiles/setup_profile.py [workload ...]"""

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


def main(names):
    import torch

    import bench
    from paper_2002_06790_b200 import sweep_variants

    torch.cuda.init()
    for wl in names:
        graphs, db, configs, graph_of = bench.build_workload(0, bench.WORKLOADS[wl][1], wl)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sweep_variants(graphs, db, configs[:8], graph_of[:8])  # warm the library / context
            torch.cuda.synchronize()
            pr = cProfile.Profile()
            t0 = time.perf_counter()
            pr.enable()
            res = sweep_variants(graphs, db, configs, graph_of)
            pr.disable()
            wall = time.perf_counter() - t0
        out = io.StringIO()
        pstats.Stats(pr, stream=out).sort_stats("cumulative").print_stats(45)
        print(f"== {wl}: cold sweep_variants {wall:.3f} s for {len(configs)} candidates "
              f"({len(res.classes)} classes, best {res.best_index})")
        print(out.getvalue())


if __name__ == "__main__":
    main(sys.argv[1:] or ["resnet50-dp8", "bert-large-ps-ar", "vgg16-sweep"])

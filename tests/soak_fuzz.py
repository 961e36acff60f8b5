"""GPU soak: random DAGs x random strategy lists (plain / allreduce / parameter server, both
algorithms, overrides with ties and zeros, 1-40 devices) through sweep(), each candidate checked
bit-for-bit against the oracle; errors must agree.  Not collected by pytest.

    python tests/soak_fuzz.py <seconds> [first_seed]
"""
import sys, time, warnings, traceback
sys.path.insert(0, '.')
import numpy as np
import paper_2002_06790_b200 as fw
from oracle import dfsim_oracle as O
from paper_2002_06790_b200 import workloads as W
from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig
from paper_2002_06790_b200.ps import expand_parameter_server
t_end = time.time() + float(sys.argv[1])
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n_ok = 0
while time.time() < t_end:
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 300))
    nd = int(rng.integers(1, 40))
    g = W.random_dag(n, float(rng.uniform(0.0, 0.15)), seed=seed, num_devices=nd)
    db = W.dag_profiles(["hwA", "hwB"])
    for link in W.SYNTH_LINKS:
        W.db_insert(db, link)
    ids = sorted(g.nodes)
    cfgs = []
    for i in range(int(rng.integers(1, 40))):
        kind = int(rng.integers(0, 3))
        ov = {}
        if rng.random() < 0.3:
            for nid in rng.choice(ids, size=min(int(rng.integers(1, 6)), n), replace=False).tolist():
                ov[nid] = float(rng.choice([0.0, 1.0, 2.5]))
        if rng.random() < 0.2:
            ov[ids[int(rng.integers(0, n))][:7] + "*"] = float(rng.choice([0.0, 3.0]))
        kw = dict(hardware=("hwA", "hwB")[int(rng.integers(0, 2))], op_gap_us=float(rng.choice([0.0, 0.125, 0.3, 1e-3 * i])), overrides=ov)
        if kind:
            R = int(rng.integers(2, 9))
            kw.update(replicas=R, device_map=tuple(f"gpu{k}" for k in range(R)),
                      collective=CollectiveConfig(("RingAnalytic", "MeasuredThroughput")[int(rng.integers(0, 2))], "PCIeSwitch"),
                      gradient_markers=(ids[int(rng.integers(0, n))][:int(rng.integers(5, 10))] + "*",), sync=("allreduce", "parameter_server")[kind - 1])
            if kind == 2:
                kw["overrides"] = dict(kw["overrides"], **{"aggregate_*": 1.25})
        cfgs.append(StrategyConfig(**kw))
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                res = fw.sweep(g, db, cfgs, keep_schedules=True)
                err = None
            except Exception as e:
                res, err = None, e
            for i, cfg in enumerate(cfgs):
                try:
                    if getattr(cfg, "sync", "allreduce") == "parameter_server":
                        gx = expand_parameter_server(g, cfg, db).graph
                        table = O.estimate(gx, db, cfg)
                        entries, ms, _ = O.simulate(gx, {k: v for k, (v, _) in table.items()})
                        cp = O.critical_path(gx, {nid: f - s for nid, _, s, f in entries})[0]
                    else:
                        ms, cp, entries, _, _ = O.run_candidate(g, db, cfg)
                    oerr = None
                except Exception as e:
                    oerr = e
                if err is not None or oerr is not None:
                    # the first failing config (list order) decides the sweep's error
                    assert err is not None and oerr is not None, (seed, i, repr(err), repr(oerr))
                    break
                assert (res.makespan[i], res.cp_len[i]) == (ms, cp), (seed, i)
                assert [(e.node_id, e.device, e.start_us, e.finish_us) for e in res.schedule(i).entries] == entries, (seed, i)
        n_ok += 1
    except AssertionError:
        print("MISMATCH seed", seed, n, nd, len(cfgs)); traceback.print_exc(); break
    seed += 1
print("soak ok instances", n_ok, "last seed", seed)

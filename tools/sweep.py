"""Sweep engine knobs on one workload: python tools/sweep.py c2 'l1=vector cap=1024 groups=148,296,592,1184,2367 hub=2048'"""
import itertools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import build_graph
from paper_2602_10080_b200 import EngineConfig, L1Params, L2Params, MlmqConfig, extract_features
from paper_2602_10080_b200.engine import prepare

name = sys.argv[1]
spec = dict(kv.split("=") for kv in sys.argv[2].split())
grid = {k: v.split(",") for k, v in spec.items()}
g = build_graph(name)
f = extract_features(g)
aw = f.avg_weight if f.float_weights else max(1, round(f.avg_weight))
keys = list(grid)
e_reach = None
for vals in itertools.product(*[grid[k] for k in keys]):
    o = dict(zip(keys, vals))
    l2 = o.get("l2", "fifo")
    ds = float(o.get("d", 1))
    cfg = MlmqConfig(l1_type=o.get("l1", "vector"), l2_type=l2, l0_capacity=int(o.get("l0", 4)),
                     l1_params=L1Params(capacity=int(o.get("cap", 1024)), wb=int(o.get("wb", 8)),
                                        filter_f=float(o.get("f", 4)) * aw, delta_nf=ds * aw),
                     l2_params=L2Params(delta=ds * aw if l2 == "bucket" else None,
                                        block_size=int(o.get("bs", 64)), bmax=int(o.get("bmax", 64))),
                     num_groups=None if o.get("groups", "auto") == "auto" else int(o["groups"]),
                     lanes_per_group=int(o.get("lanes", 32)))
    eng = EngineConfig(hub_chunk=int(o.get("hub", 0)), share=o.get("share", "1") == "1",
                       fifo_park=o.get("park", "1") == "1", bucket_window=int(o.get("win", 1)),
                       read_batch=int(o.get("rb", 64)))
    try:
        cfg2, eng2, dg, ncfg = prepare(g, 0, cfg, eng, features=f)
        ms = []
        for _ in range(int(o.get("reps", 3))):
            if o.get("unit", "0") == "1":
                ncfg.unit_weights = 1
            m = dg.sssp_device(0, ncfg)
            ms.append(m.kernel_ms)
        if e_reach is None:
            e_reach = dg.reach()[1]
        print(" ".join(f"{k}={v}" for k, v in o.items()), f"G={cfg2.num_groups} ms={min(ms):.3f} med={np.median(ms):.3f}",
              f"GTEPS={e_reach/min(ms)/1e6:.2f} infl={m.relaxations/e_reach:.2f} l2w={m.l2_enqueues} hub={m.hub_items}", flush=True)
    except Exception as ex:
        print(o, "EXC", type(ex).__name__, ex, flush=True)

"""Repro + phase breakdown (run with MLMQ_DEBUG=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import *
from bench import build_graph

eng = EngineConfig(spin_timeout_s=3.0)
g = generate_graph("rmat", seed=1, scale=16, edge_factor=16, wmin=1, wmax=255)
f = extract_features(g)
want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
for cand in enumerate_candidates():
    try:
        r = sssp_solve(g, 0, cand.bind(f, num_groups=None), eng, features=f, watchdog_s=8)
        print("rmat16", cand.label(), np.array_equal(r.dist_array, want), r.kernel_ms, flush=True)
    except Exception as e:
        print("rmat16", cand.label(), "EXC", type(e).__name__, e, flush=True)
for name in sys.argv[1:]:
    g = build_graph(name)
    f = extract_features(g)
    aw = max(1, round(f.avg_weight))
    for l1, l2, ds in [("vector", "fifo", 1), ("filter", "bucket", 4), ("vector", "bucket", 1)]:
        cfg = MlmqConfig(l1_type=l1, l2_type=l2, l1_params=L1Params(capacity=256, filter_f=4 * aw),
                         l2_params=L2Params(delta=ds * aw if l2 == "bucket" else None), num_groups=None)
        try:
            r = sssp_solve(g, 0, cfg, eng, features=f, watchdog_s=20)
            print(name, l1, l2, ds, "kernel_ms", r.kernel_ms, "relax", r.metrics.relaxations, flush=True)
        except Exception as e:
            print(name, l1, l2, ds, "EXC", type(e).__name__, e, flush=True)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_10080_b200 import *
from oracle import oracle
g = generate_graph("rmat", seed=1, scale=int(sys.argv[1]) if len(sys.argv) > 1 else 12, edge_factor=16, wmin=1, wmax=255)
f = extract_features(g)
want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
for l1 in ["slf", "vector", "near_far", "filter"]:
    for cap in [1024, 64]:
        for l2 in ["fifo", "bucket"]:
            cfg = MlmqConfig(l1_type=l1, l2_type=l2, l1_params=L1Params(capacity=cap), num_groups=int(sys.argv[2]) if len(sys.argv) > 2 else 32)
            r = sssp_solve(g, 0, cfg, EngineConfig(spin_timeout_s=5), features=f, watchdog_s=60)
            print(l1, cap, l2, np.array_equal(r.dist_array, want), flush=True)

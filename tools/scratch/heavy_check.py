import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import EngineConfig, MlmqConfig, generate_graph, sssp_solve
from paper_2602_10080_b200.graph import generate_grid2d
for name, g in [("path", generate_graph("path", seed=1, n=50, wmin=1, wmax=20)),
                ("grid", generate_grid2d(8, 8, 1, 20, seed=3)),
                ("rmat8", generate_graph("rmat", seed=2, scale=8, edge_factor=8, wmin=1, wmax=255)),
                ("rmat12", generate_graph("rmat", seed=2, scale=12, edge_factor=16, wmin=1, wmax=255))]:
    want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    for groups in (1, 4, None):
        for h in (8, 32, 128):
            r = sssp_solve(g, 0, MlmqConfig(l2_type="fifo", num_groups=groups), EngineConfig(heavy_delta=h))
            bad = np.nonzero(r.dist_array != want)[0]
            print(name, groups, h, "OK" if bad.size == 0 else f"BAD {bad.size} first {bad[:5]} got {r.dist_array[bad[:5]]} want {want[bad[:5]]}", flush=True)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import generate_graph, MlmqConfig
from paper_2602_10080_b200.sharded import sssp_solve_sharded
P = int(sys.argv[1]); sc = int(sys.argv[2])
g = generate_graph("rmat", seed=1, scale=sc, edge_factor=16, wmin=1, wmax=255)
res = sssp_solve_sharded(g, 0, P, MlmqConfig(l2_type="fifo", num_groups=int(sys.argv[3]) if len(sys.argv) > 3 else None))
want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
print("P", P, "ok", np.array_equal(res.local_dist, want), "steps", res.steps, "sent", res.sent)

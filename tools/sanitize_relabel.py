"""compute-sanitizer run of the relabel path (mlmq_api.cu ensure_relabel): forced relabel
on small skewed graphs (u32, u64, f32 distances, FIFO and bucket L2), checked against the
oracle.   MLMQ_RELABEL=1 compute-sanitizer --tool memcheck python tools/sanitize_relabel.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2602_10080_b200 import EngineConfig, MlmqConfig, generate_graph, sssp_solve  # noqa: E402
from paper_2602_10080_b200.graph import with_f32_weights  # noqa: E402

os.environ["MLMQ_RELABEL"] = "1"
for l2, dm in [("fifo", "auto"), ("bucket", "auto"), ("fifo", "u64")]:
    g = generate_graph("rmat", seed=2, scale=11, edge_factor=16, wmin=1, wmax=255)
    r = sssp_solve(g, 0, MlmqConfig(l2_type=l2, num_groups=64), EngineConfig(dist_mode=dm))
    want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    assert np.array_equal(r.dist_array, want), (l2, dm)
    print("relabel", l2, dm, "OK", flush=True)
g = with_f32_weights(generate_graph("rmat", seed=2, scale=11, edge_factor=16), seed=1)
r = sssp_solve(g, 0, MlmqConfig(num_groups=64))
assert np.array_equal(r.dist_array, oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, 0))
print("relabel f32 OK", flush=True)

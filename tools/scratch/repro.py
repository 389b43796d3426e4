"""Repro helper: python tools/repro.py <kind> <scale|side> <l1> <l2> [reps] [cap] [groups]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import *
from paper_2602_10080_b200.adaptive import ConfigCandidate

kind, sz, l1, l2 = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
cap = int(sys.argv[6]) if len(sys.argv) > 6 else 1024
ng = None if len(sys.argv) <= 7 or sys.argv[7] == "auto" else int(sys.argv[7])
if kind == "rmat":
    g = generate_graph("rmat", seed=1, scale=sz, edge_factor=16, wmin=1, wmax=255)
else:
    g = generate_graph("grid2d", seed=1, rows=sz, cols=sz, wmin=1, wmax=100)
f = extract_features(g)
want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
ds = 1
if "(" in l2:
    l2, ds = l2.split("(")[0], int(l2.split("(d")[1].rstrip(")"))
cfg = ConfigCandidate(l1, l2, delta_scale=ds).bind(f, num_groups=ng)
cfg.l1_params.capacity = cap
for i in range(reps):
  try:
    r = sssp_solve(g, 0, cfg, EngineConfig(spin_timeout_s=3, share=os.environ.get("SHARE","1")=="1", fifo_park=os.environ.get("PARK","1")=="1"), features=f, watchdog_s=6)
    print(i, l1, l2, ds, np.array_equal(r.dist_array, want), round(r.kernel_ms, 3), flush=True)
  except Exception as e:
    print("EXC", i, type(e).__name__, e, flush=True)
    os._exit(3)

"""Quick GPU diagnostic: every L1 x L2 combo on small graphs vs the CPU oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2602_10080_b200 import *
from paper_2602_10080_b200.graph import generate_grid2d

def cc(l1, l2, ng=1):
    return MlmqConfig(l1_type=l1, l2_type=l2, l1_params=L1Params(capacity=64, wb=4),
                      l2_params=L2Params(block_size=16, block_num=512, bmax=32, bnum=2),
                      num_groups=ng, lanes_per_group=8)

DIAMOND = build_csr(4, [(0, 1, 10), (0, 2, 1), (2, 1, 2), (1, 3, 1), (2, 3, 9)])
combos = [(a, b) for a in ("vector", "near_far", "filter", "slf") for b in ("fifo", "bucket", "priority", "multi")]
eng = EngineConfig(spin_timeout_s=5.0)
bad = 0
for g, name, ng in [(DIAMOND, "diamond", 1), (generate_grid2d(8, 8, 1, 20, seed=3), "grid8", 2),
                    (generate_graph("rmat", seed=5, scale=10, edge_factor=8), "rmat10", 4),
                    (generate_grid2d(64, 64, 1, 100, seed=1), "grid64", 8)]:
    want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    for l1, l2 in combos:
        t = time.time()
        try:
            r = sssp_solve(g, 0, cc(l1, l2, ng), eng, watchdog_s=10)
            ok = np.array_equal(r.dist_array, want)
            m = r.metrics
            bal = (m.l0_enqueues == m.l0_dequeues, m.l1_enqueues == m.l1_dequeues, m.l2_enqueues == m.l2_dequeues)
            print(f"{name:8s} {l1:8s} {l2:8s} ok={ok} bal={bal} relax={m.relaxations} kms={r.kernel_ms:.3f} wall={time.time()-t:.3f}", flush=True)
            bad += (not ok) or (not all(bal))
        except Exception as e:
            bad += 1
            print(f"{name:8s} {l1:8s} {l2:8s} EXC {type(e).__name__}: {e}", flush=True)
# auto groups, default configs
for kind, p in [("grid2d", dict(rows=256, cols=256, wmin=1, wmax=100)), ("rmat", dict(scale=16, edge_factor=16, wmin=1, wmax=255))]:
    g = generate_graph(kind, seed=1, **p)
    f = extract_features(g)
    want = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    for cand in enumerate_candidates():
        t = time.time()
        try:
            cfg = cand.bind(f, num_groups=None)
            cfg.l1_params.capacity = 256
            r = sssp_solve(g, 0, cfg, eng, features=f, watchdog_s=20)
            ok = np.array_equal(r.dist_array, want)
            print(f"{kind:6s} {cand.label():22s} G={r.config_used.num_groups} ok={ok} relax={r.metrics.relaxations} kms={r.kernel_ms:.3f} wall={time.time()-t:.3f}", flush=True)
            bad += not ok
        except Exception as e:
            bad += 1
            print(f"{kind} {cand.label()} EXC {type(e).__name__}: {e}", flush=True)
print("BAD", bad)

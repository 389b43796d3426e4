"""Where the end-to-end sssp_solve time goes on one workload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import build_graph, solve_config
from paper_2602_10080_b200 import EngineConfig, extract_features
from paper_2602_10080_b200.engine import prepare, sssp_solve
g = build_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
f = extract_features(g)
cfg0 = solve_config(sys.argv[1] if len(sys.argv) > 1 else "c2", g, f)
eng = EngineConfig()
for i in range(6):
    t0 = time.perf_counter()
    cfg, eng2, dg, ncfg = prepare(g, 0, cfg0, eng, features=f)
    t1 = time.perf_counter()
    dist, m, gm = dg.sssp(0, ncfg, want_groups=int(cfg.num_groups))
    t2 = time.perf_counter()
    r = sssp_solve(g, 0, cfg0, eng, features=f)
    t3 = time.perf_counter()
    print(f"prepare {1e3*(t1-t0):.2f} ms  native {1e3*(t2-t1):.2f} ms (kernel {m.kernel_ms:.2f}, lib wall {m.wall_time_us/1e3:.2f})  full sssp_solve {1e3*(t3-t2):.2f} ms", flush=True)
# the result copy alone (u32 -> u64 widen + D2H), after a device-resident solve
out = None
for i in range(5):
    dg.sssp_device(0, ncfg)
    t0 = time.perf_counter()
    out = dg.last_dist()
    t1 = time.perf_counter()
    print(f"last_dist (copy + widen of {out.size} distances) {1e3*(t1-t0):.3f} ms", flush=True)

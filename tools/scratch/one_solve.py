"""Generate a workload and run N solves (for ncu): python tools/one_solve.py c2 l1 l2 dscale cap [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10080_b200 import *
from paper_2602_10080_b200.engine import prepare
from bench import build_graph
name, l1, l2, ds, cap = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), int(sys.argv[5])
n = int(sys.argv[6]) if len(sys.argv) > 6 else 2
g = build_graph(name)
f = extract_features(g)
aw = max(1, round(f.avg_weight))
cfg = MlmqConfig(l1_type=l1, l2_type=l2, l0_capacity=int(os.environ.get('L0', '4')), l1_params=L1Params(capacity=cap, filter_f=4 * aw),
                 l2_params=L2Params(delta=int(ds * aw) if l2 == "bucket" else None), num_groups=None)
cfg, eng, dg, ncfg = prepare(g, 0, cfg, EngineConfig(), features=f)
for _ in range(n):
    m = dg.sssp_device(0, ncfg)
    print("kernel_ms", m.kernel_ms, "relax", m.relaxations, flush=True)

"""One graph, several group counts: python tools/scratch/sweep_groups.py c4 1776 2220 2400 2663"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from bench import build_graph, solve_config, solve_engine
from paper_2602_10080_b200 import extract_features
from paper_2602_10080_b200.engine import prepare

name = sys.argv[1]
g = build_graph(name)
f = extract_features(g)
for G in sys.argv[2:]:
    cfg = solve_config(name, g, f)
    cfg.num_groups = int(G)
    cfg_r, eng_r, dg, ncfg = prepare(g, 0, cfg, solve_engine(name), features=f)
    ms, inf = [], []
    e = None
    for i in range(5):
        m = dg.sssp_device(0, ncfg)
        if e is None:
            _, e = dg.reach()
        ms.append(m.kernel_ms)
        inf.append(m.relaxations / e)
    print(f"{name} groups={G}: best {min(ms[1:]):.3f} median {float(np.median(ms[1:])):.3f} ms infl {np.mean(inf):.3f}", flush=True)

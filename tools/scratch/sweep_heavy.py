"""One graph, several light/heavy thresholds: python tools/scratch/sweep_heavy.py c4 12 20 32 48"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from bench import build_graph, solve_config, solve_engine
from paper_2602_10080_b200 import extract_features
from paper_2602_10080_b200.engine import prepare

name = sys.argv[1]
g = build_graph(name)
f = extract_features(g)
for hd in sys.argv[2:]:
    eng = solve_engine(name)
    hdv = float(hd) if "." in hd else int(hd)
    eng = dataclasses.replace(eng, heavy_delta=hdv)
    cfg_r, eng_r, dg, ncfg = prepare(g, 0, solve_config(name, g, f), eng, features=f)
    ms, inf = [], []
    v, e = None, None
    for i in range(5):
        m = dg.sssp_device(0, ncfg)
        if e is None:
            v, e = dg.reach()
        ms.append(m.kernel_ms)
        inf.append(m.relaxations / e)
    print(f"{name} heavy_delta={hd}: best {min(ms[1:]):.3f} median {float(np.median(ms[1:])):.3f} ms infl {np.mean(inf):.3f}", flush=True)

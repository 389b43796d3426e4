"""Golden hashes for the two BASELINE configs the reference itself cannot run (C4, C5).

Run in the build container (minutes; ~40 GB of host memory for C4):

    python tests/golden/make_big_hashes.py [c4] [c5]   -> tests/golden/big_configs.json

The reference's Python generator and oracle cannot build or solve these graphs in the
memory of this container (C4 has 1.07 B edges, ~220 B/edge in Python), so
the chain of trust is:
  * the graph comes from the native generator (csrc/host/generators.cpp), which
    reproduces the reference generator byte for byte -- pinned by the reference-produced
    csr_sha256 of RMAT s16/s20/s22 (tests/test_generators.py);
  * the distances come from the C restatement of the reference's dijkstra_oracle
    (oracle/sssp_oracle.c, engine.py:313-338), pinned against 110 reference-produced
    golden graphs plus the C1/C2/C3 reference hashes (tests/test_oracle.py).
C4 = generate_rmat(26, 16, wmin=1, wmax=255, seed=1), source 0 (BASELINE.json configs[3]).
C5 = generate_rmat(24, 16, wmin=1, wmax=1, seed=1) topology with f32 weights U[0,1)
     (graph.with_f32_weights(seed=1)), source 0; hashed as little-endian f32, +inf
     unreachable, solved by the strict-IEEE f32 Dijkstra.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2602_10080_b200 import generate_graph  # noqa: E402
from paper_2602_10080_b200.graph import with_f32_weights  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "big_configs.json")


def _csr_hash(g, f32=False):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.row_offsets, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(g.col_indices, dtype="<u4").tobytes())
    h.update(np.ascontiguousarray(g.weights, dtype="<f4" if f32 else "<u4").tobytes())
    return h.hexdigest()


def c4():
    t = time.time()
    g = generate_graph("rmat", seed=1, scale=26, edge_factor=16, wmin=1, wmax=255)
    gen = time.time() - t
    t = time.time()
    d = oracle.dijkstra_u64(g.row_offsets, g.col_indices, g.weights, 0)
    solve = time.time() - t
    v, e = oracle.reach(g.row_offsets, d)
    fin = d[d != oracle.U64_INF]
    return {"graph": "generate_rmat(scale=26, edge_factor=16, wmin=1, wmax=255, seed=1)", "source": 0,
            "n": g.num_vertices, "m": g.num_edges, "csr_sha256": _csr_hash(g),
            "dist_sha256": oracle.dist_sha256(d), "v_reach": v, "e_reach": e,
            "max_dist": int(fin.max()), "gen_s": round(gen, 1), "oracle_s": round(solve, 1)}


def c5():
    t = time.time()
    g = with_f32_weights(generate_graph("rmat", seed=1, scale=24, edge_factor=16, wmin=1, wmax=1), seed=1)
    gen = time.time() - t
    t = time.time()
    d = oracle.dijkstra_f32(g.row_offsets, g.col_indices, g.weights, 0)
    solve = time.time() - t
    reached = np.isfinite(d)
    deg = np.diff(g.row_offsets)
    return {"graph": "with_f32_weights(generate_rmat(scale=24, edge_factor=16, wmin=1, wmax=1, seed=1), seed=1)",
            "source": 0, "n": g.num_vertices, "m": g.num_edges, "csr_sha256": _csr_hash(g, f32=True),
            "dist_f32_sha256": hashlib.sha256(np.ascontiguousarray(d, dtype="<f4").tobytes()).hexdigest(),
            "v_reach": int(reached.sum()), "e_reach": int(deg[reached].sum()),
            "max_dist": float(d[reached].max()), "gen_s": round(gen, 1), "oracle_s": round(solve, 1)}


def main():
    which = sys.argv[1:] or ["c4", "c5"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for name in which:
        print(f"[{name}] ...", flush=True)
        data[name] = {"c4": c4, "c5": c5}[name]()
        print(json.dumps(data[name]), flush=True)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
            fh.write("\n")


if __name__ == "__main__":
    main()

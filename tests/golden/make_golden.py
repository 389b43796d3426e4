"""Generate tests/golden/reference_vectors.json by running the REFERENCE package.

Run in the build container only (it imports /root/reference/pkg/src, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every graph of the reference's acceptance graph set (test_acceptance.py:48-80:
25 grids, 25 paths, 25 uniform, 25 RMAT; sources 0 and Random(seed).randrange(1, n))
plus the engine-test graphs of test_engine.py, it records the reference generator's
csr_sha256 and the reference dijkstra_oracle's dist_sha256 (and the unit-weight
distances' hash for BFS).  Small graphs also store full distance lists.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import mlq_sssp  # noqa: E402  (the reference)
from mlq_sssp.engine import dijkstra_oracle, distances_blob, unit_weight_view  # noqa: E402

assert mlq_sssp.__file__.startswith(REF), mlq_sssp.__file__

GRID_DIMS = [(5, 5), (6, 10), (8, 8), (10, 12), (12, 12), (15, 20), (20, 20), (25, 25), (25, 40),
             (30, 30), (40, 40), (50, 50), (60, 60), (70, 70), (80, 80), (90, 90), (100, 100)]
PATH_SIZES = [50, 100, 200, 500, 1000, 2000, 3000, 5000, 8000, 10000]
UNIFORM_SIZES = [100, 200, 500, 1000, 2000, 3000, 5000, 8000, 10000, 10000]
RMAT_SCALES = [6, 7, 8, 9, 10, 11, 12, 13]


def acceptance_specs():
    out = []
    for i in range(25):
        r, c = GRID_DIMS[i % len(GRID_DIMS)]
        out.append((f"grid-{i:02d}", "grid2d", dict(rows=r, cols=c, wmin=1, wmax=1 if i % 3 == 0 else 100), i))
    for i in range(25):
        out.append((f"path-{i:02d}", "path", dict(n=PATH_SIZES[i % 10], wmin=1, wmax=1 if i % 3 == 0 else 50), 100 + i))
    for i in range(25):
        n = UNIFORM_SIZES[i % 10]
        out.append((f"unif-{i:02d}", "uniform", dict(n=n, m=8 * n if i % 5 == 0 else 4 * n, wmin=1,
                                                     wmax=1 if i % 3 == 0 else 100), 200 + i))
    for i in range(25):
        out.append((f"rmat-{i:02d}", "rmat", dict(scale=RMAT_SCALES[i % 8], edge_factor=8, wmin=1,
                                                  wmax=1 if i % 3 == 0 else 100), 300 + i))
    return out


def engine_specs():
    # graphs used by test_engine.py (uniform / rmat / grid / path, seeds inline)
    return [
        ("eng-grid8", "grid2d", dict(rows=8, cols=8, wmin=1, wmax=20), 3),
        ("eng-unif300", "uniform", dict(n=300, m=1500, wmin=1, wmax=40), 5),
        ("eng-rmat7", "rmat", dict(scale=7, edge_factor=6), 5),
        ("eng-grid12", "grid2d", dict(rows=12, cols=12, wmin=1, wmax=30), 5),
        ("eng-path500", "path", dict(n=500, wmin=1, wmax=9), 5),
        ("eng-unif150", "uniform", dict(n=150, m=1200, wmin=1, wmax=30), 8),
        ("eng-unif200", "uniform", dict(n=200, m=1000, wmin=1, wmax=50), 4),
        ("eng-rmat8", "rmat", dict(scale=8, edge_factor=6), 9),
        ("eng-unif250", "uniform", dict(n=250, m=1000, wmin=1, wmax=90), 12),
        ("grid256-road", "grid2d", dict(rows=256, cols=256, wmin=10, wmax=1000), 1),
    ]


def csr_sha(g):
    h = hashlib.sha256()
    h.update(np.asarray(g.row_offsets, "<u8").tobytes())
    h.update(np.asarray(g.col_indices, "<u4").tobytes())
    h.update(np.asarray(g.weights, "<u4").tobytes())
    return h.hexdigest()


def main():
    t0 = time.time()
    entries = []
    for gid, kind, params, seed in acceptance_specs() + engine_specs():
        g = mlq_sssp.generate_graph(kind, seed=seed, **params)
        sources = [0, random.Random(seed).randrange(1, g.num_vertices)]
        unit = unit_weight_view(g)
        rec = dict(id=gid, kind=kind, params=params, seed=seed, n=g.num_vertices, m=g.num_edges,
                   csr_sha256=csr_sha(g), sources=[])
        for s in sources:
            d = dijkstra_oracle(g, s)
            du = dijkstra_oracle(unit, s)
            src = dict(source=s, dist_sha256=hashlib.sha256(distances_blob(d)).hexdigest(),
                       unit_dist_sha256=hashlib.sha256(distances_blob(du)).hexdigest())
            if g.num_vertices <= 64:
                src["dist"] = [None if x == mlq_sssp.INF else x for x in d]
            rec["sources"].append(src)
        entries.append(rec)
    out = dict(generated_by="tests/golden/make_golden.py (reference mlq_sssp 0.1.0, CPython "
                            + sys.version.split()[0] + ")",
               graphs=entries)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {len(entries)} graphs to {path} in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()

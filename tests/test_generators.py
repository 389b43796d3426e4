"""Native generators + CSR builder vs the reference (graph.py:89-124, 306-420).

Byte-identity is pinned by csr_sha256 values produced by the reference itself
(tests/golden/reference_vectors.json and the SURVEY §8c table, checked in
test_oracle.py); here: validation messages, build_csr ordering rules, features.
"""
import math

import numpy as np
import pytest

from paper_2602_10080_b200 import (CsrGraph, GraphFormatError, NegativeWeightError, build_csr,
                                   extract_features, generate_graph)
from paper_2602_10080_b200.graph import with_f32_weights


def test_generator_csr_hashes_match_reference(golden):
    from oracle import oracle
    for rec in golden["graphs"]:
        g = generate_graph(rec["kind"], seed=rec["seed"], **rec["params"])
        assert (g.num_vertices, g.num_edges) == (rec["n"], rec["m"])
        assert oracle.csr_sha256(g.row_offsets, g.col_indices, g.weights) == rec["csr_sha256"]


@pytest.mark.parametrize("kind,params,msg", [
    ("grid2d", dict(rows=0, cols=3), "grid dimensions"),
    ("path", dict(n=0), "path length"),
    ("uniform", dict(n=0, m=3), "need n >= 1"),
    ("rmat", dict(scale=0), "scale must be"),
    ("rmat", dict(scale=3, edge_factor=0), "edge_factor"),
    ("rmat", dict(scale=3, a=0.5, b=0.5, c=0.5, d=0.5), "sum to 1"),
    ("mesh", dict(), "unknown generator kind"),
])
def test_generator_validation_messages(kind, params, msg):
    with pytest.raises(ValueError, match=msg):
        generate_graph(kind, **params)


def test_build_csr_keeps_source_order_and_duplicates_drops_zero_self_loops():
    g = build_csr(3, [(2, 0, 4), (0, 2, 1), (0, 1, 7), (2, 2, 0), (1, 1, 3), (0, 2, 1)])
    assert list(g.row_offsets) == [0, 3, 4, 5]
    assert list(g.col_indices) == [2, 1, 2, 1, 0]
    assert list(g.weights) == [1, 7, 1, 3, 4]
    assert g.num_edges == 5


def test_build_csr_rejects_bad_edges():
    with pytest.raises(NegativeWeightError):
        build_csr(2, [(0, 1, -1)])
    with pytest.raises(GraphFormatError):
        build_csr(2, [(0, 2, 1)])


def test_features_match_reference_formulas():
    g = generate_graph("rmat", seed=3, scale=9, edge_factor=8, wmin=1, wmax=50)
    f = extract_features(g)
    deg = [int(g.row_offsets[i + 1] - g.row_offsets[i]) for i in range(g.num_vertices)]
    w = [int(x) for x in g.weights]
    avg = sum(deg) / len(deg)
    assert f.avg_nnz == avg
    assert f.dev_nnz == math.sqrt(max(0.0, sum(d * d for d in deg) / len(deg) - avg * avg))
    aw = sum(w) / len(w)
    assert f.avg_weight == aw
    assert f.dev_weight == math.sqrt(max(0.0, sum(x * x for x in w) / len(w) - aw * aw))
    assert (f.m, f.nnz, f.max_nnz, f.max_weight) == (g.num_vertices, g.num_edges, max(deg), max(w))


def test_f32_weights_are_in_unit_interval_and_deterministic():
    g = generate_graph("rmat", seed=1, scale=8, edge_factor=4)
    a = with_f32_weights(g, seed=7)
    b = with_f32_weights(g, seed=7)
    assert a.weights.dtype == np.float32 and np.array_equal(a.weights, b.weights)
    assert float(a.weights.min()) >= 0.0 and float(a.weights.max()) < 1.0
    assert a.float_weights and extract_features(a).float_weights


def test_csrgraph_accepts_lists():
    g = CsrGraph(3, 2, [0, 1, 2, 2], [1, 2], [5, 6])
    assert g.out_degree(0) == 1 and list(g.edges()) == [(0, 1, 5), (1, 2, 6)]

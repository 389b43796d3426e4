"""Native DIMACS / Matrix Market readers (csrc/host/loaders.cpp) against
the Python restatement of the reference readers (graph.py:132-257): same graphs, same
exception classes and messages, and a fallback to Python for the inputs only Python
reads exactly."""
import os

import numpy as np
import pytest

from paper_2602_10080_b200 import GraphFormatError, NegativeWeightError, generate_graph
from paper_2602_10080_b200.graph import (_load_dimacs_py, _load_matrix_market_py, load_dimacs,
                                         load_matrix_market, save_graph)
from paper_2602_10080_b200 import _native

CASES = {
    "tiny.gr": "c tiny\np sp 5 6\na 1 2 2\na 1 3 4\na 2 4 3\na 3 4 1\na 4 5 3\na 3 5 4\n",
    "dup_selfloop.gr": "p sp 3 4\na 1 1 0\na 1 2 5\na 1 2 5\nc x\na 3 3 7\n",
    "badcount.gr": "p sp 3 2\na 1 2 1\n",
    "badvertex.gr": "p sp 2 1\na 1 3 1\n",
    "negative.gr": "p sp 2 1\na 1 2 -4\n",
    "arcfirst.gr": "a 1 2 1\np sp 2 1\n",
    "unknown.gr": "p sp 2 1\nx 1 2 1\n",
    "noint.gr": "p sp 2 1\na 1 2 1.5\n",
    "underscore.gr": "p sp 2 1\na 1 2 1_000\n",
    "bigw.gr": "p sp 2 1\na 1 2 5000000000\n",
    "general.mtx": "%%MatrixMarket matrix coordinate integer general\n% c\n3 3 3\n1 2 4\n2 3 5\n3 1 6\n",
    "symmetric.mtx": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 2\n2 2\n3 1\n",
    "real.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 2 0.0025\n2 1 0.0035\n1 1 1.5\n2 2 2.5e-3\n",
    "negreal.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 -0.5\n",
    "rect.mtx": "%%MatrixMarket matrix coordinate integer general\n2 3 1\n1 2 1\n",
    "noheader.mtx": "3 3 1\n1 2 1\n",
    "count.mtx": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 2 1\n",
}


def _run(fn, path, *a):
    try:
        g = fn(path, *a)
        return ("ok", g.num_vertices, g.row_offsets.tolist(), g.col_indices.tolist(), g.weights.tolist())
    except (GraphFormatError, NegativeWeightError, ValueError, OSError) as e:
        return (type(e).__name__, str(e))


@pytest.mark.parametrize("name", sorted(CASES))
def test_native_reader_equals_python_restatement(name, tmp_path):
    path = str(tmp_path / name)
    with open(path, "w") as fh:
        fh.write(CASES[name])
    if name.endswith(".gr"):
        assert _run(load_dimacs, path) == _run(_load_dimacs_py, path)
    else:
        assert _run(load_matrix_market, path, 1000) == _run(_load_matrix_market_py, path, 1000)


def test_fallback_inputs_are_routed_to_python(tmp_path):
    for name in ("underscore.gr", "bigw.gr"):
        path = str(tmp_path / name)
        with open(path, "w") as fh:
            fh.write(CASES[name])
        assert _native.load_csr(path, "dimacs") is None
    assert _native.load_csr(str(tmp_path / "missing.gr"), "dimacs") is None
    with pytest.raises(FileNotFoundError):
        load_dimacs(str(tmp_path / "missing.gr"))


@pytest.mark.parametrize("ext", [".gr", ".mtx"])
def test_round_trip_generated_graph(ext, tmp_path):
    g = generate_graph("rmat", seed=5, scale=12, edge_factor=8, wmin=1, wmax=255)
    path = str(tmp_path / ("g" + ext))
    save_graph(g, path)
    h = (load_dimacs if ext == ".gr" else load_matrix_market)(path)
    assert h.row_offsets == g.row_offsets and h.col_indices == g.col_indices and h.weights == g.weights

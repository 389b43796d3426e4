"""`mlq` CLI: the reference CLI's contract (pkg/src/mlq_sssp/cli.py) --
one JSON object per command, errors as {"error": ...} with exit 2, verify exit 1 on a
mismatch, distances inline (null = unreachable) or in a .distances.u64 sidecar."""
import json
import struct

import pytest

from paper_2602_10080_b200 import cli


def run(capsys, *argv):
    rc = cli.main(list(argv))
    return rc, json.loads(capsys.readouterr().out)


def test_parse_gen_spec():  # cli.py:91-124 shorthand
    assert cli.parse_gen_spec("path:30") == ("path", {"n": 30})
    assert cli.parse_gen_spec("grid2d:3x4,1,9") == ("grid2d", {"rows": 3, "cols": 4, "wmin": 1, "wmax": 9})
    assert cli.parse_gen_spec("uniform:10,20") == ("uniform", {"n": 10, "m": 20})
    assert cli.parse_gen_spec("rmat:8,4,1,255") == ("rmat", {"scale": 8, "edge_factor": 4, "wmin": 1, "wmax": 255})
    with pytest.raises(ValueError, match="unknown generator"):
        cli.parse_gen_spec("bogus:1")
    with pytest.raises(ValueError, match="bad generator spec"):
        cli.parse_gen_spec("grid2d:x")


def test_gen_features_roundtrip(tmp_path, capsys):
    path = str(tmp_path / "g.gr")
    rc, out = run(capsys, "gen", "grid2d:5x6,1,9", "--gen-seed", "3", "--out", path)
    assert rc == 0 and out["num_vertices"] == 30 and out["path"] == path
    rc, out = run(capsys, "features", "--graph", path)
    assert rc == 0 and out["features"]["m"] == 30 and out["graph"]["num_edges"] == out["features"]["nnz"]


def test_errors_are_json_exit_2(capsys):
    rc, out = run(capsys, "features", "--gen", "nope:3")
    assert rc == 2 and out["error"]["type"] == "ValueError"
    rc, out = run(capsys, "features")
    assert rc == 2 and "exactly one of" in out["error"]["message"]


@pytest.mark.gpu
def test_solve_inline_and_sidecar(tmp_path, capsys):
    rc, out = run(capsys, "solve", "--gen", "path:30", "--l1", "slf", "--l2", "bucket", "--delta", "3",
                  "--num-groups", "2")
    assert rc == 0 and out["distances"] == list(range(30)) and out["config_source"] == "explicit"
    m = out["metrics"]
    assert m["l0_enqueues"] == m["l0_dequeues"] and m["l2_enqueues"] == m["l2_dequeues"]
    side_out = str(tmp_path / "s.json")
    rc, _ = run(capsys, "solve", "--gen", "path:50", "--max-inline-distances", "10", "--out", side_out)
    rep = json.load(open(side_out))
    blob = open(rep["distances_file"], "rb").read()
    assert rc == 0 and struct.unpack("<50Q", blob) == tuple(range(50))


@pytest.mark.gpu
def test_verify_match_and_rule_based(capsys):
    rc, out = run(capsys, "verify", "--gen", "rmat:10,8,1,255", "--gen-seed", "2")
    assert rc == 0 and out["match"] is True and out["config_source"] == "rule_based"
    rc, out = run(capsys, "verify", "--gen", "grid2d:20x20,1,50", "--unit-weights", "--l2", "fifo")
    assert rc == 0 and out["match"] is True

"""Stage the reference package's own test suites for running against this drop-in.

TEST INFRASTRUCTURE.  Copies, unmodified, the reference's test modules, their fixtures
and the JSON schemas they validate against from /root/reference/pkg into
tests/reference_suite/staged/ (git-ignored: the files are the reference's, never
committed here; they travel to the GPU box with the working tree like the built .so
files).  tests/test_reference_suite.py then runs them with ``mlq_sssp`` resolving to this
repository's package (mlq_sssp/ -> paper_2602_10080_b200/).

    python tests/reference_suite/stage.py          # also called by __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import sys

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
STAGED = os.path.join(HERE, "staged")
MODULES = ("test_engine.py", "test_graph.py", "test_cli.py", "test_adaptive.py", "test_acceptance.py")


def stage(ref: str = REF) -> bool:
    """Copy the suites; False (and nothing touched) when the reference is absent."""
    if not os.path.isdir(os.path.join(ref, "tests")):
        return False
    tests = os.path.join(STAGED, "tests")
    os.makedirs(tests, exist_ok=True)
    for m in MODULES:
        shutil.copyfile(os.path.join(ref, "tests", m), os.path.join(tests, m))
    for sub, dst in (("tests/fixtures", os.path.join(tests, "fixtures")),
                     ("docs/schemas", os.path.join(STAGED, "docs", "schemas"))):
        if os.path.isdir(dst):
            shutil.rmtree(dst)
        shutil.copytree(os.path.join(ref, sub), dst)
    with open(os.path.join(STAGED, "pytest.ini"), "w") as fh:
        fh.write("[pytest]\naddopts = -p no:cacheprovider\n")
    return True


if __name__ == "__main__":
    ok = stage(sys.argv[1] if len(sys.argv) > 1 else REF)
    print("staged" if ok else "reference not found; nothing staged", STAGED)

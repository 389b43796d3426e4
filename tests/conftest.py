"""Test configuration.

Markers:
  gpu   needs a CUDA device (B200); parity tests proper, calling through libmlmq.so.
  slow  large CPU checks (C2/C3 golden hashes, minutes); run with MLMQ_SLOW=1.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200)")
    config.addinivalue_line("markers", "slow: minutes-long CPU check; set MLMQ_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("MLMQ_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow; set MLMQ_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def gpu_available():
    from paper_2602_10080_b200 import _native
    return _native.device_count() > 0

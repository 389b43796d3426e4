"""The reference package's own test suites, run unmodified against this drop-in.

SURVEY §4.4 #1 / §7.3: ``pkg/tests/test_engine.py``, ``test_graph.py``, ``test_cli.py``,
``test_adaptive.py`` and ``test_acceptance.py`` are staged (copied, not committed) from
/root/reference by tests/reference_suite/stage.py (run by ``__graft_entry__.build()`` in
the build container) and executed in a subprocess with ``mlq_sssp`` = this repository.

* CPU (``-m "not gpu"``): every test must pass except those that need a device, and
  those may fail only with this engine's "no CUDA device" EngineError (no CPU fallback).
* GPU (``-m gpu``): every staged test must pass.
"""
from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGED = os.path.join(ROOT, "tests", "reference_suite", "staged")
NO_DEVICE = "no CUDA device is visible"


def _staged(*mods):
    paths = [os.path.join(STAGED, "tests", m) for m in mods]
    missing = [p for p in paths if not os.path.exists(p)]
    if missing:
        pytest.skip("reference suites not staged (python tests/reference_suite/stage.py)")
    return paths


def _run(paths, tmp_path, extra=(), timeout=1500):
    xml = str(tmp_path / "junit.xml")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""),
               PYTHONDONTWRITEBYTECODE="1", MLMQ_NODEV_LOG=str(tmp_path / "nodev.log"))
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", os.path.join(STAGED, "pytest.ini"),
           "--rootdir", STAGED, f"--junitxml={xml}", "-o", "junit_logging=all", *extra, *paths]
    proc = subprocess.run(cmd, cwd=STAGED, env=env, capture_output=True, text=True, timeout=timeout)
    cases = []
    if os.path.exists(xml):
        for tc in ET.parse(xml).getroot().iter("testcase"):
            bad = [c for c in tc if c.tag in ("failure", "error")]
            skipped = any(c.tag == "skipped" for c in tc)
            text = " ".join((c.get("message") or "") + (c.text or "") for c in tc
                            if c.tag in ("failure", "error", "system-out", "system-err"))
            cases.append((tc.get("classname", "") + "::" + tc.get("name", ""), bool(bad), skipped, text))
    nodev = str(tmp_path / "nodev.log")
    if os.path.exists(nodev):  # tests that stopped at the missing device (PYTEST_CURRENT_TEST ids)
        with open(nodev) as fh:
            hit = {ln.strip().split("::", 1)[-1] for ln in fh if ln.strip()}
        cases = [(n, b, s, t + (f" {NO_DEVICE}" if n.split("::", 1)[-1] in hit else ""))
                 for n, b, s, t in cases]
    return proc, cases


def test_reference_suites_cpu(tmp_path):
    """On a host without a GPU every reference test passes, or fails only for want of a
    device (graph construction, loaders, generators, features, selector, CLI parsing and
    error objects, config resolution all run on the host)."""
    from paper_2602_10080_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible: the -m gpu variant runs the full suites")
    paths = _staged("test_graph.py", "test_adaptive.py", "test_cli.py", "test_engine.py")
    proc, cases = _run(paths, tmp_path)
    assert cases, proc.stdout[-3000:] + proc.stderr[-3000:]
    other = [(n, t[:300]) for n, bad, _, t in cases if bad and NO_DEVICE not in t]
    assert not other, other
    passed = sum(1 for _, bad, sk, _ in cases if not bad and not sk)
    assert passed >= 60, (passed, len(cases))


@pytest.mark.gpu
@pytest.mark.parametrize("module", ["test_engine.py", "test_graph.py", "test_cli.py", "test_adaptive.py"])
def test_reference_suite_gpu(module, tmp_path):
    proc, cases = _run(_staged(module), tmp_path)
    failed = [(n, t[:400]) for n, bad, _, t in cases if bad]
    assert cases and not failed and proc.returncode == 0, (failed, proc.stdout[-2000:])


@pytest.mark.gpu
def test_reference_acceptance_gpu(tmp_path):
    """AC1 (2400-run oracle matrix), AC2 (termination audit), AC4-AC6, AC8, AC9 of the
    reference's acceptance suite, on the GPU engine."""
    proc, cases = _run(_staged("test_acceptance.py"), tmp_path, extra=("-s",))
    failed = [n for n, bad, _, _ in cases if bad]
    report = [ln for ln in proc.stdout.splitlines() if ln.startswith("ACCEPTANCE")]
    print("\n".join(report))
    assert cases and not failed, "; ".join(failed + report)

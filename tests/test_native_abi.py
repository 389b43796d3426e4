"""The C-ABI library loads (no GPU needed) and exports every symbol include/mlmq.h
declares, with struct layouts identical to the ctypes mirror in _native.py."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2602_10080_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlmq.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mlmq_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding_table():
    assert _declared() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.mlmq_abi_version() == 1


def test_nm_shows_exported_text_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mlmq_\w+)", out))
    assert set(_declared()) <= exported


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "mlmq.h"\n'
        "int main(void){\n"
        'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(mlmq_config_t), sizeof(mlmq_metrics_t),'
        " sizeof(mlmq_gen_params_t), offsetof(mlmq_config_t, block_num),"
        " offsetof(mlmq_config_t, watchdog_s), offsetof(mlmq_metrics_t, kernel_ms),"
        " offsetof(mlmq_config_t, hub_chunk));\nreturn 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_native.Config), ctypes.sizeof(_native.Metrics),
            ctypes.sizeof(_native.GenParams), _native.Config.block_num.offset,
            _native.Config.watchdog_s.offset, _native.Metrics.kernel_ms.offset,
            _native.Config.hub_chunk.offset]
    assert got == want


def test_status_codes_map_to_reference_exceptions():
    from paper_2602_10080_b200.core import EngineError, QueueOverflowError
    with pytest.raises(ValueError):
        _native.check(_native.MLMQ_EINVAL)
    with pytest.raises(QueueOverflowError):
        _native.check(_native.MLMQ_EOVERFLOW)
    for code in (_native.MLMQ_EENGINE, _native.MLMQ_ECUDA, _native.MLMQ_ENOMEM):
        with pytest.raises(EngineError):
            _native.check(code)


def test_solve_fails_loudly_without_a_device():
    """No CPU fallback: on a machine without a GPU, sssp_solve raises EngineError."""
    from paper_2602_10080_b200 import EngineError, build_csr, sssp_solve
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(EngineError, match="no CUDA device"):
        sssp_solve(build_csr(2, [(0, 1, 1)]), 0)

"""Alias of paper_2602_10080_b200.cli under the reference module name (``mlq`` CLI)."""
import sys as _sys

from paper_2602_10080_b200 import cli as _impl

_sys.modules[__name__] = _impl

if __name__ == "__main__":
    _sys.exit(_impl.main())

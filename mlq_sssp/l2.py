"""Alias of paper_2602_10080_b200.l2 (device-backed queues) under the reference module name."""
import sys as _sys

from paper_2602_10080_b200 import l2 as _impl

_sys.modules[__name__] = _impl

"""Alias of paper_2602_10080_b200.adaptive under the reference module name."""
import sys as _sys

from paper_2602_10080_b200 import adaptive as _impl

_sys.modules[__name__] = _impl

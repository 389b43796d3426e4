"""`mlq_sssp` — the reference package name, served by paper_2602_10080_b200.

Code written against the reference (`from mlq_sssp import sssp_solve`,
`from mlq_sssp.engine import dijkstra_oracle`, ...) runs unchanged on the GPU engine.
"""
from paper_2602_10080_b200 import *  # noqa: F401,F403
from paper_2602_10080_b200 import __all__, __version__  # noqa: F401

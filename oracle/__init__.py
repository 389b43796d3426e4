"""CPU oracle for the MLMQ SSSP hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and its
``--impl reference`` arm) may import this package.  The product package
(paper_2602_10080_b200 / mlq_sssp) never imports, links or calls it.
"""

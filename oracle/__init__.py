"""ORACLE — test infrastructure only.

CPU restatement of the reference's σ_min path (pseudospec/core.py:141-168: one dense LAPACK
zgesdd per shift via numpy.linalg.svd, BLAS pinned to one thread) and the fixture generator
that pins it to the reference itself (make_golden.py). Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import this package; the product path
(paper_2605_04550_b200) never does.
"""

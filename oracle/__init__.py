"""ORACLE -- test infrastructure, NOT the product.

CPU restatement of the reference's solve-path algorithms (schwarzdd,
arXiv 2304.04876 re-creation). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package,
and only as the checker or the timed CPU baseline. The product
(paper_2304_04876_b200) never imports it and fails loudly without its CUDA
library.

Parity of the oracle itself is pinned against golden vectors produced by
running the reference (tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

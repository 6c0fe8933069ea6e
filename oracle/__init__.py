"""CPU oracle for the IMDP construction + interval-iteration hot path.

TEST INFRASTRUCTURE -- NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this package,
and only as the checker or the timed CPU baseline; the product path
(paper_2401_03555_b200) never imports it and fails loudly when its CUDA
library is missing.

It is a numpy restatement of the reference algorithm (arxiv 2401.03555's
Python `impact` package, pkg/src/impact/*.py), each function citing the
reference file:line it follows.  Parity of the restatement itself is PINNED
against fixtures produced by running the reference in the build container
(tests/golden/make_golden.py -> tests/golden/*.npz): bitwise for
construction rows and controllers where the reference is deterministic,
within 1e-12 where the reference's own bits depend on OpenBLAS threading
(`lower @ w`, feasible.py:111).

Modules
  nm         batched projected Nelder-Mead   (optimize.py:28-162)
  construct  diagonal-noise row bounds, assemble  (abstraction.py:198-659)
  lp         greedy feasible-distribution LP  (feasible.py:53-111)
  iterate    twin interval iteration, synthesis API  (synthesis.py:79-361)
"""

"""CPU oracle for the prism-DG hot path  --  TEST INFRASTRUCTURE ONLY.

This package is a from-scratch numpy restatement of the reference algorithm
(`prismdg`, /root/reference/pkg/src/prismdg) for the functions on the hot path
(SURVEY.md section 8a).  Every function cites the reference file:line it
follows.  It is pinned against golden vectors produced by the real reference
(tests/golden/, generator scripts/make_golden.py) and is used:

  * by tests/ as the parity checker for the CUDA path,
  * by __graft_entry__.smoke() as the checker of one small invocation,
  * by bench.py as the cpu_baseline leg / the `--impl reference` arm.

The product package (paper_2605_16082_b200) never imports this package.
"""

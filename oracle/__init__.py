"""CPU oracle for the block-LU hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A plain-numpy restatement of the reference algorithm (lublock 0.1.0,
/root/reference/pkg/src/lublock) used only as the checker:

* ``oracle.structure`` — symmetrize / symbolic / Alg. 2 / curve / Alg. 3 /
  partition / dependency levels (bit-exact integer and float64 restatements);
* ``oracle.numeric``   — the dense-scratch right-looking blocked LU
  (factorize.py:38-384), residual and solve;
* ``oracle.brute``     — independent brute-force oracles restating
  pkg/tests/oracles.py (set-based fill, leading-submatrix counts, scalar
  block-pivot LU, blocking scan).

Parity is PINNED: tests/test_oracle_golden.py checks this package against
fixtures that tests/golden/make_golden.py produced by running the reference
itself (importing /root/reference/pkg/src in the build container).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product package
(paper_2512_04389_b200) never does.
"""

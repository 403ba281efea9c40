"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the PHSVDS hot path.

Restates the reference's algorithm (pkg/src/itersvd, cited per function)
in plain numpy (and C, under oracle/csrc) so tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs can check and time the
GPU path against it.  Nothing in the shipped package imports this module;
it is the checker, never the thing measured or shipped.

Pinning: oracle outputs are checked against the reference's own golden
vectors (sparse_oracle.json, clustered300x200.json, rect50x30_expected.json
copied as values into tests/golden/) and against fixtures produced by
running the reference itself in the build container
(tests/golden/make_golden.py).
"""

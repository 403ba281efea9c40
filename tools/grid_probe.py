"""Per-kernel iteration timings at config 2 (bench.iteration_kernels) under
the current SVDSB_GRID_CAP (development helper)."""
import os
import sys
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal  # noqa: E402
wl, (m, n, r, c, v) = bench.workload("c2")
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side="auto")
roof, table = bench.iteration_kernels(a, pre, wl, 6500.0, 452, [60.0])
print("cap", os.environ.get("SVDSB_GRID_CAP"), " ".join("%s=%.2f" % (k["kernel"][:14], k["us_per_launch"])
                                                       for k in table["kernels"]))

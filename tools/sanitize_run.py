"""Small end-to-end workload for compute-sanitizer runs (development
helper): smoke() (SpMV vs oracle + a 24x24 two-stage solve), a config-1
solve, a down-scaled config-2 solve (graphs, fused CGS, run-ahead) and a
b = 4 block solve of a small Zipf matrix (sliced-ELL kernels, block graphs)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import __graft_entry__ as ge  # noqa: E402
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, jacobi_precond_on_normal, workloads  # noqa

ge.smoke()
m, n, r, c, v = workloads.c1_coo(nx=32)
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
print(svds_solve(a, cfg=SvdsConfig(num_svals=10, target="largest", eps=1e-10, seed=0)).sigma)
m, n, r, c, v = workloads.c2_coo(m=20000, n=10000)
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side="auto")
print(svds_solve(a, precond=pre, cfg=SvdsConfig(num_svals=5, target="smallest", eps=1e-10, seed=0)).sigma)
m, n, r, c, v = workloads.CONFIGS["c4"].build(**workloads.SMALL["c4"])
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
res = svds_solve(a, cfg=SvdsConfig(num_svals=20, target="largest", eps=1e-6, max_block_size=4, seed=0))
print(res.sigma[:4], res.status)
print("sanitize workload done")

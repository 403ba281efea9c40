"""Reproduce bench.py's e2e leg with per-step segments (development helper).

python tools/e2e_bench_probe.py [with_iter_kernels 0|1] [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import (SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, pysvds,  # noqa: E402
                                   svds_solve)

with_ik = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
wl, (m, n, r, c, v) = bench.workload("c2")
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side="auto")
cfg = lambda: SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)  # noqa
for _ in range(6):
    res = svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
if with_ik:
    bench.iteration_kernels(a, pre, wl, 6500.0, res.stats.outer_iterations, [60.0])
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    b = p2 = None
    torch.cuda.synchronize()
    td = time.perf_counter()
    b = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    p2 = jacobi_precond_on_normal(b, side="auto")
    t1 = time.perf_counter()
    sigma, u, vv, rn, st = pysvds.svds(b, k=wl.k, which="S", tol=wl.tol, seed=0, precond=p2)
    t2 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(i, "drop %.1f" % ((td - t0) * 1e3), "coo %.1f svds %.1f tail %.1f total %.1f dev %.1f ms" % (
        (t1 - td) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t3 - t0) * 1e3, e0.elapsed_time(e1)),
        "mem %.0f MB reserved" % (torch.cuda.memory_reserved() / 1e6), flush=True)

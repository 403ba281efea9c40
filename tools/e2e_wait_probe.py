"""Per-wait timing of slow e2e steps (development helper).

Runs bench.py's order (device-timed solves, the iteration-kernel table, then
e2e solves from pinned host COO) and logs every host wait on a queued
iteration inside the e2e solves: for each step, total wait, the longest
waits and the iteration they belong to.

python tools/e2e_wait_probe.py [reps] [with_ik]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import (SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, pysvds,  # noqa: E402
                                   svds_solve)
from paper_1607_01404_b200 import eigensolver as es  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
with_ik = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl, (m, n, r, c, v) = bench.workload("c2")
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side="auto")
cfg = lambda: SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)  # noqa
for _ in range(8):
    res = svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
if with_ik:
    bench.iteration_kernels(a, pre, wl, 6500.0, res.stats.outer_iterations, [60.0])
log = []
orig = es.DavidsonSolver._wait_status


def wrapped(self, g, p, slot):
    t0 = time.perf_counter()
    out = orig(self, g, p, slot)
    log.append((t0, time.perf_counter() - t0))
    return out


es.DavidsonSolver._wait_status = wrapped
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
for i in range(reps):
    torch.cuda.synchronize()
    log.clear()
    t0 = time.perf_counter()
    b = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    p2 = jacobi_precond_on_normal(b, side="auto")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sigma, u, vv, rn, st = pysvds.svds(b, k=wl.k, which="S", tol=wl.tol, seed=0, precond=p2)
    t2 = time.perf_counter()
    waits = np.array([d for _, d in log]) * 1e3
    top = np.argsort(waits)[-4:][::-1]
    first = log[0][0] if log else t1
    print(i, "coo %.1f solve %.1f ms | waits n=%d sum %.1f median %.3f ms | pre-first-wait %.1f ms | top %s" % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, len(waits), waits.sum(), np.median(waits), (first - t1) * 1e3,
        ", ".join("#%d %.1f" % (k, waits[k]) for k in top)), flush=True)

"""Time spent capturing iteration graphs inside e2e solves (a new matrix
each step re-keys every graph) -- development helper.

python tools/capture_probe.py [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, pysvds  # noqa: E402
from paper_1607_01404_b200 import eigensolver as es  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wl, (m, n, r, c, v) = bench.workload("c2")
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
log = []
orig = es.DavidsonSolver._capture


def wrapped(self, fn, **kw):
    t0 = time.perf_counter()
    out = orig(self, fn, **kw)
    log.append(time.perf_counter() - t0)
    return out


es.DavidsonSolver._capture = wrapped
from paper_1607_01404_b200 import _lib  # noqa: E402
lib = _lib.load()
_end = lib.svdsb_graph_end
endlog = []


def end_wrapped(*a):
    t0 = time.perf_counter()
    rc = _end(*a)
    endlog.append(time.perf_counter() - t0)
    return rc


lib.svdsb_graph_end = end_wrapped
for i in range(reps):
    torch.cuda.synchronize()
    log.clear()
    endlog.clear()
    t0 = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    pre = jacobi_precond_on_normal(a, side="auto")
    sigma, u, vv, rn, st = pysvds.svds(a, k=wl.k, which="S", tol=wl.tol, seed=0, precond=pre)
    t1 = time.perf_counter()
    tot = sum(log) * 1e3
    print(i, "e2e %.1f ms, %d captures, %.1f ms capturing (%.0f us each; end+instantiate %.0f us each)" % (
        (t1 - t0) * 1e3, len(log), tot, 1e3 * tot / max(1, len(log)),
        1e6 * sum(endlog) / max(1, len(endlog))), flush=True)

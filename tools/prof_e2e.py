"""Segment timing + host profile of bench.py's e2e step (development helper).

python tools/prof_e2e.py c2 [reps]
"""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, pysvds, workloads  # noqa: E402

key = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()


def step(prof=None):
    seg = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    if prof:
        prof.enable()
    a = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    torch.cuda.synchronize(); seg["from_coo"] = time.perf_counter() - t; t = time.perf_counter()
    pre = jacobi_precond_on_normal(a, side="auto") if wl.precond else None
    torch.cuda.synchronize(); seg["precond"] = time.perf_counter() - t; t = time.perf_counter()
    sigma, u, vv, rn, stats = pysvds.svds(a, k=wl.k, which="S" if wl.which == "smallest" else "L",
                                          tol=wl.tol, seed=0, precond=pre, max_block_size=wl.block)
    torch.cuda.synchronize(); seg["svds"] = time.perf_counter() - t
    if prof:
        prof.disable()
    seg = {k: round(x * 1e3, 2) for k, x in seg.items()}
    seg["total_ms"] = round(sum(seg.values()), 2)
    return seg


for i in range(reps):
    print("step", i, step(), flush=True)
prof = cProfile.Profile()
print("profiled", step(prof), flush=True)
st = pstats.Stats(prof)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(25)

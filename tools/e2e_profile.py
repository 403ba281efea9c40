"""Where the end-to-end (host COO -> host sigma/U/V) time of a config goes
(development helper): phase timings of three e2e steps plus a cProfile of
the last one.  python tools/e2e_profile.py c4"""
import cProfile
import io
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, pysvds, workloads  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
rp = torch.from_numpy(np.ascontiguousarray(r)).pin_memory()
cp = torch.from_numpy(np.ascontiguousarray(c)).pin_memory()
vp = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()


def step(prof=None):
    t0 = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rp, cp, vp)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pre = jacobi_precond_on_normal(a, side="auto") if wl.precond else None
    out = pysvds.svds(a, k=wl.k, which="S" if wl.which == "smallest" else "L", tol=wl.tol, seed=0, precond=pre,
                      max_block_size=wl.block)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, out


for i in range(4):
    if i == 3:
        pr = cProfile.Profile()
        pr.enable()
    ta, ts, out = step()
    if i == 3:
        pr.disable()
    print("step %d: from_coo %.3f s, svds %.3f s, total %.3f s" % (i, ta, ts, ta + ts), flush=True)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumtime").print_stats(40)
print(s.getvalue()[:9000])

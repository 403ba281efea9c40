"""e2e jitter probe: repeated pysvds.svds from host COO, with Python GC
pauses logged (development helper).

python tools/e2e_jitter.py c2 [reps]
"""
import gc
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, pysvds, workloads  # noqa: E402

key = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
gc_log = []
_t = {}


def cb(phase, info):
    if phase == "start":
        _t["s"] = time.perf_counter()
    else:
        gc_log.append((info["generation"], (time.perf_counter() - _t["s"]) * 1e3))


gc.callbacks.append(cb)


def step():
    torch.cuda.synchronize()
    t = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    pre = jacobi_precond_on_normal(a, side="auto") if wl.precond else None
    out = pysvds.svds(a, k=wl.k, which="S" if wl.which == "smallest" else "L", tol=wl.tol, seed=0,
                      precond=pre, max_block_size=wl.block)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, out[4]


for mode in ("gc on", "gc frozen"):
    if mode == "gc frozen":
        gc.collect()
        gc.freeze()
    ts = []
    for i in range(reps):
        del gc_log[:]
        dt, st = step()
        ts.append(dt)
        print(mode, i, round(dt, 2), "gc:", [(g, round(x, 2)) for g, x in gc_log], flush=True)
    print(mode, "median", np.median(ts), "max", np.max(ts), "mean", np.mean(ts), flush=True)

"""Config-4 C-apply (b = 4) kernel breakdown (development helper): builds
the config-4 matrix and runs the normal operator a few times so an ncu
launch list shows every sub-kernel (sliced-ELL forward, per-block
transposed slices, chunk path, fix-up).

python tools/c4_breakdown.py [reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, make_normal_operator, workloads  # noqa
from paper_1607_01404_b200 import device as dv  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
from paper_1607_01404_b200 import _lib  # noqa: E402
import os  # noqa: E402
for kv in filter(None, os.environ.get("SVDSB_TUNE", "").split(",")):   # e.g. SVDSB_TUNE=7=1
    k, v = kv.split("=")
    _lib.call("svdsb_tune_set", int(k), int(v))
t0 = time.perf_counter()
m, n, r, c, v = workloads.CONFIGS["c4"].build()
print("gen %.1f s" % (time.perf_counter() - t0), flush=True)
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
dev = a.device_csr()
op = make_normal_operator(SvdOperator.from_csr(a, check=False))
x = dv.to_device_block(np.random.default_rng(3).standard_normal((n, 4)))
y = dv.new_block(n, 4)
ym = dv.new_block(m, 4)
yy = dv.to_device_block(np.random.default_rng(4).standard_normal((m, 4)))
op.apply_into(x, y)
torch.cuda.synchronize()
# row-length statistics of A^T per column block
hp = a.row_ptr
print("A rows", m, "nnz", a.nnz, flush=True)
for i in range(reps):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    op.apply_into(x, y)
    e1.record()
    torch.cuda.synchronize()
    print("C-apply b=4: %.1f us" % (e0.elapsed_time(e1) * 1e3), flush=True)
for name, fn in (("fwd", lambda: dev.matvec(x, ym, False)), ("adj", lambda: dev.matvec(yy, y, True))):
    for i in range(reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i:
            print("%s b=4: %.1f us" % (name, e0.elapsed_time(e1) * 1e3), flush=True)
print("checksum", float(y.sum()), float(ym.sum()), flush=True)

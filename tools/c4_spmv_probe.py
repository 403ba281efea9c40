"""Config-4 SpMV launches for ncu (development helper): one warm A.X and
A^T.Y at b = 1 and b = 4 after a warm-up pass."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads
from paper_1607_01404_b200 import device as dv
wl = workloads.CONFIGS["c4"]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
dev = a.device_csr()
for b in (1, 4):
    x = dv.to_device_block(np.random.default_rng(0).standard_normal((n, b)))
    y = dv.new_block(m, b)
    yy = dv.to_device_block(np.random.default_rng(1).standard_normal((m, b)))
    z = dv.new_block(n, b)
    for _ in range(2):
        dev.matvec(x, y, False)
        dev.matvec(yy, z, True)
torch.cuda.synchronize()
print("done")

"""Time the pieces of a fresh config-4 matrix in the e2e path (development
helper): device assembly, the first b = 4 forward / transposed products
(which build the sliced-ELL copies) and the same products again."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads  # noqa: E402
from paper_1607_01404_b200 import device as dv  # noqa: E402

m, n, r, c, v = workloads.CONFIGS["c4"].build()
rp = torch.from_numpy(r).pin_memory()
cp = torch.from_numpy(c).pin_memory()
vp = torch.from_numpy(v).pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rp, cp, vp)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dev = a.device_csr()
    x = dv.to_device_block(np.ones((n, 4)))
    y = dv.new_block(m, 4)
    z = dv.new_block(n, 4)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev.matvec(x, y, False)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    dev.matvec(y, z, True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    dev.matvec(x, y, False)
    dev.matvec(y, z, True)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print("assembly %.3f  first fwd %.3f  first adj %.3f  again both %.3f" % (t1 - t0, t3 - t2, t4 - t3, t5 - t4),
          flush=True)
    del a, dev

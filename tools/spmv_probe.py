"""Run each SpMV variant of one config a couple of times (ncu target)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, make_normal_operator, workloads
from paper_1607_01404_b200 import device as dv
key = sys.argv[1]
bs = [int(b) for b in sys.argv[2].split(',')] if len(sys.argv) > 2 else [1]
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
op = make_normal_operator(SvdOperator.from_csr(a, check=False))
for b in bs:
    x = dv.to_device_block(np.random.default_rng(3).standard_normal((op.dim, b)))
    y = dv.new_block(op.dim, b)
    for _ in range(2):
        op.apply_into(x, y)
torch.cuda.synchronize()
print("ok")

"""Config-4 assembly time from pinned host COO (development helper; SVDSB_TRACE=0 prints the phases)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads
m, n, r, c, v = workloads.c4_coo()
rp, cp, vp = [torch.from_numpy(t).pin_memory() for t in (r, c, v)]
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rp, cp, vp)
    torch.cuda.synchronize(); print("from_coo %.3f s" % (time.perf_counter() - t0), flush=True)
    del a

"""Timing of the device CSR assembly from host COO (development helper).
python tools/coo_probe.py c2"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads, _lib  # noqa: E402
from paper_1607_01404_b200.device import context  # noqa: E402

wl = workloads.CONFIGS[sys.argv[1]]
m, n, r, c, v = wl.build()
rp, cp, vp = (torch.from_numpy(a).pin_memory() for a in (r, c, v))
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rd, cd, vd = (x.to("cuda", non_blocking=True) for x in (rp, cp, vp))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx = context()
    h = ctypes.c_void_p()
    _lib.call("svdsb_csr_create_coo_device", ctx.handle, m, n, rd.numel(), ctypes.c_void_p(rd.data_ptr()),
              ctypes.c_void_p(cd.data_ptr()), ctypes.c_void_p(vd.data_ptr()), _lib.SVDSB_CSR_TRANSPOSE,
              ctx.stream, ctypes.byref(h))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    _lib.call("svdsb_csr_destroy", h)
    t3 = time.perf_counter()
    a = SparseMatrixCsr.from_coo(m, n, rp, cp, vp)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print("h2d %.2f ms, create %.2f ms, destroy %.2f ms, from_coo total %.2f ms" %
          ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3))

"""Segment the host-COO assembly (development helper)."""
import sys
import time

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200.matrix import DeviceCsr  # noqa: E402

wl, (m, n, r, c, v) = bench.workload("c2")
rows = torch.from_numpy(r).pin_memory()
cols = torch.from_numpy(c).pin_memory()
vals = torch.from_numpy(v).pin_memory()
print("threads", torch.get_num_threads(), flush=True)
keep = None
for i in range(16):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    a, b = int(rows.min()), int(rows.max())
    t.append(time.perf_counter())
    a, b = int(cols.min()), int(cols.max())
    t.append(time.perf_counter())
    d = DeviceCsr.from_coo_device(m, n, rows, cols, vals)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    keep = None
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    keep = d
    del d
    print(i, " ".join("%.2f" % ((t[j + 1] - t[j]) * 1e3) for j in range(len(t) - 1)), flush=True)

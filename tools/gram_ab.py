"""Time the b = 1..4 Gram / projection kernels at config-4 size (N = 1M,
g = 35); run once per SVDSB_LIB_VARIANT for an A/B (development helper)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import device as dv  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = dv.context()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for g in (20, 35):
    V = dv.new_block(N, g)
    V.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda').t())
    for b in (1, 2, 3, 4, 14):
        y = dv.new_block(N, b)
        y.copy_(torch.randn(b, N, dtype=torch.float64, device='cuda').t())
        C = dv.small_matrix(g, b)
        nr = torch.zeros(b, dtype=torch.float64, device='cuda')
        t = timeit(lambda: dv.gram(ctx, N, [V], y, C, norms2=nr))
        print("g=%d b=%d gram %.1f us  %.0f GB/s" % (g, b, t, 8 * N * (g + b) / t / 1e3), flush=True)

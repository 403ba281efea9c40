import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1607_01404_b200 import device as dv, _lib
ctx = dv.context()
rng = np.random.default_rng(0)
for g0 in (14, 25, 34):
    g = g0 + 1
    a = rng.standard_normal((g, g)); h = a + a.T
    l0, y0 = np.linalg.eigh(h[:g0, :g0])
    H = dv.to_device_block(h); Y0 = dv.to_device_block(y0); L0 = torch.as_tensor(l0, device='cuda')
    w = torch.zeros(g, dtype=torch.float64, device='cuda'); Y = dv.small_matrix(g, g)
    for order in (0, 1):
        for _ in range(3): dv.syev_update(ctx, H, g0, 1, Y0, L0, order, 0.0, w, Y)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): dv.syev_update(ctx, H, g0, 1, Y0, L0, order, 0.0, w, Y)
        e1.record(); torch.cuda.synchronize()
        print("g0", g0, "order", order, "us/launch", e0.elapsed_time(e1) / 20 * 1e3)
    for _ in range(3): dv.syev_small(ctx, H, g, 1, 0.0, w, Y)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): dv.syev_small(ctx, H, g, 1, 0.0, w, Y)
    e1.record(); torch.cuda.synchronize()
    print("  jacobi us/launch", e0.elapsed_time(e1) / 20 * 1e3)

"""Ritz-residual kernel variants at BASELINE sizes (development helper):
config 3 (N = 4.1 M, p = 11), config 4 (N = 1 M, p = 24), config 2
(N = 100 k, p = 6) with g = 35 (25 for config 2); svdsb_tune_set key 3.

python tools/ritz_variants.py [key]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import _lib  # noqa: E402
from paper_1607_01404_b200 import device as dv  # noqa: E402

peak = 6551.0
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


ctx = dv.context()
KEY = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for name, N, g, p in (("c3", 4096000, 35, 11), ("c4", 1000000, 35, 24), ("c2", 100000, 25, 6), ("c4p20", 1000000, 35, 20)):
    gen = torch.Generator(device='cuda').manual_seed(0)
    V = dv.new_block(N, g)
    V.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda', generator=gen).t())
    W = dv.new_block(N, g)
    W.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda', generator=gen).t())
    Y = dv.to_device_block(np.linalg.qr(np.random.default_rng(2).standard_normal((g, g)))[0])
    lam = torch.randn(g, dtype=torch.float64, device='cuda', generator=gen)
    ref = None
    for val in (1, 0):
        _lib.call("svdsb_tune_set", KEY, val)
        R = dv.new_block(N, p)
        rn2 = torch.zeros(p, dtype=torch.float64, device='cuda')
        t = timeit(lambda: dv.ritz_residual(ctx, V, W, Y[:, :p], lam[:p], R, rn2=rn2))
        byt = 8 * N * (2 * g + p)
        same = None
        if ref is None:
            ref = (R.clone(), rn2.clone())
        else:
            same = bool(torch.equal(R, ref[0]))
            rel = float(((rn2 - ref[1]).abs() / ref[1]).max())
        print(name, "tune[%d]=%d" % (KEY, val), json.dumps({"us": round(t * 1e6, 1), "frac": round(byt / t / 1e9 / peak, 3),
                                                    "R_bit_equal": same,
                                                    "rn2_rel": None if same is None else rel}), flush=True)
    _lib.call("svdsb_tune_set", KEY, 0)

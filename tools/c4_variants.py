"""Config-4 kernel variants side by side (development helper): times the
forward b = 4 SpMV and the normal-operator apply under each value of a
svdsb_tune_set knob, checks the variants agree bit for bit.

python tools/c4_variants.py [key] [values...]     (default: key 0, values 0 2)
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, _lib, make_normal_operator, workloads  # noqa
from paper_1607_01404_b200 import device as dv  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 0
values = [int(a) for a in sys.argv[2:]] or [0, 2]
peak = 6551.0
t0 = time.perf_counter()
m, n, r, c, v = workloads.CONFIGS["c4"].build()
print("gen %.1f s" % (time.perf_counter() - t0), flush=True)
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
dev = a.device_csr()
nnz = a.nnz
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


b = 4
x = dv.to_device_block(np.random.default_rng(0).standard_normal((n, b)))
op = make_normal_operator(SvdOperator.from_csr(a, check=False))
out = {}
ref_y = ref_z = ref_a = None
for val in values:
    _lib.call("svdsb_tune_set", key, val)
    y = dv.new_block(m, b)
    t = timeit(lambda: dev.matvec(x, y, False))
    byt = 12 * nnz + 4 * (m + 1) + 8 * b * (m + n)
    yy = dv.to_device_block(np.random.default_rng(1).standard_normal((m, b)))
    za = dv.new_block(n, b)
    ta = timeit(lambda: dev.matvec(yy, za, True))
    same_a = ref_a is None or bool(torch.equal(za, ref_a))
    if ref_a is None:
        ref_a = za.clone()
    ba = 12 * nnz + 4 * (n + 1) + 8 * b * (m + n)
    z = dv.new_block(n, b)
    tn = timeit(lambda: op.apply_into(x, z))
    bn = 2 * (12 * nnz) + 4 * (m + n + 2) + 2 * 8 * b * (m + n)
    same_y = ref_y is None or bool(torch.equal(y, ref_y))
    same_z = ref_z is None or bool(torch.equal(z, ref_z))
    if ref_y is None:
        ref_y, ref_z = y.clone(), z.clone()
    g = 35
    V = dv.new_block(n, g)
    V.copy_(torch.randn(g, n, dtype=torch.float64, device='cuda').t())
    ctx = dv.context()
    C = dv.small_matrix(g, b)
    nr = torch.zeros(b, dtype=torch.float64, device='cuda')
    tg = timeit(lambda: dv.gram(ctx, n, [V], x, C, norms2=nr))
    bg = 8 * n * (g + b)
    xp = x.clone()
    tp = timeit(lambda: dv.project_out(ctx, n, [V], C, xp, norms2=nr))
    bp = 8 * n * (g + 2 * b)
    extra = {"gram_b4_us": tg * 1e6, "gram_frac": bg / tg / 1e9 / peak, "project_b4_us": tp * 1e6,
             "project_frac": bp / tp / 1e9 / peak, "C_head": float(C[0, 0])}
    extra.update({"adj_b4_us": ta * 1e6, "adj_frac": ba / ta / 1e9 / peak, "adj_bit_equal": same_a})
    out[val] = {**extra, "fwd_b4_us": t * 1e6, "fwd_frac": byt / t / 1e9 / peak, "normal_b4_us": tn * 1e6,
                "normal_frac": bn / tn / 1e9 / peak, "fwd_bit_equal": same_y, "normal_bit_equal": same_z}
    print("tune[%d]=%d" % (key, val), json.dumps(out[val]), flush=True)
_lib.call("svdsb_tune_set", key, 0)

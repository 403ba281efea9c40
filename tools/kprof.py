"""Each hot-path operation of a config once, between cudaProfilerStart/Stop,
for an ncu capture that maps kernels back to operations (development
helper for profiles/traffic_<cfg>.json).

    ncu --set full --profile-from-start off ... python tools/kprof.py c3L|c4

Writes gpurun_out/kprof_<cfg>_ops.json: the operations in launch order with
the number of libsvdsb launches each made and its algorithmic bytes
(SURVEY 8(d) formulas); tools/traffic_from_ncu.py sums the ncu DRAM bytes
per operation."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, make_normal_operator, workloads, _lib  # noqa: E402
from paper_1607_01404_b200 import device as dv  # noqa: E402

key = sys.argv[1]
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
nnz = a.nnz
dev = a.device_csr()
ctx = dv.context()
op = make_normal_operator(SvdOperator.from_csr(a, check=False))
b = wl.block
N, g = n, 35
p = min(wl.k + b, g)
s = 15
s2 = min(wl.k + b, 32)
gen = torch.Generator(device="cuda")
gen.manual_seed(5)


def rnd(rows, cols):
    out = dv.new_block(rows, cols)
    out.copy_(torch.randn(cols, rows, generator=gen, dtype=torch.float64, device="cuda").t())
    return out


V, W = rnd(N, g), rnd(N, g)
Y = dv.to_device_block(np.linalg.qr(np.random.default_rng(2).standard_normal((g, g)))[0])
lam = torch.randn(g, dtype=torch.float64, device="cuda", generator=gen)
xb, yb = rnd(n, b), rnd(m, b)
ym, zn = dv.new_block(m, b), dv.new_block(n, b)
R = dv.new_block(N, p)
rn2 = torch.zeros(p, dtype=torch.float64, device="cuda")
C = dv.small_matrix(g, b)
nr = torch.zeros(b, dtype=torch.float64, device="cuda")
C1 = dv.small_matrix(g, 1)
nr1 = torch.zeros(1, dtype=torch.float64, device="cuda")
y1 = rnd(N, 1)
V2 = dv.new_block(N, g)
V2.copy_(V)

spmv_f = 12 * nnz + 4 * (m + 1) + 8 * b * (m + n)
spmv_t = 12 * nnz + 4 * (n + 1) + 8 * b * (m + n)
ops = [
    ("spmv_fwd_b%d" % b, lambda: dev.matvec(xb, ym, False), spmv_f),
    ("spmv_adj_b%d" % b, lambda: dev.matvec(yb, zn, True), spmv_t),
    ("normal_b%d" % b, lambda: op.apply_into(xb, zn), spmv_f + spmv_t),
    ("gram_b%d_g35" % b, lambda: dv.gram(ctx, N, [V], W[:, :b], C, norms2=nr), 8 * N * (g + b)),
    ("project_b%d_g35" % b, lambda: dv.project_out(ctx, N, [V], C, W[:, g - b:g], norms2=nr), 8 * N * (g + 2 * b)),
    ("cgs_gram_b1_g35", lambda: dv.gram(ctx, N, [V], y1, C1, norms2=nr1), 8 * N * (g + 1)),
    ("cgs_project_b1_g35", lambda: dv.project_out(ctx, N, [V], C1, y1, norms2=nr1), 8 * N * (g + 2)),
    ("ritz_residual_g35_p%d" % p, lambda: dv.ritz_residual(ctx, V, W, Y[:, :p], lam[:p], R, rn2=rn2),
     8 * N * (2 * g + p)),
    ("restart_inplace_35to%d" % s, lambda: dv.ts_gemm(ctx, V2, Y[:, :s], V2[:, :s]), 8 * N * (g + s)),
    ("restart_inplace_35to%d" % s2, lambda: dv.ts_gemm(ctx, V2, Y[:, :s2], V2[:, :s2]), 8 * N * (g + s2)),
]
for _ in range(2):
    for _, fn, _ in ops:
        fn()
torch.cuda.synchronize()
order = []
torch.cuda.profiler.start()
for name, fn, byt in ops:
    l0 = _lib.launch_count()
    fn()
    torch.cuda.synchronize()
    order.append({"op": name, "launches": _lib.launch_count() - l0, "algorithmic_bytes": byt})
torch.cuda.profiler.stop()
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"config": key, "m": m, "n": n, "nnz": nnz, "block": b, "g": g, "p": p, "ops": order},
          open("gpurun_out/kprof_%s_ops.json" % key, "w"), indent=1)
print(json.dumps(order))

"""Standalone kernel throughput at BASELINE sizes (development helper).
python tools/kbench.py c3L|c4 ..."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads, _lib
from paper_1607_01404_b200 import device as dv

def timeit(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))

key = sys.argv[1]
peak = 6488.0
wl = workloads.CONFIGS[key]
t0 = time.perf_counter()
m, n, r, c, v = wl.build()
print(f"gen {time.perf_counter()-t0:.1f}s", flush=True)
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
dev = a.device_csr(); ctx = dv.context(); nnz = a.nnz
out = {}
for b in sorted({1, wl.block}):
    x = dv.to_device_block(np.random.default_rng(0).standard_normal((n, b)))
    y = dv.new_block(m, b)
    t = timeit(lambda: dev.matvec(x, y, False))
    byt = 12 * nnz + 4 * (m + 1) + 8 * b * (m + n)
    out[f"spmv_fwd_b{b}"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
    yy = dv.to_device_block(np.random.default_rng(1).standard_normal((m, b)))
    z = dv.new_block(n, b)
    t = timeit(lambda: dev.matvec(yy, z, True))
    byt = 12 * nnz + 4 * (n + 1) + 8 * b * (m + n)
    out[f"spmv_adj_b{b}"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
N = n; g = 35; p = min(wl.k + wl.block, g)
rng = np.random.default_rng(2)
V = dv.new_block(N, g); V.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda').t())
W = dv.new_block(N, g); W.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda').t())
Y = dv.to_device_block(np.linalg.qr(rng.standard_normal((g, g)))[0])
lam = torch.randn(g, dtype=torch.float64, device='cuda')
R = dv.new_block(N, p); rn2 = torch.zeros(p, dtype=torch.float64, device='cuda')
t = timeit(lambda: dv.ritz_residual(ctx, V, W, Y[:, :p], lam[:p], R, rn2=rn2))
byt = 8 * N * (2 * g + p); out["ritz_residual"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
for bb in sorted({1, wl.block}):
    vcol = dv.new_block(N, bb); vcol.copy_(torch.randn(bb, N, dtype=torch.float64, device='cuda').t())
    C = dv.small_matrix(g, bb); nr = torch.zeros(bb, dtype=torch.float64, device='cuda')
    t = timeit(lambda: dv.gram(ctx, N, [V], vcol, C, norms2=nr))
    byt = 8 * N * (g + bb); out[f"gram_b{bb}"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
    t = timeit(lambda: dv.project_out(ctx, N, [V], C, vcol, norms2=nr))
    byt = 8 * N * (g + 2 * bb); out[f"project_b{bb}"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
s = 15
V2 = dv.new_block(N, s)
t = timeit(lambda: dv.ts_gemm(ctx, V, Y[:, :s], V2))
byt = 8 * N * (g + s); out["ts_gemm_35x15"] = (t * 1e6, byt / t / 1e9, byt / t / 1e9 / peak)
for k, (us, gbs, frac) in out.items():
    print(f"{k:18s} {us:10.1f} us {gbs:8.1f} GB/s  {100*frac:5.1f}% of HBM")
print(json.dumps({k: {"us": v[0], "gbs": v[1], "frac": v[2]} for k, v in out.items()}))
# normal operator (both products, block operands staged row-major)
from paper_1607_01404_b200 import SvdOperator, make_normal_operator
op = make_normal_operator(SvdOperator.from_csr(a, check=False))
for b in sorted({1, wl.block}):
    x = dv.to_device_block(np.random.default_rng(3).standard_normal((op.dim, b)))
    y = dv.new_block(op.dim, b)
    t = timeit(lambda: op.apply_into(x, y))
    byt = 2 * (12 * nnz) + 4 * (m + n + 2) + 2 * 8 * b * (m + n)
    print(f"normal_apply_b{b:<6d} {t*1e6:10.1f} us {byt/t/1e9:8.1f} GB/s  {100*byt/t/1e9/peak:5.1f}% of HBM")

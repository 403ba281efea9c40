"""Warm per-kernel time of the single-column iteration kernels at a config's
size (development helper).

python tools/iter_probe.py c2 [g]

Each kernel is launched `reps` times back to back between two CUDA events
(no L2 flush: inside a solve the basis of configs 1/2 is L2-resident), so
the figure is the per-launch cost as a graph replay sees it.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, workloads, _lib  # noqa: E402
from paper_1607_01404_b200 import device as dv  # noqa: E402

key = sys.argv[1]
g = int(sys.argv[2]) if len(sys.argv) > 2 else 30
reps = 200
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
dev = a.device_csr()
ctx = dv.context()
N = n
p = min(wl.k + wl.block, g + 1)
rng = np.random.default_rng(0)


def timeit(fn):
    """Device time per call: `reps` calls captured in one CUDA graph (the
    host launch rate of eager calls would hide the kernel time)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    old = ctx._stream
    with torch.cuda.stream(cap):
        ctx._stream = cap.cuda_stream
        graph.capture_begin()
        for _ in range(reps):
            fn()
        graph.capture_end()
    ctx._stream = old
    torch.cuda.current_stream().wait_stream(cap)
    graph.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    graph.replay()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


V = dv.new_block(N, g + 1)
V.copy_(torch.linalg.qr(torch.randn(N, g + 1, dtype=torch.float64, device='cuda'))[0])
W = dv.new_block(N, g + 1)
W.copy_(torch.randn(g + 1, N, dtype=torch.float64, device='cuda').t())
col = dv.new_block(N, 1)
col.copy_(torch.randn(1, N, dtype=torch.float64, device='cuda').t())
res = dv.new_block(N, 1)
res.copy_(col)
tmp = dv.new_block(m, 1)
hc = dv.small_matrix(g + 2, 1)
H = dv.small_matrix(64, 64)
h0 = rng.standard_normal((g + 1, g + 1))
H[:g + 1, :g + 1].copy_(torch.from_numpy(h0 + h0.T))
lam0, y0 = np.linalg.eigh(h0[:g, :g] + h0[:g, :g].T)
Y0 = dv.to_device_block(y0)
L0 = torch.from_numpy(lam0).cuda()
lams = torch.zeros(64, dtype=torch.float64, device='cuda')
Y = dv.small_matrix(64, 64)
R = dv.new_block(N, p)
rn2 = torch.zeros(p, dtype=torch.float64, device='cuda')
st = torch.zeros(8, dtype=torch.float64, device='cuda')
cw = torch.zeros(1024, dtype=torch.float64, device='cuda')
pre = jacobi_precond_on_normal(a, side='auto')
nrm = torch.ones(1, dtype=torch.float64, device='cuda')

n_, ptrs, lds, cols, _ = dv._blk_args([V[:, :g]])
out = {}
out["axpby (residual copy)"] = timeit(lambda: dv.axpby(ctx, 1.0, res, 0.0, col))
out["diag_solve (precond)"] = timeit(lambda: pre._into(res, col))
out["dgks_begin"] = timeit(lambda: _lib.call("svdsb_dgks_begin", dv.P(st), ctx.stream))


st_on = torch.zeros(8, dtype=torch.float64, device='cuda')
st_on[0] = 1.0


def cgs_pass():
    st.copy_(st_on)
    _lib.call("svdsb_cgs_pass", ctx.handle, N, n_, ptrs, lds, cols, dv.P(col), dv.P(cw), dv.P(st), 1, ctx.stream)


def cgs_gated():
    st.zero_()
    _lib.call("svdsb_cgs_pass", ctx.handle, N, n_, ptrs, lds, cols, dv.P(col), dv.P(cw), dv.P(st), 0, ctx.stream)


t_zero = timeit(lambda: st.copy_(st_on))
out["cgs_pass active (gram1+project1)"] = timeit(cgs_pass) - t_zero
out["cgs_pass gated off"] = timeit(cgs_gated) - timeit(lambda: st.zero_())
out["scale (normalise)"] = timeit(lambda: dv.scale_cols(ctx, col, nrm, dv.SCALE_DIV))
out["spmv A x"] = timeit(lambda: dev.matvec(col, tmp, False))
out["spmv A^T y"] = timeit(lambda: dev.matvec(tmp, W[:, g:g + 1], True))
out["gram (H column)"] = timeit(lambda: dv.gram(ctx, N, [V[:, :g + 1]], W[:, g:g + 1], hc[:g + 1, :]))
out["h_insert"] = timeit(lambda: dv.h_insert(ctx, g, 1, hc[:g + 1, :], H))
out["syev_update"] = timeit(lambda: dv.syev_update(ctx, H, g, 1, Y0, L0, 0, 0.0, lams[:g + 1], Y[:g + 1, :g + 1]))
out["ritz_residual p=%d" % p] = timeit(lambda: dv.ritz_residual(ctx, V[:, :g + 1], W[:, :g + 1], Y[:g + 1, :p],
                                                                 lams[:p], R, rn2=rn2))
tot = 0.0
for k, us in out.items():
    print("%-36s %7.2f us" % (k, us))
    tot += us
print("%-36s %7.2f us  (N=%d, g=%d)" % ("sum (3 cgs passes: 2 active)", tot + out["cgs_pass active (gram1+project1)"]
                                        - out["cgs_pass gated off"] * 0, N, g))

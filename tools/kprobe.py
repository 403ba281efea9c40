"""One warm launch of each hot kernel at a config's size (ncu target)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, workloads
from paper_1607_01404_b200 import device as dv
key = sys.argv[1] if len(sys.argv) > 1 else 'c3L'
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
dev = a.device_csr(); ctx = dv.context()
N, g, p, s = n, 35, min(wl.k + wl.block, 35), 15
x = dv.to_device_block(np.random.default_rng(0).standard_normal((n, 1)))
y = dv.new_block(m, 1); z = dv.new_block(n, 1)
V = dv.new_block(N, g); V.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda').t())
W = dv.new_block(N, g); W.copy_(torch.randn(g, N, dtype=torch.float64, device='cuda').t())
Y = dv.to_device_block(np.linalg.qr(np.random.default_rng(2).standard_normal((g, g)))[0])
lam = torch.randn(g, dtype=torch.float64, device='cuda')
R = dv.new_block(N, p); rn2 = torch.zeros(p, dtype=torch.float64, device='cuda')
vcol = dv.new_block(N, 1); vcol.copy_(torch.randn(1, N, dtype=torch.float64, device='cuda').t())
C = dv.small_matrix(g, 1); nr = torch.zeros(1, dtype=torch.float64, device='cuda')
V2 = dv.new_block(N, s)
for _ in range(2):
    dev.matvec(x, y, False)
    dev.matvec(y, z, True)
    dv.ritz_residual(ctx, V, W, Y[:, :p], lam[:p], R, rn2=rn2)
    dv.gram(ctx, N, [V], vcol, C, norms2=nr)
    dv.project_out(ctx, N, [V], C, vcol, norms2=nr)
    dv.ts_gemm(ctx, V, Y[:, :s], V2)
torch.cuda.synchronize()
print("ok")

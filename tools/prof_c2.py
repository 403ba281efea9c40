import cProfile, pstats, sys, io, time
import torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, jacobi_precond_on_normal, workloads
wl = workloads.CONFIGS['c2']
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side='auto')
cfg = lambda: SvdsConfig(num_svals=5, target='smallest', eps=1e-10, seed=0)
svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
pr.disable()
print("wall", time.perf_counter() - t)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(25)
print(s.getvalue()[:6000])

"""cProfile of the host side of one config solve (development helper).

python tools/host_profile.py c4"""
import cProfile
import io
import pstats
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, jacobi_precond_on_normal, workloads  # noqa

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None


def cfg():
    return SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)


for _ in range(2):
    svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t)
for key_ in ("tottime", "cumtime"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key_).print_stats(30)
    print(s.getvalue()[:7000])

"""Host-side profile of one warm solve (development helper).

python tools/prof_host.py c2 [small|full] [warm_reps]
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import (SparseMatrixCsr, SvdsConfig, svds_solve,  # noqa: E402
                                   jacobi_precond_on_normal, workloads)

key = sys.argv[1]
small = len(sys.argv) > 2 and sys.argv[2] == 'small'
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build(**(workloads.SMALL[key] if small else {}))
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None


def solve():
    cfg = SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)
    return svds_solve(a, precond=pre, cfg=cfg, return_device=True)


for _ in range(warm):
    solve()
torch.cuda.synchronize()
prof = cProfile.Profile()
t = time.perf_counter()
prof.enable()
solve()
torch.cuda.synchronize()
prof.disable()
print("profiled solve %.4f s" % (time.perf_counter() - t))
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(35)
st.sort_stats("cumulative").print_stats(30)

"""Per-inner-solve log of a JDQMR solve (development helper).

JD=1 LFAC=.. ETOL=.. python tools/jd_diag.py c2 [small] [budget]
"""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, eigensolver, jacobi_precond_on_normal, svds_solve, workloads  # noqa

key = sys.argv[1]
small = len(sys.argv) > 2 and sys.argv[2] == 'small'
budget = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build(**(workloads.SMALL[key] if small else {}))
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None
jdo = {"method": "JDQMR"}
for env, key2, typ in (("LFAC", "inner_lfac", float), ("ETOL", "inner_etol_frac", float),
                       ("MAXIN", "max_inner_iterations", int)):
    if os.environ.get(env):
        jdo[key2] = typ(os.environ[env])
log = eigensolver.JD_LOG = []
res = svds_solve(a, precond=pre, cfg=SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block,
                                                 seed=0, max_matvecs=budget, stage1_opts=jdo))
print("conv", res.converged.all(), "mv", res.stats.stage1_matvecs, "inner", res.stats.inner_iterations,
      "outer", res.stats.outer_iterations, jdo)
print("reasons", collections.Counter(x[3] for x in log))
its = np.array([x[2] for x in log])
print("inner its: mean %.1f median %d max %d" % (its.mean(), np.median(its), its.max()))
for i, (th, rn, it, why, er) in enumerate(log):
    if i < 40 or i % 10 == 0:
        print("%4d theta %.10g rnorm %.3e it %3d %-10s eres %.3e ratio %.3f" % (i, th, rn, it, why, er, er / rn))

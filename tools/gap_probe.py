"""Device busy time vs gaps between graphed iterations of one warm solve
(development helper).  python tools/gap_probe.py c2"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import (SparseMatrixCsr, SvdsConfig, svds_solve,  # noqa: E402
                                   jacobi_precond_on_normal, workloads)
from paper_1607_01404_b200 import eigensolver as es  # noqa: E402

key = sys.argv[1]
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None
cfg = lambda: SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)  # noqa
for _ in range(2):
    svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()

marks = []
orig = es.DavidsonSolver._launch_iter


def wrapped(self, *args, **kw):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(self.ctx.torch_stream)
    out = orig(self, *args, **kw)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(self.ctx.torch_stream)
    marks.append((e0, e1))
    return out


es.DavidsonSolver._launch_iter = wrapped
s0 = torch.cuda.Event(enable_timing=True)
s1 = torch.cuda.Event(enable_timing=True)
s0.record()
res = svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
s1.record()
torch.cuda.synchronize()
busy = [e0.elapsed_time(e1) * 1e3 for e0, e1 in marks]
gaps = [marks[i][1].elapsed_time(marks[i + 1][0]) * 1e3 for i in range(len(marks) - 1)]
tot = s0.elapsed_time(s1) * 1e3
print("solve %.1f us, %d graph replays, busy sum %.1f us (mean %.1f), gap sum %.1f us (median %.1f, p90 %.1f)"
      % (tot, len(busy), sum(busy), np.mean(busy), sum(gaps), np.median(gaps), np.percentile(gaps, 90)))
print("outside graphs: %.1f us" % (tot - sum(busy) - sum(gaps)))

# restarts: device time between events around DavidsonSolver.restart
rmarks = []
orig_restart = es.DavidsonSolver.restart


def wrapped_restart(self, *args, **kw):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(self.ctx.torch_stream)
    out = orig_restart(self, *args, **kw)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(self.ctx.torch_stream)
    rmarks.append((e0, e1))
    return out


es.DavidsonSolver.restart = wrapped_restart
marks.clear()
s0.record()
res = svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
s1.record()
torch.cuda.synchronize()
rt = [e0.elapsed_time(e1) * 1e3 for e0, e1 in rmarks]
print("restarts: %d, total %.1f us, mean %.1f us" % (len(rt), sum(rt), np.mean(rt) if rt else 0.0))
first = marks[0][0]
print("before first graph: %.1f us; after last graph: %.1f us" % (s0.elapsed_time(first) * 1e3,
                                                                   marks[-1][1].elapsed_time(s1) * 1e3))

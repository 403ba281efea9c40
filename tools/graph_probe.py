"""GPU time of one captured Davidson iteration vs the host loop around it
(development helper).

python tools/graph_probe.py c2 [reps]

Runs one warm solve, then replays each captured iteration graph `reps`
times back to back (no host sync in between) and reports the device time
per replay next to the solve's wall time per iteration.
"""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import (SparseMatrixCsr, SvdsConfig, svds_solve,  # noqa: E402
                                   jacobi_precond_on_normal, workloads)
from paper_1607_01404_b200 import eigensolver as es  # noqa: E402

key = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None
cfg = SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = svds_solve(a, precond=pre, cfg=cfg, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
print("solve %.4f s, %d iterations, %.1f us/iteration wall" %
      (wall, res.stats.outer_iterations, 1e6 * wall / max(res.stats.outer_iterations, 1)))
rows = []
for ws_list in es._POOL.values():
    for ws in ws_list:
        for k, (graph, nl) in ws.graphs.items():
            s = torch.cuda.current_stream()
            graph.replay(torch.cuda.current_stream().cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                graph.replay(torch.cuda.current_stream().cuda_stream)
            e1.record(s)
            e1.synchronize()
            rows.append((k[3], k[2], nl, e0.elapsed_time(e1) * 1e3 / reps))
rows.sort()
for g0, kind, nl, us in rows:
    print("g0=%3d kind=%-5s kernels=%2d  %.1f us/replay" % (g0, kind, nl, us))

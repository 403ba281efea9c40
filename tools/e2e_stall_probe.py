"""Where do slow e2e steps lose their time? (development helper)

Repeats bench.py's e2e leg (pysvds.svds from pinned host COO on config 2)
and logs, per step: wall time, this thread's CPU time, voluntary and
involuntary context switches, the device span between events recorded at
the step's ends, and the box's load average; at the end the busiest other
processes on the host (from /proc).

python tools/e2e_stall_probe.py [reps]
"""
import os
import resource
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import SparseMatrixCsr, jacobi_precond_on_normal, pysvds  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
wl, (m, n, r, c, v) = bench.workload("c2")
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "load", os.getloadavg(), flush=True)


def proc_cpu():
    out = {}
    for pid in os.listdir("/proc"):
        if not pid.isdigit():
            continue
        try:
            with open("/proc/%s/stat" % pid) as f:
                s = f.read()
            name = s[s.index("(") + 1:s.rindex(")")]
            fields = s[s.rindex(")") + 2:].split()
            out[int(pid)] = (name, int(fields[11]) + int(fields[12]))
        except Exception:
            pass
    return out


p0 = proc_cpu()
t_start = time.perf_counter()
for i in range(reps):
    torch.cuda.synchronize()
    ru0 = resource.getrusage(resource.RUSAGE_THREAD)
    c0 = time.thread_time()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    a = SparseMatrixCsr.from_coo(m, n, rows_p, cols_p, vals_p)
    pre = jacobi_precond_on_normal(a, side="auto")
    t1 = time.perf_counter()
    sigma, u, vv, rn, st = pysvds.svds(a, k=wl.k, which="S", tol=wl.tol, seed=0, precond=pre)
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    c1 = time.thread_time()
    ru1 = resource.getrusage(resource.RUSAGE_THREAD)
    print(i, "wall %.1f ms (coo %.1f, svds %.1f)  thread cpu %.1f ms  dev span %.1f ms  nvcsw %d nivcsw %d  "
          "load %.2f" % ((t2 - t0) * 1e3, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (c1 - c0) * 1e3, e0.elapsed_time(e1),
                         ru1.ru_nvcsw - ru0.ru_nvcsw, ru1.ru_nivcsw - ru0.ru_nivcsw, os.getloadavg()[0]),
          flush=True)
elapsed = time.perf_counter() - t_start
p1 = proc_cpu()
hz = os.sysconf("SC_CLK_TCK")
busy = sorted(((p1[k][1] - p0.get(k, ("", 0))[1]) / hz, k, p1[k][0]) for k in p1)[-12:]
print("busiest processes over %.1f s:" % elapsed)
for cpu_s, pid, name in reversed(busy):
    print("  %8.2f cpu-s  pid %d  %s%s" % (cpu_s, pid, name, "  (this)" if pid == os.getpid() else ""))

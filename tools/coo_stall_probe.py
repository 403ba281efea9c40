"""Split from_coo's occasional long stalls into its phases (development
helper): release of the previous matrix, host-side index checks, H2D copy,
device assembly, Jacobi diagonal; Python GC pauses logged.

python tools/coo_stall_probe.py [reps]
"""
import ctypes
import gc
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, pysvds, svds_solve  # noqa
from paper_1607_01404_b200 import _lib  # noqa: E402
from paper_1607_01404_b200.matrix import DeviceCsr  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl, (m, n, r, c, v) = bench.workload("c2")
gcl = []
_t = {}


def cb(phase, info):
    if phase == "start":
        _t["s"] = time.perf_counter()
    else:
        gcl.append((info["generation"], (time.perf_counter() - _t["s"]) * 1e3))


gc.callbacks.append(cb)
rows_p = torch.from_numpy(r).pin_memory()
cols_p = torch.from_numpy(c).pin_memory()
vals_p = torch.from_numpy(v).pin_memory()
b = p2 = None
S = torch.cuda.synchronize
from cuda.bindings import runtime as rt  # noqa: E402


def pool():
    _, mp = rt.cudaDeviceGetDefaultMemPool(0)
    A = rt.cudaMemPoolAttr
    _, res = rt.cudaMemPoolGetAttribute(mp, A.cudaMemPoolAttrReservedMemCurrent)
    _, used = rt.cudaMemPoolGetAttribute(mp, A.cudaMemPoolAttrUsedMemCurrent)
    return int(res) / 1e6, int(used) / 1e6


def steal():
    with open("/proc/stat") as f:
        x = f.readline().split()[1:]
    return int(x[7]) if len(x) > 7 else 0


def throttled():
    try:
        with open("/sys/fs/cgroup/cpu.stat") as f:
            d = dict(line.split() for line in f)
        return int(d.get("nr_throttled", 0)), int(d.get("throttled_usec", 0))
    except Exception:
        return 0, 0


def live():
    return sum(1 for o in gc.get_objects() if type(o) is DeviceCsr)
for i in range(reps):
    S()
    gcl.clear()
    st0 = steal()
    th0 = throttled()
    import resource
    ru0 = resource.getrusage(resource.RUSAGE_SELF)
    T = [time.perf_counter()]
    b = p2 = None
    S(); T.append(time.perf_counter())
    ok = int(rows_p.min()) >= 0 and int(rows_p.max()) < m and int(cols_p.min()) >= 0 and int(cols_p.max()) < n
    T.append(time.perf_counter())
    dev = torch.device("cuda", 0)
    rd = rows_p.to(dev); cd = cols_p.to(dev); vd = vals_p.to(dev)
    S(); T.append(time.perf_counter())
    h = DeviceCsr.from_coo_device(m, n, rd, cd, vd)
    T.append(time.perf_counter())
    S(); T.append(time.perf_counter())
    b = SparseMatrixCsr._from_device(h)
    p2 = jacobi_precond_on_normal(b, side="auto")
    S(); T.append(time.perf_counter())
    sigma, u, vv, rn, st = pysvds.svds(b, k=wl.k, which="S", tol=wl.tol, seed=0, precond=p2)
    T.append(time.perf_counter())
    d = np.diff(T) * 1e3
    print(i, "release %.1f checks %.1f h2d %.1f create %.1f +sync %.1f jacobi %.1f solve %.1f | gc %s | pool %.0f/%.0f MB "
          "torch %.0f MB live csr %d steal %d majflt %d minflt %d nivcsw %d" % (
              *d, gcl, *pool(), torch.cuda.memory_reserved() / 1e6, live(), steal() - st0,
              resource.getrusage(resource.RUSAGE_SELF).ru_majflt - ru0.ru_majflt,
              resource.getrusage(resource.RUSAGE_SELF).ru_minflt - ru0.ru_minflt,
              resource.getrusage(resource.RUSAGE_SELF).ru_nivcsw - ru0.ru_nivcsw),
          "throttled %d x, %.1f ms" % (throttled()[0] - th0[0], (throttled()[1] - th0[1]) / 1e3),, flush=True)

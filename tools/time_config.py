"""Time one config solve on the GPU (development helper)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, jacobi_precond_on_normal, workloads, _lib

key = sys.argv[1]
small = len(sys.argv) > 2 and sys.argv[2] == 'small'
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
budget = int(sys.argv[4]) if len(sys.argv) > 4 else None
wl = workloads.CONFIGS[key]
t0 = time.perf_counter()
m, n, r, c, v = wl.build(**(workloads.SMALL[key] if small else {}))
t1 = time.perf_counter()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"{key} m={m} n={n} nnz={a.nnz} gen {t1-t0:.2f}s build {t2-t1:.2f}s", flush=True)
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None
import os
jd = os.environ.get("JD", "")          # "1", "2" or "12": stages that run JDQMR
jdo = {"method": "JDQMR"}
if os.environ.get("ETOL"):
    jdo["inner_etol_frac"] = float(os.environ["ETOL"])
if os.environ.get("LFAC"):
    jdo["inner_lfac"] = float(os.environ["LFAC"])
if os.environ.get("MAXIN"):
    jdo["max_inner_iterations"] = int(os.environ["MAXIN"])
opts = {}
if "1" in jd:
    opts["stage1_opts"] = dict(jdo)
if "2" in jd:
    opts["stage2_opts"] = dict(jdo)
for rep in range(reps):
    cfg = SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0, max_matvecs=budget, **opts)
    l0 = _lib.launch_count()
    torch.cuda.synchronize(); t = time.perf_counter()
    res = svds_solve(a, precond=pre, cfg=cfg, return_device=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    s = res.stats
    print(json.dumps({"rep": rep, "sec": round(dt, 4), "sigma": res.sigma.tolist(), "rnorms_max": float(res.rnorms.max()),
        "conv": bool(res.converged.all()), "status": res.status, "mv1": s.stage1_matvecs, "mv2": s.stage2_matvecs,
        "restarts": s.restarts, "iters": s.outer_iterations, "inner": s.inner_iterations, "jd": jd, "jdo": jdo, "syncs": s.syncs, "graphs": s.graphs_captured, "launches": _lib.launch_count() - l0}), flush=True)

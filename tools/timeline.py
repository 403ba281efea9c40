"""GPU timeline of one config solve (development helper): CUPTI kernel and
memcpy records via torch.profiler, so every libsvdsb launch is seen.

python tools/timeline.py c4 [out.json]

Prints the solve's wall time, the summed kernel time, the idle time of the
GPU between kernels (host-bound gaps), and the top kernels by total time."""
import collections
import json
import os
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, jacobi_precond_on_normal, workloads  # noqa

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline_%s.json" % key
wl = workloads.CONFIGS[key]
m, n, r, c, v = wl.build()
a = SparseMatrixCsr.from_coo(m, n, r, c, v)
del r, c, v
pre = jacobi_precond_on_normal(a, side='auto') if wl.precond else None
budget = int(os.environ["BUDGET"]) if os.environ.get("BUDGET") else None


def cfg():
    return SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0,
                      max_matvecs=budget)


for _ in range(2):
    svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    t0 = time.perf_counter()
    res = svds_solve(a, precond=pre, cfg=cfg(), return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
trace = "/tmp/trace_%s.json" % key
prof.export_chrome_trace(trace)
ev = json.load(open(trace))["traceEvents"]
kern = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
kern.sort(key=lambda e: e["ts"])
busy = 0.0
gaps = []
big = []
end = None
prev = None
for e in kern:
    if end is not None and e["ts"] > end:
        gaps.append(e["ts"] - end)
        if e["ts"] - end > 200:
            big.append((e["ts"] - end, e["ts"] - kern[0]["ts"], prev["name"][:60], e["name"][:60]))
    busy += e["dur"]
    end = max(end or 0, e["ts"] + e["dur"])
    prev = e
span = (kern[-1]["ts"] + kern[-1]["dur"] - kern[0]["ts"]) if kern else 0
tot = collections.defaultdict(lambda: [0, 0.0])
for e in kern:
    name = e["name"].split("(")[0][:90]
    tot[name][0] += 1
    tot[name][1] += e["dur"]
top = sorted(tot.items(), key=lambda kv: -kv[1][1])[:30]
gaps.sort()
summary = {
    "config": key, "wall_s": wall, "span_us": span, "kernel_busy_us": busy, "idle_us": sum(gaps),
    "n_records": len(kern), "gaps_over_20us": sum(1 for g in gaps if g > 20),
    "idle_in_gaps_over_20us": sum(g for g in gaps if g > 20),
    "gap_p50": gaps[len(gaps) // 2] if gaps else 0, "gap_p99": gaps[int(len(gaps) * 0.99)] if gaps else 0,
    "stats": {"mv1": res.stats.stage1_matvecs, "iters": res.stats.outer_iterations, "restarts": res.stats.restarts,
              "syncs": res.stats.syncs},
    "top": [{"kernel": k, "count": c, "total_us": round(t, 1), "avg_us": round(t / c, 2)} for k, (c, t) in top],
}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "top"}))
big.sort(key=lambda t: t[1])
for g in big:
    print("gap %8.1f us at %9.1f us: after %s | before %s" % g)
for t in summary["top"]:
    print("%9.1f us %6d x %8.2f  %s" % (t["total_us"], t["count"], t["avg_us"], t["kernel"]))

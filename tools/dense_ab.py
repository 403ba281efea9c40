"""A/B of the tall-skinny kernels (register-tiled vs streamed, svdsb_tune_set
key 15) at config-4 (N = 1 M) and config-3 (N = 4.1 M) basis sizes.
python tools/dense_ab.py [out.json]"""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1607_01404_b200 import _lib
from paper_1607_01404_b200 import device as dv

PEAK = json.load(open('MEASURED_PEAKS.json')).get('hbm_gbs', 6548.5)


def timeit(fn, reps=15):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


ctx = dv.context()
out = {}
SIZES = [int(x) for x in os.environ.get('DENSE_AB_N', '1000000,4096000').split(',')]
for N in SIZES:
    g = 35
    V = dv.new_block(N, g); W = dv.new_block(N, g)
    V.normal_(); W.normal_()
    for key in (1, 2, 3, 4):
        _lib.call("svdsb_tune_set", 15, key)
        tag = {1: "reg", 2: "stream", 3: "stream12w", 4: "stream16w"}[key]
        if key >= 3:
            p = 24
            Yc = dv.small_matrix(g, p); Yc.normal_()
            lam = torch.randn(p, dtype=torch.float64, device=ctx.device)
            R = dv.new_block(N, p); rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
            t = timeit(lambda: dv.ritz_residual(ctx, V, W, Yc, lam, R, rn2=rn2))
            byt = 8 * N * (2 * g + p)
            out[f"N{N}_ritz_p{p}_{tag}"] = dict(us=t * 1e6, gbs=byt / t / 1e9, frac=byt / t / 1e9 / PEAK)
            continue
        for b in (4, 2, 1):
            Y = dv.new_block(N, b); Y.normal_()
            C = dv.small_matrix(g, b); nrm = torch.zeros(b, dtype=torch.float64, device=ctx.device)
            t = timeit(lambda: dv.gram(ctx, N, [V], Y, C, norms2=nrm))
            byt = 8 * N * (g + b)
            out[f"N{N}_gram_b{b}_{tag}"] = dict(us=t * 1e6, gbs=byt / t / 1e9, frac=byt / t / 1e9 / PEAK)
            C.mul_(1e-3)
            t = timeit(lambda: dv.project_out(ctx, N, [V], C, Y, norms2=nrm))
            byt = 8 * N * (g + 2 * b)
            out[f"N{N}_project_b{b}_{tag}"] = dict(us=t * 1e6, gbs=byt / t / 1e9, frac=byt / t / 1e9 / PEAK)
        for p in (24, 11, 5):
            Yc = dv.small_matrix(g, p); Yc.normal_()
            lam = torch.randn(p, dtype=torch.float64, device=ctx.device)
            R = dv.new_block(N, p); rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
            t = timeit(lambda: dv.ritz_residual(ctx, V, W, Yc, lam, R, rn2=rn2))
            byt = 8 * N * (2 * g + p)
            out[f"N{N}_ritz_p{p}_{tag}"] = dict(us=t * 1e6, gbs=byt / t / 1e9, frac=byt / t / 1e9 / PEAK)
        for s in (15, 24):
            Cc = dv.small_matrix(g, s); Cc.normal_(); Cc.mul_(0.1)
            X = dv.new_block(N, g); X.normal_()
            t = timeit(lambda: dv.ts_gemm(ctx, X, Cc, X[:, :s]))
            byt = 8 * N * (g + s)
            out[f"N{N}_restart_s{s}_{tag}"] = dict(us=t * 1e6, gbs=byt / t / 1e9, frac=byt / t / 1e9 / PEAK)
    _lib.call("svdsb_tune_set", 15, 0)
    del V, W
for k, v in out.items():
    print(f"{k:36s} {v['us']:9.1f} us {v['gbs']:8.1f} GB/s {v['frac']:.3f}")
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], 'w'), indent=1)

"""Per-phase clock stamps of the warm Rayleigh-Ritz update kernel
(development helper).

    python tools/arrow_phases.py build      # here: nvcc a probe build
    python tools/arrow_phases.py run [g]    # on the GPU box

The probe build compiles runtime.cu + arrow.cu with -DSVDSB_PHASE_CLOCKS
into tools/_dbg/ (git-ignored .so, travels with gpurun).
"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
GROUP = os.environ.get("ARROW_GROUP", "")
OUT = os.path.join(HERE, "_dbg", "libsvdsb_phase%s.so" % GROUP)

PHASES = ["load Y0/lam", "border column + z", "norms (tid 0)", "defl + sort", "type-2 deflation (tid 0)",
          "secular roots", "Gu-Eisenstat", "eigvec fill/normalise", "rotations", "Y <- Y P", "copy T->Y",
          "ranks", "ordering + output"]
ORDER = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13]


def build():
    from paper_1607_01404_b200 import build as b
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objs = []
    for src in ("runtime.cu", "arrow.cu"):
        obj = os.path.join(os.path.dirname(OUT), src.replace(".cu", GROUP + ".o"))
        cmd = [b.NVCC, *b.ARCH, *[f for f in b.FLAGS if f != "-v" and f != "-Xptxas"], "-DSVDSB_PHASE_CLOCKS", *(["-DSVDSB_ARROW_GROUP=" + GROUP] if GROUP else []),
               "-I", os.path.join(REPO, "include"), "-c", os.path.join(b.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", OUT, *objs], check=True)
    print(OUT)


def run(g):
    import numpy as np
    import torch
    lib = ctypes.CDLL(OUT)
    lib.svdsb_syev_update.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    rng = np.random.default_rng(0)
    h0 = rng.standard_normal((g + 1, g + 1))
    h0 = h0 + h0.T
    H = torch.zeros(64, 64, dtype=torch.float64, device="cuda")  # column-major view = transpose, symmetric
    H[:g + 1, :g + 1] = torch.from_numpy(h0)
    lam0, y0 = np.linalg.eigh(h0[:g, :g])
    Y0 = torch.from_numpy(np.asfortranarray(y0).T.copy()).cuda()  # row-major of y0^T = col-major y0
    L0 = torch.from_numpy(lam0).cuda()
    W = torch.zeros(64, dtype=torch.float64, device="cuda")
    Y = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    clk = (ctypes.c_longlong * 16)()
    rows = []
    for rep in range(6):
        rc = lib.svdsb_syev_update(g, 1, H.data_ptr(), 64, Y0.data_ptr(), g, L0.data_ptr(), 0, 0.0, W.data_ptr(),
                                   Y.data_ptr(), 64, None)
        assert rc == 0, rc
        torch.cuda.synchronize()
        assert lib.svdsb_dbg_arrow_clocks(clk) == 0
        rows.append([clk[k] for k in ORDER])
    w = np.linalg.eigvalsh(h0)
    print("max |w - eigvalsh| = %.2e" % np.abs(np.sort(W[:g + 1].cpu().numpy()) - w).max())
    last = rows[-1]
    print("root iterations: max %d, total %d (accumulated over %d calls)" % (clk[14], clk[15], len(rows)))
    tot = last[-1] - last[0]
    print("G = %d, total %d cycles (%.1f us at 1.965 GHz)" % (g + 1, tot, tot / 1965.0))
    for i, name in enumerate(PHASES):
        d = last[i + 1] - last[i]
        print("  %-28s %7d cycles %6.2f us" % (name, d, d / 1965.0))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 30)

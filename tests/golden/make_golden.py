"""Generate tests/golden/*.json from the reference implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package read-only, and writes:

* ``fixtures.json``   -- the reference suite's golden singular values
  (pkg/tests/fixtures/sparse_oracle.json, clustered300x200.json,
  rect50x30_expected.json), copied as numbers;
* ``generators.json`` -- digests of matrices built by the reference's own
  generators, which oracle/gen.py and paper_1607_01404_b200.workloads must
  reproduce bit for bit;
* ``spmv.json``       -- digests of reference spmv_block outputs on seeded
  inputs (bit-exact SpMV pins for the oracle and, via the oracle, the GPU);
* ``solves.json``     -- reference svds_solve results (sigma, rnorms,
  converged, stats) on the cases the GPU parity tests replay.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import itersvd  # noqa: E402
from itersvd.matio import SparseMatrixCsr, spmv_block  # noqa: E402
import gen_fixtures  # noqa: E402

from oracle import gen as ogen  # noqa: E402
from paper_1607_01404_b200 import workloads  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digest(a):
    return ogen.csr_digest(a.row_ptr, a.col_idx, a.values)


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name)


def fixtures():
    fx = os.path.join(REF, "tests", "fixtures")
    out = {}
    for name in ("sparse_oracle.json", "clustered300x200.json", "rect50x30_expected.json"):
        with open(os.path.join(fx, name)) as f:
            out[name] = json.load(f)
    dump("fixtures.json", out)


def generators():
    out = {"sparse": {}, "configs": {}}
    for seed in ogen.SPARSE_SEEDS:
        out["sparse"][str(seed)] = csr_digest(gen_fixtures.build_sparse(seed))
    out["clustered"] = csr_digest(gen_fixtures.build_clustered())
    out["rect50x30"] = csr_digest(gen_fixtures.build_rect50x30())
    # criterion-2 style synth matrices (test_acceptance.py:103-109)
    sigma = np.geomspace(1e-3, 1.0, 60)[::-1].copy()
    out["synth2200"] = csr_digest(itersvd.synth_matrix(itersvd.SpectrumSpec(sigma=sigma, m=90, n=60, seed=2200)))
    for key, wl in workloads.CONFIGS.items():
        kw = workloads.SMALL[key]
        m, n, r, c, v = wl.build(**kw)
        out["configs"][key] = csr_digest(SparseMatrixCsr.from_coo(m, n, r, c, v))
    dump("generators.json", out)


def spmv():
    out = []
    for seed in (11, 12, 13):
        rng = np.random.default_rng(seed)
        m, n = int(rng.integers(50, 400)), int(rng.integers(50, 400))
        nnz = int(rng.integers(100, 5000))
        r, c = rng.integers(0, m, nnz), rng.integers(0, n, nnz)
        v = rng.standard_normal(nnz) * 10.0 ** rng.uniform(-6, 6, nnz)
        a = SparseMatrixCsr.from_coo(m, n, r, c, v)
        for b in (1, 4):
            x = rng.standard_normal((n, b))
            y = rng.standard_normal((m, b))
            out.append({"seed": seed, "b": b, "m": m, "n": n, "csr": csr_digest(a),
                        "fwd": digest(np.asfortranarray(spmv_block(a, x))),
                        "adj": digest(np.asfortranarray(spmv_block(a, y, transpose=True)))})
    dump("spmv.json", out)


def _solve_record(a, cfg, precond=None):
    t0 = time.perf_counter()
    res = itersvd.svds_solve(a, precond=precond, cfg=cfg)
    sec = time.perf_counter() - t0
    s = res.stats
    return {"sigma": res.sigma.tolist(), "rnorms": res.rnorms.tolist(),
            "converged": [bool(c) for c in res.converged], "status": res.status,
            "stage1_matvecs": s.stage1_matvecs, "stage2_matvecs": s.stage2_matvecs,
            "precond_applies": s.precond_applies, "restarts": s.restarts, "resets": s.resets,
            "seconds": sec}


def solves():
    out = {}
    # BASELINE config 1 at full size, and down-scaled instances of the others
    for key in ("c1", "c2", "c3L", "c3S", "c4", "c5"):
        wl = workloads.CONFIGS[key]
        m, n, r, c, v = wl.build(**workloads.SMALL[key])
        a = SparseMatrixCsr.from_coo(m, n, r, c, v)
        pre = itersvd.jacobi_precond_on_normal(a, side="auto") if wl.precond else None
        cfg = itersvd.SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0,
                                 max_matvecs=60000)
        rec = _solve_record(a, cfg, pre)
        rec.update({"m": m, "n": n, "k": wl.k, "which": wl.which, "tol": wl.tol, "block": wl.block,
                    "precond": wl.precond, "small": workloads.SMALL[key]})
        out[key] = rec
        print(key, rec["seconds"], rec["stage1_matvecs"], rec["status"])
    # stage-2 engagement: the clustered fixture at 1e-12 (test_hybrid.py:64-80)
    a = gen_fixtures.build_clustered()
    out["clustered_S"] = _solve_record(a, itersvd.SvdsConfig(num_svals=5, target="smallest", eps=1e-12, seed=0))
    # criterion 2: kappa 1e3 synth, tight smallest
    sigma = np.geomspace(1e-3, 1.0, 60)[::-1].copy()
    a = itersvd.synth_matrix(itersvd.SpectrumSpec(sigma=sigma, m=90, n=60, seed=2200))
    out["synth2200_S12"] = _solve_record(a, itersvd.SvdsConfig(num_svals=5, target="smallest", eps=1e-12,
                                                               seed=2200))
    out["synth2200_L12"] = _solve_record(a, itersvd.SvdsConfig(num_svals=5, target="largest", eps=1e-12,
                                                               seed=2200))
    # sparse oracle seeds, both targets
    for seed in (1000, 1007):
        a = gen_fixtures.build_sparse(seed)
        for target in ("largest", "smallest"):
            for eps in (1e-6, 1e-12):
                out["sparse%d_%s_%g" % (seed, target, eps)] = _solve_record(
                    a, itersvd.SvdsConfig(num_svals=5, target=target, eps=eps, seed=seed))
    dump("solves.json", out)


# Full-size config 2 (the benchmarked solve) and mid-scale instances of the
# config 3-largest and config 4 generators, solved by the reference.  Besides
# sigma / stats / residuals this records sha256 digests of the reference's
# fp64 U and V (the oracle restatement must reproduce them bit for bit) and a
# float32 copy of V (npz next to this file) for the principal-angle checks of
# the device solves: float32 rounding keeps the angle floor near 1e-7.
BIG = {
    "c2_full": ("c2", {}),
    "c3L_40": ("c3L", {"nx": 40}),
    "c4_mid": ("c4", {"m": 500_000, "n": 50_000}),
}


def big(keys=None):
    path = os.path.join(HERE, "big_solves.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    for name, (key, kw) in BIG.items():
        if keys and name not in keys:
            continue
        wl = workloads.CONFIGS[key]
        m, n, r, c, v = wl.build(**kw)
        a = SparseMatrixCsr.from_coo(m, n, r, c, v)
        pre = itersvd.jacobi_precond_on_normal(a, side="auto") if wl.precond else None
        cfg = itersvd.SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block, seed=0)
        t0 = time.perf_counter()
        res = itersvd.svds_solve(a, precond=pre, cfg=cfg)
        sec = time.perf_counter() - t0
        s = res.stats
        rec = {"sigma": res.sigma.tolist(), "rnorms": res.rnorms.tolist(),
               "converged": [bool(x) for x in res.converged], "status": res.status,
               "stage1_matvecs": s.stage1_matvecs, "stage2_matvecs": s.stage2_matvecs,
               "precond_applies": s.precond_applies, "restarts": s.restarts, "resets": s.resets,
               "seconds": sec, "config": key, "kwargs": kw, "m": m, "n": n, "nnz": int(a.nnz),
               "csr": csr_digest(a), "u_digest": digest(np.asfortranarray(res.u)),
               "v_digest": digest(np.asfortranarray(res.v)), "a_norm_fro": float(np.linalg.norm(a.values))}
        np.savez_compressed(os.path.join(HERE, "vectors_%s.npz" % name), v=res.v.astype(np.float32),
                            sigma=res.sigma)
        out[name] = rec
        print(name, "%.1f s" % sec, rec["stage1_matvecs"], rec["stage2_matvecs"], rec["status"], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    print("wrote big_solves.json")


if __name__ == "__main__":
    if sys.argv[1:2] == ["big"]:
        big(sys.argv[2:])
        sys.exit(0)
    what = sys.argv[1:] or ["fixtures", "generators", "spmv", "solves"]
    for w in what:
        globals()[w]()

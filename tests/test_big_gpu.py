"""Parity where the benchmark runs (north star tolerances):

* full-size BASELINE config 2 (the c2 bench workload) and mid-scale
  instances of the config-3-largest and config-4 generators against the
  reference's own solves (tests/golden/big_solves.json, made by
  ``make_golden.py big`` with /root/reference; the oracle reproduces those
  solves bit for bit in tests/test_oracle.py):
    - sigma within max(tol ||A||, 1e-10 sigma_max),
    - every triplet's Eq. (7) residual (hybrid.py:206-211) recomputed on the
      host <= tol ||A||,
    - principal angles between the device's and the reference's singular
      subspaces (the reference's V stored as float32, floor ~1e-7);
* the FULL config 3-largest and config 4 device solves (the two largest
  single-GPU configs; the reference needs hours for them) certified by a
  host Eq. (7) recompute of every triplet with scipy.sparse (an
  implementation independent of libsvdsb).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


def _host_csr(m, n, r, c, v):
    import scipy.sparse as sp
    a = sp.csr_matrix((v, (r, c)), shape=(m, n))
    a.sum_duplicates()
    return a


def _eq7(a, sigma, u, v):
    """sqrt(||A v - s u||^2 + ||A^T u - s v||^2) per triplet (hybrid.py:206)."""
    av = a @ v
    atu = a.T @ u
    return np.sqrt(np.linalg.norm(av - u * sigma, axis=0) ** 2 + np.linalg.norm(atu - v * sigma, axis=0) ** 2)


def _angle(a, b):
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    s = np.linalg.svd(qa.T @ qb, compute_uv=False)
    return float(np.arccos(min(1.0, s.min())))


def _cluster_angles(sigma_ref, v_dev, v_ref, merge):
    """Principal angle per cluster of reference singular values closer than
    `merge`; returns [(indices, angle, gap to the rest of the computed set)]."""
    order = np.argsort(sigma_ref)
    groups, cur = [], [order[0]]
    for i, j in zip(order[:-1], order[1:]):
        if abs(sigma_ref[j] - sigma_ref[i]) <= merge:
            cur.append(j)
        else:
            groups.append(cur)
            cur = [j]
    groups.append(cur)
    out = []
    for g in groups:
        rest = np.setdiff1d(np.arange(sigma_ref.size), g)
        gap = np.min(np.abs(sigma_ref[rest][:, None] - sigma_ref[g][None, :])) if rest.size else np.inf
        out.append((list(map(int, g)), _angle(v_dev[:, g], v_ref[:, g]), float(gap)))
    return out


def _solve(name):
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, svds_solve, workloads
    gold = load_golden("big_solves.json")[name]
    wl = workloads.CONFIGS[gold["config"]]
    m, n, r, c, v = wl.build(**gold["kwargs"])
    a = SparseMatrixCsr.from_coo(m, n, r, c, v)
    pre = jacobi_precond_on_normal(a, side="auto") if wl.precond else None
    res = svds_solve(a, precond=pre, cfg=SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol,
                                                     max_block_size=wl.block, seed=0))
    return gold, wl, (m, n, r, c, v), res


@pytest.mark.parametrize("name", ["c2_full", "c3L_40", "c4_mid"])
def test_against_reference_solve(name):
    gold, wl, (m, n, r, c, v), res = _solve(name)
    ha = _host_csr(m, n, r, c, v)
    assert ha.nnz == gold["nnz"]
    want = np.array(gold["sigma"])
    if wl.which == "largest":
        a_norm = max(want[0], res.sigma[0])
    else:
        import scipy.sparse.linalg as sla
        a_norm = float(sla.svds(ha, k=1, return_singular_vectors=False, random_state=0)[0])
    tol = wl.tol
    assert res.converged.all(), (res.rnorms, res.status)
    assert res.status == gold["status"] == "ok"
    # sigma (north star: max(tol ||A||, 1e-10 sigma_max))
    assert np.abs(res.sigma - want).max() <= max(tol * a_norm, 1e-10 * a_norm), (res.sigma, want)
    # host Eq. (7)
    r7 = _eq7(ha, res.sigma, res.u, res.v)
    assert r7.max() <= tol * a_norm, r7
    # matvec counts: config 2 follows the reference's trajectory exactly
    if name == "c2_full":
        assert res.stats.stage1_matvecs == gold["stage1_matvecs"] == 950
        assert res.stats.stage2_matvecs == gold["stage2_matvecs"] == 0
    else:
        assert abs(res.stats.stage1_matvecs - gold["stage1_matvecs"]) <= 0.25 * gold["stage1_matvecs"]
    # singular subspaces against the reference's V (float32 copy)
    vref = np.load(os.path.join(GOLDEN, "vectors_%s.npz" % name))["v"].astype(np.float64)
    merge = 1e3 * tol * a_norm
    rows = _cluster_angles(want, res.v, vref, merge)
    print(name, "angles", [(g, "%.2e" % ang, "%.2e" % gap) for g, ang, gap in rows])
    for g, ang, gap in rows:
        # Davis-Kahan: each solution's subspace is within r / gap of the
        # exact one; 1e-6 where the tolerance allows it (config 2), the
        # residual-over-gap bound otherwise, never below the float32 floor
        bound = 1e-6 if name != "c4_mid" else max(1e-6, 4.0 * tol * a_norm / gap)
        assert ang <= bound, (g, ang, bound)
    # left vectors: u_ref = A v_ref / sigma_ref
    uref = (ha @ vref) / want
    rows_u = _cluster_angles(want, res.u, uref, merge)
    for g, ang, gap in rows_u:
        assert ang <= max(1e-6, 4.0 * tol * a_norm / gap), (g, ang)


@pytest.mark.parametrize("key", ["c3L", "c4"])
def test_full_size_certified(key):
    """The full config 3-largest (160^3) and config 4 (10M x 1M Zipf) device
    solves: converged, and every triplet's Eq. (7) residual recomputed on
    the host (scipy.sparse, independent of libsvdsb) <= tol ||A||."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, workloads
    wl = workloads.CONFIGS[key]
    m, n, r, c, v = wl.build()
    a = SparseMatrixCsr.from_coo(m, n, r, c, v)
    res = svds_solve(a, cfg=SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block,
                                       seed=0))
    del a
    assert res.converged.all(), (res.rnorms, res.status)
    assert res.status == "ok"
    assert np.all(np.diff(res.sigma) <= 0)
    ha = _host_csr(m, n, r, c, v)
    del r, c, v
    r7 = _eq7(ha, res.sigma, res.u, res.v)
    a_norm = float(res.sigma[0])
    print(key, "sigma", res.sigma[:4], "max Eq7 %.3e (tol*||A|| %.3e)" % (r7.max(), wl.tol * a_norm),
          "matvecs", res.stats.stage1_matvecs, res.stats.stage2_matvecs)
    assert r7.max() <= wl.tol * a_norm, r7
    # the library's own residuals agree with the host recompute
    assert np.allclose(res.rnorms, r7, rtol=1e-3, atol=1e-3 * wl.tol * a_norm)
    # orthonormal singular vectors
    assert np.abs(res.v.T @ res.v - np.eye(wl.k)).max() <= 1e-8
    assert np.abs(res.u.T @ res.u - np.eye(wl.k)).max() <= 1e-8


@pytest.mark.skipif(not os.environ.get("SVDSB_LONG_TESTS"),
                    reason="two minutes of GPU time: set SVDSB_LONG_TESTS=1 (profiles/r02_c3S_certified.log holds a run)")
def test_config3_smallest_full_size_jdqmr_certified():
    """BASELINE config 3, k = 10 SMALLEST triplets of the 160^3 operator at
    tol 1e-8: GD+k stalls (residual 0.0245 after 400 000 matvecs), JDQMR in
    stage 1 converges (~4.2e5 matvecs, ~2 min).  Certified like the other
    full-size solves: host Eq. (7) of every triplet <= tol ||A||, with ||A||
    from an independent scipy estimate."""
    import scipy.sparse.linalg as spla
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, workloads
    wl = workloads.CONFIGS["c3S"]
    m, n, r, c, v = wl.build()
    a = SparseMatrixCsr.from_coo(m, n, r, c, v)
    res = svds_solve(a, cfg=SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol, max_block_size=wl.block,
                                       seed=0, stage1_opts={"method": "JDQMR"}))
    del a
    assert res.converged.all(), (res.rnorms, res.status)
    assert res.status == "ok"
    ha = _host_csr(m, n, r, c, v)
    del r, c, v
    a_norm = float(spla.svds(ha, k=1, return_singular_vectors=False, tol=1e-6)[0])
    r7 = _eq7(ha, res.sigma, res.u, res.v)
    print("c3S sigma", res.sigma, "max Eq7 %.3e (tol*||A|| %.3e)" % (r7.max(), wl.tol * a_norm),
          "matvecs", res.stats.stage1_matvecs, res.stats.stage2_matvecs, "inner", res.stats.inner_iterations)
    assert r7.max() <= wl.tol * a_norm, r7
    assert np.all(np.diff(res.sigma) >= 0) or np.all(np.diff(res.sigma) <= 0)
    assert np.abs(res.v.T @ res.v - np.eye(wl.k)).max() <= 1e-8
    assert np.abs(res.u.T @ res.u - np.eye(wl.k)).max() <= 1e-8

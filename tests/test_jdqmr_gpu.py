"""JDQMR on device (jdqmr.py, csrc/jdqmr.cu): the inner solve against its
NumPy restatement (oracle/jdqmr.py) step for step, the WHILE-graph path
against the step-by-step path, and whole solves that use JDQMR in stage 1
or stage 2 against the reference's own results (its GD+k solves, so parity
is by tolerance: sigma within max(tol*||A||, 1e-10*sigma_max), residuals
recomputed on the host with the oracle SpMV)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import csr as ocsr
from oracle import gen as ogen
from oracle.jdqmr import qmrs_correction

pytestmark = pytest.mark.gpu


def _normal_setup(nx=32, seed=1):
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, make_normal_operator, workloads
    m, n, r, c, v = workloads.c1_coo(nx=nx, seed=seed)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    a = SparseMatrixCsr(m, n, rp, ci, va)
    cop = make_normal_operator(SvdOperator.wrap(a))

    def host_c(z):
        return ocsr.spmv(m, n, rp, ci, va, ocsr.spmv(m, n, rp, ci, va, z), transpose=True)
    dense = np.zeros((m, n))
    dense[np.repeat(np.arange(m), np.diff(rp)), ci] = va
    cmat = dense.T @ dense
    return a, cop, host_c, cmat, (m, n, rp, ci, va)


def _dev(x):
    from paper_1607_01404_b200 import device as dv
    return dv.to_device_block(x)[:, 0]


@pytest.mark.parametrize("pre", [False, True])
@pytest.mark.parametrize("which", ["largest", "smallest"])
@pytest.mark.parametrize("locked", [0, 3])
def test_inner_solve_matches_oracle(pre, which, locked):
    from paper_1607_01404_b200 import device as dv
    from paper_1607_01404_b200.jdqmr import JdqmrInner
    a, cop, host_c, cmat, _ = _normal_setup()
    n = cmat.shape[0]
    w, v = np.linalg.eigh(cmat)
    rng = np.random.default_rng(7)
    j = n - 1 - locked if which == "largest" else locked
    lock = v[:, n - locked:] if which == "largest" else v[:, :locked]
    x = v[:, j] + 1e-3 * rng.standard_normal(n)
    if locked:
        x -= lock @ (lock.T @ x)
    x /= np.linalg.norm(x)
    th = float(x @ host_c(x))
    r = host_c(x) - th * x
    q = np.concatenate([lock, x[:, None]], axis=1)
    dg = np.diag(cmat).copy() if pre else None
    direction = 1 if which == "largest" else -1
    t_ref, info_ref = qmrs_correction(host_c, x, th, r, q=q, dg=dg, maxit=60, direction=direction)
    ctx = dv.context()
    diag = torch.from_numpy(dg).cuda() if pre else None
    outs = []
    for use_graph in (True, False):
        jd = JdqmrInner(ctx, cop, n, diag=diag, use_graph=use_graph)
        against = [dv.to_device_block(lock)] if locked else []
        t, info = jd.solve(_dev(x), th, _dev(r), float(np.linalg.norm(r)), against=against, maxit=60,
                           direction=direction)
        outs.append((t.cpu().numpy().copy(), info))
    (tg, ig), (te, ie) = outs
    assert tg.tobytes() == te.tobytes(), "graph and step-by-step paths differ"
    assert ig["iterations"] == ie["iterations"] == info_ref["iterations"]
    assert ig["reason"] == info_ref["reason"]
    assert np.linalg.norm(tg - t_ref) <= 1e-8 * np.linalg.norm(t_ref)
    assert abs(ig["eres"] - info_ref["eres"]) <= 1e-8 * max(info_ref["eres"], 1e-300)
    # the tracked estimate is the true residual of x + t
    y = x + tg
    y /= np.linalg.norm(y)
    rho = y @ host_c(y)
    assert abs(np.linalg.norm(host_c(y) - rho * y) - ig["eres"]) <= 1e-7 * ig["eres"] + 1e-12


def test_inner_solve_counts_matvecs():
    from paper_1607_01404_b200 import device as dv
    from paper_1607_01404_b200.jdqmr import JdqmrInner
    a, cop, host_c, cmat, _ = _normal_setup()
    n = cmat.shape[0]
    x = np.ones(n) / np.sqrt(n)
    th = float(x @ host_c(x))
    r = host_c(x) - th * x
    jd = JdqmrInner(dv.context(), cop, n)
    base = cop.svd_op
    mv0, ap0 = base.n_matvecs, cop.n_applies
    _, info = jd.solve(_dev(x), th, _dev(r), float(np.linalg.norm(r)), maxit=25, lfac=0.0)
    assert info["iterations"] >= 1
    assert cop.n_applies - ap0 == info["iterations"]
    assert base.n_matvecs - mv0 == 2 * info["iterations"]


def _r7(m, n, rp, ci, va, sigma, u, v):
    out = []
    for i in range(sigma.size):
        av = ocsr.spmv(m, n, rp, ci, va, v[:, i])
        atu = ocsr.spmv(m, n, rp, ci, va, u[:, i], transpose=True)
        out.append(np.sqrt(np.linalg.norm(av - sigma[i] * u[:, i]) ** 2 +
                           np.linalg.norm(atu - sigma[i] * v[:, i]) ** 2))
    return np.array(out)


def test_config1_stage1_jdqmr():
    """BASELINE config 1 with JDQMR in stage 1 against the reference's
    GD+k solve (solves.json)."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, workloads
    gold = load_golden("solves.json")["c1"]
    m, n, r, c, v = workloads.c1_coo()
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    a = SparseMatrixCsr(m, n, rp, ci, va)
    res = svds_solve(a, cfg=SvdsConfig(num_svals=10, target="largest", eps=1e-10, seed=0,
                                       stage1_opts={"method": "JDQMR"}))
    want = np.array(gold["sigma"])
    assert res.converged.all(), (res.status, res.rnorms)
    assert res.stats.inner_iterations > 0
    assert np.abs(res.sigma - want).max() <= 1e-10 * want[0]
    assert _r7(m, n, rp, ci, va, res.sigma, res.u, res.v).max() <= 1e-10 * want[0]


@pytest.mark.parametrize("stage", ["stage2", "both"])
def test_clustered_stage2_jdqmr(stage):
    """The paper's configuration: JDQMR in stage 2 (refined extraction,
    locking) on the clustered fixture that needs stage 2 at 1e-12."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve
    fx = load_golden("fixtures.json")["clustered300x200.json"]
    m, n, rp, ci, va = ogen.build_clustered()
    a = SparseMatrixCsr(m, n, rp, ci, va)
    opts = {"stage2_opts": {"method": "JDQMR"}}
    if stage == "both":
        opts["stage1_opts"] = {"method": "JDQMR"}
    res = svds_solve(a, cfg=SvdsConfig(num_svals=5, target="smallest", eps=1e-12, seed=0, **opts))
    assert res.stats.stage2_matvecs > 0
    assert res.converged.all(), (res.rnorms, res.status)
    want = np.array(fx["smallest5"])
    assert np.abs(res.sigma - want).max() <= fx["sigma_max"] * 1e-12 * 10
    assert _r7(m, n, rp, ci, va, res.sigma, res.u, res.v).max() < fx["sigma_max"] * 1e-12


@pytest.mark.parametrize("seed", [1000, 1011])
@pytest.mark.parametrize("target", ["largest", "smallest"])
def test_sparse_oracle_jdqmr(seed, target):
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve
    recs = {r["seed"]: r for r in load_golden("fixtures.json")["sparse_oracle.json"]}
    rec = recs[seed]
    m, n, rp, ci, va = ogen.build_sparse(seed)
    a = SparseMatrixCsr(m, n, rp, ci, va)
    res = svds_solve(a, cfg=SvdsConfig(num_svals=5, target=target, eps=1e-12, seed=seed,
                                       stage1_opts={"method": "JDQMR"}, stage2_opts={"method": "JDQMR"}))
    assert res.converged.all()
    assert np.abs(res.sigma - np.array(rec[target + "5"])).max() <= rec["sigma_max"] * 1e-12 * 10
    assert _r7(m, n, rp, ci, va, res.sigma, res.u, res.v).max() < rec["sigma_max"] * 1e-12


@pytest.mark.parametrize("key", ["c2", "c3S", "c5"])
def test_downscaled_smallest_jdqmr(key):
    """Down-scaled smallest-sigma configs (Jacobi-preconditioned c2/c5)
    with JDQMR in stage 1, against the reference's GD+k results."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, svds_solve, workloads
    gold = load_golden("solves.json")[key]
    wl = workloads.CONFIGS[key]
    m, n, r, c, v = wl.build(**workloads.SMALL[key])
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    a = SparseMatrixCsr(m, n, rp, ci, va)
    pre = jacobi_precond_on_normal(a, side="auto") if wl.precond else None
    res = svds_solve(a, precond=pre, cfg=SvdsConfig(num_svals=wl.k, target=wl.which, eps=wl.tol,
                                                     max_block_size=wl.block, seed=0, max_matvecs=60000,
                                                     stage1_opts={"method": "JDQMR"}))
    want = np.array(gold["sigma"])
    assert res.converged.all(), (res.status, res.rnorms)
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    a_norm = float(spla.svds(sp.csr_matrix((va, ci, rp), shape=(m, n)), k=1, return_singular_vectors=False)[0])
    assert np.abs(res.sigma - want).max() <= max(wl.tol * a_norm, 1e-10 * want.max())
    assert _r7(m, n, rp, ci, va, res.sigma, res.u, res.v).max() <= wl.tol * a_norm

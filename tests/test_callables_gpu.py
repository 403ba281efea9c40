"""Matrix-free operators through the device solve:
``SvdOperator.from_callables(..., device=True)`` with torch device blocks
in and out, and the binding's ``svds((matvec, rmatvec), m=, n=)`` with
numpy callables (/root/reference/pkg/bindings/src/pysvds/__init__.py:
69-74).  Both must give the triplets the CSR path gives for the same
matrix, and count one matvec per operator column like the reference
(operators.py:117-129)."""
import numpy as np
import pytest
import torch

from oracle import csr as ocsr

pytestmark = pytest.mark.gpu


def _problem(seed=7, m=3000, n=1200, nnz=24000):
    rng = np.random.default_rng(seed)
    rows = np.concatenate([np.arange(n), rng.integers(0, m, nnz)])
    cols = np.concatenate([np.arange(n), rng.integers(0, n, nnz)])
    vals = np.concatenate([np.full(n, 2.0), rng.standard_normal(nnz)])
    return m, n, rows, cols, vals


@pytest.mark.parametrize("target", ["largest", "smallest"])
def test_device_callables_match_csr_path(target):
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, SvdsConfig, svds_solve
    from paper_1607_01404_b200 import device as dv
    m, n, r, c, v = _problem()
    a = SparseMatrixCsr.from_coo(m, n, r, c, v)
    dev = a.device_csr()
    calls = {"fwd": 0, "adj": 0}

    def fwd(x):                      # torch (n, b) float64 on cuda -> (m, b)
        assert isinstance(x, torch.Tensor) and x.is_cuda
        calls["fwd"] += x.shape[1]
        y = dv.new_block(m, x.shape[1])
        dev.matvec(dv.as_block(x), y)
        return y

    def adj(y):
        assert isinstance(y, torch.Tensor) and y.is_cuda
        calls["adj"] += y.shape[1]
        z = dv.new_block(n, y.shape[1])
        dev.matvec(dv.as_block(y), z, transpose=True)
        return z

    cfg = SvdsConfig(num_svals=4, target=target, eps=1e-10, seed=0)
    ref = svds_solve(a, cfg=cfg)
    op = SvdOperator.from_callables(m, n, fwd, adj, device=True)
    got = svds_solve(op, cfg=SvdsConfig(num_svals=4, target=target, eps=1e-10, seed=0))
    assert got.converged.all() and ref.converged.all()
    assert np.abs(got.sigma - ref.sigma).max() <= 1e-10 * ref.sigma.max()
    assert got.stats.stage1_matvecs == ref.stats.stage1_matvecs
    assert calls["fwd"] + calls["adj"] >= got.stats.stage1_matvecs
    # residuals recomputed on the host with the oracle's SpMV (hybrid.py:206-211)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    for i, s in enumerate(got.sigma):
        av = ocsr.spmv(m, n, rp, ci, va, got.v[:, i:i + 1])[:, 0]
        atu = ocsr.spmv(m, n, rp, ci, va, got.u[:, i:i + 1], transpose=True)[:, 0]
        res = np.sqrt(np.linalg.norm(av - s * got.u[:, i]) ** 2 + np.linalg.norm(atu - s * got.v[:, i]) ** 2)
        assert res <= 1e-10 * ref.sigma.max() * 10


def test_pysvds_matvec_rmatvec_tuple():
    """The binding's callable form: numpy (dim, b) blocks in and out, m and
    n given explicitly; same triplets as the COO form, and the binding's
    errors for a missing shape or a wrong-shaped return."""
    from paper_1607_01404_b200 import pysvds
    m, n, r, c, v = _problem(seed=9)
    dense = np.zeros((m, n))
    np.add.at(dense, (r, c), v)
    calls = {"n": 0}

    def matvec(x):
        calls["n"] += x.shape[1] if x.ndim == 2 else 1
        return dense @ x

    def rmatvec(y):
        calls["n"] += y.shape[1] if y.ndim == 2 else 1
        return dense.T @ y

    s1, u1, v1, rn1, st1 = pysvds.svds((matvec, rmatvec), k=3, which="L", tol=1e-10, m=m, n=n)
    s2, u2, v2, rn2, st2 = pysvds.svds((r, c, v), k=3, which="L", tol=1e-10, m=m, n=n)
    assert np.abs(s1 - s2).max() <= 1e-10 * s2.max()
    assert calls["n"] >= st1["stage1_matvecs"]
    assert (rn1 <= 1e-10 * s2.max() * 10).all()
    with pytest.raises(pysvds.PySvdsError):
        pysvds.svds((matvec, rmatvec), k=1)
    with pytest.raises(pysvds.PySvdsError):
        pysvds.svds((lambda x: np.zeros((m + 1, 1)), rmatvec), k=1, m=m, n=n)

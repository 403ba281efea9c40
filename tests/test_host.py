"""CPU: the C-ABI library loads and exports every symbol include/svdsb.h
declares; host-side logic of the drop-in (config validation, norm
estimate, shifts, convergence predicates, binding error mapping) without
touching a GPU."""

import os
import re

import numpy as np
import pytest

from conftest import REPO


def _header_symbols():
    with open(os.path.join(REPO, "include", "svdsb.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(svdsb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_1607_01404_b200 import _lib
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.svdsb_version() >= 1


def test_library_reports_errors_without_gpu():
    """Argument validation happens before any device work."""
    from paper_1607_01404_b200 import _lib
    lib = _lib.load()
    rc = lib.svdsb_syev_small(0, None, 1, 0, 0.0, None, None, 1, None)
    assert rc == -1
    assert "out of range" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "svdsb_syev_small")


def test_package_import_is_gpu_free():
    import paper_1607_01404_b200 as p
    for name in ("svds_solve", "SvdsConfig", "eig_solve", "EigConfig", "SvdOperator", "LinearOperator",
                 "Preconditioner", "NormEstimate", "jacobi_precond_on_normal", "make_normal_operator",
                 "make_augmented_operator", "SparseMatrixCsr", "compute_svd_residual", "stage2_shifts"):
        assert hasattr(p, name)


def test_device_ops_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1607_01404_b200 import SvdsConfig, svds_solve
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        svds_solve(np.eye(3), cfg=SvdsConfig(num_svals=1))


def test_sparse_csr_validation():
    from paper_1607_01404_b200 import SparseMatrixCsr
    a = SparseMatrixCsr(2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    assert a.nnz == 2 and a.shape == (2, 3)
    assert np.array_equal(a.to_dense(), [[1.0, 0, 0], [0, 0, 2.0]])
    with pytest.raises(ValueError):
        SparseMatrixCsr(2, 3, [0, 1], [0], [1.0])
    with pytest.raises(ValueError):
        SparseMatrixCsr(2, 3, [0, 2, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        SparseMatrixCsr(2, 3, [0, 1, 2], [0, 3], [1.0, 2.0])
    d = np.array([[0.0, 1.0], [2.0, 0.0], [0.0, 0.0]])
    assert np.array_equal(SparseMatrixCsr.from_dense(d).to_dense(), d)


def test_svds_config_validation_mirrors_reference():
    from paper_1607_01404_b200 import SvdsConfig
    assert SvdsConfig(num_svals=5, target="largest").resolved_basis_sizes() == (15, 6)
    assert SvdsConfig(num_svals=10, target="largest").resolved_basis_sizes() == (35, 14)
    assert SvdsConfig(num_svals=5, target="smallest").resolved_basis_sizes() == (35, 14)
    assert SvdsConfig(num_svals=3, max_basis_size=20).resolved_basis_sizes() == (20, 6)
    with pytest.raises(ValueError):
        SvdsConfig(num_svals=4).validate(3, 3)
    with pytest.raises(ValueError):
        SvdsConfig(target="middle").validate(10, 10)
    with pytest.raises(ValueError):
        SvdsConfig(eps=1e-20).validate(10, 10)
    with pytest.raises(ValueError):
        SvdsConfig(target="closest").validate(10, 10)
    with pytest.raises(ValueError):
        SvdsConfig(ortho_left=np.zeros((5, 1))).validate(5, 5)


def test_eig_config_validation():
    from paper_1607_01404_b200 import EigConfig
    with pytest.raises(ValueError):
        EigConfig(target="closest_geq", shifts=[1.0], locking=False).validate(100)
    with pytest.raises(ValueError):
        EigConfig(extraction="refined_const_shift").validate(100)
    with pytest.raises(ValueError):
        EigConfig(max_basis_size=10, min_restart_size=9).validate(100)
    with pytest.raises(ValueError):
        EigConfig(max_basis_size=80, min_restart_size=20).validate(1000)
    EigConfig(max_basis_size=10, min_restart_size=9).validate(10)  # dense path


def test_norm_estimate():
    from paper_1607_01404_b200 import NormEstimate, update_norm_estimate
    est = NormEstimate()
    update_norm_estimate(est, [1.0, 9.0])
    assert est.c_norm == 9.0 and est.a_norm == 3.0
    update_norm_estimate(est, [4.0])
    assert est.c_norm == 9.0
    est.update_from_augmented([-5.0, 2.0])
    assert est.c_norm == 25.0
    est = NormEstimate(user_supplied=7.0)
    est.update([100.0])
    assert est.a_norm == 7.0 and est.c_norm == 49.0
    with pytest.raises(ValueError):
        NormEstimate(user_supplied=-1.0)


def test_stage_predicates():
    from paper_1607_01404_b200.eigensolver import Candidate
    from paper_1607_01404_b200.hybrid import Stage1Test, Stage2Practical, Stage2Test, stage1_convergence_test
    from paper_1607_01404_b200 import NormEstimate
    est = NormEstimate()
    est.update([100.0])
    # brute-force agreement between the class and the functional form
    rng = np.random.default_rng(3)
    t = Stage1Test(1e-8)
    for _ in range(200):
        lam = float(rng.uniform(0, 100))
        rn = float(10.0 ** rng.uniform(-14, 0))
        assert t(lam, rn, None, None, est.c_norm) == stage1_convergence_test(lam, rn, est, 1e-8)
        assert t.evaluate(Candidate(lam, rn), est.c_norm) == stage1_convergence_test(lam, rn, est, 1e-8)
    s2 = Stage2Test(5, 1e-10)
    assert not s2.evaluate(Candidate(1.0, 1.0, nv=0.7, nu=0.7, r7=0.0), 10.0)
    assert s2.evaluate(Candidate(1.0, 1e-10, nv=0.7, nu=0.7, r7=1e-10), 10.0)
    assert not s2.evaluate(Candidate(1.0, 1e-10, nv=0.0, nu=0.7, r7=0.0), 10.0)
    p2 = Stage2Practical(5)
    assert p2.evaluate(Candidate(1.0, 1e-16, nv=0.7, nu=0.6, r7=0.0), 10.0)
    assert not p2.evaluate(Candidate(1.0, 1e-16, nv=0.99, nu=0.01, r7=0.0), 10.0)


def test_stage2_shift_arithmetic():
    """sigma - sqrt(2) rc / sigma, floored, stable ascending
    (test_hybrid.py:169-172 style)."""
    import torch
    from paper_1607_01404_b200 import NormEstimate, StageBridge, stage2_shifts
    est = NormEstimate(user_supplied=2.0)
    guesses = torch.arange(12, dtype=torch.float64).reshape(3, 4).t().contiguous().t()
    br = StageBridge(sigma_tilde=np.array([1.0, 0.5, 0.0]), rc_norms=np.array([1e-8, 1e-9, np.inf]),
                     guesses=guesses, tiny=np.array([False, False, True]))
    sh = stage2_shifts(br, est)
    floor = 2.0 * 2.220446049250313e-16
    expect = np.array([floor, 0.5 - np.sqrt(2.0) * 1e-9 / 0.5, 1.0 - np.sqrt(2.0) * 1e-8])
    assert np.array_equal(sh, expect)
    assert br.order.tolist() == [2, 1, 0]
    assert br.tiny.tolist() == [True, False, False]


def test_select_interior_candidate():
    from paper_1607_01404_b200 import select_interior_candidate
    assert select_interior_candidate(np.array([-0.5, 0.2, 1.1]), 0.1) == 1
    assert select_interior_candidate(np.array([-0.5, -0.2, -2.0]), 0.1) == 1


def test_binding_config_errors():
    from paper_1607_01404_b200.pysvds import PySvdsError, _make_config
    cfg = _make_config(3, "S", 1e-9, 4, {"max_basis_size": 20})
    assert cfg.num_svals == 3 and cfg.target == "smallest" and cfg.eps == 1e-9 and cfg.seed == 4
    with pytest.raises(PySvdsError):
        _make_config(1, "X", 1e-9, 0, {})
    with pytest.raises(PySvdsError):
        _make_config(1, "L", 1e-9, 0, {"eps": 1e-3})
    with pytest.raises(PySvdsError):
        _make_config(1, "L", 1e-9, 0, {"bogus": 1})
    assert issubclass(PySvdsError, ValueError)


def test_workload_shapes():
    from paper_1607_01404_b200 import workloads
    m, n, r, c, v = workloads.c1_coo()
    assert (m, n) == (4096, 4096) and r.size == 4096 + 4 * 63 * 64
    m, n, r, c, v = workloads.c2_coo(m=2000, n=1000)
    assert r.size == 8 * 2000 + 1000
    m, n, r, c, v = workloads.c3_coo(nx=10)
    assert (m, n) == (1000, 1000) and r.size == 1000 + 6 * 9 * 100

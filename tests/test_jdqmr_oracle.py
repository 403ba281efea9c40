"""CPU checks of the JDQMR inner-solve restatement (oracle/jdqmr.py) that
the device kernels are tested against: the tracked eigen-residual of x + t
equals the true residual, the correction stays orthogonal to Q, and the
stopping rules fire as specified."""
import numpy as np
import pytest

from oracle.jdqmr import qmrs_correction


def _problem(n=300, seed=0, noise=1e-2, which=0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = (a + a.T) / 2 + np.diag(np.linspace(0, 50, n))
    w, v = np.linalg.eigh(a)
    x = v[:, which] + noise * rng.standard_normal(n)
    x /= np.linalg.norm(x)
    th = float(x @ a @ x)
    return a, w, v, x, th, a @ x - th * x


@pytest.mark.parametrize("pre", [False, True])
@pytest.mark.parametrize("which", [0, 299])
def test_tracked_residual_is_exact(pre, which):
    a, w, v, x, th, r = _problem(which=which)
    dg = np.abs(np.diag(a)) + 1.0 if pre else None
    t, info = qmrs_correction(lambda z: a @ z, x, th, r, q=x[:, None], dg=dg, maxit=200)
    assert info["iterations"] > 0
    assert abs(x @ t) < 1e-12 * np.linalg.norm(t)
    y = (x + t) / np.linalg.norm(x + t)
    rho = y @ a @ y
    true = np.linalg.norm(a @ y - rho * y)
    assert abs(info["eres"] - true) <= 1e-9 * max(true, 1e-12)
    assert true < 0.2 * np.linalg.norm(r)


def test_stop_on_outer_tolerance():
    a, w, v, x, th, r = _problem(noise=1e-4)
    tol = 1e-3 * np.linalg.norm(r)
    t, info = qmrs_correction(lambda z: a @ z, x, th, r, q=x[:, None], tol_e=tol, maxit=500, lfac=0.0)
    assert info["reason"] == "converged"
    assert info["eres"] <= tol


def test_stop_on_etol_and_maxit():
    a, w, v, x, th, r = _problem()
    _, info = qmrs_correction(lambda z: a @ z, x, th, r, q=x[:, None], etol_frac=0.5, maxit=500)
    assert info["reason"] == "etol" and info["eres"] <= 0.5 * np.linalg.norm(r)
    _, info = qmrs_correction(lambda z: a @ z, x, th, r, q=x[:, None], maxit=2, lfac=0.0)
    assert info["iterations"] == 2 and info["reason"] == "maxit"


def test_empty_rhs():
    a, w, v, x, th, r = _problem()
    t, info = qmrs_correction(lambda z: a @ z, x, th, np.zeros_like(r), q=x[:, None])
    assert info["reason"] == "empty" and info["iterations"] == 0 and not t.any()


@pytest.mark.parametrize("which", [0, 299])
def test_rq_reversal_stop(which):
    """Extreme targets: the Rayleigh quotient of x + t only moves toward the
    wanted end while the inner solve runs; it stops at the first reversal."""
    a, w, v, x, th, r = _problem(which=which, noise=0.3)
    direction = -1 if which == 0 else 1
    t, info = qmrs_correction(lambda z: a @ z, x, th, r, q=x[:, None], maxit=300, lfac=0.0,
                              direction=direction)
    assert info["reason"] == "rq_reversal"
    # the correction still expands the search space usefully: Rayleigh-Ritz
    # on span{x, t} moves past theta toward the wanted end
    qb, _ = np.linalg.qr(np.stack([x, t], axis=1))
    ritz = np.linalg.eigvalsh(qb.T @ a @ qb)
    best = ritz[0] if direction < 0 else ritz[-1]
    assert direction * (best - th) > 0

"""Synthetic matrices with a prescribed spectrum (the reference's
``SpectrumSpec`` / ``synth_matrix``, pkg/src/itersvd/matio.py:306-362),
used by the CLI's ``--synth spectrum:`` / ``cond:`` inputs.

A host generator, not part of the solve: diag(sigma) is mixed by 20 seeded
Householder reflectors with sparse supports per side, so the result keeps
the exact singular values (to rounding) and stays sparse.  The draws and
the arithmetic follow the published construction in the same order, so the
matrices are bit-identical to the reference's (tests/test_cli.py checks the
digest of the clustered fixture pinned in tests/golden/generators.json).
"""

import numpy as np

from .matrix import SparseMatrixCsr

SYNTH_REFLECTORS = 20   # matio.py:333-335


class SpectrumSpec:
    """matio.py:306-330: singular values sorted descending, length min(m, n)."""

    def __init__(self, sigma, m, n, seed=0):
        self.sigma = np.array(sorted(sigma, reverse=True), dtype=np.float64)
        self.m = int(m)
        self.n = int(n)
        self.seed = int(seed)
        if self.m <= 0 or self.n <= 0:
            raise ValueError("matrix dimensions must be positive")
        if self.sigma.shape[0] != min(self.m, self.n):
            raise ValueError("need exactly min(m, n) singular values")
        if np.any(self.sigma < 0.0):
            raise ValueError("singular values must be nonnegative")


def _mix_rows(a, dim, rng):
    """Left-multiply by SYNTH_REFLECTORS reflectors I - 2 w w^T, each on a
    random support of max(2, dim // 10) rows (matio.py:338-344)."""
    width = min(dim, max(2, dim // 10))
    for _ in range(SYNTH_REFLECTORS):
        rows = rng.choice(dim, size=width, replace=False)
        w = rng.standard_normal(width)
        w /= np.linalg.norm(w)
        a[rows, :] -= 2.0 * np.outer(w, w @ a[rows, :])


def synth_dense(spec):
    rng = np.random.default_rng(spec.seed)
    a = np.zeros((spec.m, spec.n))
    k = spec.sigma.shape[0]
    a[np.arange(k), np.arange(k)] = spec.sigma
    _mix_rows(a, spec.m, rng)
    at = np.ascontiguousarray(a.T)
    _mix_rows(at, spec.n, rng)
    return at.T


def synth_matrix(spec):
    """matio.py:347-362: the spec's matrix as a SparseMatrixCsr."""
    return SparseMatrixCsr.from_dense(synth_dense(spec))

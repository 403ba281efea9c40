"""Seeded synthetic workloads of BASELINE.json's five configs (SURVEY.md
section 8(d)).  BASELINE.json names no public dataset, so these generated
matrices are the benchmark; every config also has a down-scaled variant
used by the parity tests.

Generators return host COO triplets (int64 rows/cols, fp64 values) drawn
from numpy.random.default_rng(seed) in the documented order; assembly to
CSR happens on device (SparseMatrixCsr.from_coo, duplicates summed like
matio.py:63-92), or on the host by the oracle for parity checks.
"""

from dataclasses import dataclass, field

import numpy as np


def stencil_coo(shape, diag, offdiag_draw, rng):
    """Grid Laplacian-type stencil on a row-major grid (index i*nx + j,
    z*ny*nx + y*nx + x in 3D): the diagonal first, then one block per
    neighbour direction in the order +axis0, -axis0, +axis1, -axis1
    [, +axis2, -axis2], each block's values drawn in one call."""
    shape = tuple(int(s) for s in shape)
    npts = int(np.prod(shape))
    idx = np.arange(npts, dtype=np.int64).reshape(shape)
    rows = [idx.ravel()]
    cols = [idx.ravel()]
    vals = [np.full(npts, float(diag))]
    for ax in range(len(shape)):
        for sgn in (+1, -1):
            sl_src = [slice(None)] * len(shape)
            sl_dst = [slice(None)] * len(shape)
            if sgn > 0:
                sl_src[ax] = slice(0, shape[ax] - 1)
                sl_dst[ax] = slice(1, shape[ax])
            else:
                sl_src[ax] = slice(1, shape[ax])
                sl_dst[ax] = slice(0, shape[ax] - 1)
            r = idx[tuple(sl_src)].ravel()
            c = idx[tuple(sl_dst)].ravel()
            rows.append(r)
            cols.append(c)
            vals.append(offdiag_draw(rng, r.shape[0]))
    return npts, npts, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def c1_coo(nx=64, seed=1):
    """2D 5-point convection-diffusion: diag 4, off-diagonals
    -1 + 0.1 U(-1, 1)."""
    rng = np.random.default_rng(seed)
    return stencil_coo((nx, nx), 4.0, lambda g, k: -1.0 + 0.1 * g.uniform(-1.0, 1.0, k), rng)


def c2_coo(m=200_000, n=100_000, per_row=8, seed=2):
    """Random rectangular: per_row N(0,1) entries per row at uniform
    columns, plus 1.0 on the leading n x n diagonal (full column rank)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(m, dtype=np.int64), per_row)
    cols = rng.integers(0, n, per_row * m).astype(np.int64)
    vals = rng.standard_normal(per_row * m)
    d = np.arange(n, dtype=np.int64)
    return m, n, np.concatenate([rows, d]), np.concatenate([cols, d]), np.concatenate([vals, np.ones(n)])


def c3_coo(nx=160, seed=3):
    """3D 7-point Laplacian, diag 6, off-diagonals -(1 + 0.05 N(0,1))."""
    rng = np.random.default_rng(seed)
    return stencil_coo((nx, nx, nx), 6.0, lambda g, k: -(1.0 + 0.05 * g.standard_normal(k)), rng)


def c4_coo(m=10_000_000, n=1_000_000, per_row=20, a=1.1, seed=4):
    """Tall power-law: per_row entries per row with Zipf(a) columns
    (draws >= n redrawn in order until all < n), values U(-1, 1) drawn
    after the rejection loop."""
    rng = np.random.default_rng(seed)
    cols = rng.zipf(a, per_row * m) - 1
    bad = np.flatnonzero(cols >= n)
    while bad.size:
        cols[bad] = rng.zipf(a, bad.size) - 1
        bad = bad[cols[bad] >= n]
    rows = np.repeat(np.arange(m, dtype=np.int64), per_row)
    vals = rng.uniform(-1.0, 1.0, per_row * m)
    return m, n, rows, cols.astype(np.int64), vals


def c5_coo(gpus=1, nx=4096, ny_per_gpu=4096, seed=5):
    """Weak-scaling 2D 5-point Laplacian, nx x (ny_per_gpu * G) points,
    diag 4, off-diagonals -(1 + 0.1 U(-1, 1))."""
    rng = np.random.default_rng(seed)
    return stencil_coo((ny_per_gpu * gpus, nx), 4.0, lambda g, k: -(1.0 + 0.1 * g.uniform(-1.0, 1.0, k)), rng)


@dataclass
class Workload:
    name: str
    coo: object            # callable -> (m, n, rows, cols, vals)
    k: int
    which: str             # "largest" | "smallest"
    tol: float
    block: int = 1
    precond: bool = False
    note: str = ""
    kwargs: dict = field(default_factory=dict)

    def build(self, **overrides):
        kw = dict(self.kwargs)
        kw.update(overrides)
        return self.coo(**kw)


CONFIGS = {
    "c1": Workload("c1", c1_coo, 10, "largest", 1e-10, note="64x64 conv-diff, k=10 largest"),
    "c2": Workload("c2", c2_coo, 5, "smallest", 1e-10, precond=True,
                   note="200000x100000 random sparse, k=5 smallest, Jacobi"),
    "c3L": Workload("c3L", c3_coo, 10, "largest", 1e-8, note="160^3 7-pt, k=10 largest"),
    "c3S": Workload("c3S", c3_coo, 10, "smallest", 1e-8, note="160^3 7-pt, k=10 smallest"),
    "c4": Workload("c4", c4_coo, 20, "largest", 1e-6, block=4,
                   note="10Mx1M Zipf(1.1), k=20 largest, block 4"),
    "c5": Workload("c5", c5_coo, 5, "smallest", 1e-8, precond=True,
                   note="4096 x 4096G 5-pt, k=5 smallest, Jacobi"),
}

# down-scaled instances of the same generators (parity runs on CPU oracle)
SMALL = {
    "c1": {},
    "c2": {"m": 20_000, "n": 10_000},
    "c3L": {"nx": 24},
    "c3S": {"nx": 12},
    "c4": {"m": 100_000, "n": 10_000},
    "c5": {"nx": 32, "ny_per_gpu": 32},
}

"""TEST INFRASTRUCTURE ONLY.  Restated test-input generators of the
reference suite, so the GPU box (which has no /root/reference) can rebuild
the exact matrices the reference's golden values were computed for.

* ``sparse_random_coo`` restates pkg/tests/oracles.py:222-254 (seeded
  positions without replacement, N(0,1) values, deterministic patch-up of
  empty rows/columns).
* ``synth_matrix`` restates pkg/src/itersvd/matio.py:306-362 (prescribed
  spectrum mixed by 20 seeded sparse Householder reflectors per side).
* ``build_sparse`` / ``build_clustered`` / ``cluster_sigma`` follow
  pkg/tests/gen_fixtures.py:39-70.

tests/golden/make_golden.py checks each against the reference itself
(checksums stored in tests/golden/generators.json).
"""

import numpy as np

from . import csr as ocsr

SPARSE_SHAPE = (400, 250)
SPARSE_DENSITY = 0.02
SPARSE_SEEDS = list(range(1000, 1020))
CLUSTER_SEED = 77
RECT_SEED = 1230
SYNTH_REFLECTORS = 20


def sparse_random_coo(m, n, density, seed):
    rng = np.random.default_rng(seed)
    target = max(int(round(m * n * density)), 1)
    picks = rng.choice(m * n, size=min(target, m * n), replace=False)
    rows = (picks // n).astype(np.int64)
    cols = (picks % n).astype(np.int64)
    seen = set(zip(rows.tolist(), cols.tolist()))
    add_r, add_c = [], []
    for i in sorted(set(range(m)) - set(rows.tolist())):
        j = int(rng.integers(n))
        add_r.append(i)
        add_c.append(j)
        seen.add((i, j))
    for j in sorted(set(range(n)) - set(cols.tolist())):
        i = int(rng.integers(m))
        if (i, j) not in seen:
            add_r.append(i)
            add_c.append(j)
            seen.add((i, j))
    if add_r:
        rows = np.concatenate([rows, np.array(add_r, dtype=np.int64)])
        cols = np.concatenate([cols, np.array(add_c, dtype=np.int64)])
    vals = rng.standard_normal(rows.shape[0])
    return rows, cols, vals


def _reflect_rows(a, dim, rng):
    width = min(dim, max(2, dim // 10))
    for _ in range(SYNTH_REFLECTORS):
        support = rng.choice(dim, size=width, replace=False)
        w = rng.standard_normal(width)
        w /= np.linalg.norm(w)
        a[support, :] -= 2.0 * np.outer(w, w @ a[support, :])


def synth_dense(sigma, m, n, seed):
    """Dense matrix with singular values ``sigma`` (sorted descending,
    length min(m, n))."""
    sigma = np.array(sorted(sigma, reverse=True), dtype=np.float64)
    rng = np.random.default_rng(int(seed))
    a = np.zeros((m, n))
    k = sigma.shape[0]
    a[np.arange(k), np.arange(k)] = sigma
    _reflect_rows(a, m, rng)
    at = np.ascontiguousarray(a.T)
    _reflect_rows(at, n, rng)
    return at.T


def synth_csr(sigma, m, n, seed):
    """CSR (row_ptr, col_idx, values) of SparseMatrixCsr.from_dense of the
    synthetic matrix (matio.py:94-98)."""
    d = synth_dense(sigma, m, n, seed)
    rows, cols = np.nonzero(d)
    return ocsr.csr_from_coo(m, n, rows, cols, d[rows, cols])


def build_sparse(seed):
    m, n = SPARSE_SHAPE
    rows, cols, vals = sparse_random_coo(m, n, SPARSE_DENSITY, seed)
    return (m, n) + ocsr.csr_from_coo(m, n, rows, cols, vals)


def cluster_sigma(p=200, count=5, base=1e-3, rel_gap=5e-5):
    bottom = base * (1.0 + rel_gap * np.arange(count))
    rest = np.geomspace(1e-2, 1.0, p - count)
    return np.sort(np.concatenate([bottom, rest]))[::-1]


def build_clustered():
    return (300, 200) + synth_csr(cluster_sigma(), 300, 200, CLUSTER_SEED)


def build_rect50x30():
    rows, cols, vals = sparse_random_coo(50, 30, 0.15, RECT_SEED)
    return (50, 30) + ocsr.csr_from_coo(50, 30, rows, cols, vals)


def csr_digest(row_ptr, col_idx, values):
    """Order-sensitive checksum of a CSR (for pinning generators)."""
    import hashlib
    h = hashlib.sha256()
    for arr in (np.asarray(row_ptr, np.int64), np.asarray(col_idx, np.int64), np.asarray(values, np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def build_spec(spec):
    """Host CSR (m, n, row_ptr, col_idx, values) of a spec."""
    k = spec["kind"]
    if k == "crit9":
        inner = np.linspace(0.3, 0.7, 38)
        sigma = np.sort(np.concatenate([[1.0 / spec["kappa"]], inner, [1.0]]))[::-1].copy()
        return (60, 40) + synth_csr(sigma, 60, 40, spec["seed"])
    if k == "synth":
        sigma = np.geomspace(spec["lo"], 1.0, spec["p"])[::-1].copy()
        return (spec["m"], spec["n"]) + synth_csr(sigma, spec["m"], spec["n"], spec["seed"])
    if k == "diag":
        d = np.asarray(spec["d"])
        n = d.shape[0]
        return (n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), d.astype(np.float64))
    if k == "zero_col":
        rng = np.random.default_rng(spec["seed"])
        dense = rng.standard_normal((spec["m"], spec["n"]))
        dense[:, spec["col"]] = 0.0
        rows, cols = np.nonzero(dense)
        return (spec["m"], spec["n"]) + ocsr.csr_from_coo(spec["m"], spec["n"], rows, cols, dense[rows, cols])
    if k == "sparse":
        return build_sparse(spec["seed"])
    raise ValueError(k)

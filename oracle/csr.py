"""TEST INFRASTRUCTURE ONLY.  Numpy restatement of the reference's CSR
assembly and block SpMV (pkg/src/itersvd/matio.py).

Every function reproduces the reference's floating-point operation order,
so its outputs are bit-identical to the reference's (checked against the
reference itself by tests/golden/make_golden.py fixtures).
"""

import numpy as np


def csr_from_coo(m, n, rows, cols, vals):
    """SparseMatrixCsr.from_coo (matio.py:63-92): stable (row, col) sort,
    duplicates summed in ascending input order into zeros, row_ptr by count
    and cumsum.  Returns (row_ptr, col_idx, values) int64/int64/fp64."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if not (rows.shape == cols.shape == vals.shape):
        raise ValueError("triplet arrays must have equal length")
    if rows.size:
        if rows.min() < 0 or rows.max() >= m:
            raise ValueError("row index out of range")
        if cols.min() < 0 or cols.max() >= n:
            raise ValueError("column index out of range")
    perm = np.lexsort((cols, rows))
    r, c, v = rows[perm], cols[perm], vals[perm]
    if r.size:
        key = r * np.int64(n) + c
        head = np.ones(key.shape[0], dtype=bool)
        head[1:] = key[1:] != key[:-1]
        seg = np.cumsum(head) - 1
        acc = np.zeros(int(head.sum()))
        np.add.at(acc, seg, v)        # sequential, ascending input order
        r, c, v = r[head], c[head], acc
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return row_ptr, c, v


def csr_transpose(m, n, row_ptr, col_idx, vals):
    """CSR(A^T) == from_coo(n, m, col_idx, rows, vals): the build stores it
    explicitly where the reference scatters (matio.py:150-154)."""
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(row_ptr))
    return csr_from_coo(n, m, col_idx, rows, vals)


def _pairwise(a):
    """NumPy's DOUBLE_pairwise_sum (what np.add.reduceat applies to the
    tail of each segment), restated in Python floats."""
    n = len(a)
    if n < 8:
        r = 0.0
        for t in a:
            r += t
        return r
    if n <= 128:
        acc = [a[i] for i in range(8)]
        i = 8
        lim = n - (n % 8)
        while i < lim:
            for j in range(8):
                acc[j] += a[i + j]
            i += 8
        res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
        while i < n:
            res += a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a[:n2]) + _pairwise(a[n2:])


def spmv(m, n, row_ptr, col_idx, vals, x, transpose=False):
    """spmv_block (matio.py:126-155) with the same summation order:
    forward y[r] = p0 + pairwise(p1..) (np.add.reduceat); transpose by the
    sequential scatter of np.add.at.  x: (rows, b) array."""
    x = np.asarray(x, dtype=np.float64)
    squeeze = x.ndim == 1
    if squeeze:
        x = x[:, None]
    b = x.shape[1]
    if not transpose:
        if x.shape[0] != n:
            raise ValueError("operand has wrong leading dimension")
        y = np.zeros((m, b), order="F")
        if vals.size:
            prod = vals[:, None] * x[col_idx, :]
            nonempty = np.flatnonzero(np.diff(row_ptr) > 0)
            if nonempty.size:
                y[nonempty, :] = np.add.reduceat(prod, row_ptr[nonempty], axis=0)
    else:
        if x.shape[0] != m:
            raise ValueError("operand has wrong leading dimension")
        y = np.zeros((n, b), order="F")
        if vals.size:
            rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(row_ptr))
            prod = vals[:, None] * x[rows, :]
            np.add.at(y, col_idx, prod)
    return y[:, 0] if squeeze else y


def spmv_loop(m, n, row_ptr, col_idx, vals, x, transpose=False):
    """Same products, written as explicit per-row folds (pure Python, small
    sizes): the order the CUDA kernel implements, used to pin `spmv`."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    if transpose:
        t_rp, t_ci, t_va = csr_transpose(m, n, row_ptr, col_idx, vals)
        out = np.zeros((n, x.shape[1]))
        for j in range(n):
            for c in range(x.shape[1]):
                s = 0.0
                for k in range(t_rp[j], t_rp[j + 1]):
                    s += t_va[k] * x[t_ci[k], c]
                out[j, c] = s
        return out
    out = np.zeros((m, x.shape[1]))
    for i in range(m):
        lo, hi = row_ptr[i], row_ptr[i + 1]
        for c in range(x.shape[1]):
            p = [vals[k] * x[col_idx[k], c] for k in range(lo, hi)]
            if not p:
                continue
            out[i, c] = p[0] if len(p) == 1 else p[0] + _pairwise(p[1:])
    return out


def column_sq_norms(m, n, row_ptr, col_idx, vals):
    """matio.py:115-118 (np.bincount order)."""
    return np.bincount(col_idx, weights=vals ** 2, minlength=n)


def row_sq_norms(m, n, row_ptr, col_idx, vals):
    """matio.py:120-123."""
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(row_ptr))
    return np.bincount(rows, weights=vals ** 2, minlength=m)


def jacobi_diag(m, n, row_ptr, col_idx, vals, side="cols"):
    """operators.py:240-248: squared norms clamped at EPS * max."""
    eps = 2.220446049250313e-16
    if side == "auto":
        side = "cols" if m >= n else "rows"
    d = column_sq_norms(m, n, row_ptr, col_idx, vals) if side == "cols" \
        else row_sq_norms(m, n, row_ptr, col_idx, vals)
    return np.maximum(d, eps * d.max())

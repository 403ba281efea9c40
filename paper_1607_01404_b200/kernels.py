"""Device versions of the reference's dense building blocks
(pkg/src/itersvd/kernels.py), same names and contracts, operands are
column-major fp64 device blocks (torch tensors from ``device.new_block``).

The solver does not call these wrappers -- its iteration uses the same
libsvdsb kernels with device-resident state -- but they expose the
bookkeeping of SURVEY 8(a) rows a10-a12 on their own, so the reference's
tests for them (criterion 7, test_acceptance.py:241-265; test_kernels.py)
replay on the GPU against the reference's semantics:

* ``qr_append``  (kernels.py:160-222): iterated CGS of the new column
  against Q (Gram + projection kernels), coefficients accumulated into R's
  new column, nonnegative diagonal, random replacement when deficient;
* ``qr_restart`` (kernels.py:225-242): ``svdsb_qr_small`` (QR of R Y with
  signs absorbed) and ``svdsb_ts_gemm`` (Q Qy);
* ``qr_factor``  (kernels.py:245-252): column-by-column ``qr_append``;
* ``sym_eig``    (kernels.py:136-145): ``svdsb_syev_small`` in ascending
  order.

The host reads one pair of norms per CGS pass, exactly the scalars the
reference branches on.
"""

import numpy as np
import torch

from . import device as dv

REORTH_FACTOR = 1.0 / np.sqrt(2.0)     # kernels.py:24
DEFICIENT_TOL = 1e-14                  # kernels.py:28
_MAX_REORTH_PASSES = 6                 # kernels.py:30


def _norm2(ctx, v, out):
    dv.col_norms2(ctx, v, out)
    return float(np.sqrt(dv.fetch(ctx, [out])[0][0]))


def qr_append(q, r, new_col, rng=None):
    """Thin QR of [Q R, new_col] (kernels.py:160-222).  ``q`` (rows x g)
    and ``r`` (g x g) are device blocks; returns fresh ``(q2, r2,
    deficient)`` device blocks."""
    ctx = dv.context()
    rows = new_col.shape[0]
    g = q.shape[1] if q is not None else 0
    if q is not None and (q.shape[0] != rows or tuple(r.shape) != (g, g)):
        raise ValueError("inconsistent QR dimensions")
    if rng is None:
        rng = np.random.default_rng(0)
    q2 = dv.new_block(rows, g + 1)
    if g:
        q2[:, :g].copy_(q)
    v = q2[:, g:g + 1]
    v.copy_(dv.as_block(new_col).reshape(rows, 1))
    coef = dv.small_matrix(max(g, 1), 1)
    c = dv.small_matrix(max(g, 1), 1)
    nrm = torch.zeros(2, dtype=torch.float64, device=q2.device)
    orig = _norm2(ctx, v, nrm[:1])
    prev = orig
    deficient = orig == 0.0
    collapses = 1 if deficient else 0
    if not deficient:
        for _ in range(_MAX_REORTH_PASSES):
            if g:
                dv.gram(ctx, rows, [q2[:, :g]], v, c[:g])
                dv.axpby(ctx, 1.0, c[:g], 1.0, coef[:g])
                dv.project_out(ctx, rows, [q2[:, :g]], c[:g], v, norms2=nrm[1:2])
                cur = float(np.sqrt(dv.fetch(ctx, [nrm[1:2]])[0][0]))
            else:
                cur = _norm2(ctx, v, nrm[1:2])
            if cur < DEFICIENT_TOL * orig:
                collapses += 1
                if collapses >= 2:
                    deficient = True
                    break
            elif cur > REORTH_FACTOR * prev:
                break
            else:
                collapses = 0
            prev = cur
        else:
            deficient = True
    r2 = dv.small_matrix(g + 1, g + 1)
    if g:
        r2[:g, :g].copy_(r)
        r2[:g, g:g + 1].copy_(coef[:g])
    if deficient:
        fill = torch.from_numpy(rng.standard_normal(rows)).to(q2.device)
        v.copy_(fill.reshape(rows, 1))
        for _ in range(2):
            if g:
                dv.gram(ctx, rows, [q2[:, :g]], v, c[:g])
                dv.project_out(ctx, rows, [q2[:, :g]], c[:g], v)
        dv.col_norms2(ctx, v, nrm[:1])
        dv.scale_cols(ctx, v, nrm[:1], dv.SCALE_DIV_SQRT)
        r2[g, g] = 0.0
    else:
        cur = _norm2(ctx, v, nrm[:1])
        dv.scale_cols(ctx, v, nrm[:1], dv.SCALE_DIV_SQRT)
        r2[g, g] = cur
    return q2, r2, deficient


def qr_restart(q, r, y):
    """QR of the compressed block (Q R) Y without touching the tall block
    twice (kernels.py:225-242): (Qy, Ry) = qr(R Y) with nonnegative
    diag(Ry) on device, then Q2 = Q Qy."""
    ctx = dv.context()
    g = q.shape[1]
    if tuple(r.shape) != (g, g) or y.shape[0] != g:
        raise ValueError("inconsistent restart dimensions")
    s = y.shape[1]
    yd = dv.to_device_block(np.asarray(y)) if isinstance(y, np.ndarray) else y
    qy = dv.small_matrix(g, s)
    ry = dv.small_matrix(s, s)
    dv.qr_small(ctx, r, g, yd, s, qy, ry)
    q2 = dv.new_block(q.shape[0], s)
    dv.ts_gemm(ctx, q, qy, q2)
    return q2, ry


def qr_factor(m, rng=None):
    """Thin QR of a device block, built column by column (kernels.py:245)."""
    q, r = None, None
    for j in range(m.shape[1]):
        q, r, _ = qr_append(q, r, m[:, j:j + 1], rng=rng)
    return q, r


def sym_eig(h):
    """Ascending eigenpairs of a small symmetric matrix (kernels.py:136)."""
    ctx = dv.context()
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError("sym_eig expects a square matrix")
    g = h.shape[0]
    hd = dv.to_device_block(h)
    w = torch.zeros(g, dtype=torch.float64, device=hd.device)
    y = dv.small_matrix(g, g)
    dv.syev_small(ctx, hd, g, 0, 0.0, w, y)
    return dv.to_host(w), dv.to_host(y)

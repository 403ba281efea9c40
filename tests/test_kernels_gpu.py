"""Kernel parity on the GPU: CSR build / transpose / SpMV / preconditioner
diagonal bit-exact against the oracle (the reference's own summation
order), tall-skinny kernels against fp64 numpy within 1e-13 relative, and
the single-CTA small dense kernels against LAPACK."""

import numpy as np
import pytest
import torch

from oracle import csr as ocsr

pytestmark = pytest.mark.gpu


def _dev():
    from paper_1607_01404_b200 import device as dv
    return dv


def _rand_coo(rng, m, n, nnz, dup=True, scale_spread=True):
    rows = rng.integers(0, m, nnz)
    cols = rng.integers(0, n, nnz)
    vals = rng.standard_normal(nnz)
    if scale_spread:
        vals *= 10.0 ** rng.uniform(-4, 4, nnz)
    if not dup:
        key = np.unique(rows * n + cols)
        rows, cols = key // n, key % n
        vals = vals[:key.size]
    return rows, cols, vals


def _csr(m, n, rows, cols, vals):
    from paper_1607_01404_b200 import SparseMatrixCsr
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    return SparseMatrixCsr(m, n, rp, ci, va), (rp, ci, va)


@pytest.fixture(autouse=True)
def _exact_mid_rows():
    """The kernel tests below check the transposed products bit for bit
    against np.add.at's order for every row up to a tile, which needs the
    serial fold for 65-2048-nonzero rows (svdsb_tune_set key 8 = 1); the
    default lane-parallel sums of those rows are checked separately
    (test_spmv_transpose_mid_rows_default)."""
    from paper_1607_01404_b200 import _lib
    _lib.call("svdsb_tune_set", 8, 1)
    yield
    _lib.call("svdsb_tune_set", 8, 0)


SHAPES = [(1, 1, 1), (7, 5, 12), (300, 40, 3000), (40, 300, 3000), (2000, 1500, 30000), (513, 257, 0)]


@pytest.mark.parametrize("m,n,nnz", SHAPES)
def test_transpose_build_bit_exact(m, n, nnz, rng):
    rows, cols, vals = _rand_coo(rng, m, n, nnz)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    dev = a.device_csr()
    t_rp, t_ci, t_va = dev.export(transpose=True)
    e_rp, e_ci, e_va = ocsr.csr_transpose(m, n, rp, ci, va)
    assert np.array_equal(t_rp, e_rp)
    assert np.array_equal(t_ci, e_ci)
    assert np.array_equal(t_va.view(np.int64), e_va.view(np.int64))
    f_rp, f_ci, f_va = dev.export(transpose=False)
    assert np.array_equal(f_rp, rp) and np.array_equal(f_ci, ci) and np.array_equal(f_va, va)


@pytest.mark.parametrize("m,n,nnz", [(5, 4, 30), (300, 40, 3000), (1000, 2000, 50000)])
def test_from_coo_device_bit_exact(m, n, nnz, rng):
    from paper_1607_01404_b200 import SparseMatrixCsr
    rows, cols, vals = _rand_coo(rng, m, n, nnz)
    # force explicit duplicates
    rows = np.concatenate([rows, rows[:nnz // 3]])
    cols = np.concatenate([cols, cols[:nnz // 3]])
    vals = np.concatenate([vals, rng.standard_normal(nnz // 3)])
    a = SparseMatrixCsr.from_coo(m, n, rows, cols, vals)
    e_rp, e_ci, e_va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    assert a.nnz == e_va.size
    assert np.array_equal(a.row_ptr, e_rp)
    assert np.array_equal(a.col_idx, e_ci)
    assert np.array_equal(a.values.view(np.int64), e_va.view(np.int64))


def _spmv_dev(a, x, transpose):
    dv = _dev()
    dev = a.device_csr()
    xb = dv.to_device_block(x)
    rows = a.n if transpose else a.m
    y = dv.new_block(rows, xb.shape[1])
    dev.matvec(xb, y, transpose=transpose)
    return dv.to_host(y)


@pytest.mark.parametrize("m,n,nnz", SHAPES[:5])
@pytest.mark.parametrize("b", [1, 3, 4])
def test_spmv_bit_exact(m, n, nnz, b, rng):
    rows, cols, vals = _rand_coo(rng, m, n, nnz)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    x = rng.standard_normal((n, b)) * 10.0 ** rng.uniform(-3, 3, (n, b))
    y = rng.standard_normal((m, b))
    got = _spmv_dev(a, x, False)
    want = ocsr.spmv(m, n, rp, ci, va, x)
    assert np.array_equal(got, want)
    got_t = _spmv_dev(a, y, True)
    want_t = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    assert np.array_equal(got_t, want_t)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_spmv_forward_b4_variants_bit_exact(variant, rng):
    """Forward b = 4 products of short-row matrices (sliced ELL, warp-staged
    CSR, thread-per-row, four lanes per row; svdsb_tune_set key 0) against
    the oracle: ragged rows of 0..120 nonzeros (tails below, at and above
    numpy's 8-term block), a row count that is not a multiple of 32, and
    32-row groups larger than the warp stage (global fallback)."""
    from paper_1607_01404_b200 import _lib
    m, n = 4133, 3001
    lens = rng.integers(0, 24, m)
    lens[rng.random(m) < 0.02] = 0
    lens[1000:1064] = rng.integers(90, 121, 64)
    rows = np.repeat(np.arange(m), lens)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.uniform(-3, 3, rows.size)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    x = rng.standard_normal((n, 4)) * 10.0 ** rng.uniform(-3, 3, (n, 4))
    try:
        _lib.call("svdsb_tune_set", 0, variant)
        got = _spmv_dev(a, x, False)
    finally:
        _lib.call("svdsb_tune_set", 0, 0)
    assert np.array_equal(got, ocsr.spmv(m, n, rp, ci, va, x))


@pytest.mark.parametrize("order", [0, 2])
def test_gram_b4_grid_orders(order, rng):
    """b = 4 Gram in both grid orders (svdsb_tune_set key 1) against numpy,
    column counts that leave a partial group of eight."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim = 200003
    a = rng.standard_normal((dim, 35))
    y = rng.standard_normal((dim, 4))
    X, Y = dv.to_device_block(a), dv.to_device_block(y)
    C = dv.small_matrix(35, 4)
    nrm = torch.zeros(4, dtype=torch.float64, device=ctx.device)
    try:
        _lib.call("svdsb_tune_set", 1, order)
        dv.gram(ctx, dim, [X], Y, C, norms2=nrm)
    finally:
        _lib.call("svdsb_tune_set", 1, 0)
    want = a.T @ y
    assert np.abs(dv.to_host(C) - want).max() <= 1e-13 * np.abs(want).max() * np.sqrt(dim)
    assert np.allclose(nrm.cpu().numpy(), (y ** 2).sum(0), rtol=1e-13)


@pytest.mark.parametrize("p", [6, 11, 16, 20, 24, 32])
def test_ritz_residual_variants(p, rng):
    """Ritz residuals R = W Y - V Y diag(lam) and |R_j|^2 for one and two
    threads per row, the latter with one or two rows per thread
    (svdsb_tune_set key 3; dim odd so a pair tail exists): R bit-identical
    between the variants (same fma order), all against fp64 numpy."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim, g = 30011, 35
    vh, wh = rng.standard_normal((dim, g)), rng.standard_normal((dim, g))
    yh = np.linalg.qr(rng.standard_normal((g, g)))[0][:, :p]
    lh = rng.standard_normal(p)
    V, W, Y = dv.to_device_block(vh), dv.to_device_block(wh), dv.to_device_block(yh)
    lam = torch.from_numpy(lh).to(ctx.device)
    want = wh @ yh - (vh @ yh) * lh
    outs = []
    try:
        for variant in (1, 2, 4, 0):
            _lib.call("svdsb_tune_set", 3, variant)
            R = dv.new_block(dim, p)
            rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
            dv.ritz_residual(ctx, V, W, Y, lam, R, rn2=rn2)
            outs.append((dv.to_host(R), rn2.cpu().numpy()))
    finally:
        _lib.call("svdsb_tune_set", 3, 0)
    for got, n2 in outs:
        assert np.array_equal(got, outs[0][0])
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
        assert np.allclose(n2, (want ** 2).sum(0), rtol=1e-12)


@pytest.mark.parametrize("g,p", [(35, 6), (35, 11), (26, 16), (35, 24), (40, 32), (5, 3)])
def test_ritz_residual_dmma(g, p, rng):
    """Ritz residuals of an HBM-scale basis (N >= 2^20 rows) on the fp64
    tensor cores (DMMA m8n8k4, svdsb_tune_set key 11 = 1) against fp64
    NumPy and the FMA kernels (key 11 = 0, the default): R to rounding (the tensor cores
    accumulate in their own order), the squared norms, the x / W y outputs;
    a row count that is not a multiple of the 8-row fragment."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim = (1 << 20) + 13
    vh, wh = rng.standard_normal((dim, g)), rng.standard_normal((dim, g))
    yh = np.linalg.qr(rng.standard_normal((g, g)))[0][:, :p]
    lh = rng.standard_normal(p)
    V, W, Y = dv.to_device_block(vh), dv.to_device_block(wh), dv.to_device_block(yh)
    lam = torch.from_numpy(lh).to(ctx.device)
    xw = vh @ yh
    ow = wh @ yh
    want = ow - xw * lh
    outs = []
    try:
        for key in (1, 0):
            _lib.call("svdsb_tune_set", 11, key)
            R, X, OX = dv.new_block(dim, p), dv.new_block(dim, p), dv.new_block(dim, p)
            rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
            dv.ritz_residual(ctx, V, W, Y, lam, R, X, OX, rn2)
            outs.append((dv.to_host(R), dv.to_host(X), dv.to_host(OX), rn2.cpu().numpy()))
    finally:
        _lib.call("svdsb_tune_set", 11, 0)
    (r0, x0, o0, n0), (r1, x1, o1, n1) = outs
    scale = np.abs(want).max()
    assert np.abs(r0 - want).max() <= 1e-12 * scale
    assert np.abs(r0 - r1).max() <= 1e-13 * scale
    assert np.abs(x0 - xw).max() <= 1e-13 * np.abs(xw).max()
    assert np.abs(o0 - ow).max() <= 1e-13 * np.abs(ow).max()
    assert np.allclose(n0, (want ** 2).sum(0), rtol=1e-12)
    assert np.allclose(n0, n1, rtol=1e-12)


@pytest.mark.parametrize("variant", [0, 1])
def test_spmv_transpose_b4_variants(variant, rng):
    """Transposed b = 4 products (svdsb_tune_set key 5: length-sorted sliced
    ELL for rows <= 64 + one warp per row up to 2048, or the CSR tiles)
    against the oracle: bit-exact on rows up to a tile, chunked rows
    (> 2048) within rounding, empty rows zero."""
    from paper_1607_01404_b200 import _lib
    m, n = 9000, 700
    cols = np.concatenate([rng.integers(0, n, 20000),          # short rows of A^T
                           rng.integers(0, 40, 15000),         # ~375-nonzero rows
                           np.full(2600, 650), np.full(3000, 651)])  # beyond a tile
    cols[cols == 699] = 698                                    # one empty row
    rows = rng.integers(0, m, cols.size)
    vals = rng.standard_normal(cols.size) * 10.0 ** rng.uniform(-3, 3, cols.size)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    y = rng.standard_normal((m, 4))
    try:
        _lib.call("svdsb_tune_set", 5, variant)
        got = _spmv_dev(a, y, True)
    finally:
        _lib.call("svdsb_tune_set", 5, 0)
    want = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    t_rp = ocsr.csr_transpose(m, n, rp, ci, va)[0]
    lens = np.diff(t_rp)
    assert lens.max() > 2048 and ((lens > 64) & (lens <= 2048)).any() and (lens == 0).any()
    ok = lens <= 2048
    assert np.array_equal(got[ok], want[ok])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("m", [1, 31, 33, 70_001])
def test_spmv_forward_b4_tma_ring_bit_exact(m, rng):
    """The TMA-staged sliced-ELL forward b = 4 kernel (rows <= 20 nonzeros,
    svdsb_tune_set key 7 = 0) against the direct-load sliced-ELL kernel
    (key 7 = 1) and the oracle, bit for bit: ragged rows of 0..20 nonzeros
    (every tail length below, at and above numpy's 8-term block), empty
    rows, slices of width 1, row counts around the 32-row slice, and enough
    slices per warp to wrap the two-stage ring many times."""
    from paper_1607_01404_b200 import _lib
    n = 5000
    lens = rng.integers(0, 21, m)
    lens[rng.random(m) < 0.05] = 0
    if m >= 64:
        lens[32:64] = rng.integers(0, 2, 32)        # a slice of width <= 1
    rows = np.repeat(np.arange(m), lens)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.uniform(-3, 3, rows.size)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    assert np.diff(rp).max() <= 20
    x = rng.standard_normal((n, 4)) * 10.0 ** rng.uniform(-3, 3, (n, 4))
    want = ocsr.spmv(m, n, rp, ci, va, x)
    got = {}
    for key in (0, 1, 4):
        try:
            _lib.call("svdsb_tune_set", 7, key)
            got[key] = _spmv_dev(a, x, False)
        finally:
            _lib.call("svdsb_tune_set", 7, 0)
    for key in got:
        assert np.array_equal(got[key], want), key


@pytest.mark.parametrize("m", [33, 70_001])
def test_spmv_forward_b4_hot_rows_bit_exact(m, rng):
    """The forward b = 4 ring kernel with the part's 1280 most referenced
    columns read from a shared-memory copy of their operand rows
    (svdsb_tune_set key 12 = 1; built when those columns carry at least a
    fifth of the nonzeros) against the all-global kernel (key 12 = 0) and
    the oracle, bit for bit: Zipf-like column ids whose hot set is not the
    lowest indices, ties in the column counts, rows of 0..20 nonzeros."""
    from paper_1607_01404_b200 import _lib
    n = 30_000
    lens = rng.integers(0, 21, m)
    rows = np.repeat(np.arange(m), lens)
    scramble = rng.permutation(n)
    cols = scramble[np.minimum(rng.zipf(1.2, rows.size) - 1, n - 1)]
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.uniform(-3, 3, rows.size)
    x = rng.standard_normal((n, 4)) * 10.0 ** rng.uniform(-3, 3, (n, 4))
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    want = ocsr.spmv(m, n, rp, ci, va, x)
    for key, nhot in ((1, 1280 if rows.size >= 32 * 1280 else 0), (0, 0)):
        try:
            _lib.call("svdsb_tune_set", 12, key)
            a, _ = _csr(m, n, rows, cols, vals)        # a fresh handle: the copies are built on first use
            got = _spmv_dev(a, x, False)
            assert a.device_csr().layout_info(1) == nhot
        finally:
            _lib.call("svdsb_tune_set", 12, 0)
        assert np.array_equal(got, want), key
    # uniform columns: the hot copy is not worth building
    try:
        _lib.call("svdsb_tune_set", 12, 1)
        a, (rp, ci, va) = _csr(m, n, rows, rng.integers(0, n, rows.size), vals)
        got = _spmv_dev(a, x, False)
        assert a.device_csr().layout_info(1) == 0
    finally:
        _lib.call("svdsb_tune_set", 12, 0)
    assert np.array_equal(got, ocsr.spmv(m, n, rp, ci, va, x))


@pytest.mark.parametrize("variant", [0, 2])
def test_spmv_transpose_b4_tma_ring(variant, rng):
    """The TMA-staged transposed b = 4 kernel (svdsb_tune_set key 7 = 2:
    length-sorted slices streamed in 8-column chunks, mid rows one warp per
    row) against the direct-load kernel and the oracle: bit-exact up to a
    tile, chunked rows within rounding, empty rows zero; both with a fresh
    output and accumulating over the column blocks of a tall matrix."""
    import os
    from paper_1607_01404_b200 import _lib
    m, n = 9000, 700
    cols = np.concatenate([rng.integers(0, n, 20000), rng.integers(0, 40, 15000),
                           np.full(2600, 650), np.full(3000, 651)])
    cols[cols == 699] = 698
    rows = rng.integers(0, m, cols.size)
    vals = rng.standard_normal(cols.size) * 10.0 ** rng.uniform(-3, 3, cols.size)
    y = rng.standard_normal((m, 4))
    want = ocsr.spmv(m, n, *ocsr.csr_from_coo(m, n, rows, cols, vals), y, transpose=True)
    old = os.environ.get("SVDSB_T_BLOCK_ROWS")
    got = {}
    try:
        for blocked in (False, True):
            if blocked:
                os.environ["SVDSB_T_BLOCK_ROWS"] = "2500"     # 4 column blocks: accumulating path
            a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
            _lib.call("svdsb_tune_set", 7, variant)
            got[blocked] = _spmv_dev(a, y, True)
            _lib.call("svdsb_tune_set", 7, 0)
    finally:
        _lib.call("svdsb_tune_set", 7, 0)
        if old is None:
            os.environ.pop("SVDSB_T_BLOCK_ROWS", None)
        else:
            os.environ["SVDSB_T_BLOCK_ROWS"] = old
    lens = np.diff(ocsr.csr_transpose(m, n, rp, ci, va)[0])
    ok = lens <= 2048
    for g in got.values():
        assert np.array_equal(g[ok], want[ok])
        assert np.abs(g - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("b", [2, 3])
def test_spmv_b23_padded_to_b4(b, rng):
    """2- and 3-column products of short-row matrices run the 4-column
    sliced-ELL kernels on a zero-padded operand (svdsb_tune_set key 6 = 0)
    or the b-column CSR tiles (key 6 = 1): bit-identical to each other, to
    the oracle for rows up to a tile, and so is the normal operator."""
    from paper_1607_01404_b200 import _lib, make_normal_operator, SvdOperator
    dv = _dev()
    m, n = 9000, 700
    cols = np.concatenate([rng.integers(0, n, 60000), rng.integers(0, 40, 15000), np.full(2600, 650)])
    rows = np.concatenate([np.arange(m).repeat(6), rng.integers(0, m, cols.size - 6 * m)])
    vals = rng.standard_normal(cols.size)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    x = rng.standard_normal((n, b))
    y = rng.standard_normal((m, b))
    op = make_normal_operator(SvdOperator.from_csr(a, check=False))
    out = {}
    for key in (0, 1):
        try:
            _lib.call("svdsb_tune_set", 6, key)
            z = dv.new_block(n, b)
            op.apply_into(dv.to_device_block(x), z)
            out[key] = (_spmv_dev(a, x, False), _spmv_dev(a, y, True), dv.to_host(z))
        finally:
            _lib.call("svdsb_tune_set", 6, 0)
    for u, v in zip(out[0], out[1]):
        assert np.array_equal(u, v)
    assert np.array_equal(out[0][0], ocsr.spmv(m, n, rp, ci, va, x))
    want_t = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    lens = np.diff(ocsr.csr_transpose(m, n, rp, ci, va)[0])
    ok = lens <= 2048
    assert np.array_equal(out[0][1][ok], want_t[ok])
    assert np.abs(out[0][1] - want_t).max() <= 1e-12 * np.abs(want_t).max()


@pytest.mark.parametrize("b", [1, 2, 4])
def test_spmv_transpose_mid_rows_default(b, rng):
    """Default transposed products (svdsb_tune_set key 8 = 0): rows of at
    most 64 nonzeros bit-exact, rows of 65-2048 summed lane-parallel with a
    fixed xor tree -- deterministic and within 1e-13 relative of the
    sequential sum -- in the plain and the column-blocked (accumulating)
    layout."""
    import os
    from paper_1607_01404_b200 import _lib
    _lib.call("svdsb_tune_set", 8, 0)
    m, n = 9000, 700
    cols = np.concatenate([rng.integers(0, n, 20000), rng.integers(0, 40, 15000),
                           np.full(2600, 650)])
    rows = rng.integers(0, m, cols.size)
    vals = rng.standard_normal(cols.size)
    y = rng.standard_normal((m, b))
    want = ocsr.spmv(m, n, *ocsr.csr_from_coo(m, n, rows, cols, vals), y, transpose=True)
    old = os.environ.get("SVDSB_T_BLOCK_ROWS")
    try:
        for blocked in (False, True):
            if blocked:
                os.environ["SVDSB_T_BLOCK_ROWS"] = "2500"
            a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
            g1 = _spmv_dev(a, y, True)
            g2 = _spmv_dev(a, y, True)
            assert np.array_equal(g1, g2)
            lens = np.diff(ocsr.csr_transpose(m, n, rp, ci, va)[0])
            assert ((lens > 64) & (lens <= 2048)).any()
            scale = np.abs(want).max()
            assert np.abs(g1 - want).max() <= 1e-13 * scale * 10
            if b == 1:
                assert np.array_equal(g1[lens <= 2048], want[lens <= 2048])   # b = 1 kernels stay serial
            else:
                assert np.array_equal(g1[lens <= 64], want[lens <= 64])
    finally:
        if old is None:
            os.environ.pop("SVDSB_T_BLOCK_ROWS", None)
        else:
            os.environ["SVDSB_T_BLOCK_ROWS"] = old


@pytest.mark.parametrize("blocked", [False, True])
def test_spmv_transpose_long_rows_head_tiles(blocked, rng):
    """Long rows (> 2048 nonzeros) of transposed b = 4 products: operand
    tiles staged in shared memory (svdsb_tune_set key 9 = 1, several tiles
    and pieces per row, a row count that is not a tile multiple) against the
    L2-gathering chunks (key 9 = 1) and the oracle: deterministic, within
    1e-13 relative of the sequential sum, short rows untouched (bit-exact)."""
    import os
    from paper_1607_01404_b200 import _lib
    m, n = 11000, 300
    cols = np.concatenate([rng.integers(0, n, 30000), np.full(9000, 7), np.full(4000, 123),
                           rng.integers(0, 3, 9000)])
    rows = rng.integers(0, m, cols.size)
    vals = rng.standard_normal(cols.size)
    y = rng.standard_normal((m, 4))
    rp_, ci_, va_ = ocsr.csr_from_coo(m, n, rows, cols, vals)
    want = ocsr.spmv(m, n, rp_, ci_, va_, y, transpose=True)
    lens = np.diff(ocsr.csr_transpose(m, n, rp_, ci_, va_)[0])
    assert (lens > 2048).sum() >= 3
    old = os.environ.get("SVDSB_T_BLOCK_ROWS")
    got = {}
    try:
        if blocked:
            os.environ["SVDSB_T_BLOCK_ROWS"] = "3001"
        a, _ = _csr(m, n, rows, cols, vals)
        for key in (0, 1, 1):
            _lib.call("svdsb_tune_set", 9, key)
            g = _spmv_dev(a, y, True)
            if key in got:
                assert np.array_equal(g, got[key])       # deterministic
            got[key] = g
    finally:
        _lib.call("svdsb_tune_set", 9, 0)
        if old is None:
            os.environ.pop("SVDSB_T_BLOCK_ROWS", None)
        else:
            os.environ["SVDSB_T_BLOCK_ROWS"] = old
    scale = np.abs(want).max()
    for g in got.values():
        assert np.abs(g - want).max() <= 1e-13 * scale * 10
        assert np.array_equal(g[lens <= 64], want[lens <= 64])


def test_sell_copies_device_build_matches_host(rng):
    """The sliced-ELL copies built on the device (CUB select / stable radix
    sort by length / scan; svdsb_tune_set key 10 = 0) and on the host (key
    10 = 1) give the same products bit for bit, forward and transposed, on
    ragged rows: short, mid (65-2048) and long rows, empty rows."""
    from paper_1607_01404_b200 import _lib
    m, n = 7000, 500
    cols = np.concatenate([rng.integers(0, n, 30000), rng.integers(0, 30, 6000), np.full(2500, 400)])
    cols[cols == 499] = 498
    rows = np.concatenate([np.repeat(np.arange(m), 2), rng.integers(0, m, cols.size - 2 * m)])
    vals = rng.standard_normal(cols.size)
    x = rng.standard_normal((n, 4))
    y = rng.standard_normal((m, 4))
    out = {}
    try:
        for key in (1, 0):
            _lib.call("svdsb_tune_set", 10, key)
            a, _ = _csr(m, n, rows, cols, vals)           # a fresh matrix: copies built under this key
            out[key] = (_spmv_dev(a, x, False), _spmv_dev(a, y, True))
    finally:
        _lib.call("svdsb_tune_set", 10, 0)
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_spmv_bulk_copy_path_bit_exact(rng):
    """Matrices of >= 64 MB stream through the cp.async.bulk tile ring
    (csr_tile_bulk_kernel); it must reproduce the reference's summation
    order bit for bit like the register pipeline: a 100^3 7-point stencil
    (1M rows, 6.9M nnz, 83 MB) for A x and A^T y, plus a scattered
    rectangular matrix whose tiles take the strided path."""
    from paper_1607_01404_b200 import workloads
    m, n, r, c, v = workloads.c3_coo(nx=100)
    a, (rp, ci, va) = _csr(m, n, r, c, v)
    assert 12 * va.size >= 64 << 20
    x = rng.standard_normal((n, 1))
    assert np.array_equal(_spmv_dev(a, x, False), ocsr.spmv(m, n, rp, ci, va, x))
    y = rng.standard_normal((m, 1))
    assert np.array_equal(_spmv_dev(a, y, True), ocsr.spmv(m, n, rp, ci, va, y, transpose=True))
    m2, n2 = 600000, 50000
    rows = np.repeat(np.arange(m2), 12)
    cols = rng.integers(0, n2, rows.size)
    a2, (rp2, ci2, va2) = _csr(m2, n2, rows, cols, rng.standard_normal(rows.size))
    assert 12 * va2.size >= 64 << 20
    x2 = rng.standard_normal((n2, 1))
    assert np.array_equal(_spmv_dev(a2, x2, False), ocsr.spmv(m2, n2, rp2, ci2, va2, x2))


def test_spmv_long_rows_and_dead_rows(rng):
    """Rows longer than one tile (2048 nnz) take the chunked path: results
    are deterministic and within fp64 rounding of the sequential sum."""
    m, n = 20000, 64
    rows = np.concatenate([rng.integers(0, m, 60000), np.arange(0, m, 3)])
    cols = np.concatenate([rng.integers(0, 4, 60000), rng.integers(0, n, (m + 2) // 3)])
    vals = rng.standard_normal(rows.size)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    assert np.diff(ocsr.csr_transpose(m, n, rp, ci, va)[0]).max() > 2048
    y = rng.standard_normal((m, 2))
    got1 = _spmv_dev(a, y, True)
    got2 = _spmv_dev(a, y, True)
    assert np.array_equal(got1, got2)
    want = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    scale = np.abs(va)[:, None] * np.abs(y[np.repeat(np.arange(m), np.diff(rp))])
    bound = 1e-14 * np.sqrt(np.bincount(ci, weights=scale[:, 0] ** 2, minlength=n)).max() * 50
    assert np.abs(got1 - want).max() <= max(bound, 1e-12)
    # the short rows (fewer than a tile) are still bit-exact
    t_rp = ocsr.csr_transpose(m, n, rp, ci, va)[0]
    short = np.flatnonzero(np.diff(t_rp) <= 2048)
    assert np.array_equal(got1[short], want[short])


def test_spmv_identity_permutation_dead_row():
    """test_matio.py:99-112 known answers."""
    from paper_1607_01404_b200 import SparseMatrixCsr
    a = SparseMatrixCsr.from_dense(np.array([[0.0, 1.0], [1.0, 0.0], [0.0, 0.0]]))
    assert np.array_equal(_spmv_dev(a, np.array([[2.0], [5.0]]), False)[:, 0], [5.0, 2.0, 0.0])
    assert np.array_equal(_spmv_dev(a, np.array([[7.0], [11.0], [13.0]]), True)[:, 0], [11.0, 7.0])
    eye = SparseMatrixCsr.from_dense(np.eye(3))
    x = np.random.default_rng(0).standard_normal((3, 2))
    assert np.array_equal(_spmv_dev(eye, x, False), x)


@pytest.mark.parametrize("side", ["cols", "rows"])
def test_jacobi_diag_bit_exact(side, rng):
    from paper_1607_01404_b200 import jacobi_precond_on_normal
    m, n = 400, 250
    rows, cols, vals = _rand_coo(rng, m, n, 4000)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    pre = jacobi_precond_on_normal(a, side=side)
    want = ocsr.jacobi_diag(m, n, rp, ci, va, side=side)
    got = pre.diagonal.cpu().numpy()
    assert np.array_equal(got, want)
    x = rng.standard_normal((want.size, 2))
    y = _dev().to_host(pre.apply(_dev().to_device_block(x)))
    assert np.array_equal(y, x / want[:, None])


def test_normal_and_augmented_operators(rng):
    from paper_1607_01404_b200 import SvdOperator, make_augmented_operator, make_normal_operator
    m, n = 300, 200
    rows, cols, vals = _rand_coo(rng, m, n, 3000, scale_spread=False)
    a, (rp, ci, va) = _csr(m, n, rows, cols, vals)
    op = SvdOperator.from_csr(a)
    d = a.to_dense()
    c = make_normal_operator(op)
    x = rng.standard_normal((n, 3))
    got = _dev().to_host(c.apply(_dev().to_device_block(x)))
    ref = d.T @ (d @ x)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert op.n_matvecs == 6
    b = make_augmented_operator(op)
    z = rng.standard_normal((n + m, 2))
    got = _dev().to_host(b.apply(_dev().to_device_block(z)))
    ref = np.vstack([d.T @ z[n:], d @ z[:n]])
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert op.n_matvecs == 10


# ------------------------------------------------------------ tall-skinny

@pytest.mark.parametrize("dim", [1, 100, 5000, 300001])
def test_gram_project_tsgemm(dim, rng):
    dv = _dev()
    ctx = dv.context()
    a1 = rng.standard_normal((dim, 7))
    a2 = rng.standard_normal((dim, 30))
    y = rng.standard_normal((dim, 4))
    X1, X2, Y = dv.to_device_block(a1), dv.to_device_block(a2), dv.to_device_block(y)
    for b in (1, 2, 3, 4):
        C = dv.small_matrix(37, b)
        nrm = torch.zeros(b, dtype=torch.float64, device=ctx.device)
        dv.gram(ctx, dim, [X1, X2], Y[:, :b], C, norms2=nrm)
        want = np.hstack([a1, a2]).T @ y[:, :b]
        got = dv.to_host(C)
        assert np.abs(got - want).max() <= 1e-13 * max(1.0, np.abs(want).max()) * np.sqrt(dim)
        assert np.allclose(nrm.cpu().numpy(), (y[:, :b] ** 2).sum(0), rtol=1e-13)
        Yc = Y[:, :b].clone()
        Yc = dv.to_device_block(y[:, :b])
        nrm2 = torch.zeros(b, dtype=torch.float64, device=ctx.device)
        dv.project_out(ctx, dim, [X1, X2], C, Yc, norms2=nrm2)
        want_y = y[:, :b] - np.hstack([a1, a2]) @ got
        assert np.abs(dv.to_host(Yc) - want_y).max() <= 1e-12 * max(1.0, np.abs(want_y).max())
        assert np.allclose(nrm2.cpu().numpy(), (want_y ** 2).sum(0), rtol=1e-10, atol=1e-20)
    cm = rng.standard_normal((30, 15))
    out = dv.new_block(dim, 15)
    dv.ts_gemm(ctx, X2, dv.to_device_block(cm), out)
    want = a2 @ cm
    assert np.abs(dv.to_host(out) - want).max() <= 1e-13 * np.abs(want).max() * 4


@pytest.mark.parametrize("dim", [7, 100003])
@pytest.mark.parametrize("g,s", [(35, 15), (40, 32), (3, 1)])
def test_ts_gemm_inplace_matches_out_of_place(dim, g, s, rng):
    """The in-place restart V <- V C is bit-identical to the out-of-place
    product (same fma order per row)."""
    dv = _dev()
    ctx = dv.context()
    a = rng.standard_normal((dim, g))
    cm = dv.to_device_block(rng.standard_normal((g, s)))
    x = dv.to_device_block(a)
    ref = dv.new_block(dim, s)
    dv.ts_gemm(ctx, x, cm, ref)
    dv.ts_gemm(ctx, x, cm, x[:, :s])
    assert np.array_equal(dv.to_host(x[:, :s]), dv.to_host(ref))
    assert np.array_equal(dv.to_host(x[:, s:]), a[:, s:])
    if g >= 3:
        # in place with more outputs than inputs is rejected, not raced
        with pytest.raises(ValueError):
            dv.ts_gemm(ctx, x[:, :2], dv.to_device_block(rng.standard_normal((2, 3))), x[:, :3])


@pytest.mark.parametrize("dim", [50, 100003, 250001])   # 250001: HBM-streamed bulk-copy path
@pytest.mark.parametrize("p", [1, 11, 24])
def test_ritz_residual(dim, p, rng):
    dv = _dev()
    ctx = dv.context()
    g = 35
    v = rng.standard_normal((dim, g))
    w = rng.standard_normal((dim, g))
    yc = rng.standard_normal((g, p))
    lam = rng.standard_normal(p)
    V, W = dv.to_device_block(v), dv.to_device_block(w)
    R, X, OX = dv.new_block(dim, p), dv.new_block(dim, p), dv.new_block(dim, p)
    rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
    dv.ritz_residual(ctx, V, W, dv.to_device_block(yc), torch.as_tensor(lam, device=ctx.device), R, X, OX, rn2)
    x = v @ yc
    ox = w @ yc
    r = ox - x * lam
    tol = 1e-13 * np.abs(ox).max() * 4
    assert np.abs(dv.to_host(X) - x).max() <= tol
    assert np.abs(dv.to_host(OX) - ox).max() <= tol
    assert np.abs(dv.to_host(R) - r).max() <= tol * 4
    assert np.allclose(rn2.cpu().numpy(), (r ** 2).sum(0), rtol=1e-12)


def test_split_residual_matches_direct(rng):
    dv = _dev()
    ctx = dv.context()
    n, m, p = 700, 1100, 3
    x = rng.standard_normal((n + m, p))
    x[:n] *= 0.8
    lam = np.array([1.5, -0.7, 2.0])
    r = rng.standard_normal((n + m, p)) * 1e-3
    R, X = dv.to_device_block(r), dv.to_device_block(x)
    lam_d = torch.as_tensor(lam, device=ctx.device)
    st = torch.zeros(6 * p, dtype=torch.float64, device=ctx.device)
    out = torch.zeros(p, dtype=torch.float64, device=ctx.device)
    dv.split_stats(ctx, n, R, X, st)
    dv.split_residual(ctx, n, R, X, lam_d, st, out)
    bx = r + x * lam
    for j in range(p):
        nv, nu = np.linalg.norm(x[:n, j]), np.linalg.norm(x[n:, j])
        sg = abs(lam[j])
        e1 = bx[n:, j] / nv - sg * x[n:, j] / nu
        e2 = bx[:n, j] / nu - sg * x[:n, j] / nv
        want = e1 @ e1 + e2 @ e2
        assert abs(out[j].item() - want) <= 1e-12 * max(want, 1e-300) + 1e-26
        s = st[6 * j:6 * j + 6].cpu().numpy()
        assert np.allclose(s[[2, 5]], [nv ** 2, nu ** 2], rtol=1e-13)


# ------------------------------------------------------------ small dense

@pytest.mark.parametrize("g", [1, 2, 3, 15, 35, 64])
def test_syev_small(g, rng):
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    a = rng.standard_normal((g, g))
    h = a + a.T
    if g > 3:
        h[0, 0] = h[1, 1]  # some structure
    H = dv.to_device_block(h)
    w = torch.zeros(g, dtype=torch.float64, device=ctx.device)
    Y = dv.small_matrix(g, g)
    ref_w, ref_v = np.linalg.eigh(h)
    for order, expect in ((_lib.ORDER_ASC, np.arange(g)), (_lib.ORDER_DESC, np.argsort(-ref_w, kind="stable"))):
        dv.syev_small(ctx, H, g, order, 0.0, w, Y)
        got_w = w.cpu().numpy()
        got_y = dv.to_host(Y)
        assert np.abs(got_w - ref_w[expect]).max() <= 1e-13 * np.abs(ref_w).max() * g
        assert np.abs(got_y.T @ got_y - np.eye(g)).max() <= 1e-13 * g
        res = h @ got_y - got_y * got_w
        assert np.abs(res).max() <= 1e-13 * np.abs(ref_w).max() * g
    shift = float(np.median(ref_w)) + 1e-3
    dv.syev_small(ctx, H, g, _lib.ORDER_INTERIOR, shift, w, Y)
    below = ref_w < shift
    key = np.where(below, shift - ref_w, ref_w - shift)
    expect = np.lexsort((key, below.astype(np.int64)))
    assert np.abs(w.cpu().numpy() - ref_w[expect]).max() <= 1e-13 * np.abs(ref_w).max() * g


@pytest.mark.parametrize("g", [2, 9, 35])
def test_refined_small(g, rng):
    dv = _dev()
    ctx = dv.context()
    r = np.triu(rng.standard_normal((g, g)))
    r[g - 1, g - 1] = 1e-9
    h = rng.standard_normal((g, g))
    h = h + h.T
    y = torch.zeros(g, dtype=torch.float64, device=ctx.device)
    lam = torch.zeros(1, dtype=torch.float64, device=ctx.device)
    sv = torch.zeros(g, dtype=torch.float64, device=ctx.device)
    dv.refined_small(ctx, dv.to_device_block(r), dv.to_device_block(h), g, y, lam, sv)
    _, s, vt = np.linalg.svd(r)
    yv = y.cpu().numpy()
    assert abs(abs(yv @ vt[-1]) - 1.0) <= 1e-10
    assert np.allclose(sv.cpu().numpy(), s, rtol=1e-12, atol=1e-14 * s[0])
    assert abs(lam.item() - yv @ h @ yv) <= 1e-12 * np.abs(h).max() * g


@pytest.mark.parametrize("g,s", [(5, 3), (35, 15), (20, 20)])
def test_qr_small(g, s, rng):
    dv = _dev()
    ctx = dv.context()
    r = np.triu(rng.standard_normal((g, g)))
    yc, _ = np.linalg.qr(rng.standard_normal((g, s)))
    qy = dv.small_matrix(g, s)
    ry = dv.small_matrix(s, s)
    dv.qr_small(ctx, dv.to_device_block(r), g, dv.to_device_block(yc), s, qy, ry)
    qw, rw = np.linalg.qr(r @ yc)
    sign = np.where(np.diag(rw) < 0.0, -1.0, 1.0)
    qw, rw = qw * sign, rw * sign[:, None]
    assert np.abs(dv.to_host(qy) - qw).max() <= 1e-12
    assert np.abs(dv.to_host(ry) - rw).max() <= 1e-12 * np.abs(rw).max()


def _coef_gs_ref(columns, limit, against):
    kept = []
    for col in columns:
        if len(kept) >= limit:
            break
        c = np.array(col, dtype=np.float64, copy=True)
        for _ in range(2):
            for b in against:
                c -= b * (b @ c)
            for b in kept:
                c -= b * (b @ c)
        nrm = np.linalg.norm(c)
        if nrm > 1e-8:
            kept.append(c / nrm)
    return kept


def test_restart_coefs(rng):
    dv = _dev()
    ctx = dv.context()
    g, gmax = 35, 35
    h = rng.standard_normal((g, g))
    _, y = np.linalg.eigh(h + h.T)
    yfirst = rng.standard_normal(g)
    yfirst /= np.linalg.norm(yfirst)
    excl = y[:, 3].copy()
    prev = rng.standard_normal((30, 1))
    out = dv.small_matrix(g, g)
    cnt = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    dv.restart_coefs(ctx, g, gmax, torch.as_tensor(yfirst, device=ctx.device), dv.to_device_block(y), g, 14,
                     torch.as_tensor(excl, device=ctx.device), dv.to_device_block(prev), 1, 30, 1, out, cnt)
    s = int(cnt.item())
    sel = _coef_gs_ref([yfirst] + [y[:, j] for j in range(g)], 14, [excl])
    padded = np.zeros(g)
    padded[:30] = prev[:, 0]
    plus = _coef_gs_ref([padded], 1, [excl] + sel)
    want = np.array(sel + plus).T
    assert s == want.shape[1] == 15
    assert np.abs(dv.to_host(out)[:, :s] - want).max() <= 1e-12


def test_launch_counter_moves():
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    before = _lib.launch_count()
    x = dv.to_device_block(np.ones((10, 1)))
    out = torch.zeros(1, dtype=torch.float64, device=ctx.device)
    dv.col_norms2(ctx, x, out)
    assert _lib.launch_count() == before + 1
    assert out.item() == 10.0


@pytest.mark.parametrize("g0,b", [(0, 1), (1, 1), (14, 1), (34, 1), (20, 4), (30, 5), (60, 4)])
@pytest.mark.parametrize("kind", ["prev", "diag", "degenerate"])
def test_syev_update_matches_eigh(g0, b, kind, rng):
    """Warm arrowhead update of a bordered projection vs LAPACK."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    g = g0 + b
    a = rng.standard_normal((g, g))
    h = a + a.T
    if kind == "degenerate" and g0 >= 4:
        # repeated leading eigenvalues and an (almost) decoupled direction
        w0, q0 = np.linalg.eigh(h[:g0, :g0])
        w0[1] = w0[0]
        w0[3] = w0[2] + 1e-17
        h[:g0, :g0] = (q0 * w0) @ q0.T
        h[:g0, g0] = q0[:, 0] * 1e-20 + h[:g0, g0] * (np.arange(g0) % 2)
        h[g0, :g0] = h[:g0, g0]
    if kind == "diag":
        h[:g0, :g0] = np.diag(np.sort(rng.standard_normal(g0)))
    H = dv.to_device_block(h)
    w = torch.zeros(g, dtype=torch.float64, device=ctx.device)
    Y = dv.small_matrix(g, g)
    if kind == "diag" or g0 == 0:
        y0 = l0 = None
    else:
        l0h, y0h = np.linalg.eigh(h[:g0, :g0])
        y0 = dv.to_device_block(y0h)
        l0 = torch.as_tensor(l0h, device=ctx.device)
    ref_w = np.linalg.eigh(h)[0]
    scale = max(1.0, np.abs(ref_w).max())
    for order in (_lib.ORDER_ASC, _lib.ORDER_DESC):
        dv.syev_update(ctx, H, g0, b, y0, l0, order, 0.0, w, Y)
        got_w = w.cpu().numpy()
        got_y = dv.to_host(Y)
        exp = ref_w if order == _lib.ORDER_ASC else ref_w[::-1]
        assert np.abs(got_w - exp).max() <= 1e-13 * scale * g
        assert np.abs(got_y.T @ got_y - np.eye(g)).max() <= 1e-13 * g
        assert np.abs(h @ got_y - got_y * got_w).max() <= 1e-13 * scale * g


@pytest.mark.parametrize("accum", [0, 1])
@pytest.mark.parametrize("b", [1, 2, 4])
def test_column_blocked_transpose(b, accum, rng, monkeypatch):
    """A^T through row blocks of A (tall scattered matrices) keeps the
    reference's left-to-right order across blocks: bit-exact for short rows,
    deterministic within rounding for long (chunked) rows.  Running sums in
    the result (svdsb_tune_set key 13 = 0) or in the row-major scratch block
    (1); columns that occur in one block only (their rows are empty in the
    other blocks and must keep their sums) and columns that never occur."""
    monkeypatch.setenv("SVDSB_T_BLOCK_ROWS", "997")
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, make_normal_operator, _lib
    m, n = 5000, 320
    rows = np.concatenate([np.repeat(np.arange(m), 3), rng.integers(0, m, 6000), rng.integers(1000, 1500, 40)])
    cols = np.concatenate([rng.integers(0, 300, 3 * m), rng.integers(0, 3, 6000),   # 3 heavy columns
                           rng.integers(300, 310, 40)])                             # one-block columns
    vals = rng.standard_normal(rows.size)
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    a = SparseMatrixCsr(m, n, rp, ci, va)
    y = rng.standard_normal((m, b))
    _lib.call("svdsb_tune_set", 13, accum)
    try:
        got = _spmv_dev(a, y, True)
        assert a.device_csr().layout_info(2) == 6
        _test_column_blocked_rest(a, rp, ci, va, m, n, b, y, got, rng)
    finally:
        _lib.call("svdsb_tune_set", 13, 0)


def test_column_blocked_transpose_long_rows_first(rng, monkeypatch):
    """Kernel order of a transposed b = 4 part (svdsb_tune_set key 16): long
    rows before short rows gives the same bits (disjoint rows per part)."""
    monkeypatch.setenv("SVDSB_T_BLOCK_ROWS", "997")
    from paper_1607_01404_b200 import SparseMatrixCsr, _lib
    m, n, b = 5000, 320, 4
    rows = np.concatenate([np.repeat(np.arange(m), 3), rng.integers(0, m, 9000)])
    cols = np.concatenate([rng.integers(0, 300, 3 * m), rng.integers(0, 3, 9000)])   # 3 heavy (chunked) columns
    vals = rng.standard_normal(rows.size)
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    y = rng.standard_normal((m, b))
    outs = []
    for key in (0, 1):
        a = SparseMatrixCsr(m, n, rp, ci, va)
        _lib.call("svdsb_tune_set", 16, key)
        try:
            outs.append(_spmv_dev(a, y, True))
        finally:
            _lib.call("svdsb_tune_set", 16, 0)
    assert np.array_equal(outs[0], outs[1])
    want = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    assert np.abs(outs[1] - want).max() <= 1e-12 * np.abs(want).max()


def _test_column_blocked_rest(a, rp, ci, va, m, n, b, y, got, rng):
    from paper_1607_01404_b200 import SvdOperator, make_normal_operator
    want = ocsr.spmv(m, n, rp, ci, va, y, transpose=True)
    t_rp = ocsr.csr_transpose(m, n, rp, ci, va)[0]
    long_rows = np.flatnonzero(np.diff(t_rp) > 2048)
    short = np.setdiff1d(np.arange(n), long_rows)
    assert np.array_equal(got[short], want[short])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    op = make_normal_operator(SvdOperator.from_csr(a, check=False))
    x = rng.standard_normal((n, b))
    c = _dev().to_host(op.apply(_dev().to_device_block(x)))
    ref = ocsr.spmv(m, n, rp, ci, va, ocsr.spmv(m, n, rp, ci, va, x), transpose=True)
    assert np.abs(c - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("dim", [5, 100003])
def test_gather_cols_device_index(dim, rng):
    """Device-indexed column gather: plain copy, and divided by a diagonal
    bit-identically to svdsb_diag_solve; the limit clips the column range."""
    import torch
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    x = rng.standard_normal((dim, 6))
    d = rng.uniform(0.5, 2.0, dim)
    X = dv.to_device_block(x)
    D = torch.from_numpy(d).cuda()
    first = torch.tensor([2], dtype=torch.int32, device="cuda")
    Y = dv.new_block(dim, 3)
    dv.gather_cols(ctx, X, first, 3, 4, Y)
    got = dv.to_host(Y)
    assert np.array_equal(got[:, :2], x[:, 2:4])
    assert np.all(got[:, 2] == 0.0)           # column 4 is past the limit
    dv.set_int(ctx, first, 5)
    dv.gather_cols(ctx, X, first, 1, 6, Y[:, :1], d=D)
    ref = dv.new_block(dim, 1)
    _lib.call("svdsb_diag_solve", dim, dv.P(D), dv.P(X[:, 5:6]), dv.ld_of(X), dv.P(ref), dv.ld_of(ref), 1,
              ctx.stream)
    assert np.array_equal(dv.to_host(Y[:, :1]), dv.to_host(ref))
    assert np.array_equal(dv.to_host(ref)[:, 0], x[:, 5] / d)


@pytest.mark.parametrize("dim,g", [(7, 3), (5000, 30), (300001, 40), (300001, 1)])
@pytest.mark.parametrize("precond", [False, True])
def test_cgs_fused_matches_pass_by_pass(dim, g, precond, rng):
    """svdsb_cgs_fused (one launch, software grid barrier) against the
    pass-by-pass kernels: same selected column, +k copy, DGKS pass count and
    orthonormalised vector to rounding."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    q, _ = np.linalg.qr(rng.standard_normal((dim, g)))
    V = dv.to_device_block(q)
    R = dv.to_device_block(rng.standard_normal((dim, 3)) + 0.5 * q[:, :1])
    d = torch.from_numpy(rng.uniform(0.5, 2.0, dim)).cuda() if precond else None
    ci = torch.tensor([1], dtype=torch.int32, device="cuda")
    Y = dv.to_device_block(rng.standard_normal((g, g)))
    kk = 2
    n_, ptrs, lds, cols, _ = dv._blk_args([V])
    outs = []
    for fused in (True, False):
        x = dv.new_block(dim, 1)
        prev = dv.small_matrix(g, kk)
        st = torch.zeros(8, dtype=torch.float64, device="cuda")
        if fused:
            _lib.call("svdsb_cgs_fused", ctx.handle, dim, n_, ptrs, lds, cols, dv.P(R), dv.ld_of(R), dv.P(ci),
                      None if d is None else dv.P(d), dv.P(x), dv.P(Y), dv.ld_of(Y), g, kk, dv.P(prev),
                      dv.ld_of(prev), 3, dv.P(st), ctx.stream)
        else:
            cw = torch.zeros(256, dtype=torch.float64, device="cuda")
            dv.gather_cols(ctx, Y, ci, kk, g, prev)
            dv.gather_cols(ctx, R, ci, 1, 3, x, d=d)
            _lib.call("svdsb_dgks_begin", dv.P(st), ctx.stream)
            for p in range(3):
                _lib.call("svdsb_cgs_pass", ctx.handle, dim, n_, ptrs, lds, cols, dv.P(x), dv.P(cw), dv.P(st),
                          1 if p == 0 else 0, ctx.stream)
            dv.scale_cols(ctx, x, st[5:6], dv.SCALE_DIV)
        outs.append((dv.to_host(x)[:, 0], dv.to_host(prev), st.cpu().numpy()))
    (xf, pf, sf), (xr, pr, sr) = outs
    assert np.array_equal(pf[:, :1], pr[:, :1]) and np.array_equal(pf, pr)
    assert sf[0] == sr[0] == 0.0 and sf[1] == sr[1] and sf[5] > 0.0
    assert abs(sf[5] - sr[5]) <= 1e-12 * sr[5]
    assert np.abs(xf - xr).max() <= 1e-12
    assert abs(np.linalg.norm(xf) - 1.0) <= 1e-13
    assert np.abs(q.T @ xf).max() <= 1e-13


@pytest.mark.parametrize("g,s", [(20, 3), (35, 8), (35, 15), (35, 20), (40, 32)])
def test_restart_inplace_product_variants(g, s, rng):
    """Thick-restart V <- V C in place: the vectorised kernel
    (ts_gemm_inplace_vec_kernel) and the generic one (svdsb_tune_set key
    4 = 2) give the same bits, equal to X C within rounding, on an odd row
    count; the columns past s are untouched."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim = 200_001
    x0 = rng.standard_normal((dim, g))
    c = rng.standard_normal((g, s))
    outs = []
    for key in (0, 2):
        X = dv.to_device_block(x0)
        C = dv.to_device_block(c)
        try:
            _lib.call("svdsb_tune_set", 4, key)
            dv.ts_gemm(ctx, X, C, X[:, :s])
        finally:
            _lib.call("svdsb_tune_set", 4, 0)
        outs.append(dv.to_host(X))
    assert np.array_equal(outs[0], outs[1])
    want = x0 @ c
    assert np.abs(outs[0][:, :s] - want).max() <= 1e-13 * np.abs(want).max() * g
    assert np.array_equal(outs[0][:, s:], x0[:, s:])


@pytest.mark.parametrize("b", [2, 3, 4])
def test_cgs_block_matches_column_loop(b, rng):
    """svdsb_cgs_block (first CGS pass batched over the block's columns)
    against the reference's column loop run on the host with NumPy
    (kernels.py:54-133): the same DGKS pass counts, the same vectors to
    rounding, an orthonormal block orthogonal to the basis; a column that
    repeats an earlier one is reported collapsed (state[5] == 0) so the
    solver redoes the block on the host path."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim, g = 400_000, 27
    q, _ = np.linalg.qr(rng.standard_normal((dim, g)))
    S = rng.standard_normal((dim, b)) + q[:, :b] * 3.0
    V = dv.to_device_block(q)
    n_, ptrs, lds, cols, _ = dv._blk_args([V])
    for collapse in (False, True):
        src = S.copy()
        if collapse:
            src[:, b - 1] = src[:, 0]
        X = dv.to_device_block(src)
        st = torch.zeros(8 * b, dtype=torch.float64, device="cuda")
        cw = torch.zeros(1024, dtype=torch.float64, device="cuda")
        _lib.call("svdsb_cgs_block", ctx.handle, dim, n_, ptrs, lds, cols, dv.P(X), dv.ld_of(X), b, dv.P(cw),
                  dv.P(st), 3, ctx.stream)
        got, rec = dv.to_host(X), st.cpu().numpy().reshape(b, 8)
        # host column loop (the reference's algorithm)
        want = src.copy()
        passes = []
        for j in range(b):
            prior = np.concatenate([q, want[:, :j]], axis=1)
            v = want[:, j]
            orig = prev = np.linalg.norm(v)
            hits, npass, final = 0, 0, 0.0
            for _ in range(3):
                v -= prior @ (prior.T @ v)
                npass += 1
                cur = np.linalg.norm(v)
                if cur < 1e-14 * orig:
                    hits += 1
                    if hits >= 2:
                        break
                elif cur > 2 ** -0.5 * prev:
                    final = cur
                    break
                else:
                    hits = 0
                prev = cur
            passes.append(npass)
            if final > 0:
                v /= final
        if not collapse:
            assert (rec[:, 0] == 0.0).all() and (rec[:, 5] > 0.0).all()
            assert list(rec[:, 1].astype(int)) == passes
            assert np.abs(got - want).max() <= 1e-12
            assert np.abs(got.T @ got - np.eye(b)).max() <= 1e-13
            assert np.abs(q.T @ got).max() <= 1e-13
        else:
            assert rec[b - 1, 5] == 0.0 or rec[b - 1, 0] != 0.0


def test_grid_barrier_and_ticket_reductions_stress(rng):
    """Race evidence for the synchronisation the kernels build themselves
    (compute-sanitizer is closed on the GPU pool): the software grid
    barrier of svdsb_cgs_fused and the last-CTA ticket folds of the Gram /
    projection / Ritz kernels, 300 times each while a second stream keeps
    the SMs busy with independent work (so CTA scheduling and completion
    order vary between repetitions).  Every repetition must give the same
    bits: a lost update, a stale partial or a barrier passed early shows up
    as a different result."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    dim, g = 300_000, 33
    q, _ = np.linalg.qr(rng.standard_normal((dim, g)))
    V = dv.to_device_block(q)
    W = dv.to_device_block(rng.standard_normal((dim, g)))
    R = dv.to_device_block(rng.standard_normal((dim, 3)) + 0.5 * q[:, :1])
    Y = dv.to_device_block(np.linalg.qr(rng.standard_normal((g, g)))[0])
    lam = torch.from_numpy(rng.standard_normal(g)).cuda()
    ci = torch.tensor([1], dtype=torch.int32, device="cuda")
    n_, ptrs, lds, cols, _ = dv._blk_args([V])
    noise = torch.randn(1 << 24, device="cuda")
    side = torch.cuda.Stream()
    ref = None
    for rep in range(300):
        with torch.cuda.stream(side):
            for _ in range(3):
                noise.mul_(1.0000001).add_(1e-7)
        x = dv.new_block(dim, 1)
        prev = dv.small_matrix(g, 2)
        st = torch.zeros(8, dtype=torch.float64, device="cuda")
        _lib.call("svdsb_cgs_fused", ctx.handle, dim, n_, ptrs, lds, cols, dv.P(R), dv.ld_of(R), dv.P(ci), None,
                  dv.P(x), dv.P(Y), dv.ld_of(Y), g, 2, dv.P(prev), dv.ld_of(prev), 3, dv.P(st), ctx.stream)
        c = dv.small_matrix(g, 4)
        nr = torch.zeros(4, dtype=torch.float64, device="cuda")
        dv.gram(ctx, dim, [V], W[:, :4], c, norms2=nr)
        y4 = W[:, 4:8].clone()
        dv.project_out(ctx, dim, [V], c, y4)
        r = dv.new_block(dim, 12)
        rn2 = torch.zeros(12, dtype=torch.float64, device="cuda")
        dv.ritz_residual(ctx, V, W, Y[:, :12], lam[:12], r, rn2=rn2)
        got = [t.cpu().numpy().copy() for t in (x, st, c, nr, y4, rn2)] + [float(r.sum())]
        if ref is None:
            ref = got
            assert ref[1][0] == 0.0 and ref[1][5] > 0.0
        else:
            for a, b in zip(ref[:-1], got[:-1]):
                assert np.array_equal(a, b), rep
            assert ref[-1] == got[-1], rep
    torch.cuda.synchronize()


def test_config4_shape_b4_products_at_hbm_scale(rng):
    """Config 4's generator at a fifth of its size (2 M x 200 k, ~35 M nnz,
    every operand larger than L2): the sliced-ELL forward b = 4 product
    against the oracle bit for bit, and the transposed b = 4 product on the
    length-sorted sliced ELL against the CSR-tile kernel bit for bit (the
    oracle's add.at is too slow at this size), with the C-apply passing the
    adjoint identity <A x, A x> = <x, A^T A x>."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdOperator, _lib, make_normal_operator, workloads
    dv = _dev()
    m, n, r, c, v = workloads.c4_coo(m=2_000_000, n=200_000)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    del r, c, v
    a = SparseMatrixCsr(m, n, rp, ci, va)
    x = rng.standard_normal((n, 4))
    assert np.array_equal(_spmv_dev(a, x, False), ocsr.spmv(m, n, rp, ci, va, x))
    y = rng.standard_normal((m, 4))
    try:
        _lib.call("svdsb_tune_set", 5, 1)
        ref_t = _spmv_dev(a, y, True)
    finally:
        _lib.call("svdsb_tune_set", 5, 0)
    assert np.array_equal(_spmv_dev(a, y, True), ref_t)
    op = make_normal_operator(SvdOperator.from_csr(a, check=False))
    cx = dv.to_host(op.apply(dv.to_device_block(x)))
    ax = ocsr.spmv(m, n, rp, ci, va, x)
    lhs, rhs = (ax * ax).sum(0), (x * cx).sum(0)
    assert np.all(np.abs(lhs - rhs) <= 1e-11 * np.abs(lhs))


def test_config3_full_size_adjoint_identity(rng):
    """Config 3 at its full size (160^3, 28.5 M nnz): A x bit-exact against
    the oracle and <A x, y> = <x, A^T y> within rounding."""
    from paper_1607_01404_b200 import SparseMatrixCsr, workloads
    m, n, r, c, v = workloads.c3_coo()
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    del r, c, v
    a = SparseMatrixCsr(m, n, rp, ci, va)
    x = rng.standard_normal((n, 1))
    y = rng.standard_normal((m, 1))
    ax = _spmv_dev(a, x, False)
    assert np.array_equal(ax, ocsr.spmv(m, n, rp, ci, va, x))
    aty = _spmv_dev(a, y, True)
    lhs, rhs = float((ax * y).sum()), float((x * aty).sum())
    assert abs(lhs - rhs) <= 1e-12 * np.sqrt(n) * np.abs(ax).max() * np.abs(y).max()


def test_from_coo_range_checks():
    """Index validation of SparseMatrixCsr.from_coo (matio.py:41-52), done on
    the device copies: ValueError for rows >= m, negative columns, columns
    >= n; equal-length check on the host."""
    from paper_1607_01404_b200 import SparseMatrixCsr
    ok = (np.array([0, 1]), np.array([0, 2]), np.array([1.0, 2.0]))
    SparseMatrixCsr.from_coo(2, 3, *ok)
    with pytest.raises(ValueError, match="row index"):
        SparseMatrixCsr.from_coo(2, 3, np.array([0, 2]), ok[1], ok[2])
    with pytest.raises(ValueError, match="column index"):
        SparseMatrixCsr.from_coo(2, 3, ok[0], np.array([-1, 0]), ok[2])
    with pytest.raises(ValueError, match="column index"):
        SparseMatrixCsr.from_coo(2, 3, ok[0], np.array([0, 3]), ok[2])
    with pytest.raises(ValueError, match="equal length"):
        SparseMatrixCsr.from_coo(2, 3, ok[0], ok[1], np.array([1.0]))


# ---------------------------------------------------------------- streamed
# (cp.async.bulk ring) tall-skinny kernels, svdsb_tune_set key 15


@pytest.mark.parametrize("dim", [1, 255, 257, 70_001, 300_002])
@pytest.mark.parametrize("g,p", [(35, 24), (35, 11), (8, 3), (40, 32), (17, 16), (5, 7)])
def test_ritz_residual_streamed_bit_identical(dim, g, p, rng):
    """ts_stream_kernel<2, PQ, true> against the register-tiled Ritz kernels:
    R, X = V Y and OpX = W Y bit for bit (same fma chain), |R_j|^2 to
    rounding, on odd / sub-tile / multi-tile row counts and partial column
    chunks; the status copy is exercised by the solver tests."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    vh, wh = rng.standard_normal((dim, g)), rng.standard_normal((dim, g))
    yh = rng.standard_normal((g, p))
    lh = rng.standard_normal(p)
    V, W, Y = dv.to_device_block(vh), dv.to_device_block(wh), dv.to_device_block(yh)
    lam = torch.from_numpy(lh).to(ctx.device)
    outs = []
    try:
        for key in (1, 2, 3, 4):   # 3 / 4: the twelve- / sixteen-warp variants for 16 < p <= 24
            _lib.call("svdsb_tune_set", 15, key)
            R, X, OX = dv.new_block(dim, p), dv.new_block(dim, p), dv.new_block(dim, p)
            rn2 = torch.zeros(p, dtype=torch.float64, device=ctx.device)
            dv.ritz_residual(ctx, V, W, Y, lam, R, x=X, ox=OX, rn2=rn2)
            outs.append((dv.to_host(R), dv.to_host(X), dv.to_host(OX), rn2.cpu().numpy()))
    finally:
        _lib.call("svdsb_tune_set", 15, 0)
    for k in range(3):
        assert np.array_equal(outs[0][k], outs[1][k])
        assert np.array_equal(outs[0][k], outs[2][k])
        assert np.array_equal(outs[0][k], outs[3][k])
    assert np.allclose(outs[2][3], outs[1][3], rtol=1e-12)
    assert np.allclose(outs[3][3], outs[1][3], rtol=1e-12)
    want = wh @ yh - (vh @ yh) * lh
    assert np.abs(outs[1][0] - want).max() <= 1e-12 * max(np.abs(want).max(), 1.0)
    assert np.allclose(outs[1][3], (want ** 2).sum(0), rtol=1e-12)


@pytest.mark.parametrize("dim", [1, 257, 200_001])
@pytest.mark.parametrize("g,s", [(20, 3), (35, 15), (35, 20), (40, 32), (9, 9)])
def test_restart_inplace_streamed_bit_identical(dim, g, s, rng):
    """In-place V <- V C through the streamed kernel equals the vectorised
    register kernel bit for bit; columns past s untouched."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    x0 = rng.standard_normal((dim, g))
    c = rng.standard_normal((g, s))
    outs = []
    for key in (1, 2):
        X = dv.to_device_block(x0)
        C = dv.to_device_block(c)
        try:
            _lib.call("svdsb_tune_set", 15, key)
            dv.ts_gemm(ctx, X, C, X[:, :s])
        finally:
            _lib.call("svdsb_tune_set", 15, 0)
        outs.append(dv.to_host(X))
    assert np.array_equal(outs[0], outs[1])
    want = x0 @ c
    assert np.abs(outs[1][:, :s] - want).max() <= 1e-13 * np.abs(want).max() * g
    assert np.array_equal(outs[1][:, s:], x0[:, s:])


@pytest.mark.parametrize("dim", [1, 127, 129, 70_001, 300_002])
@pytest.mark.parametrize("g,b", [(35, 4), (40, 4), (7, 2), (20, 3), (1, 4), (33, 7), (35, 1), (3, 1)])
def test_gram_streamed(dim, g, b, rng):
    """gram_stream_kernel against fp64 numpy and the register-tiled kernel
    (different summation trees: rounding-level agreement), norms included;
    two calls give identical bits (fixed tile ranges and trees)."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    a = rng.standard_normal((dim, g))
    y = rng.standard_normal((dim, b))
    X, Y = dv.to_device_block(a), dv.to_device_block(y)
    outs = []
    try:
        for key in (1, 2, 2):
            _lib.call("svdsb_tune_set", 15, key)
            C = dv.small_matrix(g, b)
            nrm = torch.zeros(b, dtype=torch.float64, device=ctx.device)
            dv.gram(ctx, dim, [X], Y, C, norms2=nrm)
            outs.append((dv.to_host(C), nrm.cpu().numpy()))
    finally:
        _lib.call("svdsb_tune_set", 15, 0)
    want = a.T @ y
    tol = 1e-13 * max(np.abs(want).max(), 1.0) * np.sqrt(dim)
    for got, n2 in outs:
        assert np.abs(got - want).max() <= tol
        assert np.allclose(n2, (y ** 2).sum(0), rtol=1e-13)
    assert np.array_equal(outs[1][0], outs[2][0]) and np.array_equal(outs[1][1], outs[2][1])


@pytest.mark.parametrize("dim", [1, 255, 257, 70_001, 300_002])
@pytest.mark.parametrize("g1,g2,b", [(35, 0, 1), (7, 30, 4), (40, 0, 2), (3, 5, 3), (1, 0, 1), (20, 13, 6)])
def test_project_streamed_bit_identical(dim, g1, g2, b, rng):
    """project_stream_kernel against the register kernels: Y -= X C bit for
    bit (same fma chain, basis index ascending, one or two basis blocks),
    |Y_j|^2 to rounding; b = 6 runs as 4 + 2 columns."""
    from paper_1607_01404_b200 import _lib
    dv = _dev()
    ctx = dv.context()
    a1 = rng.standard_normal((dim, g1))
    a2 = rng.standard_normal((dim, max(g2, 1)))
    y = rng.standard_normal((dim, b))
    c = rng.standard_normal((g1 + g2, b)) * 0.1
    X1, X2 = dv.to_device_block(a1), dv.to_device_block(a2)
    blocks = [X1, X2] if g2 else [X1]
    outs = []
    try:
        for key in (1, 2):
            _lib.call("svdsb_tune_set", 15, key)
            Y = dv.to_device_block(y)
            C = dv.to_device_block(c)
            nrm = torch.zeros(b, dtype=torch.float64, device=ctx.device)
            dv.project_out(ctx, dim, blocks, C, Y, norms2=nrm)
            outs.append((dv.to_host(Y), nrm.cpu().numpy()))
    finally:
        _lib.call("svdsb_tune_set", 15, 0)
    assert np.array_equal(outs[0][0], outs[1][0])
    want = y - np.hstack([a1, a2[:, :g2]]) @ c
    assert np.abs(outs[1][0] - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    assert np.allclose(outs[1][1], (want ** 2).sum(0), rtol=1e-12, atol=1e-300)
    assert np.allclose(outs[1][1], outs[0][1], rtol=1e-12, atol=1e-300)


def test_from_coo_values_copied_on_side_stream(rng):
    """from_coo of large host arrays copies the values on a side stream
    while the indices are sorted (svdsb_csr_create_coo_device_ev waits for
    the copy's event before the duplicate sums): the assembled CSR and its
    stored transpose equal the oracle's bit for bit, pinned or pageable
    inputs, three times in a row (the side stream and buffers get reused)."""
    from paper_1607_01404_b200 import SparseMatrixCsr
    m, n, nt = 200_000, 50_000, (1 << 22) + 12_345
    rows = rng.integers(0, m, nt)
    cols = rng.integers(0, n, nt)
    cols[: nt // 8] = rng.integers(0, 4, nt // 8)          # hot columns: duplicates to sum, long A^T rows
    vals = rng.standard_normal(nt)
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    trp, tci, tva = ocsr.csr_from_coo(n, m, cols, rows, vals)
    pinned = [torch.from_numpy(a).pin_memory() for a in (rows, cols, vals)]
    for rep in range(3):
        src = pinned if rep != 1 else (rows, cols, vals)
        a = SparseMatrixCsr.from_coo(m, n, *src)
        grp, gci, gva = a.device_csr().export()
        assert np.array_equal(grp, rp) and np.array_equal(gci, ci) and np.array_equal(gva, va)
        g2 = a.device_csr().export(transpose=True)
        assert np.array_equal(g2[0], trp) and np.array_equal(g2[1], tci) and np.array_equal(g2[2], tva)

"""Matrix Market ingestion.

Same functions, arguments, results and errors as the reference's
pkg/src/itersvd/matio.py:158-276 (``read_matrix_market``,
``write_matrix_market``, ``write_dense_market``, ``read_dense_market``,
``MatrixMarketError``).  Parsing runs in the native library
(csrc/mmio.cpp, one pass over the file in C++); the triplets then go to the
device CSR assembly, which sums duplicates in input order exactly like the
reference's ``SparseMatrixCsr.from_coo``.  ``read_matrix_market_coo``
returns the parsed (and symmetric-expanded) triplets without assembling.

Binary CSR cache (an addition of this build):
``read_matrix_market(path, cache=True)`` keeps the assembled CSR next to
the file (``<path>.csrb``, keyed on the source's size and mtime) and later
reads skip parsing and assembly; ``save_csr`` / ``load_csr`` read and
write the format directly.
"""

import ctypes
import os

import numpy as np

from . import _lib
from .matrix import SparseMatrixCsr


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; carries the offending line number
    (matio.py:12-19)."""

    def __init__(self, message, line=None):
        if line is not None:
            message = "line %d: %s" % (line, message)
        super().__init__(message)
        self.line = line


def _path(path):
    return os.fsencode(os.fspath(path))


def _check(rc, err_line, what):
    if rc == 0:
        return
    if rc == -5:
        raise MatrixMarketError(_lib.last_error(), line=int(err_line.value))
    _lib.check(rc, what)


def read_matrix_market_coo(path):
    """(m, n, rows, cols, vals, is_array) of a Matrix Market file: 0-based
    int64 indices, symmetric storage expanded as the reference does
    (stored entries first, then the mirrored off-diagonal ones), stored zeros
    of array files dropped (matio.py:170-241)."""
    lib = _lib.load()
    m, n, entries = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    is_array, symmetric = ctypes.c_int(), ctypes.c_int()
    err = ctypes.c_int64()
    p = _path(path)
    rc = lib.svdsb_mm_read_header(p, ctypes.byref(m), ctypes.byref(n), ctypes.byref(entries),
                                  ctypes.byref(is_array), ctypes.byref(symmetric), ctypes.byref(err))
    _check(rc, err, "svdsb_mm_read_header")
    cnt = int(entries.value)
    rows = np.empty(cnt, dtype=np.int64)
    cols = np.empty(cnt, dtype=np.int64)
    vals = np.empty(cnt, dtype=np.float64)
    rc = lib.svdsb_mm_read_entries(p, cnt, _lib.np_ptr(rows), _lib.np_ptr(cols), _lib.np_ptr(vals),
                                   ctypes.byref(err))
    _check(rc, err, "svdsb_mm_read_entries")
    if symmetric.value:
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    if is_array.value:
        # dense storage forces zeros in; the reference drops them after
        # assembly (no duplicates exist in array storage, so before is equal)
        keep = vals != 0.0
        if not keep.all():
            rows, cols, vals = rows[keep], cols[keep], vals[keep]
    return int(m.value), int(n.value), rows, cols, vals, bool(is_array.value)


def read_matrix_market(path, device=None, cache=None):
    """Read a real Matrix Market file into a (device-assembled) CSR matrix
    (matio.py:170-241).  ``coordinate real/integer/double general|symmetric``
    and ``array real general``; anything else raises MatrixMarketError with
    the reference's message and line number.

    cache: None/False (the reference's behaviour), True (``<path>.csrb``) or
    a cache file path.  A cache written for the same source size and mtime
    is loaded instead of parsing; otherwise the file is parsed, assembled
    and the cache (re)written."""
    cpath = None
    if cache:
        cpath = os.fspath(path) + ".csrb" if cache is True else os.fspath(cache)
        key = _source_key(path)
        hit = _load_csr_arrays(cpath, expect_key=key)
        if hit is not None:
            m, n, rp, ci, va = hit
            return SparseMatrixCsr(m, n, rp, ci, va)
    m, n, rows, cols, vals, _ = read_matrix_market_coo(path)
    if rows.size == 0 or m == 0 or n == 0:
        a = SparseMatrixCsr(m, n, np.zeros(m + 1, dtype=np.int64), np.zeros(0, dtype=np.int64),
                            np.zeros(0, dtype=np.float64))
    else:
        a = SparseMatrixCsr.from_coo(m, n, rows, cols, vals, device=device)
    if cpath is not None:
        save_csr(cpath, a, source_key=key)
    return a


# ------------------------------------------------------------ CSR cache
_MAGIC = b"SVDSBCSR"
_VERSION = 1
_HDR = np.dtype([("magic", "S8"), ("version", "<u4"), ("idx32", "<u4"), ("m", "<i8"), ("n", "<i8"),
                 ("nnz", "<i8"), ("src_size", "<i8"), ("src_mtime_ns", "<i8")])


def _source_key(path):
    st = os.stat(path)
    return int(st.st_size), int(st.st_mtime_ns)


def save_csr(path, a, source_key=(-1, -1)):
    """Write a SparseMatrixCsr in the binary cache format: a 56-byte header
    (magic, version, index width, m, n, nnz, source size / mtime), then
    row_ptr (int64, m+1), col_idx (int32 when n < 2^31, else int64) and
    values (float64), little endian.  Written to a temporary name and
    renamed, so a reader never sees a partial file."""
    rp = np.ascontiguousarray(a.row_ptr, dtype="<i8")
    idx32 = a.n < 2 ** 31
    ci = np.ascontiguousarray(a.col_idx, dtype="<i4" if idx32 else "<i8")
    va = np.ascontiguousarray(a.values, dtype="<f8")
    hdr = np.zeros(1, dtype=_HDR)
    hdr[0] = (_MAGIC, _VERSION, int(idx32), a.m, a.n, va.shape[0], source_key[0], source_key[1])
    tmp = "%s.tmp%d" % (os.fspath(path), os.getpid())
    with open(tmp, "wb") as fh:
        fh.write(hdr.tobytes())
        fh.write(rp.tobytes())
        fh.write(ci.tobytes())
        fh.write(va.tobytes())
    os.replace(tmp, path)


def _load_csr_arrays(path, expect_key=None):
    try:
        fh = open(path, "rb")
    except OSError:
        return None
    with fh:
        raw = fh.read(_HDR.itemsize)
        if len(raw) != _HDR.itemsize:
            return None
        h = np.frombuffer(raw, dtype=_HDR)[0]
        if h["magic"] != _MAGIC or int(h["version"]) != _VERSION:
            return None
        if expect_key is not None and (int(h["src_size"]), int(h["src_mtime_ns"])) != tuple(expect_key):
            return None
        m, n, nnz = int(h["m"]), int(h["n"]), int(h["nnz"])
        rp = np.fromfile(fh, dtype="<i8", count=m + 1)
        ci = np.fromfile(fh, dtype="<i4" if int(h["idx32"]) else "<i8", count=nnz)
        va = np.fromfile(fh, dtype="<f8", count=nnz)
    if rp.shape[0] != m + 1 or ci.shape[0] != nnz or va.shape[0] != nnz:
        return None   # truncated: treat as a miss
    return m, n, rp, ci.astype(np.int64, copy=False), va


def load_csr(path):
    """Read a binary CSR cache file (any source key) as a SparseMatrixCsr;
    ValueError when the file is not a complete cache file."""
    got = _load_csr_arrays(path)
    if got is None:
        raise ValueError("%s is not a complete svdsb CSR cache file" % (os.fspath(path),))
    m, n, rp, ci, va = got
    return SparseMatrixCsr(m, n, rp, ci, va)


def write_matrix_market(path, a):
    """``coordinate real general`` with %.17g values (matio.py:244-251)."""
    rp = _lib.as_i64(a.row_ptr)
    ci = _lib.as_i64(a.col_idx)
    va = _lib.as_f64(a.values)
    rc = _lib.load().svdsb_mm_write_coo(_path(path), int(a.m), int(a.n), int(va.shape[0]), _lib.np_ptr(rp),
                                        _lib.np_ptr(ci), _lib.np_ptr(va))
    _lib.check(rc, "svdsb_mm_write_coo")


def write_dense_market(path, a):
    """``array real general``, column major (matio.py:254-262); ``a`` may be
    a host array or a device tensor."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError("dense block must be two-dimensional")
    rc = _lib.load().svdsb_mm_write_array(_path(path), int(a.shape[0]), int(a.shape[1]), _lib.np_ptr(a),
                                          max(int(a.shape[0]), 1))
    _lib.check(rc, "svdsb_mm_write_array")


def read_dense_market(path):
    """An ``array real general`` file as a dense column-major host block
    (matio.py:265-268)."""
    m, n, rows, cols, vals, _ = read_matrix_market_coo(path)
    out = np.zeros((m, n), dtype=np.float64, order="F")
    # duplicates only arise from coordinate files: summed in input order,
    # as the reference's CSR assembly does before densifying
    np.add.at(out, (rows, cols), vals)
    return out

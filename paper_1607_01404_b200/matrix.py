"""CSR matrix: host container in the reference layout, device-resident
storage of A and its stored transpose for the kernels.

Mirrors ``SparseMatrixCsr`` (pkg/src/itersvd/matio.py:22-123): int64
``row_ptr``/``col_idx`` and fp64 ``values`` with strictly increasing columns
per row and duplicates summed at assembly.  The difference is where the
data lives: the device copy (int32 indices, plus CSR(A^T) built on device
by a stable radix sort, bit-identical to ``from_coo(n, m, cols, rows,
vals)``) is what every product uses; the host arrays are materialised
lazily only when someone asks for them.
"""

import ctypes
import itertools

import numpy as np
import torch

from . import _lib
from .device import context, require_cuda

# When set to a list, every SpMV appends (kind, block, start_event,
# end_event) with kind in fwd / adj / normal (both products) recorded on the launching stream (bench.py's roofline probe).
SPMV_PROFILER = None

_UIDS = itertools.count(1)


_SIDE = {}


def _side_stream(device):
    """One extra stream per device for copies that overlap the assembly."""
    key = torch.device(device).index
    st = _SIDE.get(key)
    if st is None:
        st = _SIDE[key] = torch.cuda.Stream(device=device)
    return st


class DeviceCsr:
    """Owning handle to a libsvdsb CSR (A and A^T) on one device."""

    def __init__(self, handle, ctx, m, n, nnz):
        # process-unique id: a freed handle's address can be reused by the
        # next matrix, so captured graphs are keyed by this instead
        self.uid = next(_UIDS)
        self.handle = handle
        self.ctx = ctx
        self.m, self.n, self.nnz = int(m), int(n), int(nnz)

    @classmethod
    def from_host(cls, m, n, row_ptr, col_idx, values, device=None, transpose=True):
        ctx = context(device)
        rp = _lib.as_i64(row_ptr)
        ci = _lib.as_i64(col_idx)
        va = _lib.as_f64(values)
        h = ctypes.c_void_p()
        flags = _lib.SVDSB_CSR_TRANSPOSE if transpose else 0
        with torch.cuda.device(ctx.device):
            _lib.call("svdsb_csr_create_host", ctx.handle, int(m), int(n), int(va.shape[0]),
                      _lib.np_ptr(rp), _lib.np_ptr(ci), _lib.np_ptr(va), flags, ctx.stream,
                      ctypes.byref(h))
        return cls(h, ctx, m, n, va.shape[0])

    @classmethod
    def from_coo_device(cls, m, n, rows, cols, vals, device=None, transpose=True, vals_ready=None):
        """rows/cols int64, vals fp64, all torch device tensors.  vals_ready:
        a recorded torch.cuda.Event after which `vals` is complete (its copy
        may still run on another stream while the indices are sorted)."""
        ctx = context(device)
        rows = rows.to(device=ctx.device, dtype=torch.int64).contiguous()
        cols = cols.to(device=ctx.device, dtype=torch.int64).contiguous()
        vals = vals.to(device=ctx.device, dtype=torch.float64).contiguous()
        h = ctypes.c_void_p()
        flags = _lib.SVDSB_CSR_TRANSPOSE if transpose else 0
        with torch.cuda.device(ctx.device):
            ev = ctypes.c_void_p(vals_ready.cuda_event) if vals_ready is not None else None
            _lib.call("svdsb_csr_create_coo_device_ev", ctx.handle, int(m), int(n), int(rows.numel()),
                      ctypes.c_void_p(rows.data_ptr()), ctypes.c_void_p(cols.data_ptr()),
                      ctypes.c_void_p(vals.data_ptr()), ev, flags, ctx.stream, ctypes.byref(h))
        nnz = ctypes.c_int64()
        _lib.call("svdsb_csr_shape", h, None, None, ctypes.byref(nnz))
        return cls(h, ctx, m, n, nnz.value)

    def layout_info(self, key):
        """Derived-layout counters (svdsb_csr_layout_info; tests and tools)."""
        out = ctypes.c_int64()
        _lib.call("svdsb_csr_layout_info", self.handle, int(key), ctypes.byref(out))
        return out.value

    def export(self, transpose=False):
        """(row_ptr, col_idx, values) of A (or A^T) in the reference layout."""
        rows = self.n if transpose else self.m
        rp = np.empty(rows + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int64)
        va = np.empty(self.nnz, dtype=np.float64)
        _lib.call("svdsb_csr_export_host", self.handle, int(bool(transpose)), _lib.np_ptr(rp),
                  _lib.np_ptr(ci), _lib.np_ptr(va))
        return rp, ci, va

    def device_arrays(self, transpose=False):
        """(row_ptr int32, col int32, val fp64) device pointers as ints."""
        rp, ci, va = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("svdsb_csr_device_arrays", self.handle, int(bool(transpose)), ctypes.byref(rp),
                  ctypes.byref(ci), ctypes.byref(va))
        return rp.value, ci.value, va.value

    def fro_norm(self):
        """||A||_F from the device values (one reduction)."""
        from .device import DTYPE
        _, _, va = self.device_arrays()
        out = torch.zeros(1, dtype=DTYPE, device=self.ctx.device)
        if self.nnz:
            _lib.call("svdsb_col_norms2", self.ctx.handle, self.nnz, ctypes.c_void_p(va), self.nnz, 1,
                      ctypes.c_void_p(out.data_ptr()), self.ctx.stream)
        return float(torch.sqrt(out).item())

    def matvec(self, x, y, transpose=False):
        """y = A x (or A^T x) on column-major device blocks (PRIMME
        matrixMatvec)."""
        from .device import P, ld_of, as_block
        x, y = as_block(x), as_block(y)
        prof = SPMV_PROFILER
        if prof is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        _lib.call("svdsb_matvec", self.ctx.handle, self.handle, int(bool(transpose)), P(x), ld_of(x),
                  P(y), ld_of(y), x.shape[1], self.ctx.stream)
        if prof is not None:
            e1.record()
            prof.append(("adj" if transpose else "fwd", int(x.shape[1]), e0, e1))

    def scratch(self, rows, cols):
        """Grow-only column-major scratch block owned by the matrix (the
        inner product of the normal operator)."""
        from .device import new_block
        # single columns get their own never-reallocated buffer: captured
        # CUDA graphs of the one-column iteration bake its address in
        attr = "_scratch1" if cols <= 1 else "_scratch"
        buf = getattr(self, attr, None)
        if buf is None or buf.shape[0] != rows or buf.shape[1] < cols:
            buf = new_block(rows, max(cols, 1), device=self.ctx.device, zero=False)
            setattr(self, attr, buf)
        return buf[:, :cols]

    def col_sq_norms(self, out):
        """Unclamped squared column norms (matio.py:115-118) into out[n]."""
        from .device import P
        _lib.call("svdsb_row_sq", self.ctx.handle, self.handle, 0, P(out), self.ctx.stream)

    def precond_diag(self, side, out):
        from .device import P
        _lib.call("svdsb_precond_diag", self.ctx.handle, self.handle, int(side), P(out),
                  self.ctx.stream)

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib._lib is not None:
                if _lib.CAPTURING[0]:
                    _lib.DEFERRED.append(self.handle)   # destroyed after the capture
                else:
                    _lib._lib.svdsb_csr_destroy(self.handle)
                    _lib.flush_deferred()
        except Exception:
            pass


class SparseMatrixCsr:
    """Compressed sparse row matrix (reference type, matio.py:22-123).

    Construct from CSR arrays (validated like the reference's __init__) or
    with :meth:`from_coo` (assembled on device).  ``row_ptr``, ``col_idx``
    and ``values`` are host numpy arrays, produced on first access when the
    matrix was assembled on device.
    """

    def __init__(self, m, n, row_ptr, col_idx, values):
        self.m = int(m)
        self.n = int(n)
        rp = np.asarray(row_ptr, dtype=np.int64)
        ci = np.asarray(col_idx, dtype=np.int64)
        va = np.asarray(values, dtype=np.float64)
        # matio.py:41-52
        if self.m < 0 or self.n < 0:
            raise ValueError("negative matrix dimension")
        if rp.shape != (self.m + 1,):
            raise ValueError("row_ptr has wrong length")
        if rp[0] != 0 or rp[-1] != va.shape[0]:
            raise ValueError("row_ptr endpoints inconsistent with nnz")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be nondecreasing")
        if ci.shape != va.shape:
            raise ValueError("col_idx / values length mismatch")
        if ci.size and (ci.min() < 0 or ci.max() >= self.n):
            raise ValueError("column index out of range")
        self._host = (rp, ci, va)
        self._nnz = int(va.shape[0])
        self._dev = None

    @classmethod
    def _from_device(cls, dev):
        obj = cls.__new__(cls)
        obj.m, obj.n = dev.m, dev.n
        obj._host = None
        obj._nnz = dev.nnz
        obj._dev = dev
        return obj

    @classmethod
    def from_coo(cls, m, n, rows, cols, values, device=None):
        """Assemble from triplets, duplicates summed in ascending input order
        (matio.py:63-92), on the GPU."""
        require_cuda()
        def t(a, dt):
            if isinstance(a, torch.Tensor):
                return a
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt))
        rows = t(rows, np.int64)
        cols = t(cols, np.int64)
        values = t(values, np.float64)
        if not (rows.shape == cols.shape == values.shape):
            raise ValueError("triplet arrays must have equal length")
        ctx = context(device)
        rows = rows.to(device=ctx.device, dtype=torch.int64, non_blocking=True)
        cols = cols.to(device=ctx.device, dtype=torch.int64, non_blocking=True)
        ready = None
        if values.device.type == "cpu" and values.dtype == torch.float64 and values.numel() >= (1 << 22):
            # large host value arrays: copied on a side stream behind the index
            # copies, so the transfer overlaps the key build / sort / scans of
            # the assembly, which waits for it only before the duplicate sums
            main = torch.cuda.current_stream(ctx.device)
            side = _side_stream(ctx.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                values = values.to(device=ctx.device, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(side)
            values.record_stream(main)
        else:
            values = values.to(device=ctx.device, dtype=torch.float64, non_blocking=True)
        # the range checks of matio.py:74-78 run inside the device assembly
        # (svdsb_csr_create_coo_device: same messages, ValueError)
        dev = DeviceCsr.from_coo_device(m, n, rows, cols, values, device=ctx.device, vals_ready=ready)
        return cls._from_device(dev)

    @classmethod
    def from_dense(cls, a):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("matrix must be two-dimensional")
        rows, cols = np.nonzero(a)
        m, n = a.shape
        # np.nonzero is row-major ordered and duplicate free: CSR directly
        row_ptr = np.zeros(m + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        np.cumsum(row_ptr, out=row_ptr)
        return cls(m, n, row_ptr, cols, a[rows, cols])

    # ------------------------------------------------------------ access
    def _materialize(self):
        if self._host is None:
            self._host = self._dev.export(transpose=False)
        return self._host

    @property
    def row_ptr(self):
        return self._materialize()[0]

    @property
    def col_idx(self):
        return self._materialize()[1]

    @property
    def values(self):
        return self._materialize()[2]

    @property
    def nnz(self):
        return self._nnz

    @property
    def shape(self):
        return (self.m, self.n)

    def device_csr(self, device=None):
        """The device copy (uploaded on first use)."""
        if self._dev is None:
            rp, ci, va = self._host
            self._dev = DeviceCsr.from_host(self.m, self.n, rp, ci, va, device=device)
        return self._dev

    def to_dense(self):
        rp, ci, va = self._materialize()
        a = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.m, dtype=np.int64), np.diff(rp))
        a[rows, ci] = va
        return a

    def fro_norm(self):
        if self._host is not None:
            return float(np.linalg.norm(self._host[2]))
        return self._dev.fro_norm()

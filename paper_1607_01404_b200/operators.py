"""Operator plugin API on device blocks.

Mirrors pkg/src/itersvd/operators.py: ``SvdOperator`` (:50-136) is the
rectangular matrix with forward/transpose products and matvec counting,
``LinearOperator`` (:28-47) a square operator, ``make_normal_operator``
(:163-172) / ``make_augmented_operator`` (:175-190) derive C = A^T A (or
A A^T) and B = [0 A^T; A 0] without forming them, ``Preconditioner``
(:193-222) / ``jacobi_precond_on_normal`` (:225-249) the point-Jacobi
preconditioner, ``NormEstimate`` (:252-292) the running ||A|| estimate.

Operands are column-major fp64 CUDA tensors (rows, cols) with strides
(1, ld).  Built-in operators write into caller-provided outputs
(``apply_into``), the PRIMME ``matrixMatvec(x, ldx, y, ldy, blockSize)``
contract; ``apply`` returns a fresh block like the reference.  Callables
supplied by the user keep the reference contract (numpy block in, block
out) unless created with ``device=True`` (torch device block in/out).
"""

import warnings

import numpy as np
import torch

from . import device as dv
from .device import DTYPE
from .matrix import SparseMatrixCsr

EPS = 2.220446049250313e-16   # kernels.py:20
_PROBE_COUNT = 10             # operators.py:24
_PROBE_TOL = 1e-12            # operators.py:25


def _user_call(fn, x, rows_out, on_device):
    """Run a user callable on a device block, returning a device block."""
    if on_device:
        y = fn(x)
        if not isinstance(y, torch.Tensor):
            y = torch.as_tensor(np.asarray(y, dtype=np.float64))
        y = y.to(device=x.device, dtype=DTYPE)
    else:
        xh = np.asfortranarray(x.detach().cpu().numpy())
        y = torch.from_numpy(np.ascontiguousarray(np.asarray(fn(xh), dtype=np.float64)))
        y = y.to(device=x.device)
    if y.dim() == 1:
        y = y.unsqueeze(1)
    if y.shape != (rows_out, x.shape[1]):
        raise ValueError("operator returned shape %r, expected %r" % (tuple(y.shape), (rows_out, x.shape[1])))
    return y


class LinearOperator:
    """Square operator on device blocks (operators.py:28-47)."""

    def __init__(self, dim, apply_fn=None, symmetric=True, device=False, into=None):
        self.dim = int(dim)
        self._apply = apply_fn
        self._into = into          # native out-parameter form, if any
        self._on_device = device
        self.symmetric = symmetric
        self.n_applies = 0

    def apply_into(self, x, y):
        """y[:, :b] = Op x (counts b applications)."""
        x = dv.as_block(x)
        if x.shape[0] != self.dim:
            raise ValueError("operand has wrong leading dimension")
        self.n_applies += x.shape[1]
        if self._into is not None:
            self._into(x, y)
        else:
            y.copy_(_user_call(self._apply, x, self.dim, self._on_device))
        return y

    def apply(self, x):
        xt = x if isinstance(x, torch.Tensor) else dv.to_device_block(x)
        squeeze = xt.dim() == 1
        xb = dv.as_block(xt)
        y = dv.new_block(self.dim, xb.shape[1], device=xb.device, zero=False)
        self.apply_into(xb, y)
        return y[:, 0] if squeeze else y


class SvdOperator:
    """A rectangular matrix with forward and transpose products
    (operators.py:50-136).  One matvec is counted per column per product."""

    def __init__(self, m, n, apply_fn=None, apply_t_fn=None, explicit=None, check=True, device=False,
                 into=None, into_t=None):
        self.m = int(m)
        self.n = int(n)
        if self.m <= 0 or self.n <= 0:
            raise ValueError("matrix dimensions must be positive")
        self._apply = apply_fn
        self._apply_t = apply_t_fn
        self._into = into
        self._into_t = into_t
        self._on_device = device
        self.explicit = explicit
        self.n_matvecs = 0
        if check and explicit is not None:
            self._check_transpose_pair()

    @classmethod
    def from_csr(cls, a, check=True, device=None):
        dev = a.device_csr(device)
        op = cls(a.m, a.n, explicit=a, check=check,
                 into=lambda x, y: dev.matvec(x, y, transpose=False),
                 into_t=lambda x, y: dev.matvec(x, y, transpose=True))
        op._csr_dev = dev
        return op

    @classmethod
    def from_dense(cls, arr, check=True):
        return cls.from_csr(SparseMatrixCsr.from_dense(arr), check=check)

    @classmethod
    def from_callables(cls, m, n, apply_fn, apply_t_fn, device=False):
        return cls(m, n, apply_fn, apply_t_fn, device=device)

    @classmethod
    def wrap(cls, a):
        if isinstance(a, SvdOperator):
            return a
        if isinstance(a, SparseMatrixCsr):
            return cls.from_csr(a)
        return cls.from_dense(np.asarray(a, dtype=np.float64))

    @property
    def ctx(self):
        return dv.context()

    def _check_transpose_pair(self):
        """<y, A x> == <A^T y, x> on 10 random probes (operators.py:95-106),
        drawn on device from a generator seeded like the reference's."""
        ctx = dv.context()
        scale = self.explicit.fro_norm()
        gen = torch.Generator(device=ctx.device)
        gen.manual_seed(2 ** 20 + self.m * 31 + self.n)
        x = dv.new_block(self.n, _PROBE_COUNT)
        y = dv.new_block(self.m, _PROBE_COUNT)
        x.copy_(torch.randn((_PROBE_COUNT, self.n), generator=gen, device=ctx.device, dtype=DTYPE).t())
        y.copy_(torch.randn((_PROBE_COUNT, self.m), generator=gen, device=ctx.device, dtype=DTYPE).t())
        ax = dv.new_block(self.m, _PROBE_COUNT)
        aty = dv.new_block(self.n, _PROBE_COUNT)
        self._raw(x, ax, False)
        self._raw(y, aty, True)
        stats = torch.zeros(4 * _PROBE_COUNT, dtype=DTYPE, device=ctx.device)
        dv.col_dots(ctx, y, ax, stats[0:_PROBE_COUNT])
        dv.col_dots(ctx, aty, x, stats[_PROBE_COUNT:2 * _PROBE_COUNT])
        dv.col_norms2(ctx, x, stats[2 * _PROBE_COUNT:3 * _PROBE_COUNT])
        dv.col_norms2(ctx, y, stats[3 * _PROBE_COUNT:])
        lhs, rhs, nx2, ny2 = dv.fetch(ctx, [stats[i * _PROBE_COUNT:(i + 1) * _PROBE_COUNT] for i in range(4)])
        bound = _PROBE_TOL * max(1.0, scale) * np.sqrt(nx2) * np.sqrt(ny2)
        if np.any(np.abs(lhs - rhs) > bound):
            raise ValueError("forward and transpose products disagree")

    def _raw(self, x, y, transpose):
        if transpose:
            if self._into_t is not None:
                self._into_t(x, y)
            else:
                y.copy_(_user_call(self._apply_t, x, self.n, self._on_device))
        else:
            if self._into is not None:
                self._into(x, y)
            else:
                y.copy_(_user_call(self._apply, x, self.m, self._on_device))

    def apply_into(self, x, y):
        x = dv.as_block(x)
        if x.shape[0] != self.n:
            raise ValueError("operand has wrong leading dimension")
        self.n_matvecs += x.shape[1]
        self._raw(x, dv.as_block(y), False)
        return y

    def apply_t_into(self, x, y):
        x = dv.as_block(x)
        if x.shape[0] != self.m:
            raise ValueError("operand has wrong leading dimension")
        self.n_matvecs += x.shape[1]
        self._raw(x, dv.as_block(y), True)
        return y

    def _fresh(self, x, rows, fn):
        xt = x if isinstance(x, torch.Tensor) else dv.to_device_block(x)
        squeeze = xt.dim() == 1
        xb = dv.as_block(xt)
        y = dv.new_block(rows, xb.shape[1], device=xb.device, zero=False)
        fn(xb, y)
        return y[:, 0] if squeeze else y

    def apply(self, x):
        return self._fresh(x, self.m, self.apply_into)

    def apply_t(self, y):
        return self._fresh(y, self.n, self.apply_t_into)

    def transposed(self):
        return _TransposedSvdOperator(self)

    def reset_counter(self):
        self.n_matvecs = 0


class _TransposedSvdOperator:
    """Transposed view sharing the base counter (operators.py:139-160)."""

    def __init__(self, base):
        self.base = base
        self.m = base.n
        self.n = base.m
        self.explicit = None

    @property
    def n_matvecs(self):
        return self.base.n_matvecs

    def apply_into(self, x, y):
        return self.base.apply_t_into(x, y)

    def apply_t_into(self, x, y):
        return self.base.apply_into(x, y)

    def apply(self, x):
        return self.base.apply_t(x)

    def apply_t(self, y):
        return self.base.apply(y)

    def transposed(self):
        return self.base

    def reset_counter(self):
        self.base.reset_counter()


class _Scratch:
    """Grow-only scratch block cache keyed by (rows, name)."""

    def __init__(self):
        self._bufs = {}

    def get(self, name, rows, cols, device):
        buf = self._bufs.get(name)
        if buf is None or buf.shape[0] != rows or buf.shape[1] < cols or buf.device != device:
            buf = dv.new_block(rows, max(cols, 1), device=device, zero=False)
            self._bufs[name] = buf
        return buf[:, :cols]


def make_normal_operator(a):
    """x -> A^T (A x) of dimension n when m >= n, else x -> A (A^T x)
    (operators.py:163-172).  Two matvecs per column; the inner m x b (or
    n x b) product goes through a cached scratch block in HBM."""
    scratch = _Scratch()
    from .dist import DistSvdOperator
    if isinstance(a, DistSvdOperator):
        # row-sharded: all-gather, two local products, reduce-scatter
        op = LinearOperator(a.n_loc, into=lambda x, y: a.normal_into(x, y))
        op.svd_op = a
        op.kind = "normal"
        op.comm = a.comm
        op.dim_global = a.n
        op.local_slice = a.n_slice
        op.local_row0 = a.c0
        return op
    base = a.base if isinstance(a, _TransposedSvdOperator) else a
    dev = getattr(base, "_csr_dev", None)
    if dev is not None:
        # one C call: both products, block operands staged row-major inside
        side = 0 if (a.m >= a.n) == (base is a) else 1
        dim = a.n if a.m >= a.n else a.m
        inner = a.m if a.m >= a.n else a.n

        # the inner m x b (or n x b) product lives with the matrix, so its
        # address is stable across solves (graphs captured by the solver
        # bake it in)
        def raw_into(x, y):
            from . import _lib
            b = x.shape[1]
            t = dev.scratch(inner, b)
            _lib.call("svdsb_apply_normal", dev.ctx.handle, dev.handle, side, dv.P(x), dv.ld_of(x), dv.P(y),
                      dv.ld_of(y), b, dv.P(t), dv.ld_of(t), dev.ctx.stream)

        def into_native(x, y):
            from . import matrix
            base.n_matvecs += 2 * x.shape[1]
            prof = matrix.SPMV_PROFILER
            if prof is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            raw_into(x, y)
            if prof is not None:
                e1.record()
                prof.append(("normal", x.shape[1], e0, e1))

        op = LinearOperator(dim, into=into_native)
        op.svd_op = a
        op.kind = "normal"
        op.raw_into = raw_into
        # for the native iteration entry point (svdsb_gdk_iteration)
        op.native_normal = (dev, side, inner)
        # evaluated at capture / replay time: includes the scratch address
        op.graph_key = lambda: ("normal", dev.uid, side, dev.scratch(inner, 1).data_ptr())
        op.count_svd_matvecs = lambda cols: setattr(base, "n_matvecs", base.n_matvecs + 2 * cols)
        return op
    if a.m >= a.n:
        def into(x, y):
            t = scratch.get("t", a.m, x.shape[1], x.device)
            a.apply_into(x, t)
            a.apply_t_into(t, y)
        dim = a.n
    else:
        def into(x, y):
            t = scratch.get("t", a.n, x.shape[1], x.device)
            a.apply_t_into(x, t)
            a.apply_into(t, y)
        dim = a.m
    op = LinearOperator(dim, into=into)
    op.svd_op = a
    op.kind = "normal"
    return op


def make_augmented_operator(a):
    """Stacked operator on [v (n); u (m)]: [A^T u; A v]
    (operators.py:175-190, layout SPEC.md:174)."""
    from .dist import DistSvdOperator
    if isinstance(a, DistSvdOperator):
        # local stacked layout: [v rows of this rank (n_loc); u rows (m_loc)]
        nl, ml = a.n_loc, a.m_loc

        def into_d(x, y):
            a.apply_t_into(x[nl:, :], y[:nl, :])
            a.apply_into(x[:nl, :], y[nl:, :])

        op = LinearOperator(nl + ml, into=into_d)
        op.svd_op = a
        op.kind = "augmented"
        op.comm = a.comm
        op.dim_global = a.n + a.m
        op.local_slice = lambda full: np.concatenate([full[a.c0:a.c1], full[a.n + a.r0:a.n + a.r1]], axis=0)
        op.split_local = nl
        return op
    n, m = a.n, a.m

    def into(x, y):
        a.apply_t_into(x[n:, :], y[:n, :])
        a.apply_into(x[:n, :], y[n:, :])

    op = LinearOperator(n + m, into=into)
    op.svd_op = a
    op.kind = "augmented"
    op.split_local = n
    return op


class Preconditioner:
    """Approximate inverse applied to residuals before expansion
    (operators.py:193-222).  ``mode`` in AtA / AAt / augmented / none."""

    MODES = ("AtA", "AAt", "augmented", "none")

    def __init__(self, mode, apply_fn=None, device=False, into=None):
        if mode not in self.MODES:
            raise ValueError("unknown preconditioner mode %r" % (mode,))
        self.mode = mode
        self._apply = apply_fn
        self._into = into
        self._on_device = device
        self.n_applies = 0

    def apply_into(self, x, y):
        x = dv.as_block(x)
        self.n_applies += x.shape[1]
        if self.mode == "none" or (self._apply is None and self._into is None):
            if y.data_ptr() != x.data_ptr():
                y.copy_(x)
        elif self._into is not None:
            self._into(x, y)
        else:
            y.copy_(_user_call(self._apply, x, x.shape[0], self._on_device))
        return y

    def apply(self, x):
        xt = x if isinstance(x, torch.Tensor) else dv.to_device_block(x)
        squeeze = xt.dim() == 1
        xb = dv.as_block(xt)
        y = dv.new_block(xb.shape[0], xb.shape[1], device=xb.device, zero=False)
        self.apply_into(xb, y)
        return y[:, 0] if squeeze else y


def jacobi_precond_on_normal(a, side="cols"):
    """Point Jacobi for the normal operator (operators.py:225-249): the
    squared column (or row) norms, clamped below at EPS * max, computed on
    device bit-identically to the reference; applied as x ./ d."""
    csr = a.explicit if isinstance(a, SvdOperator) else a
    if csr is None:
        raise ValueError("point Jacobi needs explicit matrix storage")
    if csr.nnz == 0:
        raise ValueError("empty matrix has no usable diagonal")
    if side == "auto":
        side = "cols" if csr.m >= csr.n else "rows"
    if side == "cols":
        mode, dim, s = "AtA", csr.n, 0
    elif side == "rows":
        mode, dim, s = "AAt", csr.m, 1
    else:
        raise ValueError("side must be 'cols', 'rows' or 'auto'")
    dev = csr.device_csr()
    d = torch.empty(dim, dtype=DTYPE, device=dev.ctx.device)
    dev.precond_diag(s, d)

    def into(x, y):
        from . import _lib
        _lib.call("svdsb_diag_solve", x.shape[0], dv.P(d), dv.P(x), dv.ld_of(x), dv.P(y), dv.ld_of(y),
                  x.shape[1], dv.context(x.device).stream)

    pre = Preconditioner(mode, into=into)
    pre.diagonal = d
    pre.graph_key = ("jacobi", d.data_ptr())
    return pre


class NormEstimate:
    """Running estimate of ||A||^2 from observed Ritz values
    (operators.py:252-292).  Host scalars only."""

    def __init__(self, user_supplied=None):
        if user_supplied is not None and user_supplied <= 0.0:
            raise ValueError("a user-supplied norm must be positive")
        self.user_supplied = user_supplied
        self._c_running = 0.0

    @property
    def c_norm(self):
        if self.user_supplied is not None:
            return self.user_supplied ** 2
        return self._c_running

    @property
    def a_norm(self):
        if self.user_supplied is not None:
            return self.user_supplied
        return float(np.sqrt(self._c_running))

    def update(self, ritz_values):
        values = np.atleast_1d(np.asarray(ritz_values, dtype=np.float64))
        if values.size:
            peak = float(np.abs(values).max())
            if peak > self._c_running:
                self._c_running = peak
        return self

    def update_from_augmented(self, ritz_values):
        values = np.atleast_1d(np.asarray(ritz_values, dtype=np.float64))
        if values.size:
            self.update(float(np.abs(values).max()) ** 2)
        return self


def update_norm_estimate(est, ritz_values):
    return est.update(ritz_values)


def select_preconditioner(precond, wanted_mode):
    """``precond`` if it matches the stage, else None with a warning
    (operators.py:300-309)."""
    if precond is None or precond.mode == "none":
        return None
    if precond.mode != wanted_mode:
        warnings.warn("preconditioner mode %r does not match stage mode %r; ignoring it"
                      % (precond.mode, wanted_mode), stacklevel=2)
        return None
    return precond

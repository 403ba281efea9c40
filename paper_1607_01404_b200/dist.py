"""Row-sharded multi-GPU execution (the paper's SPMD model,
PAPER.md:584-599, 645-657).

* A (oriented tall, m >= n) is split into G contiguous row blocks balanced
  by nnz: start_p = lower_bound(row_ptr, ceil(p * nnz / G)), computed on the
  host in int64 (bit-exact, ``partition_rows``).  Rank p stores CSR(A_p) and
  its transpose (A^T column-partitioned, spanning all n rows).
* n-space vectors (stage 1) are split evenly (``even_split``); stage-2
  stacked vectors [v; u] hold the rank's v chunk followed by its u rows.
* A C-apply is: all-gather x (n x b) -> local A_p x -> local A_p^T y_p ->
  reduce-scatter of the partial n x b result (``DistSvdOperator``).  When
  every rank's rows only touch columns of its own chunk and its two
  neighbours' (grid stencils: configs 3 and 5, square, column chunks = row
  blocks) the all-gather becomes a halo exchange (x rows [lo, c0) from
  rank-1, [c1, hi) from rank+1, P2P sends) and the reduce-scatter a
  reverse halo (the partial sums of the neighbours' rows travel back and
  are added): O(halo) bytes per C-apply instead of O(n).
* ``DistSvdOperator.from_coo``: each rank selects and assembles only its
  own row block's triplets on its device (``partition_coo``).
* Every Gram / norm partial is finished by ``Comm.allreduce_`` -- PRIMME's
  globalSumDouble -- over NCCL on the kernels' stream.
  Small state is replicated and all-reduce returns identical bits on every
  rank, so host decisions stay in lock-step.
"""

import numpy as np
import torch
import torch.distributed as tdist


def partition_rows(row_ptr, parts):
    """nnz-balanced contiguous row blocks: bounds[p] = first row whose
    row_ptr >= ceil(p * nnz / parts).  Host int64, bit-exact."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    nnz = int(row_ptr[-1])
    m = row_ptr.shape[0] - 1
    bounds = np.empty(parts + 1, dtype=np.int64)
    for p in range(parts + 1):
        target = -(-p * nnz // parts)  # ceil in exact integer arithmetic
        bounds[p] = np.searchsorted(row_ptr, target, side="left")
    bounds[0] = 0
    bounds[parts] = m
    return np.minimum(bounds, m)


def partition_coo(comm, m, n, rows):
    """Row blocks balanced by the triplet counts of the rows (for a
    duplicate-free COO -- every BASELINE generator but config 4 -- these are
    the CSR row pointers, so the bounds equal ``partition_rows``'; with
    duplicates the balance is by triplets; host int64, deterministic).
    Square matrices split their columns like their rows (so a grid
    stencil's coupling stays between neighbouring ranks), tall ones evenly.
    Returns (this rank's triplet selection, row bounds, column bounds)."""
    rows = np.asarray(rows)
    counts = np.bincount(rows, minlength=m).astype(np.int64) if rows.size else np.zeros(m, np.int64)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    rb = partition_rows(rp, comm.world)
    cb = rb.copy() if m == n else even_split(n, comm.world)
    r0, r1 = int(rb[comm.rank]), int(rb[comm.rank + 1])
    if rows.size and bool(np.all(rows[1:] >= rows[:-1])):
        sel = slice(int(np.searchsorted(rows, r0, "left")), int(np.searchsorted(rows, r1, "left")))
    else:
        sel = np.flatnonzero((rows >= r0) & (rows < r1))
    return sel, rb, cb


def even_split(n, parts):
    """Contiguous chunks of sizes differing by at most one."""
    base, extra = divmod(int(n), parts)
    sizes = [base + (1 if p < extra else 0) for p in range(parts)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


class Comm:
    """globalSumDouble and the two collectives of a sharded C-apply."""

    def __init__(self, group=None, world=None, rank=None):
        self.group = group
        if world is None:
            world = tdist.get_world_size(group) if tdist.is_available() and tdist.is_initialized() else 1
        if rank is None:
            rank = tdist.get_rank(group) if tdist.is_available() and tdist.is_initialized() else 0
        self.world, self.rank = int(world), int(rank)

    @property
    def distributed(self):
        return self.world > 1

    def allreduce_(self, t):
        """In-place sum over ranks (no-op on one rank)."""
        if self.world > 1 and t.numel():
            if t.is_contiguous():
                tdist.all_reduce(t, op=tdist.ReduceOp.SUM, group=self.group)
            elif t.dim() == 2 and t.t().is_contiguous():  # column-major small matrix
                tdist.all_reduce(t.t(), op=tdist.ReduceOp.SUM, group=self.group)
            else:
                tmp = t.contiguous()
                tdist.all_reduce(tmp, op=tdist.ReduceOp.SUM, group=self.group)
                t.copy_(tmp)
        return t

    def allgather_rows(self, local, bounds, out):
        """Column-major (local_rows, b) blocks -> full (rows, b) block."""
        if self.world == 1:
            out.copy_(local)
            return out
        b = local.shape[1]
        sizes = [int(bounds[p + 1] - bounds[p]) for p in range(self.world)]
        cols_ok = all(t[:, j].is_contiguous() for t in (local, out) for j in range(b))
        if cols_ok and b <= 4:
            # column-major blocks: every column of the result is one contiguous
            # vector, so each rank's slice of it is gathered in place (no
            # slab transposes or staging copies; b collectives of rows*8 bytes)
            for j in range(b):
                col = out[:, j]
                views = [col[int(bounds[p]):int(bounds[p + 1])] for p in range(self.world)]
                tdist.all_gather(views, local[:, j], group=self.group)
            return out
        # gather contiguous (b, rows_p) row-major slabs, then place them
        mine = local.t().contiguous()
        slabs = [torch.empty((b, s), dtype=local.dtype, device=local.device) for s in sizes]
        tdist.all_gather(slabs, mine, group=self.group)
        for p, slab in enumerate(slabs):
            out[int(bounds[p]):int(bounds[p + 1]), :].copy_(slab.t())
        return out

    def reduce_scatter_rows(self, full, bounds, out):
        """Sum the full (rows, b) partials over ranks and keep this rank's
        rows in ``out``."""
        if self.world == 1:
            out.copy_(full)
            return out
        b = full.shape[1]
        cols_ok = all(t[:, j].is_contiguous() for t in (full, out) for j in range(b))
        if cols_ok and b <= 4:
            # as allgather_rows: slices of contiguous columns reduced straight
            # into this rank's column (no transposes or staging copies)
            for j in range(b):
                col = full[:, j]
                views = [col[int(bounds[p]):int(bounds[p + 1])] for p in range(self.world)]
                tdist.reduce_scatter(out[:, j], views, op=tdist.ReduceOp.SUM, group=self.group)
            return out
        slabs = [full[int(bounds[p]):int(bounds[p + 1]), :].t().contiguous() for p in range(self.world)]
        mine = torch.empty_like(slabs[self.rank])
        tdist.reduce_scatter(mine, slabs, op=tdist.ReduceOp.SUM, group=self.group)
        out.copy_(mine.t())
        return out

    def _exchange(self, ops):
        if ops:
            for req in tdist.batch_isend_irecv(ops):
                req.wait()

    def halo_gather(self, x_loc, col_bounds, ext, ext_all, out):
        """out (rows [lo, hi) of the global vector) = own chunk + the halo
        rows from the two neighbours.  ext = (lo, hi) of this rank,
        ext_all[p] = (lo_p, hi_p) of every rank."""
        r, world = self.rank, self.world
        lo, hi = ext
        c0, c1 = int(col_bounds[r]), int(col_bounds[r + 1])
        out[c0 - lo:c1 - lo].copy_(x_loc)
        b = x_loc.shape[1]
        ops, recvs = [], []
        if r > 0 and lo < c0:
            t = torch.empty((b, c0 - lo), dtype=x_loc.dtype, device=x_loc.device)
            ops.append(tdist.P2POp(tdist.irecv, t, r - 1, self.group))
            recvs.append((t, 0, c0 - lo))
        if r + 1 < world and hi > c1:
            t = torch.empty((b, hi - c1), dtype=x_loc.dtype, device=x_loc.device)
            ops.append(tdist.P2POp(tdist.irecv, t, r + 1, self.group))
            recvs.append((t, c1 - lo, hi - lo))
        # what the neighbours need from this chunk
        if r > 0 and int(ext_all[r - 1][1]) > c0:
            k1 = int(ext_all[r - 1][1])
            ops.append(tdist.P2POp(tdist.isend, x_loc[0:k1 - c0].t().contiguous(), r - 1, self.group))
        if r + 1 < world and int(ext_all[r + 1][0]) < c1:
            k0 = int(ext_all[r + 1][0])
            ops.append(tdist.P2POp(tdist.isend, x_loc[k0 - c0:c1 - c0].t().contiguous(), r + 1, self.group))
        self._exchange(ops)
        for t, a, bnd in recvs:
            out[a:bnd].copy_(t.t())
        return out

    def halo_reduce(self, z_ext, col_bounds, ext, ext_all, out):
        """out (this rank's chunk) = own partial sums + the neighbours'
        partial sums of this chunk's rows (the reverse of halo_gather)."""
        r, world = self.rank, self.world
        lo, hi = ext
        c0, c1 = int(col_bounds[r]), int(col_bounds[r + 1])
        out.copy_(z_ext[c0 - lo:c1 - lo])
        b = z_ext.shape[1]
        ops, recvs = [], []
        if r > 0 and lo < c0:
            ops.append(tdist.P2POp(tdist.isend, z_ext[0:c0 - lo].t().contiguous(), r - 1, self.group))
        if r + 1 < world and hi > c1:
            ops.append(tdist.P2POp(tdist.isend, z_ext[c1 - lo:hi - lo].t().contiguous(), r + 1, self.group))
        if r > 0 and int(ext_all[r - 1][1]) > c0:
            k1 = int(ext_all[r - 1][1])
            t = torch.empty((b, k1 - c0), dtype=z_ext.dtype, device=z_ext.device)
            ops.append(tdist.P2POp(tdist.irecv, t, r - 1, self.group))
            recvs.append((t, 0, k1 - c0))
        if r + 1 < world and int(ext_all[r + 1][0]) < c1:
            k0 = int(ext_all[r + 1][0])
            t = torch.empty((b, c1 - k0), dtype=z_ext.dtype, device=z_ext.device)
            ops.append(tdist.P2POp(tdist.irecv, t, r + 1, self.group))
            recvs.append((t, k0 - c0, c1 - c0))
        self._exchange(ops)
        for t, a, bnd in recvs:
            out[a:bnd] += t.t()
        return out

    def allgather_host(self, arr):
        """Concatenate host numpy arrays (rows) from all ranks in rank order."""
        if self.world == 1:
            return arr
        objs = [None] * self.world
        tdist.all_gather_object(objs, arr, group=self.group)
        return np.concatenate(objs, axis=0)


LOCAL = Comm(world=1, rank=0)


class DistSvdOperator:
    """Row-sharded A (m >= n) with forward / transpose products on local
    blocks.  ``local_fwd(x_full, y_loc)`` computes A_p x_full;
    ``local_adj(y_loc, z_full)`` computes the partial A_p^T y_loc over all n
    rows.  The factory ``from_host_csr`` binds them to device CSR kernels.

    Vector layout: n-space blocks hold rows [col_bounds[r], col_bounds[r+1])
    of the global vector, m-space blocks rows [row_bounds[r], row_bounds[r+1]).
    """

    def __init__(self, comm, m, n, row_bounds, col_bounds, local_fwd, local_adj, alloc=None, halo=None):
        if m < n:
            raise ValueError("DistSvdOperator expects an oriented (tall) matrix")
        self.comm = comm
        self.m, self.n = int(m), int(n)
        self.row_bounds = np.asarray(row_bounds, dtype=np.int64)
        self.col_bounds = np.asarray(col_bounds, dtype=np.int64)
        r = comm.rank
        self.r0, self.r1 = int(self.row_bounds[r]), int(self.row_bounds[r + 1])
        self.c0, self.c1 = int(self.col_bounds[r]), int(self.col_bounds[r + 1])
        self.m_loc, self.n_loc = self.r1 - self.r0, self.c1 - self.c0
        self._fwd, self._adj = local_fwd, local_adj
        self._alloc = alloc
        # halo = (ext, ext_all): the global column range [lo, hi) this rank's
        # rows touch, and every rank's; local products then work on rows
        # [lo, hi) of x / z instead of all n
        self.halo = halo
        self._bufs = {}
        self.n_matvecs = 0
        self.explicit = None

    def _buf(self, name, rows, b, like):
        key = (name, rows, b)
        t = self._bufs.get(key)
        if t is None:
            if self._alloc is not None:
                t = self._alloc(rows, b)
            else:
                t = torch.zeros((b, rows), dtype=like.dtype, device=like.device).t()
            self._bufs[key] = t
        return t

    # -- local pieces of global vectors
    def n_slice(self, full):
        return full[self.c0:self.c1]

    def m_slice(self, full):
        return full[self.r0:self.r1]

    # -- products (one matvec counted per column, on every rank alike)
    def apply_into(self, x_loc, y_loc):
        """y_loc = (A x)[r0:r1] from the local n-chunk of x."""
        b = x_loc.shape[1]
        self.n_matvecs += b
        if self.halo is not None:
            (lo, hi), ext_all = self.halo
            x_ext = self._buf("xext", hi - lo, b, x_loc)
            self.comm.halo_gather(x_loc, self.col_bounds, (lo, hi), ext_all, x_ext)
            self._fwd(x_ext, y_loc)
            return y_loc
        x_full = self._buf("xfull", self.n, b, x_loc)
        self.comm.allgather_rows(x_loc, self.col_bounds, x_full)
        self._fwd(x_full, y_loc)
        return y_loc

    def apply_t_into(self, y_loc, z_loc):
        """z_loc = (A^T y)[c0:c1] from the local m-rows of y."""
        b = y_loc.shape[1]
        self.n_matvecs += b
        if self.halo is not None:
            (lo, hi), ext_all = self.halo
            z_ext = self._buf("zext", hi - lo, b, y_loc)
            self._adj(y_loc, z_ext)
            self.comm.halo_reduce(z_ext, self.col_bounds, (lo, hi), ext_all, z_loc)
            return z_loc
        z_full = self._buf("zfull", self.n, b, y_loc)
        self._adj(y_loc, z_full)
        self.comm.reduce_scatter_rows(z_full, self.col_bounds, z_loc)
        return z_loc

    def normal_into(self, x_loc, z_loc):
        """C x = A^T (A x) on the n-chunk: all-gather, two local products,
        reduce-scatter."""
        b = x_loc.shape[1]
        y_loc = self._buf("yloc", self.m_loc, b, x_loc)
        self.apply_into(x_loc, y_loc)
        self.apply_t_into(y_loc, z_loc)
        return z_loc

    @classmethod
    def from_host_csr(cls, comm, m, n, row_ptr, col_idx, values, device=None):
        """Shard a host CSR (reference layout) over the ranks of ``comm``;
        each rank uploads only its row block."""
        from . import device as dv
        from .matrix import DeviceCsr
        row_ptr = np.asarray(row_ptr, dtype=np.int64)
        rb = partition_rows(row_ptr, comm.world)
        cb = even_split(n, comm.world)
        r0, r1 = int(rb[comm.rank]), int(rb[comm.rank + 1])
        lo, hi = int(row_ptr[r0]), int(row_ptr[r1])
        local = DeviceCsr.from_host(r1 - r0, n, row_ptr[r0:r1 + 1] - lo, np.asarray(col_idx)[lo:hi],
                                    np.asarray(values)[lo:hi], device=device)

        def fwd(x_full, y_loc):
            local.matvec(x_full, y_loc, transpose=False)

        def adj(y_loc, z_full):
            local.matvec(y_loc, z_full, transpose=True)

        op = cls(comm, m, n, rb, cb, fwd, adj, alloc=lambda rows, b: dv.new_block(rows, b, device=device))
        op.local_csr = local
        return op


def column_extent(comm, col_bounds, cols):
    """(lo, hi) of the global columns this rank's triplets touch (its own
    chunk always included), every rank's extents, and whether a halo
    exchange covers them (each extent within the neighbours' chunks)."""
    r = comm.rank
    c0, c1 = int(col_bounds[r]), int(col_bounds[r + 1])
    if len(cols):
        cmin = int(cols.min()) if not isinstance(cols, torch.Tensor) else int(cols.min().item())
        cmax = int(cols.max()) if not isinstance(cols, torch.Tensor) else int(cols.max().item())
        lo, hi = min(c0, cmin), max(c1, cmax + 1)
    else:
        lo, hi = c0, c1
    ext = np.array([[lo, hi]], dtype=np.int64)
    ext_all = comm.allgather_host(ext) if comm.distributed else ext
    ok = True
    for p in range(comm.world):
        plo, phi = int(ext_all[p][0]), int(ext_all[p][1])
        lo_lim = int(col_bounds[max(p - 1, 0)])
        hi_lim = int(col_bounds[min(p + 2, comm.world)])
        ok &= lo_lim <= plo and phi <= hi_lim
    return (lo, hi), [tuple(int(v) for v in e) for e in ext_all], ok


def _from_coo(cls, comm, m, n, rows, cols, vals, device=None, bounds=None):
    from .matrix import SparseMatrixCsr
    from . import device as dv
    if bounds is None:
        sel, rb, cb = partition_coo(comm, m, n, np.asarray(rows))
        rows, cols, vals = rows[sel], cols[sel], vals[sel]
    else:
        rb, cb = bounds
    r0, r1 = int(rb[comm.rank]), int(rb[comm.rank + 1])
    (lo, hi), ext_all, use_halo = column_extent(comm, cb, cols)
    shift = lo if use_halo else 0
    ncols = (hi - lo) if use_halo else n
    local = SparseMatrixCsr.from_coo(r1 - r0, ncols, rows - r0, cols - shift if shift else cols, vals,
                                     device=device).device_csr(device)

    def fwd(x, y_loc):
        local.matvec(x, y_loc, transpose=False)

    def adj(y_loc, z):
        local.matvec(y_loc, z, transpose=True)

    op = cls(comm, m, n, rb, cb, fwd, adj, alloc=lambda nr, b: dv.new_block(nr, b, device=device),
             halo=((lo, hi), ext_all) if use_halo else None)
    op.local_csr = local
    op.local_nnz = local.nnz
    tot = torch.tensor([local.nnz], dtype=torch.int64)
    if comm.distributed and tdist.get_backend(comm.group) == "nccl":
        tot = tot.to(local.ctx.device)
    op.nnz_global = int(comm.allreduce_(tot).item())
    return op


DistSvdOperator.from_coo = classmethod(_from_coo)


def dist_jacobi_diag(op, part):
    """This rank's chunk of the Jacobi diagonal from its rows' partial
    squared column norms ``part`` (length hi - lo with a halo, n otherwise):
    summed over the ranks sharing a column, clamped below at EPS times the
    global maximum (operators.py:225-249)."""
    part = part.reshape(-1, 1)
    d = torch.zeros((1, op.n_loc), dtype=part.dtype, device=part.device).t()
    if op.halo is not None:
        (lo, hi), ext_all = op.halo
        op.comm.halo_reduce(part, op.col_bounds, (lo, hi), ext_all, d)
    else:
        op.comm.reduce_scatter_rows(part, op.col_bounds, d)
    mx = d.max().reshape(1) if d.numel() else torch.zeros(1, dtype=d.dtype, device=d.device)
    if op.comm.distributed:
        tdist.all_reduce(mx, op=tdist.ReduceOp.MAX, group=op.comm.group)
    eps = float(np.finfo(np.float64).eps)
    return torch.maximum(d[:, 0], mx * eps).contiguous()


def dist_jacobi(op):
    """Point-Jacobi preconditioner of the sharded normal operator: squared
    column norms of this rank's rows on device (svdsb_row_sq), reduced over
    ranks by ``dist_jacobi_diag`` -- no rank holds the whole matrix.  The
    cross-rank additions round differently from the single-GPU bincount
    order (not bit-exact with it)."""
    from . import _lib
    from . import device as dv
    from .operators import Preconditioner
    local = op.local_csr
    part = dv.new_block(local.n, 1, device=local.ctx.device)
    local.col_sq_norms(part[:, 0])
    d = dist_jacobi_diag(op, part[:, 0])

    def into(x, y):
        _lib.call("svdsb_diag_solve", x.shape[0], dv.P(d), dv.P(x), dv.ld_of(x), dv.P(y), dv.ld_of(y), x.shape[1],
                  dv.context(x.device).stream)

    pre = Preconditioner("AtA", into=into)
    pre.diagonal = d
    return pre


def local_jacobi(op, csr):
    """Point-Jacobi preconditioner of the sharded normal operator: the
    global squared-column-norm diagonal (operators.py:225-249, computed on
    device from the full CSR), restricted to this rank's n-chunk."""
    from . import _lib
    from . import device as dv
    from .operators import Preconditioner, jacobi_precond_on_normal
    full = jacobi_precond_on_normal(csr, side="cols")
    d = full.diagonal[op.c0:op.c1].contiguous()

    def into(x, y):
        _lib.call("svdsb_diag_solve", x.shape[0], dv.P(d), dv.P(x), dv.ld_of(x), dv.P(y), dv.ld_of(y), x.shape[1],
                  dv.context(x.device).stream)

    pre = Preconditioner("AtA", into=into)
    pre.diagonal = d
    return pre

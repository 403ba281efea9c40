"""Row-sharded multi-GPU execution (the paper's SPMD model,
PAPER.md:584-599, 645-657).

* A (oriented tall, m >= n) is split into G contiguous row blocks balanced
  by nnz: start_p = lower_bound(row_ptr, ceil(p * nnz / G)), computed on the
  host in int64 (bit-exact, ``partition_rows``).  Rank p stores CSR(A_p) and
  its transpose (A^T column-partitioned, spanning all n rows).
* n-space vectors (stage 1) are split evenly (``even_split``); stage-2
  stacked vectors [v; u] hold the rank's v chunk followed by its u rows.
* A C-apply is: all-gather x (n x b) -> local A_p x -> local A_p^T y_p ->
  reduce-scatter of the partial n x b result (``DistSvdOperator``).
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
        slabs = [full[int(bounds[p]):int(bounds[p + 1]), :].t().contiguous() for p in range(self.world)]
        mine = torch.empty_like(slabs[self.rank])
        tdist.reduce_scatter(mine, slabs, op=tdist.ReduceOp.SUM, group=self.group)
        out.copy_(mine.t())
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

    def __init__(self, comm, m, n, row_bounds, col_bounds, local_fwd, local_adj, alloc=None):
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
        x_full = self._buf("xfull", self.n, b, x_loc)
        self.comm.allgather_rows(x_loc, self.col_bounds, x_full)
        self._fwd(x_full, y_loc)
        return y_loc

    def apply_t_into(self, y_loc, z_loc):
        """z_loc = (A^T y)[c0:c1] from the local m-rows of y."""
        b = y_loc.shape[1]
        self.n_matvecs += b
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

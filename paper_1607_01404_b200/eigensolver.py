"""GD+k Davidson eigensolver with every N-sized operation on the GPU.

Host-side control flow mirrors pkg/src/itersvd/eigensolver.py (cited per
method); the state it drives -- the basis V, its image W = Op V, the
projection H, the refined QR factors, the locked vectors -- lives in
device memory and is touched only by libsvdsb kernels.  Per outer
iteration the host reads one small status record (Ritz values, candidate
residual norms, stage-2 split residuals; < 2 KB) in a single
synchronisation, plus one norm per Gram-Schmidt pass of the expansion
vector: exactly the scalars the reference's branches depend on.

Small g x g work (Rayleigh-Ritz eigenproblem, refined SVD, restart
coefficient selection, H <- C^T H C, QR of R Y) runs in single-CTA device
kernels; random draws come from the same numpy Generator streams as the
reference so trajectories track it.
"""

import ctypes
import gc
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv
from .device import DTYPE
from .operators import NormEstimate

EPS = 2.220446049250313e-16
TARGET_LARGEST = "largest_algebraic"
TARGET_SMALLEST = "smallest_algebraic"
TARGET_CLOSEST_GEQ = "closest_geq"
EXTRACT_RR = "rayleigh_ritz"
EXTRACT_REFINED = "refined_const_shift"
PRACTICAL_FLOOR_FACTOR = 10.0          # eigensolver.py:43
METHOD_GDK = "GD+k"                    # the reference's method in both stages
METHOD_JDQMR = "JDQMR"                 # PRIMME's JDQMR; jdqmr.py
JD_LOG = None                          # diagnostics: a list collects every inner solve
_IMPROVE_FACTOR = 0.999                # eigensolver.py:47
REORTH_FACTOR = 1.0 / np.sqrt(2.0)     # kernels.py:24
DEFICIENT_TOL = 1e-14                  # kernels.py:28
_MAX_REORTH_PASSES = 6                 # kernels.py:30
_MAX_RANDOM_RETRIES = 20               # kernels.py:31


class BasisCollapseError(RuntimeError):
    """Every expansion direction was dependent several times in a row."""


@dataclass
class EigConfig:
    """Solver knobs (eigensolver.py:54-107); same fields and validation."""

    num_evals: int = 1
    target: str = TARGET_LARGEST
    shifts: tuple = ()
    max_basis_size: int = 15
    min_restart_size: int = 6
    plus_k: int = 1
    max_block_size: int = 1
    locking: bool = False
    extraction: str = EXTRACT_RR
    convergence_test: object = None
    practical_test: object = None
    max_matvecs: int = None
    deactivate_krylov_init: bool = False
    seed: int = 0
    disable_reset: bool = False
    stagnation_window: int = 250
    iteration_hook: object = None
    # expansion method: GD+k (preconditioned residual, the reference's) or
    # JDQMR (QMRs on the correction equation, device inner solver)
    method: str = METHOD_GDK
    max_inner_iterations: int = 200
    inner_etol_frac: float = 0.0
    inner_lfac: float = 0.1

    def validate(self, dim):
        if self.num_evals < 0:
            raise ValueError("num_evals must be nonnegative")
        if self.method not in (METHOD_GDK, METHOD_JDQMR):
            raise ValueError("method must be %r or %r" % (METHOD_GDK, METHOD_JDQMR))
        if self.max_inner_iterations < 0 or not (0.0 <= self.inner_etol_frac < 1.0) or self.inner_lfac < 0.0:
            raise ValueError("bad JDQMR inner-solver settings")
        if self.target not in (TARGET_LARGEST, TARGET_SMALLEST, TARGET_CLOSEST_GEQ):
            raise ValueError("unknown target %r" % (self.target,))
        if self.extraction not in (EXTRACT_RR, EXTRACT_REFINED):
            raise ValueError("unknown extraction %r" % (self.extraction,))
        if self.target == TARGET_CLOSEST_GEQ:
            if not len(self.shifts):
                raise ValueError("closest_geq needs at least one shift")
            if not self.locking:
                raise ValueError("interior targets require locking")
        elif self.extraction == EXTRACT_REFINED:
            raise ValueError("refined extraction is tied to interior targets")
        if dim <= self.max_basis_size:
            return
        if not (0 < self.min_restart_size < self.max_basis_size):
            raise ValueError("need 0 < min_restart_size < max_basis_size")
        if self.plus_k < 0 or self.max_block_size < 1:
            raise ValueError("bad plus_k or max_block_size")
        if self.min_restart_size + self.plus_k >= self.max_basis_size:
            raise ValueError("min_restart_size + plus_k must stay below max_basis_size")
        if self.num_evals > self.max_basis_size - 2:
            raise ValueError("num_evals too large for the basis size")
        if self.max_basis_size > _lib.SMALL_MAX:
            raise ValueError("max_basis_size above %d is not supported on device" % _lib.SMALL_MAX)


@dataclass
class EigStats:
    matvecs: int = 0
    precond_applies: int = 0
    restarts: int = 0
    resets: int = 0
    outer_iterations: int = 0
    syncs: int = 0
    graphs_captured: int = 0
    inner_iterations: int = 0
    inner_solves: int = 0
    device_rng: bool = False   # initial block from svdsb_randn (not the reference's numpy stream)


@dataclass
class EigResult:
    """eigenvalues/residual_norms/converged on host; eigenvectors a
    column-major device block (dim x t)."""

    eigenvalues: np.ndarray
    eigenvectors: object
    residual_norms: np.ndarray
    converged: np.ndarray
    stats: EigStats
    status: str = "ok"

    @property
    def num_converged(self):
        return int(self.converged.sum())


def select_interior_candidate(lams, shift):
    """eigensolver.py:133-145."""
    lams = np.asarray(lams, dtype=np.float64)
    if lams.size == 0:
        raise ValueError("no pairs to select from")
    above = np.flatnonzero(lams >= shift)
    if above.size:
        return int(above[np.argmin(lams[above])])
    return int(np.argmax(lams))


class Candidate:
    """Per-candidate view handed to convergence tests: host scalars plus
    lazily materialised device vectors."""

    __slots__ = ("lam", "rnorm", "x", "opx", "nv", "nu", "r7")

    def __init__(self, lam, rnorm, x=None, opx=None, nv=None, nu=None, r7=None):
        self.lam, self.rnorm, self.x, self.opx = lam, rnorm, x, opx
        self.nv, self.nu, self.r7 = nv, nu, r7


def _run_test(test, cand, op_norm):
    fast = getattr(test, "evaluate", None)
    if fast is not None:
        return bool(fast(cand, op_norm))
    return bool(test(cand.lam, cand.rnorm, cand.x, cand.opx, op_norm))


def _test_needs(test):
    """(needs x/opx vectors, needs split statistics) for a test."""
    if test is None:
        return False, False
    if getattr(test, "evaluate", None) is not None:
        return False, bool(getattr(test, "split_n", None) is not None)
    return True, False


class Orthonormalizer:
    """Iterated classical Gram-Schmidt with the DGKS 1/sqrt(2) test and
    random replacement of collapsed columns (kernels.py:54-133), one column
    at a time on device; the host sees two norms per pass.

    Distributed: block rows are this rank's slice of the global vectors;
    every partial inner product is finished by ``comm.allreduce_`` (the
    globalSum of PAPER.md:727), and replacement draws are global-length
    draws sliced by ``local_slice`` so all ranks agree."""

    def __init__(self, ctx, comm=None, global_rows=None, local_slice=None):
        from .dist import LOCAL
        self.ctx = ctx
        self.comm = comm if comm is not None else LOCAL
        self.global_rows = global_rows
        self.local_slice = local_slice
        self.c = torch.zeros(4 * _lib.SMALL_MAX * 4, dtype=DTYPE, device=ctx.device)
        self.nrm = torch.zeros(2, dtype=DTYPE, device=ctx.device)
        self.syncs = 0

    def draw(self, rng, rows):
        """A standard-normal column of the GLOBAL length, this rank's rows."""
        if self.local_slice is None or self.global_rows is None:
            return rng.standard_normal(rows)
        return self.local_slice(rng.standard_normal(self.global_rows))

    def _pass(self, prior, v):
        ctx = self.ctx
        if prior:
            total = sum(b.shape[1] for b in prior)
            c = self.c[:total]
            dv.gram(ctx, v.shape[0], prior, v, c.unsqueeze(1), norms2=self.nrm[0:1])
            if self.comm.distributed:
                self.comm.allreduce_(self.c[:total])
            dv.project_out(ctx, v.shape[0], prior, c.unsqueeze(1), v, norms2=self.nrm[1:2])
        else:
            dv.col_norms2(ctx, v, self.nrm[0:1])
            dv.col_norms2(ctx, v, self.nrm[1:2])
        if self.comm.distributed:
            # nrm[0] reduced before the projection was already summed only
            # locally; one reduction finishes both entries
            self.comm.allreduce_(self.nrm)
        before2, after2 = dv.fetch(ctx, [self.nrm])[0]
        self.syncs += 1
        return float(np.sqrt(before2)), float(np.sqrt(after2))

    def column(self, v, prior):
        """DGKS loop on one column; returns the final norm (0 on collapse)
        and leaves v normalised when it is > 0."""
        final = 0.0
        prev = orig = None
        collapses = 0
        for p in range(_MAX_REORTH_PASSES):
            before, cur = self._pass(prior, v)
            if p == 0:
                orig = prev = before
                if orig == 0.0:
                    break
            if cur < DEFICIENT_TOL * orig:
                collapses += 1
                if collapses >= 2:
                    break
            elif cur > REORTH_FACTOR * prev:
                final = cur
                break
            else:
                collapses = 0
            prev = cur
        if final > 0.0:
            dv.scale_cols(self.ctx, v, self.nrm[1:2], dv.SCALE_DIV_SQRT)
        return final

    def resume(self, v, prior, st):
        """Continue a DGKS loop started on device (state st, see
        svdsb_cgs_pass) with host-checked passes; returns the final norm."""
        p, collapses, orig, prev = int(st[1]), int(st[2]), float(st[3]), float(st[4])
        final = 0.0
        while p < _MAX_REORTH_PASSES:
            _, cur = self._pass(prior, v)
            p += 1
            if cur < DEFICIENT_TOL * orig:
                collapses += 1
                if collapses >= 2:
                    break
            elif cur > REORTH_FACTOR * prev:
                final = cur
                break
            else:
                collapses = 0
            prev = cur
        if final > 0.0:
            dv.scale_cols(self.ctx, v, self.nrm[1:2], dv.SCALE_DIV_SQRT)
        return final

    def __call__(self, block, against=None, start_col=0, rng=None):
        rows, cols = block.shape
        ext = [b for b in (against or []) if b is not None and b.shape[1] > 0]
        n_ext = sum(b.shape[1] for b in ext)
        for b in ext:
            if b.shape[0] != rows:
                raise ValueError("dimension mismatch between block and against")
        grows = self.global_rows if self.global_rows is not None else rows
        if n_ext + cols > grows:
            raise ValueError("more columns than the space can hold")
        if rng is None:
            rng = np.random.default_rng(0)
        replaced = []
        for j in range(start_col, cols):
            prior = ext + ([block[:, :j]] if j > 0 else [])
            v = block[:, j:j + 1]
            flagged = False
            for _ in range(_MAX_RANDOM_RETRIES):
                if self.column(v, prior) > 0.0:
                    break
                if not flagged:
                    replaced.append(j)
                    flagged = True
                v.copy_(torch.from_numpy(np.ascontiguousarray(self.draw(rng, rows))).unsqueeze(1))
            else:
                raise np.linalg.LinAlgError("orthonormalize could not produce an independent column")
        return replaced


class _NativeGraph:
    """An instantiated CUDA graph (svdsb_graph_end), replayed with
    svdsb_graph_launch on the solver's stream."""

    __slots__ = ("exec",)

    def __init__(self, ex):
        self.exec = ex

    def replay(self, stream):
        rc = _lib.load().svdsb_graph_launch(self.exec, stream)
        if rc:
            _lib.check(rc, "svdsb_graph_launch")

    def __del__(self):
        try:
            if self.exec and _lib._lib is not None:
                _lib._lib.svdsb_graph_destroy(self.exec)
        except Exception:
            pass


class _Workspace:
    """Device buffers of one solver shape, pooled per device so repeated
    solves of the same shape reuse memory -- and with it the CUDA graphs
    captured for their iterations (graphs bake device pointers).

    The per-iteration outputs (Ritz values and coefficients, candidate
    residuals, status scalars, DGKS state, the pinned status copy) come in
    two slots: a graphed iteration reads slot s and writes slot 1 - s, so
    the next iteration can be queued before the host has decided on the
    current one (see DavidsonSolver._expand_graphed)."""

    def __init__(self, key, n, gm, pmax, bs, plus_k):
        dev = dv.context().device
        self.key = key
        self.v = dv.new_block(n, gm)
        self.w = dv.new_block(n, gm)
        self.v2 = dv.new_block(n, gm)
        self.w2 = dv.new_block(n, gm)
        self.h = dv.small_matrix(gm, gm)
        self.lams = [torch.zeros(gm, dtype=DTYPE, device=dev) for _ in range(2)]
        self.y = [dv.small_matrix(gm, gm) for _ in range(2)]
        self.rbuf = [dv.new_block(n, pmax) for _ in range(2)]
        self.stat = [torch.zeros(8 * pmax + 4, dtype=DTYPE, device=dev) for _ in range(2)]
        # one 8-double DGKS record per column of a block expansion
        self.dgks = [torch.zeros(8 * max(bs, 1), dtype=DTYPE, device=dev) for _ in range(2)]
        self.status = [torch.zeros(2 * gm + 8 * max(bs, 1) + 32, dtype=DTYPE, pin_memory=True) for _ in range(2)]
        # preconditioned expansion block of a speculative block expansion
        # (kept so a rejected speculation can be redone on the host path)
        self.src = [dv.new_block(n, bs) for _ in range(2)] if bs > 1 else None
        self.hcb = dv.small_matrix(gm + bs, bs)
        self.events = [torch.cuda.Event() for _ in range(2)]
        self.coefs = dv.small_matrix(gm, gm)
        self.count = torch.zeros(1, dtype=torch.int32, device=dev)
        self.prev = dv.small_matrix(gm, max(plus_k, 1))
        self.yref = torch.zeros(gm, dtype=DTYPE, device=dev)
        self.excl = torch.zeros(gm, dtype=DTYPE, device=dev)
        self.dgks_eager = torch.zeros(8 * max(bs, 1), dtype=DTYPE, device=dev)
        self.hc1 = dv.small_matrix(gm + 1, 1)
        self.ci = torch.zeros(1, dtype=torch.int32, device=dev)   # selected candidate (device copy)
        self.zero_i = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ci_host = None                                        # its value in stream order
        self.orthoc = torch.zeros(4 * _lib.SMALL_MAX * 4, dtype=DTYPE, device=dev)
        self.graphs = {}
        self.graph_shape = {}   # key without the operator identity -> current key
        self.graph_owner = None

    def reset(self):
        self.h.zero_()


_POOL = {}


def _acquire_workspace(n, gm, pmax, bs, plus_k):
    ctx = dv.context()
    key = (ctx.index, int(n), int(gm), int(pmax), int(bs), int(plus_k))
    free = _POOL.setdefault(key, [])
    ws = free.pop() if free else _Workspace(key, n, gm, pmax, bs, plus_k)
    ws.reset()
    return ws


def _release_workspace(ws):
    if ws is not None:
        _POOL.setdefault(ws.key, []).append(ws)


class DavidsonSolver:
    """One solve (eigensolver.py:157-785); create it, then call run()."""

    # capture single-column iterations as CUDA graphs (SVDSB_GRAPHS=0 disables)
    use_graphs = os.environ.get("SVDSB_GRAPHS", "1") != "0"

    def __init__(self, op, cfg, guesses=None, ortho_constraints=None, precond=None, est=None,
                 est_mode="normal"):
        cfg.validate(op.dim)
        self.ctx = dv.context()
        ctx = self.ctx
        if hasattr(ctx, "refresh_stream"):
            ctx.refresh_stream()
        self.op = op
        self.cfg = cfg
        self.precond = precond
        self.est = est if est is not None else NormEstimate()
        if est_mode not in ("normal", "augmented"):
            raise ValueError("est_mode must be 'normal' or 'augmented'")
        self.est_mode = est_mode
        self.rng = np.random.default_rng(cfg.seed)
        self.stats = EigStats()
        self.status = "ok"
        self.n = op.dim
        # distributed operators expose the global length and the slicing of
        # a global host vector to this rank's rows; single-GPU is the
        # identity
        from .dist import LOCAL
        self.comm = getattr(op, "comm", LOCAL)
        self.n_global = int(getattr(op, "dim_global", self.n))
        self._slice = getattr(op, "local_slice", None)
        self.ortho = Orthonormalizer(ctx, self.comm, self.n_global, self._slice)

        self.ext = []
        if ortho_constraints is not None and ortho_constraints.shape[1] > 0:
            c = ortho_constraints if isinstance(ortho_constraints, torch.Tensor) else \
                dv.to_device_block(self._local_rows(np.asarray(ortho_constraints, dtype=np.float64)))
            self.ortho(c, rng=self.rng)
            self.ext.append(c)
        self.n_ext = sum(b.shape[1] for b in self.ext)

        self.wanted = max(min(cfg.num_evals, self.n_global - self.n_ext), 0)
        self.dense = self.n_global <= cfg.max_basis_size
        if self.dense and self.comm.distributed:
            raise ValueError("problems smaller than the basis are not distributed")
        gmax = self.n - self.n_ext if self.dense else cfg.max_basis_size
        self.gmax = gmax
        gm = max(gmax, 1)
        bs = cfg.max_block_size

        pmax = max(min(self.wanted + bs, gm), 1)
        self.pmax = pmax
        self._ws = None
        if getattr(ctx, "handle", None) is not None:
            ws = self._ws = _acquire_workspace(self.n, gm, pmax, bs, cfg.plus_k)
            self.v, self.w, self._v2, self._w2 = ws.v, ws.w, ws.v2, ws.w2
            self.h = ws.h
            self._use_slot(0)
            self.coefs, self.count_d = ws.coefs, ws.count
            self.prev_d, self.yref, self.excl = ws.prev, ws.yref, ws.excl
            ws.ci_host = None
            self.ortho.c = ws.orthoc
            # graphs of a previous operator stay as update targets: their
            # keys carry that operator's identity, so they are never
            # replayed for this one (_launch_iter updates them in place)
            gk = getattr(op, "graph_key", None)
            ws.graph_owner = gk() if gk is not None else None
        else:
            self.v = dv.new_block(self.n, gm)
            self.w = dv.new_block(self.n, gm)
            self._v2 = None
            self._w2 = None
            self.h = dv.small_matrix(gm, gm)
            self.lams_d = torch.zeros(gm, dtype=DTYPE, device=ctx.device)
            self.y_d = dv.small_matrix(gm, gm)
            self.rbuf = dv.new_block(self.n, pmax)
            # status scratch: rn2 | split stats (6 per col) | r7^2 | refined lam
            self.stat_d = torch.zeros(8 * pmax + 4, dtype=DTYPE, device=ctx.device)
            self.coefs = dv.small_matrix(gm, gm)
            self.count_d = torch.zeros(1, dtype=torch.int32, device=ctx.device)
            self.prev_d = dv.small_matrix(gm, max(cfg.plus_k, 1))
            self.yref = torch.zeros(gm, dtype=DTYPE, device=ctx.device)
            self.excl = torch.zeros(gm, dtype=DTYPE, device=ctx.device)
        self.g = 0
        self.xbuf = None
        self.oxbuf = None
        self._pending = None   # graphed iteration queued, status not yet read
        self._ahead = None     # next graphed iteration queued speculatively
        self._ahead_used = False
        self._graph_base = None
        self._graph_static = None

        self.locked_vecs = dv.new_block(self.n, 0)
        self._locked_buf = dv.new_block(self.n, max(self.wanted, 1)) if cfg.locking else None
        self.locked_vals = []
        self.locked_rnorms = []
        self.locked_user = []

        self.q = None
        self.rfac = None
        self.tau = None

        self.restarts_since_reset = 0
        self.prev_coefs = None          # number of stored previous columns
        self.prev_coefs_g = 0
        self.collapse_streak = 0
        self._slot_progress = {}
        self._finished = self.wanted == 0
        self._warm = None           # (kind, g0) of the last known decomposition of H
        self.warm_start = True
        self.speculate = True       # device-decided DGKS for single-column expansions
        self._spec = None
        self._dgks_state = self._ws.dgks_eager if self._ws is not None else torch.zeros(
            8 * max(bs, 1), dtype=DTYPE, device=ctx.device)

        need_v1, split1 = _test_needs(cfg.convergence_test)
        need_v2, split2 = _test_needs(cfg.practical_test)
        self._need_vecs = need_v1 or need_v2 or cfg.iteration_hook is not None
        self._split_n = None
        for t in (cfg.convergence_test, cfg.practical_test):
            if t is not None and getattr(t, "split_n", None) is not None:
                self._split_n = int(t.split_n)
        if self._split_n is not None and hasattr(op, "split_local"):
            self._split_n = int(op.split_local)
        if self._need_vecs or self._split_n is not None or cfg.locking:
            self.xbuf = dv.new_block(self.n, pmax)
        if self._need_vecs:
            self.oxbuf = dv.new_block(self.n, pmax)

        if not self._finished:
            self._init_basis(guesses)
            if self.g == 0:
                self._finished = True
            elif self.cfg.extraction == EXTRACT_REFINED and not self.dense:
                self._rebuild_qr()

    # ------------------------------------------------------------ plumbing
    def _use_slot(self, s):
        """Point the per-iteration buffers at workspace slot s."""
        ws = self._ws
        self._slot = s
        self.lams_d, self.y_d, self.rbuf, self.stat_d = ws.lams[s], ws.y[s], ws.rbuf[s], ws.stat[s]

    @property
    def op_norm(self):
        return self.est.a_norm if self.est_mode == "augmented" else self.est.c_norm

    def _observe(self, lams):
        if self.est_mode == "augmented":
            self.est.update_from_augmented(lams)
        else:
            self.est.update(lams)

    def _budget_left(self):
        if self.cfg.max_matvecs is None:
            return 10 ** 18
        return self.cfg.max_matvecs - self.stats.matvecs

    def _apply_op(self, x, y):
        self.stats.matvecs += x.shape[1]
        self.op.apply_into(x, y)

    def _active_shift(self):
        shifts = self.cfg.shifts
        i = min(len(self.locked_vals), len(shifts) - 1)
        return float(shifts[i])

    def _against(self):
        blocks = list(self.ext)
        if self.locked_vecs.shape[1]:
            blocks.append(self.locked_vecs)
        return blocks

    def _order_mode(self):
        if self.cfg.target == TARGET_LARGEST:
            return _lib.ORDER_DESC, 0.0
        if self.cfg.target == TARGET_SMALLEST:
            return _lib.ORDER_ASC, 0.0
        return _lib.ORDER_INTERIOR, self._active_shift()

    def _user_test(self, cand):
        test = self.cfg.convergence_test
        if test is None:
            return cand.rnorm <= max(1e-12 * self.op_norm, PRACTICAL_FLOOR_FACTOR * EPS * self.op_norm)
        return _run_test(test, cand, self.op_norm)

    def _practical_test(self, cand):
        if self.cfg.practical_test is not None:
            return _run_test(self.cfg.practical_test, cand, self.op_norm)
        return self.op_norm > 0.0 and cand.rnorm <= PRACTICAL_FLOOR_FACTOR * EPS * self.op_norm

    def _sync_fetch(self, tensors):
        self.stats.syncs += 1
        return dv.fetch(self.ctx, tensors)

    def _upload_normal(self, block, draws):
        """Copy a C-order (rows, cols) numpy draw into a column-major block."""
        block.copy_(torch.from_numpy(np.ascontiguousarray(draws)))

    def _local_rows(self, arr):
        return arr if self._slice is None else self._slice(arr)

    def _draw(self, cols):
        """rng.standard_normal((N, cols)) of the GLOBAL length N (the same
        stream on every rank), this rank's rows."""
        return self._local_rows(self.rng.standard_normal((self.n_global, cols)))

    # Initial blocks of at least this many draws come from the device
    # counter RNG (svdsb_randn) instead of the host draw of the reference's
    # numpy stream: a 10 M x 20 host draw alone costs ~0.2 s (config 4).
    # Smaller problems keep the reference's stream, so their iterates and
    # matvec counts match the reference's; SVDSB_DEVICE_RNG_MIN overrides.
    device_rng_min = int(os.environ.get("SVDSB_DEVICE_RNG_MIN", str(1 << 22)))

    def _draw_into(self, block, cols):
        """block[:, :cols] = the initial standard-normal block
        (eigensolver.py:283-292)."""
        row0 = 0
        if self.comm.distributed:
            row0 = getattr(self.op, "local_row0", None)
        if (row0 is not None and getattr(self.ctx, "handle", None) is not None
                and self.n_global * cols >= self.device_rng_min):
            seed = (int(self.cfg.seed) * 0x9E3779B97F4A7C15 + 0x5FD) & ((1 << 64) - 1)
            blk = block[:, :cols]
            _lib.call("svdsb_randn", seed, int(row0), self.n, int(cols), dv.P(blk), dv.ld_of(blk), self.ctx.stream)
            self.stats.device_rng = True
            return
        self._upload_normal(block[:, :cols], self._draw(cols))

    def _red(self, *tensors):
        """Finish local partial sums across ranks (globalSum)."""
        if self.comm.distributed:
            for t in tensors:
                self.comm.allreduce_(t)

    def orthonormalize(self, block, against=None, start_col=0):
        r = self.ortho(block, against=against, start_col=start_col, rng=self.rng)
        self.stats.syncs = self.stats.syncs  # ortho keeps its own count
        return r

    # ------------------------------------------------------ initialization
    def _init_basis(self, guesses):
        """eigensolver.py:278-347."""
        cfg = self.cfg
        if self.dense:
            free = self.gmax
            self._upload_normal(self.v[:, :free], self._draw(free))
            self.orthonormalize(self.v[:, :free], against=self.ext)
            self.g = free
            take = min(free, max(self._budget_left(), 0))
            if take:
                self._apply_op(self.v[:, :take], self.w[:, :take])
            if take < free:
                self.status = "budget"
                self.g = take
            self._update_h_full()
            return
        g0 = 0
        if guesses is not None and guesses.shape[1] > 0:
            take = min(guesses.shape[1], self.gmax - 1)
            src = guesses if isinstance(guesses, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(self._local_rows(np.asarray(guesses, dtype=np.float64))))
            self.v[:, :take].copy_(src[:, :take])
            self.orthonormalize(self.v[:, :take], against=self._against())
            g0 = take
        if g0 == 0:
            b0 = min(max(cfg.max_block_size, cfg.num_evals), self.gmax - 1)
            self._draw_into(self.v, b0)
            self.orthonormalize(self.v[:, :b0], against=self._against())
            g0 = b0
        if cfg.deactivate_krylov_init:
            init_target = g0
        else:
            free = self.n_global - self.n_ext
            init_target = min(max(cfg.min_restart_size, g0), self.gmax - 1, free)
        if g0 > 1:
            take = min(g0 - 1, max(self._budget_left(), 0))
            if take:
                self._apply_op(self.v[:, :take], self.w[:, :take])
            if take < g0 - 1:
                self.status = "budget"
                self.g = take
                self._update_h_full()
                return
        j = g0 - 1
        skip_apply = False
        if (self.spec_fill and self.speculate and self.q is None and not self.comm.distributed
                and getattr(self.ctx, "handle", None) is not None and init_target - j >= 2
                and self._budget_left() >= init_target - j):
            # the whole Krylov fill with device-decided DGKS, one host sync
            resume = self._krylov_fill_speculative(j, init_target)
            if resume is None:
                self.g = init_target
                self._update_h_full()
                return
            j, skip_apply = resume, True
        while True:
            if self._budget_left() < 1:
                self.status = "budget"
                self.g = j
                self._update_h_full()
                return
            if not skip_apply:
                self._apply_op(self.v[:, j:j + 1], self.w[:, j:j + 1])
            skip_apply = False
            if j + 1 >= init_target:
                break
            dv.axpby(self.ctx, 1.0, self.w[:, j:j + 1], 0.0, self.v[:, j + 1:j + 2])
            self.orthonormalize(self.v[:, :j + 2], against=self._against(), start_col=j + 1)
            j += 1
        self.g = init_target
        self._update_h_full()

    def _krylov_fill_speculative(self, j0, target):
        """Krylov fill of eigensolver.py:320-346 (v_{j+1} = orthonormalised
        Op v_j) with every column's DGKS passes decided on the device and a
        single status read at the end.  Returns None when every column was
        accepted, else the column j whose successor must be redone on the
        host path (W[:, j] is valid and counted; later products are
        uncounted)."""
        nspec = target - 1 - j0
        states = torch.zeros((nspec, 8), dtype=DTYPE, device=self.ctx.device)
        for k in range(nspec):
            jj = j0 + k
            self._apply_op(self.v[:, jj:jj + 1], self.w[:, jj:jj + 1])
            prior = self._against() + [self.v[:, :jj + 1]]
            self._spec_cgs(prior, self.w[:, jj:jj + 1], self.v[:, jj + 1:jj + 2], states[k])
        self._apply_op(self.v[:, target - 1:target], self.w[:, target - 1:target])
        st = states.cpu().numpy()
        self.stats.syncs += 1
        for k in range(nspec):
            if not (st[k, 0] == 0.0 and st[k, 5] > 0.0):
                self._uncount_products(target - 1 - (j0 + k))
                return j0 + k
        return None

    def _uncount_products(self, ncols):
        """Undo the matvec accounting of ncols discarded operator columns."""
        self.stats.matvecs -= ncols
        self.op.n_applies -= ncols
        svd_op = getattr(self.op, "svd_op", None)
        if svd_op is not None:
            getattr(svd_op, "base", svd_op).n_matvecs -= 2 * ncols

    def _spec_cgs(self, prior, src, dst, st, d=None):
        """dst = src (./ d) orthonormalised against the prior blocks with
        device-decided DGKS passes (state into st, no host sync): the one
        launch of the graphed iterations while the basis is L2-resident,
        else the pass-by-pass kernels."""
        total = sum(b.shape[1] for b in prior)
        ws = self._ws
        if (ws is not None and self._use_fused_cgs(total) and len(prior) <= _lib.MAX_BLOCKS):
            n, ptrs, lds, cols, _ = dv._blk_args(prior)
            blk = dv.as_block(src)
            _lib.call("svdsb_cgs_fused", self.ctx.handle, self.n, n, ptrs, lds, cols, dv.P(blk), dv.ld_of(blk),
                      dv.P(ws.zero_i), None if d is None else dv.P(d), dv.P(dst), None, 1, total, 1, None, 1,
                      self.SPEC_PASSES, dv.P(st), self.ctx.stream)
            return
        if d is not None:
            _lib.call("svdsb_diag_solve", dst.shape[0], dv.P(d), dv.P(src), dv.ld_of(src), dv.P(dst), dv.ld_of(dst),
                      1, self.ctx.stream)
        else:
            dv.axpby(self.ctx, 1.0, src, 0.0, dst)
        _lib.call("svdsb_dgks_begin", dv.P(st), self.ctx.stream)
        n, ptrs, lds, cols, _ = dv._blk_args(prior)
        for p in range(self.SPEC_PASSES):
            _lib.call("svdsb_cgs_pass", self.ctx.handle, self.n, n, ptrs, lds, cols, dv.P(dst),
                      dv.P(self.ortho.c), dv.P(st), 1 if p == 0 else 0, self.ctx.stream)
        dv.scale_cols(self.ctx, dst, st[5:6], dv.SCALE_DIV)

    def _update_h_full(self):
        """H = sym(V^T W) (eigensolver.py:349-352)."""
        g = self.g
        self._warm = None
        if g == 0:
            return
        hg = dv.small_matrix(g, g)
        dv.gram(self.ctx, self.n, [self.v[:, :g]], self.w[:, :g], hg)
        self._red(hg)
        dv.h_symmetrize(self.ctx, g, hg, self.h[:g, :g])

    def _ensure_qr(self):
        if self.q is None:
            gm = max(self.gmax, 1)
            self.q = dv.new_block(self.n, gm)
            self._q2 = dv.new_block(self.n, gm)
            self.rfac = dv.small_matrix(gm, gm)
            self._qtmp = dv.new_block(self.n, 1)
            self._qy = dv.small_matrix(gm, gm)
            self._ry = dv.small_matrix(gm, gm)

    def _rebuild_qr(self):
        """Q R = W - tau V column by column (eigensolver.py:354-357)."""
        self._ensure_qr()
        self.tau = self._active_shift()
        self.rfac.zero_()
        self.qg = 0
        for j in range(self.g):
            self._qr_append_col(self.w[:, j:j + 1], self.v[:, j:j + 1])

    def _qr_append_col(self, wcol, vcol):
        """qr_append of (w - tau v) (kernels.py:160-222) into column qg."""
        ctx = self.ctx
        g = self.qg
        v = self.q[:, g:g + 1]
        dv.axpby(ctx, 1.0, wcol, 0.0, v)
        dv.axpby(ctx, -self.tau, vcol, 1.0, v)
        coef = self.rfac[:g, g:g + 1]
        self.rfac[:g + 1, g].zero_()
        prior = [self.q[:, :g]] if g > 0 else []
        orth = self.ortho
        # the reference's loop: orig, then passes with coefficient accumulation
        orig = None
        prev = None
        deficient = False
        collapses = 0
        for p in range(_MAX_REORTH_PASSES):
            if prior:
                c = orth.c[:g].unsqueeze(1)
                dv.gram(ctx, self.n, prior, v, c, norms2=orth.nrm[0:1])
                self._red(orth.c[:g])
                dv.project_out(ctx, self.n, prior, c, v, norms2=orth.nrm[1:2])
                dv.axpby(ctx, 1.0, c, 1.0, coef)
            else:
                dv.col_norms2(ctx, v, orth.nrm[0:1])
                dv.col_norms2(ctx, v, orth.nrm[1:2])
            self._red(orth.nrm)
            before2, after2 = dv.fetch(ctx, [orth.nrm])[0]
            orth.syncs += 1
            before, cur = float(np.sqrt(before2)), float(np.sqrt(after2))
            if p == 0:
                orig = prev = before
                if orig == 0.0:
                    deficient = True
                    break
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
        if deficient:
            v.copy_(torch.from_numpy(np.ascontiguousarray(self._draw(1))))
            self.ortho(v, against=prior, rng=self.rng)
            self.rfac[g, g] = 0.0
        else:
            dv.scale_cols(ctx, v, orth.nrm[1:2], dv.SCALE_DIV_SQRT)
            self.rfac[g:g + 1, g].copy_(torch.sqrt(orth.nrm[1:2]))
        self.qg = g + 1
        return deficient

    # ---------------------------------------------------------- extraction
    def extract_rayleigh_ritz(self):
        """Ritz values/vectors of H[:g,:g] in target order (device).

        Warm path: when H only grew by bordering columns since the last
        extraction (or since a Ritz-vector restart left it diagonal), the
        new decomposition is an O(g^2) secular-equation update of the known
        one; otherwise a cold Jacobi solve."""
        order, shift = self._order_mode()
        g = self.g
        warm = self._warm if self.warm_start else None
        if warm is not None and 0 < g - warm[1] <= 8:
            kind, g0 = warm
            y0 = self.y_d[:g0, :g0] if kind == "prev" else None
            l0 = self.lams_d[:g0] if kind == "prev" else None
            dv.syev_update(self.ctx, self.h, g0, g - g0, y0, l0, order, shift, self.lams_d[:g], self.y_d[:g, :g])
        else:
            dv.syev_small(self.ctx, self.h[:g, :g], g, order, shift, self.lams_d[:g], self.y_d[:g, :g])
        self._warm = ("prev", g)
        return self.lams_d[:g], self.y_d[:g, :g]

    def _candidates(self, y, lam, p, need_x, need_ox):
        """R = W Y - V Y diag(lam) for p columns, norms and optional split
        statistics (eigensolver.py:385-394); returns device views."""
        g = self.g
        r = self.rbuf[:, :p]
        x = self.xbuf[:, :p] if need_x else None
        ox = self.oxbuf[:, :p] if need_ox else None
        rn2 = self.stat_d[:p]
        dv.ritz_residual(self.ctx, self.v[:, :g], self.w[:, :g], y, lam, r, x, ox, rn2)
        self._red(rn2)
        split = None
        if self._split_n is not None:
            pm = self.pmax
            st = self.stat_d[pm:pm + 6 * p]
            r7 = self.stat_d[7 * pm:7 * pm + p]
            dv.split_stats(self.ctx, self._split_n, r, x, st)
            self._red(st)
            dv.split_residual(self.ctx, self._split_n, r, x, lam, st, r7)
            self._red(r7)
            split = (st, r7)
        return r, x, ox, rn2, split

    def _make_cands(self, lams, rn2, split_h, p, x, ox):
        cands = []
        rn = np.sqrt(np.maximum(rn2[:p], 0.0)).tolist()
        lv = lams[:p].tolist()
        for i in range(p):
            c = Candidate(lv[i], rn[i])
            if x is not None:
                c.x = x[:, i]
            if ox is not None:
                c.opx = ox[:, i]
            if split_h is not None:
                st, r7 = split_h
                c.nv = float(np.sqrt(st[6 * i + 2]))
                c.nu = float(np.sqrt(st[6 * i + 5]))
                c.r7 = float(np.sqrt(r7[i])) if np.isfinite(r7[i]) else np.inf
            cands.append(c)
        return cands

    # ---------------------------------------------------- reset, stagnation
    def maybe_reset(self, rnorm):
        """eigensolver.py:396-416."""
        if self.cfg.disable_reset:
            return False
        threshold = np.sqrt(self.restarts_since_reset) * self.op_norm * EPS
        if rnorm >= threshold:
            return False
        g = self.g
        if self._budget_left() < g:
            return False
        self.orthonormalize(self.v[:, :g], against=self._against())
        self._apply_op(self.v[:, :g], self.w[:, :g])
        self._update_h_full()
        if self.q is not None:
            self._rebuild_qr()
        self.restarts_since_reset = 0
        self.prev_coefs = None
        self.stats.resets += 1
        return True

    def _note_progress(self, slot, rnorm, lam):
        """eigensolver.py:418-433."""
        rec = self._slot_progress.get(slot)
        if rec is None:
            self._slot_progress[slot] = [rnorm, 0, lam]
            return 0
        best, stale, lam_ref = rec
        moved = abs(lam - lam_ref) > 100.0 * EPS * max(abs(lam), abs(lam_ref))
        if rnorm < best * _IMPROVE_FACTOR or moved:
            self._slot_progress[slot] = [min(rnorm, best), 0, lam]
            return 0
        rec[1] = stale + 1
        return stale + 1

    # ------------------------------------------------ restarting and locking
    def _reseed_basis(self):
        """eigensolver.py:471-483."""
        self._upload_normal(self.v[:, :1], self._draw(1))
        self.orthonormalize(self.v[:, :1], against=self._against())
        self.g = 1
        if self._budget_left() < 1:
            self.status = "budget"
            self._finished = True
            self.w[:, 0].zero_()
        else:
            self._apply_op(self.v[:, :1], self.w[:, :1])
        self._update_h_full()

    def _swap_basis(self, s):
        g = self.g
        c = self.coefs[:g, :s]
        if s <= 32:
            # row-local in-place V <- V C: the basis keeps its address, so the
            # captured iteration graphs do not come in two copies
            dv.ts_gemm(self.ctx, self.v[:, :g], c, self.v[:, :s])
            dv.ts_gemm(self.ctx, self.w[:, :g], c, self.w[:, :s])
            return
        if self._v2 is None:
            self._v2 = dv.new_block(self.n, max(self.gmax, 1))
            self._w2 = dv.new_block(self.n, max(self.gmax, 1))
        dv.ts_gemm(self.ctx, self.v[:, :g], c, self._v2[:, :s])
        dv.ts_gemm(self.ctx, self.w[:, :g], c, self._w2[:, :s])
        self.v, self._v2 = self._v2, self.v
        self.w, self._w2 = self._w2, self.w

    def restart(self, conv_count, exclude=None, y_first=None):
        """Thick restart keeping target-ordered Ritz vectors plus the
        previous candidate coefficients (eigensolver.py:485-536).  Uses the
        ordered Ritz coefficients of the current extraction (self.y_d)."""
        cfg = self.cfg
        g = self.g
        retain_target = max(cfg.min_restart_size, conv_count + 1)
        retain_target = max(min(retain_target, g - 1 if g > 1 else 1, self.gmax - 2), 1)
        prev = None
        nprev = 0
        if self.prev_coefs is not None and self.prev_coefs_g <= g:
            prev = self.prev_d
            nprev = self.prev_coefs
        dv.restart_coefs(self.ctx, g, self.gmax, y_first, self.y_d[:g, :g], g, retain_target, exclude,
                         prev, nprev, self.prev_coefs_g, cfg.plus_k, self.coefs[:g, :], self.count_d)
        self.stats.syncs += 1
        s = int(self.count_d.item())
        self.stats.restarts += 1
        self.restarts_since_reset += 1
        self.prev_coefs = None
        if s == 0:
            self._reseed_basis()
            if self.q is not None and not self._finished:
                self._rebuild_qr()
            return self.g
        self._swap_basis(s)
        dv.project_small(self.ctx, self.h[:g, :g], g, self.coefs[:g, :s], s, self.h[:s, :s])
        # Kept Ritz vectors plus a +k direction orthogonal to them make
        # C^T H C diagonal (to rounding): the next extraction starts from
        # (diag(H), I).  A refined head vector or an excluded direction breaks
        # that, so those restarts fall back to a cold solve.
        self._warm = ("diag", s) if (y_first is None and exclude is None) else None
        if self.q is not None:
            dv.qr_small(self.ctx, self.rfac[:g, :g], g, self.coefs[:g, :s], s, self._qy[:g, :s],
                        self._ry[:s, :s])
            dv.ts_gemm(self.ctx, self.q[:, :g], self._qy[:g, :s], self._q2[:, :s])
            self.q, self._q2 = self._q2, self.q
            self.rfac[:s, :s].copy_(self._ry[:s, :s])
            self.qg = s
        self.g = s
        return s

    def lock_candidate(self, lam, y, x, rnorm, user_flag):
        """eigensolver.py:538-558; y: device coefficient vector, x: device
        candidate vector."""
        cols = self.locked_vecs.shape[1]
        slot = self._locked_buf[:, cols:cols + 1]
        dv.col_norms2(self.ctx, x, self.stat_d[-1:])
        self._red(self.stat_d[-1:])
        dv.scale_cols(self.ctx, x, self.stat_d[-1:], dv.SCALE_DIV_SQRT, slot)
        self.locked_vecs = self._locked_buf[:, :cols + 1]
        self.orthonormalize(self.locked_vecs, against=self.ext, start_col=cols)
        self.locked_vals.append(float(lam))
        self.locked_rnorms.append(float(rnorm))
        self.locked_user.append(bool(user_flag))
        if len(self.locked_vals) >= self.wanted:
            self._finished = True
            return
        self.excl[:self.g].copy_(y)
        self.restart(0, exclude=self.excl[:self.g])
        if self.q is not None and not self._finished:
            self._rebuild_qr()

    # ------------------------------------------------------------ main loop
    def step(self):
        """One outer iteration (eigensolver.py:563-664)."""
        cfg = self.cfg
        self.stats.outer_iterations += 1
        info = {"restarted": False, "reset": False, "locked": False, "done": False}
        g = self.g
        refined = cfg.extraction == EXTRACT_REFINED
        need_x = self.xbuf is not None
        need_ox = self._need_vecs
        if self._pending is not None:
            # extraction, candidates and the status copy were queued (graph)
            # together with the previous expansion; only wait for them
            pend, self._pending = self._pending, None
            p = pend["p"]
            self._use_slot(pend["slot"])
            lams_d, y_d = self.lams_d[:g], self.y_d[:g, :g]
            r, x, ox, split = self.rbuf[:, :p], None, None, None
            got = self._wait_status(g, p, pend["slot"], pend["b"])
            st = got.pop()
            if not self._resolve_speculation(st):
                # the queued next iteration was built on the collapsed column
                self._ahead = None
                self.stats.outer_iterations -= 1
                return self.step()
            lams, rn2_h, split_h = got[0], got[1], None
            self._observe(lams)
            self._ahead_used = False
            try:
                return self._step_decide(info, g, lams, y_d, rn2_h, split_h, r, x, ox, p, refined)
            finally:
                if not self._ahead_used:
                    # the host decided differently from the speculation: the
                    # queued iteration only wrote buffers nobody reads now
                    self._ahead = None
        lams_d, y_d = self.extract_rayleigh_ritz()
        if refined:
            lamref = self.stat_d[-2:-1]
            dv.refined_small(self.ctx, self.rfac[:g, :g], self.h[:g, :g], g, self.yref[:g], lamref)
            p = 1
            r, x, ox, rn2, split = self._candidates(self.yref[:g].unsqueeze(1), lamref, 1, need_x, need_ox)
            fetch = [lams_d, rn2, lamref]
        else:
            p = 1 if cfg.locking else min(self.wanted + cfg.max_block_size, g)
            r, x, ox, rn2, split = self._candidates(y_d[:, :p], lams_d[:p], p, need_x, need_ox)
            fetch = [lams_d, rn2]
        if split is not None:
            fetch += [split[0], split[1]]
        spec = self._spec is not None
        if spec:
            fetch.append(self._dgks_state)
        got = self._sync_fetch(fetch)
        if spec:
            st = got.pop()
            if not self._resolve_speculation(st):
                # the previous expansion was redone: extract again
                self.stats.outer_iterations -= 1
                return self.step()
        lams = got[0]
        rn2_h = got[1]
        split_h = (got[-2], got[-1]) if split is not None else None
        self._observe(lams)
        self._lam_ref_h = float(got[2][0]) if refined else None
        return self._step_decide(info, g, lams, y_d, rn2_h, split_h, r, x, ox, p, refined)

    def _step_decide(self, info, g, lams, y_d, rn2_h, split_h, r, x, ox, p, refined):
        """Host half of an outer iteration: convergence tests, reset,
        locking, stagnation, budget, restart and expansion
        (eigensolver.py:586-664) on the fetched status."""
        cfg = self.cfg
        if refined:
            lam_ref = self._lam_ref_h
            cands = self._make_cands(np.array([lam_ref]), rn2_h, split_h, 1, x, ox)
            cand = cands[0]
            conv_count = 0
            ci = 0
            y_first = self.yref[:g]
            y_c = self.yref[:g]
        else:
            cands = self._make_cands(lams, rn2_h, split_h, p, x, ox)
            conv_count = 0
            if not cfg.locking:
                for i in range(min(self.wanted, p)):
                    if not (self._user_test(cands[i]) or self._practical_test(cands[i])):
                        break
                    conv_count += 1
            ci = min(conv_count, p - 1)
            cand = cands[ci]
            y_first = None
            y_c = y_d[:, ci]
        lam_c, rnorm_c = cand.lam, cand.rnorm
        x_c = x[:, ci:ci + 1] if x is not None else None
        res_block = r[:, ci:min(ci + cfg.max_block_size, p)]

        slot = len(self.locked_vals) if cfg.locking else conv_count
        info.update(lam=lam_c, rnorm=rnorm_c, x=x_c, conv_count=conv_count, g=g, slot=slot,
                    tau=self.tau if self.q is not None else None)
        if cfg.iteration_hook is not None:
            yfull = dv.to_host(y_d)
            yref_h = self.yref[:g].cpu().numpy() if refined else None
            cfg.iteration_hook(self, dict(info, rr_values=lams, rr_coefs=yfull, y_refined=yref_h))

        if self.maybe_reset(rnorm_c):
            info["reset"] = True
            return info
        if not cfg.locking and conv_count >= self.wanted:
            self._finished = True
            info["done"] = True
            return info
        if cfg.locking:
            ok_user = self._user_test(cand)
            if ok_user or self._practical_test(cand):
                self.lock_candidate(lam_c, y_c, x_c, rnorm_c, ok_user)
                info["locked"] = True
                info["done"] = self._finished
                return info
        if cfg.stagnation_window is not None and \
                self._note_progress(slot, rnorm_c, lam_c) > cfg.stagnation_window:
            self.status = "stagnated"
            self._finished = True
            info["done"] = True
            return info
        if self._budget_left() < cfg.max_block_size:
            self.status = "budget"
            self._finished = True
            info["done"] = True
            return info

        restarted = False
        if self.g >= self.gmax:
            # keep the candidate coefficients we still need after the restart
            self.restart(conv_count, y_first=y_first)
            restarted = True
            info["restarted"] = True
            if self._finished:
                info["done"] = True
                return info
        if not restarted:
            # saved before the expansion: a graphed expansion also runs the
            # next extraction, which overwrites the Ritz coefficients
            if refined:
                dv.axpby(self.ctx, 1.0, self.yref[:g].unsqueeze(1), 0.0, self.prev_d[:g, :1])
                self.prev_coefs = 1
            else:
                hi = min(conv_count + max(cfg.plus_k, 1), g)
                k = hi - conv_count
                # a graphed expansion copies the same columns on device
                # (selected by the device-side candidate index)
                if k > 0 and not (ci == conv_count and self._graph_ok(min(res_block.shape[1],
                                                                          self.gmax - self.g))):
                    dv.axpby(self.ctx, 1.0, y_d[:, conv_count:hi], 0.0, self.prev_d[:g, :k])
                self.prev_coefs = k
            self.prev_coefs_g = info["g"]
        if cfg.method == METHOD_JDQMR:
            corr = self._jd_corrections(res_block, ci, cands, y_d, refined)
            if corr is not None:
                self._expand(corr, ci, graph=False, precondition=False)
                return info
        self._expand(res_block, ci, graph=refined or ci == conv_count)
        return info

    # ------------------------------------------------------------ JDQMR
    def _jd_direction(self):
        if self.cfg.target == TARGET_LARGEST:
            return 1
        if self.cfg.target == TARGET_SMALLEST:
            return -1
        return 0

    def _jd_threshold(self, cand):
        """Eigen-residual at which the candidate would pass the outer test
        (the inner solve stops there)."""
        test = self.cfg.convergence_test
        if test is None:
            return max(1e-12 * self.op_norm, PRACTICAL_FLOOR_FACTOR * EPS * self.op_norm)
        fn = getattr(test, "threshold", None)
        return float(fn(cand.lam, self.op_norm)) if fn is not None else 0.0

    def _jd_corrections(self, res_block, ci, cands, y_d, refined):
        """JDQMR expansion block: for each block column the device inner
        solve of the correction equation of its Ritz pair (jdqmr.py);
        None when a GD step is taken instead (nothing to correct)."""
        from .jdqmr import JdqmrInner
        cfg = self.cfg
        b = min(res_block.shape[1], self.gmax - self.g)
        if b <= 0:
            return None
        jd = getattr(self, "_jd", None)
        if jd is None:
            diag = getattr(self.precond, "diagonal", None) if self.precond is not None else None
            if self.precond is not None and diag is None:
                raise ValueError("JDQMR supports the point-Jacobi preconditioner or none")
            jd = self._jd = JdqmrInner(self.ctx, self.op, self.n, diag=diag,
                                       use_graph=self.use_graphs and not self.comm.distributed)
            jd.log = JD_LOG
            self._jd_x = dv.new_block(self.n, 1)
            self._jd_out = dv.new_block(self.n, cfg.max_block_size)
        if self.comm.distributed:
            raise ValueError("JDQMR is single-GPU in this build")
        g = self.g
        out = self._jd_out[:, :b]
        any_inner = False
        for j in range(b):
            if refined:
                ycol, cand = self.yref[:g], cands[0]
            else:
                ycol, cand = y_d[:g, ci + j], cands[ci + j]
            r = res_block[:, j:j + 1]
            budget = self._budget_left() - (b - j)
            maxit = max(min(cfg.max_inner_iterations, budget), 0)
            if cand.rnorm <= 0.0 or maxit == 0:
                dv.axpby(self.ctx, 1.0, r, 0.0, out[:, j:j + 1])
                continue
            dv.ts_gemm(self.ctx, self.v[:, :g], ycol.reshape(g, 1), self._jd_x)
            t, info = jd.solve(self._jd_x, cand.lam, r, cand.rnorm, against=self._against(), maxit=maxit,
                               tol_e=self._jd_threshold(cand), etol_frac=cfg.inner_etol_frac,
                               lfac=cfg.inner_lfac, direction=self._jd_direction())
            it = info["iterations"]
            self.stats.matvecs += it
            self.stats.inner_iterations += it
            self.stats.inner_solves += 1
            if self.precond is not None:
                self.precond.n_applies += it + 1
                self.stats.precond_applies += it + 1
            if it == 0:
                # breakdown before the first step: plain residual
                dv.axpby(self.ctx, 1.0, r, 0.0, out[:, j:j + 1])
            else:
                any_inner = True
                dv.axpby(self.ctx, 1.0, t.unsqueeze(1), 0.0, out[:, j:j + 1])
        if not any_inner and self.precond is not None:
            return None
        return out

    # ------------------------------------------------ speculative expansion
    # A single new column is orthonormalised by device-decided CGS passes
    # (svdsb_cgs_pass) and the iteration proceeds without waiting for the
    # pass norms; the DGKS state rides along with the next status read.  In
    # the rare case the column collapsed (or needs more than SPEC_PASSES
    # passes) the expansion is rolled back and redone on the host path,
    # which reproduces the reference's random-replacement sequence.
    SPEC_PASSES = 3

    def _can_speculate(self, b):
        return ((b == 1 or (self._ws is not None and self._ws.src is not None and b <= self.cfg.max_block_size))
                and self.speculate and self.q is None and not self.comm.distributed
                and self.g >= 1 and getattr(self.ctx, "handle", None) is not None)

    def _use_fused_cgs(self, cols):
        """The one-launch CGS wins while the basis is L2-resident (latency
        bound: configs 1 and 2); HBM-streamed bases run the separate
        Gram / projection kernels, which stream at 82-86 % of HBM."""
        return (self.fused_cgs and cols <= 40 and 8 * self.n * cols <= (64 << 20)
                and _lib.cgs_fused_supported())

    def _expand_speculative(self, block, precondition=True):
        if block.shape[1] > 1:
            self._expand_speculative_block(block, precondition)
            return
        g = self.g
        dst = self.v[:, g:g + 1]
        prior = [b for b in self._against()] + [self.v[:, :g]]
        total = sum(b.shape[1] for b in prior)
        ws = self._ws
        pre = self.precond if precondition else None
        d = getattr(pre, "diagonal", None) if pre is not None else None
        if (ws is not None and self._use_fused_cgs(total) and len(prior) <= _lib.MAX_BLOCKS
                and (pre is None or d is not None)):
            # same single launch as the graphed iterations (bit-identical)
            if pre is not None:
                self.precond.n_applies += 1
                self.stats.precond_applies += 1
            st = self._dgks_state
            n, ptrs, lds, cols, _ = dv._blk_args(prior)
            blk = dv.as_block(block)
            _lib.call("svdsb_cgs_fused", self.ctx.handle, self.n, n, ptrs, lds, cols, dv.P(blk), dv.ld_of(blk),
                      dv.P(ws.zero_i), None if d is None else dv.P(d), dv.P(dst), None, 1, g, 1, None, 1,
                      self.SPEC_PASSES, dv.P(st), self.ctx.stream)
            self._apply_op(dst, self.w[:, g:g + 1])
            hc = dv.small_matrix(g + 1, 1)
            dv.gram(self.ctx, self.n, [self.v[:, :g + 1]], self.w[:, g:g + 1], hc)
            dv.h_insert(self.ctx, g, 1, hc, self.h)
            self._spec = {"g0": g}
            self.g = g + 1
            return
        if pre is not None:
            pre.apply_into(block, dst)
            self.stats.precond_applies += 1
        else:
            dv.axpby(self.ctx, 1.0, block, 0.0, dst)
        st = self._dgks_state
        _lib.call("svdsb_dgks_begin", dv.P(st), self.ctx.stream)
        prior = [b for b in self._against()] + [self.v[:, :g]]
        n, ptrs, lds, cols, total = dv._blk_args(prior)
        for p in range(self.SPEC_PASSES):
            _lib.call("svdsb_cgs_pass", self.ctx.handle, self.n, n, ptrs, lds, cols, dv.P(dst),
                      dv.P(self.ortho.c), dv.P(st), 1 if p == 0 else 0, self.ctx.stream)
        dv.scale_cols(self.ctx, dst, st[5:6], dv.SCALE_DIV)
        self._apply_op(dst, self.w[:, g:g + 1])
        hc = dv.small_matrix(g + 1, 1)
        dv.gram(self.ctx, self.n, [self.v[:, :g + 1]], self.w[:, g:g + 1], hc)
        dv.h_insert(self.ctx, g, 1, hc, self.h)
        self._spec = {"g0": g}
        self.g = g + 1

    def _expand_speculative_block(self, block, precondition=True, slot=None):
        """Block expansion (eigensolver.py:666-700 with b > 1) with every
        column's DGKS passes decided on the device: column j is
        orthonormalised against the basis and the new columns before it, as
        the reference's column loop does, with no host round trip; the b
        DGKS records ride along with the next status read."""
        g = self.g
        b = block.shape[1]
        ws = self._ws
        src = ws.src[self._slot if slot is None else slot][:, :b]
        if self.precond is not None and precondition:
            self.precond.apply_into(block, src)
            self.stats.precond_applies += b
        else:
            dv.axpby(self.ctx, 1.0, block, 0.0, src)
        st = self._dgks_state
        self._block_cgs(self._against() + [self.v[:, :g]], src, self.v[:, g:g + b], st)
        self._apply_op(self.v[:, g:g + b], self.w[:, g:g + b])
        hc = ws.hcb[:g + b, :b]
        dv.gram(self.ctx, self.n, [self.v[:, :g + b]], self.w[:, g:g + b], hc)
        dv.h_insert(self.ctx, g, b, hc, self.h)
        self._spec = {"g0": g, "b": b, "src": src}
        self.g = g + b

    # block CGS: batched first pass (svdsb_cgs_block); SVDSB_BLOCK_CGS=0 runs
    # the columns one by one through _spec_cgs instead
    block_cgs = os.environ.get("SVDSB_BLOCK_CGS", "1") != "0"

    def _block_cgs(self, prior, src, dst, st):
        """dst = src orthonormalised column by column against the prior
        blocks and the block's earlier columns, DGKS decided on the device
        (b records in st)."""
        b = dst.shape[1]
        total = sum(p_.shape[1] for p_ in prior)
        if (not self.block_cgs or len(prior) + 1 >= _lib.MAX_BLOCKS
                or total * b + 3 * b + total > self.ortho.c.numel() or total + b > 256):
            g0 = prior[-1].shape[1]
            for j in range(b):
                self._spec_cgs(prior[:-1] + [self.v[:, :g0 + j]], src[:, j:j + 1], dst[:, j:j + 1],
                               st[8 * j:8 * j + 8])
            return
        dv.axpby(self.ctx, 1.0, src, 0.0, dst)
        n, ptrs, lds, cols, _ = dv._blk_args(prior)
        _lib.call("svdsb_cgs_block", self.ctx.handle, self.n, n, ptrs, lds, cols, dv.P(dst), dv.ld_of(dst), b,
                  dv.P(self.ortho.c), dv.P(st), self.SPEC_PASSES, self.ctx.stream)

    def _resolve_block(self, spec, st):
        """Resolve a speculative block expansion: it stands when every
        column was accepted by DGKS within SPEC_PASSES; otherwise the whole
        block is redone on the host path from the kept preconditioned
        directions (the reference's column loop, random replacement
        included)."""
        g, b, src = spec["g0"], spec["b"], spec["src"]
        rec = np.asarray(st[:8 * b]).reshape(b, 8)
        if np.all(rec[:, 0] == 0.0) and np.all(rec[:, 5] > 0.0):
            self.collapse_streak = 0
            return True
        self.g = g
        self._uncount_products(b)
        dv.axpby(self.ctx, 1.0, src, 0.0, self.v[:, g:g + b])
        replaced = self.orthonormalize(self.v[:, :g + b], against=self._against(), start_col=g)
        if len(replaced) == b:
            self.collapse_streak += 1
            if self.collapse_streak >= 3:
                raise BasisCollapseError("no independent expansion direction after 3 retries")
        else:
            self.collapse_streak = 0
        self._apply_op(self.v[:, g:g + b], self.w[:, g:g + b])
        hc = dv.small_matrix(g + b, b)
        dv.gram(self.ctx, self.n, [self.v[:, :g + b]], self.w[:, g:g + b], hc)
        dv.h_insert(self.ctx, g, b, hc, self.h)
        self.g = g + b
        self._warm = None
        return False

    def _resolve_speculation(self, st):
        """Called with the fetched DGKS state; True if the speculative
        expansion stands, else it has been redone on the host path."""
        spec, self._spec = self._spec, None
        if spec.get("b", 1) > 1:
            return self._resolve_block(spec, st)
        if st[0] == 0.0 and st[5] > 0.0:
            self.collapse_streak = 0
            return True
        # roll back the product of the speculative column
        g = spec["g0"]
        self.g = g
        self.stats.matvecs -= 1
        self.op.n_applies -= 1
        svd_op = getattr(self.op, "svd_op", None)
        if svd_op is not None:
            getattr(svd_op, "base", svd_op).n_matvecs -= 2
        v = self.v[:, g:g + 1]
        prior = self._against() + [self.v[:, :g]]
        replaced = False
        final = 0.0
        if st[0] != 0.0:
            # still iterating after SPEC_PASSES: continue the same DGKS loop
            final = self.ortho.resume(v, prior, st)
        if final == 0.0:
            replaced = True
            for _ in range(_MAX_RANDOM_RETRIES):
                v.copy_(torch.from_numpy(np.ascontiguousarray(self._draw(1))))
                if self.ortho.column(v, prior) > 0.0:
                    break
            else:
                raise np.linalg.LinAlgError("orthonormalize could not produce an independent column")
        if replaced:
            self.collapse_streak += 1
            if self.collapse_streak >= 3:
                raise BasisCollapseError("no independent expansion direction after 3 retries")
        else:
            self.collapse_streak = 0
        self._apply_op(v, self.w[:, g:g + 1])
        hc = dv.small_matrix(g + 1, 1)
        dv.gram(self.ctx, self.n, [self.v[:, :g + 1]], self.w[:, g:g + 1], hc)
        dv.h_insert(self.ctx, g, 1, hc, self.h)
        self.g = g + 1
        self._warm = None
        return False

    # ------------------------------------------------- graphed iterations
    # The device work between two host decisions of a plain single-column
    # Rayleigh-Ritz iteration -- expansion (preconditioner, device-decided
    # CGS passes, the C-apply, the H column), the next warm extraction, the
    # candidate residuals and the status copy -- depends only on (g, p, warm
    # state, buffers); the selected candidate is a device-side index.  It is
    # captured once as a CUDA graph and replayed: one launch instead of ~17,
    # no Python in between.
    #
    # Iterations are also queued one ahead: right after iteration k's graph,
    # iteration k+1's graph is launched on the guess that the host will
    # decide on k the way it usually does (no new convergence, no reset, no
    # stop -- so the same candidate index, and no restart since the basis is
    # not full).  The host then decides on k while the GPU already runs k+1.
    # k+1 reads slot s and writes slot 1-s, so a wrong guess costs only the
    # wasted GPU work: nothing the host path reads was overwritten, and the
    # counters are only advanced when the queued iteration is accepted.

    run_ahead = os.environ.get("SVDSB_AHEAD", "1") != "0"
    # Krylov fill of the initial basis with device-decided DGKS (SVDSB_SPEC_FILL=0: host-driven)
    spec_fill = os.environ.get("SVDSB_SPEC_FILL", "1") != "0"
    fused_cgs = os.environ.get("SVDSB_CGS_FUSED", "1") != "0"

    def _graph_ok(self, b):
        static = self._graph_static
        if static is None:
            # the parts fixed for the whole solve, evaluated once
            static = self._graph_static = bool(
                self.use_graphs and self._ws is not None and not self.comm.distributed
                and getattr(self.ctx, "handle", None) is not None
                and not self.cfg.locking and self.cfg.extraction == EXTRACT_RR
                and self._split_n is None and not self._need_vecs and self.cfg.iteration_hook is None
                and not self.ext and getattr(self.op, "graph_key", None) is not None
                and (self.precond is None or getattr(self.precond, "diagonal", None) is not None))
        return (static and (b == 1 or (self._ws.src is not None and b <= self.cfg.max_block_size))
                and self.speculate and self.q is None and self.g >= 1 and self.warm_start
                and self._warm is not None and self.locked_vecs.shape[1] == 0)

    def _iter_device(self, g, kind, g0, p, order, shift, sin, sout, b=1):
        """Launch-only body of a graphed iteration (no host bookkeeping):
        expand with candidate *ws.ci of slot sin, extract into slot sout."""
        if b > 1:
            self._iter_device_block(g, kind, g0, p, order, shift, sin, sout, b)
            return
        ctx = self.ctx
        ws = self._ws
        dst = self.v[:, g:g + 1]
        y_in, l_in = ws.y[sin], ws.lams[sin]
        y_out, l_out, r_out, s_out = ws.y[sout], ws.lams[sout], ws.rbuf[sout], ws.stat[sout]
        kk = max(self.cfg.plus_k, 1)
        d = self.precond.diagonal if self.precond is not None else None
        st = ws.dgks[sout]
        nat = getattr(self.op, "native_normal", None)
        if nat is not None and self._use_fused_cgs(g):
            # the whole launch sequence in one native call (csrc/gdk.cu)
            dev, side, inner = nat
            tmp = dev.scratch(inner, 1)
            gn = g + 1
            y0 = y_in if kind == "prev" else None
            a = _lib.GdkIterArgs(
                n=self.n, v=self.v.data_ptr(), ldv=dv.ld_of(self.v), w=self.w.data_ptr(), ldw=dv.ld_of(self.w), g=g,
                rsrc=ws.rbuf[sin].data_ptr(), ldr=dv.ld_of(ws.rbuf[sin]), ci=ws.ci.data_ptr(),
                d=None if d is None else d.data_ptr(), yin=y_in.data_ptr(), ldyin=dv.ld_of(y_in), kk=kk,
                prev=self.prev_d.data_ptr(), ldprev=dv.ld_of(self.prev_d), passes=self.SPEC_PASSES,
                dgks=st.data_ptr(), csr=dev.handle, side=side, tmp=tmp.data_ptr(), ldtmp=dv.ld_of(tmp),
                hc=ws.hc1.data_ptr(), ldhc=dv.ld_of(ws.hc1), h=self.h.data_ptr(), ldh=dv.ld_of(self.h),
                g0=g0, y0=None if y0 is None else y0.data_ptr(), ldy0=dv.ld_of(y0) if y0 is not None else 1,
                l0=None if y0 is None else l_in.data_ptr(), order=int(order), shift=float(shift),
                lout=l_out.data_ptr(), yout=y_out.data_ptr(), ldyout=dv.ld_of(y_out), p=p,
                rout=r_out.data_ptr(), ldrout=dv.ld_of(r_out), rn2=s_out.data_ptr(),
                status_host=ws.status[sout].data_ptr())
            _lib.call("svdsb_gdk_iteration", ctx.handle, ctypes.byref(a), ctx.stream)
            return
        n_, ptrs, lds, cols, _ = dv._blk_args([self.v[:, :g]])
        if self._use_fused_cgs(g):
            # select + precondition + +k copy + device-decided CGS passes +
            # normalise, one launch (svdsb_cgs_fused)
            rin, yb = ws.rbuf[sin], y_in[:g, :g]
            _lib.call("svdsb_cgs_fused", ctx.handle, self.n, n_, ptrs, lds, cols, dv.P(rin), dv.ld_of(rin),
                      dv.P(ws.ci), None if d is None else dv.P(d), dv.P(dst), dv.P(yb), dv.ld_of(yb), g, kk,
                      dv.P(self.prev_d), dv.ld_of(self.prev_d), self.SPEC_PASSES, dv.P(st), ctx.stream)
        else:
            # +k coefficients kept for the next restart (eigensolver.py:520-527)
            dv.gather_cols(ctx, y_in[:g, :g], ws.ci, kk, g, self.prev_d[:g, :kk])
            # the selected residual, preconditioned (x ./ d as svdsb_diag_solve)
            dv.gather_cols(ctx, ws.rbuf[sin], ws.ci, 1, self.pmax, dst, d=d)
            _lib.call("svdsb_dgks_begin", dv.P(st), ctx.stream)
            for p_ in range(self.SPEC_PASSES):
                _lib.call("svdsb_cgs_pass", ctx.handle, self.n, n_, ptrs, lds, cols, dv.P(dst),
                          dv.P(self.ortho.c), dv.P(st), 1 if p_ == 0 else 0, ctx.stream)
            dv.scale_cols(ctx, dst, st[5:6], dv.SCALE_DIV)
        self.op.raw_into(dst, self.w[:, g:g + 1])
        hc = ws.hc1[:g + 1, :]
        dv.gram(ctx, self.n, [self.v[:, :g + 1]], self.w[:, g:g + 1], hc)
        dv.h_insert(ctx, g, 1, hc, self.h)
        gn = g + 1
        y0 = y_in[:g0, :g0] if kind == "prev" else None
        l0 = l_in[:g0] if kind == "prev" else None
        dv.syev_update(ctx, self.h, g0, gn - g0, y0, l0, order, shift, l_out[:gn], y_out[:gn, :gn])
        dv.ritz_residual(ctx, self.v[:, :gn], self.w[:, :gn], y_out[:gn, :p], l_out[:p],
                         r_out[:, :p], rn2=s_out[:p])
        # status straight into the pinned host slot (one kernel, no copies)
        _lib.call("svdsb_status_pack", dv.P(l_out), gn, dv.P(s_out), p, dv.P(st), ws.status[sout].data_ptr(),
                  ctx.stream)

    def _iter_device_block(self, g, kind, g0, p, order, shift, sin, sout, b):
        """_iter_device for a block expansion of b columns (candidates
        *ws.ci .. *ws.ci + b - 1): the +k copy, the preconditioned residual
        block, device-decided CGS column by column, the b-column operator
        product, the H border, the warm b-border RR update, the candidate
        residuals and the status record with b DGKS records."""
        ctx = self.ctx
        ws = self._ws
        y_in, l_in = ws.y[sin], ws.lams[sin]
        y_out, l_out, r_out, s_out = ws.y[sout], ws.lams[sout], ws.rbuf[sout], ws.stat[sout]
        kk = max(self.cfg.plus_k, 1)
        d = self.precond.diagonal if self.precond is not None else None
        st = ws.dgks[sout]
        src = ws.src[sout][:, :b]
        dv.gather_cols(ctx, y_in[:g, :g], ws.ci, kk, g, self.prev_d[:g, :kk])
        dv.gather_cols(ctx, ws.rbuf[sin], ws.ci, b, self.pmax, src, d=d)
        self._block_cgs([self.v[:, :g]], src, self.v[:, g:g + b], st)
        self.op.raw_into(self.v[:, g:g + b], self.w[:, g:g + b])
        hc = ws.hcb[:g + b, :b]
        dv.gram(ctx, self.n, [self.v[:, :g + b]], self.w[:, g:g + b], hc)
        dv.h_insert(ctx, g, b, hc, self.h)
        gn = g + b
        y0 = y_in[:g0, :g0] if kind == "prev" else None
        l0 = l_in[:g0] if kind == "prev" else None
        dv.syev_update(ctx, self.h, g0, gn - g0, y0, l0, order, shift, l_out[:gn], y_out[:gn, :gn])
        dv.ritz_residual(ctx, self.v[:, :gn], self.w[:, :gn], y_out[:gn, :p], l_out[:p],
                         r_out[:, :p], rn2=s_out[:p])
        _lib.call("svdsb_status_pack_n", dv.P(l_out), gn, dv.P(s_out), p, dv.P(st), b, ws.status[sout].data_ptr(),
                  ctx.stream)

    def _capture(self, fn, reuse=None):
        """Record fn's libsvdsb launches as a CUDA graph on a side stream
        (capture needs a non-default stream) and instantiate it -- or, with
        `reuse` (a _NativeGraph of the same iteration shape, e.g. captured
        for the previous matrix), update that executable in place, which
        costs a fraction of an instantiation."""
        ctx = self.ctx
        cap = getattr(ctx, "capture_stream", None)
        if cap is None:
            cap = ctx.capture_stream = torch.cuda.Stream(ctx.device)
        old = ctx._stream
        lib = _lib.load()
        ex = ctypes.c_void_p()
        # no cyclic garbage collection while capturing: a finaliser that
        # frees device memory (a previous matrix) would invalidate the
        # capture; matrix finalisers run anyway are deferred (_lib.CAPTURING)
        gc_on = gc.isenabled()
        gc.disable()
        _lib.CAPTURING[0] += 1
        try:
            _lib.check(lib.svdsb_graph_begin(cap.cuda_stream), "svdsb_graph_begin")
            try:
                ctx._stream = cap.cuda_stream
                fn()
            finally:
                ctx._stream = old
                if reuse is None:
                    rc = lib.svdsb_graph_end(cap.cuda_stream, ctypes.byref(ex))
                else:
                    rc = lib.svdsb_graph_end_update(cap.cuda_stream, reuse.exec, ctypes.byref(ex))
        finally:
            _lib.CAPTURING[0] -= 1
            if gc_on:
                gc.enable()
            _lib.flush_deferred()
        _lib.check(rc, "svdsb_graph_end")
        if reuse is not None and ex.value == reuse.exec:
            reuse.exec = None   # ownership moves to the returned graph
        return _NativeGraph(ex.value)

    def _launch_iter(self, g, kind, g0, sin, ci, b=1):
        """Replay (capturing on first use) the iteration graph that expands
        a basis of size g by b columns from slot sin; returns the
        queued-iteration record."""
        ws = self._ws
        sout = 1 - sin
        p = min(self.wanted + self.cfg.max_block_size, g + b)
        order, shift = self._order_mode()
        base = self._graph_base
        if base is None:
            # operator / preconditioner identity: fixed for the solve
            base = self._graph_base = (self.op.graph_key(),
                                       None if self.precond is None else self.precond.diagonal.data_ptr())
        key = (self.v.data_ptr(), self.w.data_ptr(), kind, g0, g, b, p, sin, order, shift, base)
        entry = ws.graphs.get(key)
        if entry is None:
            # one graph per iteration shape: the one captured for another
            # operator / preconditioner (a new matrix) is updated in place
            skey = key[:-1]
            old_key = ws.graph_shape.get(skey)
            old = ws.graphs.pop(old_key, None) if old_key is not None else None
            before = _lib.launch_count()
            graph = self._capture(lambda: self._iter_device(g, kind, g0, p, order, shift, sin, sout, b),
                                  reuse=None if old is None else old[0])
            entry = (graph, _lib.launch_count() - before)
            ws.graphs[key] = entry
            ws.graph_shape[skey] = key
            self.stats.graphs_captured += 1
        entry[0].replay(self.ctx._stream)
        ws.events[sout].record(self.ctx.torch_stream)
        _lib.load().svdsb_note_launches(entry[1])
        return {"p": p, "slot": sout, "sin": sin, "g": g, "ci": ci, "b": b}

    def _block_width(self, ci, g):
        """Columns of the expansion that follows an extraction at basis size
        g with candidate ci (eigensolver.py:650-656: the residual block
        res[:, ci:ci+b] of p candidates, cut to the free basis columns)."""
        bs = self.cfg.max_block_size
        p = min(self.wanted + bs, g)
        return min(min(ci + bs, p) - ci, self.gmax - g)

    def _expand_graphed(self, ci, b=1):
        ws = self._ws
        g = self.g
        sin = self._slot
        ahead, self._ahead = self._ahead, None
        self._ahead_used = True
        if ahead is not None and ahead["g"] == g and ahead["ci"] == ci and ahead["sin"] == sin \
                and ahead["b"] == b and self._warm == ("prev", g):
            pend = ahead          # already running: the guess was right
        else:
            if ws.ci_host != ci:
                dv.set_int(self.ctx, ws.ci, ci)
                ws.ci_host = ci
            kind, g0 = self._warm
            if kind == "diag" and sin == 1:
                # a restart cycle always starts from slot 0 (the diag-warm
                # iteration reads only the chosen residual), so each basis
                # size maps to one slot and half as many graphs get captured
                dv.axpby(self.ctx, 1.0, ws.rbuf[1][:, ci:ci + b], 0.0, ws.rbuf[0][:, ci:ci + b])
                sin = 0
            pend = self._launch_iter(g, kind, g0, sin, ci, b)
        # host bookkeeping of what the graph does
        if self.precond is not None:
            self.precond.n_applies += b
            self.stats.precond_applies += b
        self.stats.matvecs += b
        self.op.n_applies += b
        self.op.count_svd_matvecs(b)
        self._spec = {"g0": g, "b": b, "src": ws.src[pend["slot"]][:, :b] if b > 1 else None}
        self.g = g + b
        self._warm = ("prev", g + b)
        self._pending = pend
        # queue the next iteration on the usual decision; with a full basis
        # the host would restart instead, so only while g + b < gmax
        if self.run_ahead and g + b < self.gmax:
            b_next = self._block_width(ci, g + b)
            if b_next >= 1:
                self._ahead = self._launch_iter(g + b, "prev", g + b, pend["slot"], ci, b_next)

    def _wait_status(self, g, p, slot, b=1):
        """Wait for the queued iteration that writes `slot` (not for a
        later one queued behind it) and read its status."""
        ws = self._ws
        ws.events[slot].synchronize()
        self.stats.syncs += 1
        host = ws.status[slot].numpy()
        return [host[:g].copy(), host[g:g + p].copy(), host[g + p:g + p + 8 * b].copy()]

    def _expand(self, res_block, ci=0, graph=True, precondition=True):
        """eigensolver.py:666-700.  precondition=False: the block is already
        the expansion direction (JDQMR corrections)."""
        b = min(res_block.shape[1], self.gmax - self.g)
        if b <= 0:
            return
        if graph and precondition and self._graph_ok(b):
            self._expand_graphed(ci, b)
            return
        block = res_block[:, :b]
        if self._can_speculate(b):
            self._expand_speculative(block, precondition)
            return
        g = self.g
        dst = self.v[:, g:g + b]
        if self.precond is not None and precondition:
            self.precond.apply_into(block, dst)
            self.stats.precond_applies += b
        else:
            dv.axpby(self.ctx, 1.0, block, 0.0, dst)
        replaced = self.orthonormalize(self.v[:, :g + b], against=self._against(), start_col=g)
        if len(replaced) == b:
            self.collapse_streak += 1
            if self.collapse_streak >= 3:
                raise BasisCollapseError("no independent expansion direction after 3 retries")
        else:
            self.collapse_streak = 0
        self._apply_op(self.v[:, g:g + b], self.w[:, g:g + b])
        hc = dv.small_matrix(g + b, b)
        dv.gram(self.ctx, self.n, [self.v[:, :g + b]], self.w[:, g:g + b], hc)
        self._red(hc)
        dv.h_insert(self.ctx, g, b, hc, self.h)
        if self.q is not None:
            for j in range(b):
                self._qr_append_col(self.w[:, g + j:g + j + 1], self.v[:, g + j:g + j + 1])
        self.g = g + b

    # ---------------------------------------------------------- finalization
    def _final_pairs(self, x, wx, z_d, lam_d, t):
        """x2 = x z, wx2 = wx z, res = wx2 - x2 lam, norms (+split)."""
        x2 = dv.new_block(self.n, t)
        rbuf = dv.new_block(self.n, t)
        ox2 = dv.new_block(self.n, t) if self._need_vecs else None
        rn2 = torch.zeros(t, dtype=DTYPE, device=self.ctx.device)
        dv.ritz_residual(self.ctx, x, wx, z_d, lam_d, rbuf, x2, ox2, rn2)
        self._red(rn2)
        fetch = [lam_d, rn2]
        if self._split_n is not None:
            st = torch.zeros(6 * t, dtype=DTYPE, device=self.ctx.device)
            r7 = torch.zeros(t, dtype=DTYPE, device=self.ctx.device)
            dv.split_stats(self.ctx, self._split_n, rbuf, x2, st)
            self._red(st)
            dv.split_residual(self.ctx, self._split_n, rbuf, x2, lam_d, st, r7)
            self._red(r7)
            fetch += [st, r7]
        got = self._sync_fetch(fetch)
        split_h = (got[2], got[3]) if self._split_n is not None else None
        cands = self._make_cands(got[0], got[1], split_h, t, x2, ox2)
        conv = np.array([self._user_test(cands[i]) for i in range(t)], dtype=bool)
        rnorms = np.array([c.rnorm for c in cands], dtype=np.float64)
        return np.asarray(got[0], dtype=np.float64), x2, rnorms, conv

    def finalize_soft_locked(self):
        """Extra RR over the leading pairs with fresh products
        (eigensolver.py:705-724)."""
        _, y_d = self.extract_rayleigh_ritz()
        t = min(self.wanted, self.g)
        if t == 0:
            return np.zeros(0), dv.new_block(self.n, 0), np.zeros(0), np.zeros(0, dtype=bool)
        x = dv.new_block(self.n, t)
        dv.ts_gemm(self.ctx, self.v[:, :self.g], y_d[:, :t], x)
        wx = dv.new_block(self.n, t)
        self._apply_op(x, wx)
        h2 = dv.small_matrix(t, t)
        dv.gram(self.ctx, self.n, [x], wx, h2)
        self._red(h2)
        order, shift = self._order_mode()
        lam2 = torch.zeros(t, dtype=DTYPE, device=self.ctx.device)
        z = dv.small_matrix(t, t)
        dv.syev_small(self.ctx, h2, t, order, shift, lam2, z)
        return self._final_pairs(x, wx, z, lam2, t)

    def _finalize_locked(self):
        """eigensolver.py:726-739."""
        t = len(self.locked_vals)
        if t == 0:
            return np.zeros(0), dv.new_block(self.n, 0), np.zeros(0), np.zeros(0, dtype=bool)
        x = self.locked_vecs[:, :t]
        wx = dv.new_block(self.n, t)
        self._apply_op(x, wx)
        lam = torch.zeros(t, dtype=DTYPE, device=self.ctx.device)
        dv.col_dots(self.ctx, x, wx, lam)
        self._red(lam)
        eye = dv.small_matrix(t, t)
        eye.copy_(torch.eye(t, dtype=DTYPE))
        return self._final_pairs(x, wx, eye, lam, t)

    def _run_dense(self):
        """Exact solve once the basis spans the admissible space
        (eigensolver.py:741-768)."""
        g = self.g
        lams_all_d = torch.zeros(max(g, 1), dtype=DTYPE, device=self.ctx.device)
        y_all = dv.small_matrix(max(g, 1), max(g, 1))
        if g:
            dv.syev_small(self.ctx, self.h[:g, :g], g, _lib.ORDER_ASC, 0.0, lams_all_d[:g], y_all[:g, :g])
        lams_all = self._sync_fetch([lams_all_d[:g]])[0]
        self._observe(lams_all)
        if self.cfg.target == TARGET_CLOSEST_GEQ:
            shifts = self.cfg.shifts
            chosen = []
            open_idx = list(range(lams_all.shape[0]))
            for i in range(min(self.wanted, lams_all.shape[0])):
                s = float(shifts[min(i, len(shifts) - 1)])
                pick = open_idx[select_interior_candidate(lams_all[open_idx], s)]
                open_idx.remove(pick)
                chosen.append(pick)
        else:
            if self.cfg.target == TARGET_LARGEST:
                order = np.argsort(-lams_all, kind="stable")
            else:
                order = np.argsort(lams_all, kind="stable")
            chosen = list(order[:self.wanted])
        t = len(chosen)
        if t == 0:
            return EigResult(np.zeros(0), dv.new_block(self.n, 0), np.zeros(0), np.zeros(0, dtype=bool),
                             self.stats, self.status)
        idx = torch.tensor(chosen, dtype=torch.long, device=self.ctx.device)
        ysel = dv.small_matrix(g, t)
        ysel.copy_(y_all[:g, :g].index_select(1, idx))
        lam_sel = lams_all_d[:g].index_select(0, idx).contiguous()
        lam, x, rnorms, conv = self._final_pairs(self.v[:, :g], self.w[:, :g], ysel, lam_sel, t)
        return EigResult(lam, x, rnorms, conv, self.stats, self.status)

    def run(self):
        if self.wanted == 0:
            return EigResult(np.zeros(0), dv.new_block(self.n, 0), np.zeros(0), np.zeros(0, dtype=bool),
                             self.stats, self.status)
        if self.dense:
            return self._run_dense()
        while not self._finished:
            self.step()
        if self.cfg.locking:
            lam, x, rnorms, conv = self._finalize_locked()
        else:
            lam, x, rnorms, conv = self.finalize_soft_locked()
        self.stats.syncs += self.ortho.syncs
        return EigResult(np.asarray(lam, dtype=np.float64), x, np.asarray(rnorms, dtype=np.float64), conv,
                         self.stats, self.status)


def eig_solve(op, cfg, guesses=None, ortho_constraints=None, precond=None, est=None, est_mode="normal"):
    """Compute cfg.num_evals eigenpairs of a symmetric device operator
    (eigensolver.py:788-821)."""
    solver = DavidsonSolver(op, cfg, guesses=guesses, ortho_constraints=ortho_constraints, precond=precond,
                            est=est, est_mode=est_mode)
    try:
        return solver.run()
    finally:
        # results never alias the pooled buffers (finalisation writes fresh
        # blocks), so the workspace -- and its captured graphs -- can serve
        # the next solve of the same shape
        _release_workspace(solver._ws)
        solver._ws = None

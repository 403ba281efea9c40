"""PHSVDS two-stage driver on device (Algorithm 1 of arXiv:1607.01404).

Mirrors pkg/src/itersvd/hybrid.py:465-631 (``svds_solve``) and its helpers:
stage 1 is GD+k on C = A^T A (or A A^T), its triplets are post-processed
and certified with the two-sided residual (Eq. 7); only the uncertified
ones seed stage 2 on B = [0 A^T; A 0] with refined extraction at shifts
just below each value.  Every vector lives on the GPU; the host sees the
scalars the algorithm branches on.
"""

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from .device import DTYPE
from .eigensolver import (EXTRACT_REFINED, EXTRACT_RR, PRACTICAL_FLOOR_FACTOR, TARGET_CLOSEST_GEQ,
                          TARGET_LARGEST, TARGET_SMALLEST, EigConfig, eig_solve)
from .operators import (NormEstimate, SvdOperator, make_augmented_operator, make_normal_operator,
                        select_preconditioner)

EPS = 2.220446049250313e-16
TARGETS = ("largest", "smallest", "closest")
METHODS = ("hybrid", "normal", "augmented")
_BASIS_SMALL = (15, 6)   # hybrid.py:43
_BASIS_LARGE = (35, 14)  # hybrid.py:44


@dataclass
class SvdsConfig:
    """Parameters of svds_solve (hybrid.py:47-117), same fields."""

    num_svals: int = 1
    target: str = "largest"
    target_values: tuple = ()
    eps: float = 1e-12
    max_basis_size: int = None
    min_restart_size: int = None
    max_block_size: int = 1
    method: str = "hybrid"
    a_norm: float = None
    max_matvecs: int = None
    initial_left: np.ndarray = None
    initial_right: np.ndarray = None
    ortho_left: np.ndarray = None
    ortho_right: np.ndarray = None
    seed: int = 0
    stage1_opts: dict = None
    stage2_opts: dict = None

    def resolved_basis_sizes(self):
        if self.target == "largest" and self.num_svals < 10:
            mbs, mrs = _BASIS_SMALL
        else:
            mbs, mrs = _BASIS_LARGE
        if self.max_basis_size is not None:
            mbs = int(self.max_basis_size)
            mrs = max(1, min(mrs, mbs // 2 - 1))
        if self.min_restart_size is not None:
            mrs = int(self.min_restart_size)
        return mbs, mrs

    def validate(self, m, n):
        if self.num_svals < 0 or self.num_svals > min(m, n):
            raise ValueError("num_svals must lie in [0, min(m, n)]")
        if self.target not in TARGETS:
            raise ValueError("unknown target %r" % (self.target,))
        if self.target == "closest" and not len(self.target_values):
            raise ValueError("closest target needs target_values")
        if self.method not in METHODS:
            raise ValueError("unknown method %r" % (self.method,))
        if not EPS <= self.eps < 1.0:
            raise ValueError("eps must lie in [%g, 1)" % EPS)
        if self.a_norm is not None and self.a_norm <= 0:
            raise ValueError("a_norm must be positive when given")
        mbs, mrs = self.resolved_basis_sizes()
        if self.num_svals > max(mbs - 2, 0) and self.num_svals < min(m, n):
            raise ValueError("num_svals needs a larger max_basis_size")
        have_l = self.ortho_left is not None and self.ortho_left.shape[1] > 0
        have_r = self.ortho_right is not None and self.ortho_right.shape[1] > 0
        if have_l != have_r or (have_l and self.ortho_left.shape[1] != self.ortho_right.shape[1]):
            raise ValueError("ortho_left/ortho_right must pair up")


@dataclass
class SvdsStats:
    stage1_matvecs: int = 0
    stage2_matvecs: int = 0
    precond_applies: int = 0
    restarts: int = 0
    resets: int = 0
    seconds: float = 0.0
    outer_iterations: int = 0
    syncs: int = 0
    graphs_captured: int = 0
    inner_iterations: int = 0


@dataclass
class SvdsResult:
    """Triplets in target order (hybrid.py:130-150).  ``u``/``v`` are host
    F-ordered arrays unless svds_solve(..., return_device=True), in which
    case they are column-major device blocks."""

    sigma: np.ndarray
    u: object
    v: object
    rnorms: np.ndarray
    converged: np.ndarray
    stats: SvdsStats
    status: str = "ok"
    stage1_rnorms: np.ndarray = None

    @property
    def converged_count(self):
        return int(self.converged.sum())


@dataclass
class StageBridge:
    """hybrid.py:153-168; ``guesses`` is a device block (n+m) x k."""

    sigma_tilde: np.ndarray
    rc_norms: np.ndarray
    guesses: object
    tiny: np.ndarray
    shifts: np.ndarray = None
    order: np.ndarray = None


@dataclass
class _Provisional:
    sigma: np.ndarray
    u: object
    v: object
    r7: np.ndarray
    conv: np.ndarray

    def permute(self, order):
        idx = torch.as_tensor(np.asarray(order), dtype=torch.long, device=self.u.device)
        self.sigma = self.sigma[order]
        self.u = _colsel(self.u, idx)
        self.v = _colsel(self.v, idx)
        self.r7 = self.r7[order]
        self.conv = self.conv[order]


def _colsel(block, idx):
    if not block.is_cuda:  # host-side bookkeeping tests only permute columns
        return block.index_select(1, idx.to(block.device))
    out = dv.new_block(block.shape[0], int(idx.numel()), device=block.device, zero=False)
    if idx.numel():
        out.copy_(block.index_select(1, idx))
    return out


# ------------------------------------------------------- convergence tests

class Stage1Test:
    """||r_C|| <= max(sqrt(|lam| ||C||) delta, eps ||C||) (hybrid.py:214-223,
    Alg. 1 line 2)."""

    split_n = None

    def __init__(self, delta):
        self.delta = float(delta)

    def evaluate(self, cand, op_norm):
        return cand.rnorm <= max(np.sqrt(abs(cand.lam) * op_norm) * self.delta, EPS * op_norm)

    def threshold(self, lam, op_norm):
        return max(np.sqrt(abs(lam) * op_norm) * self.delta, EPS * op_norm)

    def __call__(self, lam, rnorm, x, opx, op_norm):
        return rnorm <= max(np.sqrt(abs(lam) * op_norm) * self.delta, EPS * op_norm)


class Stage2Test:
    """Two-level stage-2 acceptance (hybrid.py:408-411 + :226-241): the
    eigenresidual test, then Eq. (7) on the normalised halves, evaluated from
    device split statistics."""

    def __init__(self, n, delta):
        self.split_n = int(n)
        self.delta = float(delta)

    def threshold(self, lam, op_norm):
        return np.sqrt(2.0) * op_norm * self.delta

    def evaluate(self, cand, op_norm):
        if not cand.rnorm < np.sqrt(2.0) * op_norm * self.delta:
            return False
        if cand.nv == 0.0 or cand.nu == 0.0:
            return False
        return bool(cand.r7 < op_norm * self.delta)


class Stage2Practical:
    """Practical floor with the null-space guard (hybrid.py:413-423)."""

    def __init__(self, n):
        self.split_n = int(n)

    def evaluate(self, cand, op_norm):
        if not (op_norm > 0.0 and cand.rnorm <= PRACTICAL_FLOOR_FACTOR * EPS * op_norm):
            return False
        if cand.nv == 0.0 or cand.nu == 0.0:
            return False
        return min(cand.nv, cand.nu) >= 0.1 * max(cand.nv, cand.nu)


def stage1_convergence_test(lam, rnorm, est, delta):
    """hybrid.py:214-223."""
    c = est.c_norm
    return rnorm <= max(np.sqrt(abs(lam) * c) * delta, EPS * c)


# ------------------------------------------------------------- utilities

def _comm(op):
    from .dist import LOCAL
    return getattr(op, "comm", LOCAL)


def _red(op, *tensors):
    c = _comm(op)
    if c.distributed:
        for t in tensors:
            c.allreduce_(t)


def _local_n(op):
    return getattr(op, "n_loc", op.n)


def _local_m(op):
    return getattr(op, "m_loc", op.m)


def orient_problem(a):
    """Rows >= cols; hybrid.py:197-203."""
    from .dist import DistSvdOperator
    if isinstance(a, DistSvdOperator):
        return a, False   # sharded operators are built oriented
    a = SvdOperator.wrap(a)
    if a.m < a.n:
        return a.transposed(), True
    return a, False


def _dev(x):
    if isinstance(x, torch.Tensor):
        return dv.as_block(x) if x.dim() == 2 else x.unsqueeze(1)
    return dv.to_device_block(x)


def _svd_residual_block(ctx, a, sigma_d, u, v):
    """r7^2 per column: ||A v - s u||^2 + ||A^T u - s v||^2 (2 matvecs per
    column, hybrid.py:206-211) -> device vector."""
    k = u.shape[1]
    ml, nl = _local_m(a), _local_n(a)
    av = dv.new_block(ml, k, zero=False)
    atu = dv.new_block(nl, k, zero=False)
    a.apply_into(v, av)
    a.apply_t_into(u, atu)
    eye = dv.small_matrix(k, k)
    eye.copy_(torch.eye(k, dtype=DTYPE))
    r1 = dv.new_block(ml, k, zero=False)
    r2 = dv.new_block(nl, k, zero=False)
    n1 = torch.zeros(k, dtype=DTYPE, device=ctx.device)
    n2 = torch.zeros(k, dtype=DTYPE, device=ctx.device)
    dv.ritz_residual(ctx, u, av, eye, sigma_d, r1, rn2=n1)
    dv.ritz_residual(ctx, v, atu, eye, sigma_d, r2, rn2=n2)
    _red(a, n1, n2)
    return n1, n2


def compute_svd_residual(a, sigma, u, v):
    """Two-sided residual sqrt(||A v - s u||^2 + ||A^T u - s v||^2)
    (hybrid.py:206-211) on device."""
    ctx = dv.context()
    ub, vb = _dev(u), _dev(v)
    s = torch.full((1,), float(sigma), dtype=DTYPE, device=ctx.device)
    n1, n2 = _svd_residual_block(ctx, a, s, ub, vb)
    h1, h2 = dv.fetch(ctx, [n1, n2])
    return float(np.sqrt(h1[0] + h2[0]))


def stage1_postprocess(eig, a, est, k=None, rng=None):
    """Provisional triplets and bridge data from stage-1 pairs
    (hybrid.py:268-337), as block operations on device."""
    ctx = dv.context()
    if rng is None:
        rng = np.random.default_rng(0)
    m, n = a.m, a.n
    ml, nl = _local_m(a), _local_n(a)
    comm = _comm(a)
    m_slice = getattr(a, "m_slice", lambda full: full)
    n_slice = getattr(a, "n_slice", lambda full: full)
    got = eig.eigenvalues.shape[0]
    if k is None:
        k = got
    t = min(got, k)
    sigma = np.zeros(k)
    u = dv.new_block(ml, k)
    v = dv.new_block(nl, k)
    rc = np.full(k, np.inf)
    r7 = np.full(k, np.inf)
    tiny = np.zeros(k, dtype=bool)
    conv = np.zeros(k, dtype=bool)
    floor = est.a_norm * EPS * max(m, n)
    if t:
        x = eig.eigenvectors[:, :t]
        nrm = torch.zeros(t, dtype=DTYPE, device=ctx.device)
        dv.col_norms2(ctx, x, nrm)
        _red(a, nrm)
        dv.scale_cols(ctx, x, nrm, dv.SCALE_DIV_SQRT, v[:, :t])
        lam = eig.eigenvalues[:t]
        sig = np.sqrt(np.maximum(lam, 0.0))
        av = dv.new_block(ml, t, zero=False)
        a.apply_into(v[:, :t], av)
        nav_d = torch.zeros(t, dtype=DTYPE, device=ctx.device)
        dv.col_norms2(ctx, av, nav_d)
        _red(a, nav_d)
        nav = np.sqrt(dv.fetch(ctx, [nav_d])[0])
        dv.scale_cols(ctx, av, nav_d, dv.SCALE_DIV_SQRT, u[:, :t])
        for i in range(t):
            if sig[i] < floor:
                tiny[i] = True
                sigma[i] = 0.0
                if not nav[i] > 0.0:
                    u[:, i].copy_(torch.from_numpy(np.ascontiguousarray(m_slice(rng.standard_normal(m)))))
                    from .eigensolver import Orthonormalizer
                    Orthonormalizer(ctx, comm, m, m_slice)(u[:, :i + 1], start_col=i, rng=rng)
            else:
                sigma[i] = sig[i]
        sig_d = torch.as_tensor(sigma[:t], dtype=DTYPE, device=ctx.device)
        atu = dv.new_block(nl, t, zero=False)
        a.apply_t_into(u[:, :t], atu)
        eye = dv.small_matrix(t, t)
        eye.copy_(torch.eye(t, dtype=DTYPE))
        r1 = dv.new_block(ml, t, zero=False)
        r2 = dv.new_block(nl, t, zero=False)
        n1 = torch.zeros(t, dtype=DTYPE, device=ctx.device)
        n2 = torch.zeros(t, dtype=DTYPE, device=ctx.device)
        dv.ritz_residual(ctx, u[:, :t], av, eye, sig_d, r1, rn2=n1)
        dv.ritz_residual(ctx, v[:, :t], atu, eye, sig_d, r2, rn2=n2)
        _red(a, n1, n2)
        h1, h2 = dv.fetch(ctx, [n1, n2])
        r7[:t] = np.sqrt(h1 + h2)
        rc[:t] = eig.residual_norms[:t]
        conv[:t] = eig.converged[:t]
    if t < k:
        from .eigensolver import Orthonormalizer
        orth_v = Orthonormalizer(ctx, comm, n, n_slice)
        orth_u = Orthonormalizer(ctx, comm, m, m_slice)
        for i in range(t, k):
            v[:, i].copy_(torch.from_numpy(np.ascontiguousarray(n_slice(rng.standard_normal(n)))))
            u[:, i].copy_(torch.from_numpy(np.ascontiguousarray(m_slice(rng.standard_normal(m)))))
            orth_v(v[:, :i + 1], start_col=i, rng=rng)
            orth_u(u[:, :i + 1], start_col=i, rng=rng)
    guesses = dv.new_block(nl + ml, k)
    s2 = 1.0 / np.sqrt(2.0)
    dv.axpby(ctx, s2, v, 0.0, guesses[:nl, :])
    dv.axpby(ctx, s2, u, 0.0, guesses[nl:, :])
    bridge = StageBridge(sigma_tilde=sigma.copy(), rc_norms=rc, guesses=guesses, tiny=tiny)
    prov = _Provisional(sigma=sigma, u=u, v=v, r7=r7, conv=conv)
    return bridge, prov


def stage2_shifts(bridge, est):
    """Interior shifts sigma - sqrt(2) rc / sigma, floored, sorted stably
    (hybrid.py:340-364)."""
    k = bridge.sigma_tilde.shape[0]
    floor = est.a_norm * EPS
    shifts = np.full(k, floor)
    for i in range(k):
        sig = bridge.sigma_tilde[i]
        rc = bridge.rc_norms[i]
        if bridge.tiny[i] or sig <= 0.0 or not np.isfinite(rc):
            continue
        shifts[i] = max(sig - np.sqrt(2.0) * rc / sig, floor)
    order = np.argsort(shifts, kind="stable")
    bridge.shifts = shifts[order]
    bridge.order = order
    bridge.sigma_tilde = bridge.sigma_tilde[order]
    bridge.rc_norms = bridge.rc_norms[order]
    idx = torch.as_tensor(order, dtype=torch.long, device=bridge.guesses.device)
    bridge.guesses = _colsel(bridge.guesses, idx)
    bridge.tiny = bridge.tiny[order]
    return bridge.shifts


def _random_bridge(op, k, rng):
    """hybrid.py:367-373."""
    from .eigensolver import Orthonormalizer
    m, n = op.m, op.n
    nl, ml = _local_n(op), _local_m(op)
    draw = rng.standard_normal((n + m, k))
    if _comm(op).distributed:
        draw = np.concatenate([draw[op.c0:op.c1], draw[n + op.r0:n + op.r1]], axis=0)

        def sl(full):
            return np.concatenate([full[op.c0:op.c1], full[n + op.r0:n + op.r1]], axis=0)
    else:
        sl = None
    guesses = dv.new_block(nl + ml, k)
    guesses.copy_(torch.from_numpy(np.ascontiguousarray(draw)))
    Orthonormalizer(dv.context(), _comm(op), n + m, sl)(guesses, rng=rng)
    return StageBridge(sigma_tilde=np.zeros(k), rc_norms=np.full(k, np.inf), guesses=guesses,
                       tiny=np.zeros(k, dtype=bool))


def _eig_overrides(cfg_eig, opts):
    for key, value in (opts or {}).items():
        if not hasattr(cfg_eig, key):
            raise ValueError("unknown eigensolver option %r" % (key,))
        setattr(cfg_eig, key, value)
    return cfg_eig


def _stage1_eig_config(cfg, delta, mbs, mrs, budget_ops):
    """hybrid.py:384-404."""
    if cfg.target == "closest":
        shifts = tuple(sorted(float(s) ** 2 for s in cfg.target_values))
        target, locking, extraction = TARGET_CLOSEST_GEQ, True, EXTRACT_REFINED
    elif cfg.target == "smallest":
        shifts, target, locking, extraction = (), TARGET_SMALLEST, False, EXTRACT_RR
    else:
        shifts, target, locking, extraction = (), TARGET_LARGEST, False, EXTRACT_RR
    e = EigConfig(num_evals=cfg.num_svals, target=target, shifts=shifts, max_basis_size=mbs,
                  min_restart_size=mrs, plus_k=1, max_block_size=cfg.max_block_size, locking=locking,
                  extraction=extraction, convergence_test=Stage1Test(delta), max_matvecs=budget_ops,
                  seed=cfg.seed)
    return _eig_overrides(e, cfg.stage1_opts)


def _stage2_eig_config(cfg, delta, n, mbs, mrs, num, shifts, budget_ops):
    """hybrid.py:407-440."""
    test = Stage2Test(n, delta)
    practical = Stage2Practical(n)
    if cfg.target == "largest":
        e = EigConfig(num_evals=num, target=TARGET_LARGEST, max_basis_size=mbs, min_restart_size=mrs,
                      plus_k=1, max_block_size=cfg.max_block_size, locking=False, extraction=EXTRACT_RR,
                      convergence_test=test, practical_test=practical, max_matvecs=budget_ops,
                      deactivate_krylov_init=True, seed=cfg.seed + 1)
    else:
        e = EigConfig(num_evals=num, target=TARGET_CLOSEST_GEQ, shifts=tuple(shifts), max_basis_size=mbs,
                      min_restart_size=mrs, plus_k=1, max_block_size=cfg.max_block_size, locking=True,
                      extraction=EXTRACT_REFINED, convergence_test=test, practical_test=practical,
                      max_matvecs=budget_ops, deactivate_krylov_init=True, seed=cfg.seed + 1)
    return _eig_overrides(e, cfg.stage2_opts)


def _final_order(cfg, sigma):
    if cfg.target == "largest":
        return np.argsort(-sigma, kind="stable")
    return np.argsort(sigma, kind="stable")


def _status_merge(statuses, all_conv):
    if all_conv:
        return "ok"
    for s in ("budget", "stagnated"):
        if s in statuses:
            return s
    return "ok"


def _stack_pairs(ctx, vs, us):
    """[v; u] / sqrt(2) columns (hybrid.py:263-265)."""
    k = vs.shape[1]
    out = dv.new_block(vs.shape[0] + us.shape[0], k)
    s2 = 1.0 / np.sqrt(2.0)
    dv.axpby(ctx, s2, vs, 0.0, out[:vs.shape[0], :])
    dv.axpby(ctx, s2, us, 0.0, out[vs.shape[0]:, :])
    return out


def _add_stats(stats, r):
    stats.restarts += r.stats.restarts
    stats.resets += r.stats.resets
    stats.outer_iterations += r.stats.outer_iterations
    stats.syncs += r.stats.syncs
    stats.graphs_captured += r.stats.graphs_captured
    stats.inner_iterations += r.stats.inner_iterations


def svds_solve(a, precond=None, cfg=None, return_device=False):
    """Compute cfg.num_svals singular triplets of ``a`` (hybrid.py:465-631).

    ``a``: SvdOperator, SparseMatrixCsr or dense array.  Returns an
    SvdsResult whose ``u``/``v`` are F-ordered numpy arrays (the
    reference's contract) or device blocks with ``return_device=True``.
    """
    t0 = time.perf_counter()
    cfg = cfg if cfg is not None else SvdsConfig()
    from .dist import DistSvdOperator
    if not isinstance(a, DistSvdOperator):
        a = SvdOperator.wrap(a)
    cfg.validate(a.m, a.n)
    ctx = dv.context()
    stats = SvdsStats()
    k = cfg.num_svals
    if k == 0:
        stats.seconds = time.perf_counter() - t0
        u0, v0 = dv.new_block(a.m, 0), dv.new_block(a.n, 0)
        if not return_device:
            u0, v0 = dv.to_host(u0), dv.to_host(v0)
        return SvdsResult(sigma=np.zeros(0), u=u0, v=v0, rnorms=np.zeros(0),
                          converged=np.zeros(0, dtype=bool), stats=stats, status="ok",
                          stage1_rnorms=np.zeros(0))

    op, swapped = orient_problem(a)
    m, n = op.m, op.n
    nl, ml = _local_n(op), _local_m(op)
    comm = _comm(op)

    def _dev_n(x):  # host guesses / constraints of global length -> local rows
        if isinstance(x, torch.Tensor):
            return _dev(x)
        return _dev(getattr(op, "n_slice", lambda f: f)(np.asarray(x, dtype=np.float64)))

    def _dev_m(x):
        if isinstance(x, torch.Tensor):
            return _dev(x)
        return _dev(getattr(op, "m_slice", lambda f: f)(np.asarray(x, dtype=np.float64)))
    delta = float(cfg.eps)
    est = NormEstimate(cfg.a_norm)
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 0x5fd]))
    mbs, mrs = cfg.resolved_basis_sizes()

    left_g, right_g = cfg.initial_left, cfg.initial_right
    ortho_l, ortho_r = cfg.ortho_left, cfg.ortho_right
    if swapped:
        left_g, right_g = right_g, left_g
        ortho_l, ortho_r = ortho_r, ortho_l

    budget = cfg.max_matvecs
    mv0 = op.n_matvecs

    def ops_left():
        if budget is None:
            return None
        return max((budget - (op.n_matvecs - mv0)) // 2, 0)

    statuses = []
    # ---------------------------------------------------------- stage 1
    if cfg.method in ("hybrid", "normal"):
        c_op = make_normal_operator(op)
        e1 = _stage1_eig_config(cfg, delta, mbs, mrs, ops_left())
        pre1 = select_preconditioner(precond, "AAt" if swapped else "AtA")
        pre1_before = pre1.n_applies if pre1 is not None else 0
        guess = _dev_n(right_g) if right_g is not None else None
        ortho = _dev_n(ortho_r) if ortho_r is not None else None
        r1 = eig_solve(c_op, e1, guesses=guess, ortho_constraints=ortho, precond=pre1, est=est,
                       est_mode="normal")
        statuses.append(r1.status)
        _add_stats(stats, r1)
        if pre1 is not None:
            stats.precond_applies += pre1.n_applies - pre1_before
        bridge, prov = stage1_postprocess(r1, op, est, k=k, rng=rng)
    else:
        bridge = _random_bridge(op, k, rng)
        prov = _Provisional(sigma=np.zeros(k), u=dv.new_block(ml, k), v=dv.new_block(nl, k),
                            r7=np.full(k, np.inf), conv=np.zeros(k, dtype=bool))
    stats.stage1_matvecs = op.n_matvecs - mv0

    a_norm = est.a_norm
    passed = prov.r7 < a_norm * delta
    run_stage2 = cfg.method == "augmented" or (cfg.method == "hybrid" and not passed.all())

    # ---------------------------------------------------------- stage 2
    mv1 = op.n_matvecs
    if run_stage2:
        if cfg.target != "largest":
            stage2_shifts(bridge, est)
            prov.permute(bridge.order)
            passed = passed[bridge.order]
        active = np.flatnonzero(~bridge.tiny & ~passed)
        if active.size:
            b_op = make_augmented_operator(op)
            pre2 = select_preconditioner(precond, "augmented")
            pre2_before = pre2.n_applies if pre2 is not None else 0
            frozen = []
            if ortho_l is not None and ortho_l.shape[1] > 0:
                frozen.append(_stack_pairs(ctx, _dev_n(ortho_r), _dev_m(ortho_l)))
            fz = np.flatnonzero(bridge.tiny | passed)
            if fz.size:
                frozen.append(_colsel(bridge.guesses, torch.as_tensor(fz, device=ctx.device)))
            ortho_b = None
            if frozen:
                tot = sum(f.shape[1] for f in frozen)
                ortho_b = dv.new_block(nl + ml, tot)
                c0 = 0
                for f in frozen:
                    ortho_b[:, c0:c0 + f.shape[1]].copy_(f)
                    c0 += f.shape[1]
            shifts2 = bridge.shifts[active] if bridge.shifts is not None else ()
            e2 = _stage2_eig_config(cfg, delta, nl, mbs, mrs, active.size, shifts2, ops_left())
            guesses2 = _colsel(bridge.guesses, torch.as_tensor(active, device=ctx.device))
            r2 = eig_solve(b_op, e2, guesses=guesses2, ortho_constraints=ortho_b, precond=pre2, est=est,
                           est_mode="augmented")
            statuses.append(r2.status)
            _add_stats(stats, r2)
            if pre2 is not None:
                stats.precond_applies += pre2.n_applies - pre2_before
            a_norm = est.a_norm
            got = r2.eigenvalues.shape[0]
            nj = min(got, active.size)
            if nj:
                x = r2.eigenvectors[:, :nj]
                nvd = torch.zeros(nj, dtype=DTYPE, device=ctx.device)
                nud = torch.zeros(nj, dtype=DTYPE, device=ctx.device)
                dv.col_norms2(ctx, x[:nl, :], nvd)
                dv.col_norms2(ctx, x[nl:, :], nud)
                _red(op, nvd, nud)
                nv2, nu2 = dv.fetch(ctx, [nvd, nud])
                keep = [j for j in range(nj) if nv2[j] > 0.0 and nu2[j] > 0.0]
                for j in keep:
                    slot = active[j]
                    prov.sigma[slot] = abs(float(r2.eigenvalues[j]))
                    dv.scale_cols(ctx, x[:nl, j:j + 1], nvd[j:j + 1], dv.SCALE_DIV_SQRT,
                                  prov.v[:, slot:slot + 1])
                    dv.scale_cols(ctx, x[nl:, j:j + 1], nud[j:j + 1], dv.SCALE_DIV_SQRT,
                                  prov.u[:, slot:slot + 1])
                if keep:
                    slots = torch.as_tensor(active[keep], dtype=torch.long, device=ctx.device)
                    us = _colsel(prov.u, slots)
                    vs = _colsel(prov.v, slots)
                    sd = torch.as_tensor(prov.sigma[active[keep]], dtype=DTYPE, device=ctx.device)
                    n1, n2 = _svd_residual_block(ctx, op, sd, us, vs)
                    h1, h2 = dv.fetch(ctx, [n1, n2])
                    prov.r7[active[keep]] = np.sqrt(h1 + h2)
    stats.stage2_matvecs = op.n_matvecs - mv1

    # --------------------------------------------------------- assemble
    stage1_r7 = prov.r7.copy() if not run_stage2 else None
    conv = prov.r7 < a_norm * delta
    order = _final_order(cfg, prov.sigma)
    sigma = prov.sigma[order]
    idx = torch.as_tensor(order, dtype=torch.long, device=ctx.device)
    u = _colsel(prov.u, idx)
    v = _colsel(prov.v, idx)
    rnorms = prov.r7[order]
    conv = conv[order]
    if run_stage2:
        if cfg.method == "augmented":
            stage1_r7 = np.full(k, np.nan)
        else:
            stage1_r7_full = np.where(bridge.tiny | passed, prov.r7, np.inf)
            for i in np.flatnonzero(~bridge.tiny & ~passed):
                sig = bridge.sigma_tilde[i]
                if sig > 0 and np.isfinite(bridge.rc_norms[i]):
                    stage1_r7_full[i] = bridge.rc_norms[i] / sig
            stage1_r7 = stage1_r7_full
        stage1_r7 = stage1_r7[order]
    else:
        stage1_r7 = stage1_r7[order]
    if swapped:
        u, v = v, u
    if not return_device:
        u, v = dv.to_host(u), dv.to_host(v)
        if comm.distributed:
            # local row chunks, rank order == row order
            u = np.asfortranarray(comm.allgather_host(np.ascontiguousarray(u)))
            v = np.asfortranarray(comm.allgather_host(np.ascontiguousarray(v)))
    else:
        torch.cuda.current_stream(ctx.device).synchronize()
    stats.seconds = time.perf_counter() - t0
    return SvdsResult(sigma=sigma, u=u, v=v, rnorms=rnorms, converged=conv, stats=stats,
                      status=_status_merge(statuses, bool(conv.all())), stage1_rnorms=stage1_r7)


# ------------------------------------------------- condition-number mode

@dataclass
class CondResult:
    """hybrid.py:187-194."""

    kappa: float
    sigma_max: float
    sigma_min: float
    infinite: bool
    lower_bound: bool
    stats: SvdsStats


class _RelativeTest:
    """||r_C|| <= rel_tol |lam| (the loose rule of hybrid.py:667-668)."""

    split_n = None

    def __init__(self, rel_tol):
        self.rel_tol = float(rel_tol)

    def evaluate(self, cand, op_norm):
        return cand.rnorm <= abs(cand.lam) * self.rel_tol

    def threshold(self, lam, op_norm):
        return abs(lam) * self.rel_tol

    def __call__(self, lam, rnorm, x, opx, op_norm):
        return rnorm <= abs(lam) * self.rel_tol


def estimate_condition_number(a, precond=None, cfg=None, rel_tol=0.1):
    """sigma_max / sigma_min from two loose one-pair GD+k solves on the
    normal operator, largest then smallest (hybrid.py:634-701).  A smallest
    squared value at or below ||C|| eps max(m, n) reports kappa = inf; a
    smallest solve cut off by the budget marks the estimate a lower bound."""
    t0 = time.perf_counter()
    cfg = cfg if cfg is not None else SvdsConfig()
    from .dist import DistSvdOperator
    if not isinstance(a, DistSvdOperator):
        a = SvdOperator.wrap(a)
    if not 0.0 < rel_tol < 1.0:
        raise ValueError("rel_tol must lie in (0, 1)")
    stats = SvdsStats()
    op, swapped = orient_problem(a)
    est = NormEstimate(cfg.a_norm)
    c_op = make_normal_operator(op)
    pre = select_preconditioner(precond, "AAt" if swapped else "AtA")
    budget = cfg.max_matvecs
    mv0 = op.n_matvecs

    def ops_left():
        if budget is None:
            return None
        return max((budget - (op.n_matvecs - mv0)) // 2, 0)

    test = _RelativeTest(rel_tol)

    def one(target, seed, mbs, mrs):
        e = EigConfig(num_evals=1, target=target, max_basis_size=mbs, min_restart_size=mrs, plus_k=1,
                      max_block_size=1, convergence_test=test, max_matvecs=ops_left(), seed=seed)
        return eig_solve(c_op, e, precond=pre, est=est, est_mode="normal")

    pre_before = pre.n_applies if pre is not None else 0
    r_hi = one(TARGET_LARGEST, cfg.seed, *_BASIS_SMALL)
    stats.stage1_matvecs = op.n_matvecs - mv0
    mv1 = op.n_matvecs
    r_lo = one(TARGET_SMALLEST, cfg.seed + 1, *_BASIS_LARGE)
    stats.stage2_matvecs = op.n_matvecs - mv1
    stats.restarts = r_hi.stats.restarts + r_lo.stats.restarts
    stats.resets = r_hi.stats.resets + r_lo.stats.resets
    if pre is not None:
        stats.precond_applies = pre.n_applies - pre_before
    sigma_max = float(np.sqrt(max(r_hi.eigenvalues[0], 0.0))) if r_hi.eigenvalues.size else 0.0
    lam_min = float(r_lo.eigenvalues[0]) if r_lo.eigenvalues.size else 0.0
    sigma_min = float(np.sqrt(max(lam_min, 0.0)))
    infinite = lam_min <= est.c_norm * EPS * max(op.m, op.n)
    lower_bound = (not infinite) and (r_lo.status != "ok" or not bool(np.all(r_lo.converged)))
    kappa = np.inf if infinite else sigma_max / sigma_min
    stats.seconds = time.perf_counter() - t0
    return CondResult(kappa=kappa, sigma_max=sigma_max, sigma_min=sigma_min, infinite=infinite,
                      lower_bound=lower_bound, stats=stats)


def stage2_convergence_test(lam, x, a, est, delta):
    """Two-level stage-2 acceptance on the stacked vector x = [v; u]
    (hybrid.py:244-260): the eigenresidual test, then Eq. (7) on the
    normalised halves; a zero-norm half is rejected.  ``x`` may be a host
    array or a device vector; the two products run on device (counted)."""
    a = SvdOperator.wrap(a)
    n = a.n
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64).copy())
    xt = xt.to(device=dv.context().device, dtype=DTYPE).reshape(-1)
    xv, xu = xt[:n].contiguous(), xt[n:].contiguous()
    av = a.apply(xv).reshape(-1)
    atu = a.apply_t(xu).reshape(-1)
    lam = float(lam)
    rnorm = float(torch.sqrt(torch.sum((atu - lam * xv) ** 2) + torch.sum((av - lam * xu) ** 2)))
    a_norm = est.a_norm
    if not rnorm < np.sqrt(2.0) * a_norm * delta:
        return False
    nv, nu = float(torch.linalg.vector_norm(xv)), float(torch.linalg.vector_norm(xu))
    if nv == 0.0 or nu == 0.0:
        return False
    sigma = abs(lam)
    r7 = np.sqrt(float(torch.sum((av / nv - sigma * xu / nu) ** 2)) +
                 float(torch.sum((atu / nu - sigma * xv / nv) ** 2)))
    return bool(r7 < a_norm * delta)

"""TEST INFRASTRUCTURE ONLY.  CPU restatement (numpy) of the reference's
PHSVDS solve path -- the oracle the GPU build is checked against and the
CPU baseline bench.py times (``cpu_baseline.kind = "port"``).

Restates, in a functional layout of its own:
  * block SpMV and the normal / augmented operators
        pkg/src/itersvd/matio.py:126-155, operators.py:163-190
  * iterated CGS orthonormalisation, QR append / restart
        kernels.py:54-133, :160-252
  * the GD+k Davidson iteration (thick restart, +k, RR / refined
    extraction, soft / hard locking, reset, practical floor, stagnation,
    budget)  eigensolver.py:157-821
  * the two-stage driver  hybrid.py:214-631
using the same numpy operations in the same order, so its results track
the reference to rounding (pinned by tests/test_oracle.py against
tests/golden/solves.json, produced by the reference itself).

Nothing in paper_1607_01404_b200 imports this module.
"""

import time

import numpy as np

from . import csr as ocsr

EPS = 2.220446049250313e-16
REORTH = 1.0 / np.sqrt(2.0)
DEFICIENT = 1e-14
PASSES = 6
RETRIES = 20
FLOOR_FACTOR = 10.0
IMPROVE = 0.999


# ------------------------------------------------------------------ matrix

class Csr:
    """Host CSR with a matvec counter (SvdOperator.from_csr semantics)."""

    def __init__(self, m, n, row_ptr, col_idx, values):
        self.m, self.n = int(m), int(n)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)
        self._rows = None
        self.count = 0

    def rows(self):
        if self._rows is None:
            self._rows = np.repeat(np.arange(self.m, dtype=np.int64), np.diff(self.row_ptr))
        return self._rows

    def fwd(self, x):
        """A x for a (n, b) block (matio.py:141-149 order)."""
        y = np.zeros((self.m, x.shape[1]), order="F")
        if self.values.size:
            prod = self.values[:, None] * x[self.col_idx, :]
            live = np.flatnonzero(np.diff(self.row_ptr) > 0)
            if live.size:
                y[live, :] = np.add.reduceat(prod, self.row_ptr[live], axis=0)[:, :]
        return y

    def adj(self, y):
        """A^T y (matio.py:150-154 order)."""
        z = np.zeros((self.n, y.shape[1]), order="F")
        if self.values.size:
            np.add.at(z, self.col_idx, self.values[:, None] * y[self.rows(), :])
        return z


class View:
    """Counting view of a matrix, possibly transposed (operators.py:117-160)."""

    def __init__(self, mat, flipped=False):
        self.mat, self.flipped = mat, flipped
        self.m, self.n = (mat.n, mat.m) if flipped else (mat.m, mat.n)

    @property
    def count(self):
        return self.mat.count

    def mul(self, x):
        x = np.asarray(x, dtype=np.float64)
        one = x.ndim == 1
        xb = x[:, None] if one else x
        self.mat.count += xb.shape[1]
        y = self.mat.adj(xb) if self.flipped else self.mat.fwd(xb)
        return y[:, 0] if one else y

    def tmul(self, y):
        y = np.asarray(y, dtype=np.float64)
        one = y.ndim == 1
        yb = y[:, None] if one else y
        self.mat.count += yb.shape[1]
        x = self.mat.fwd(yb) if self.flipped else self.mat.adj(yb)
        return x[:, 0] if one else x


class SymOp:
    """Square operator; apply() counts columns (operators.py:28-47)."""

    def __init__(self, dim, fn):
        self.dim, self.fn, self.applied = int(dim), fn, 0

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        one = x.ndim == 1
        xb = x[:, None] if one else x
        self.applied += xb.shape[1]
        y = self.fn(xb)
        return y[:, 0] if one else y


def normal_op(v):
    if v.m >= v.n:
        return SymOp(v.n, lambda x: v.tmul(v.mul(x)))
    return SymOp(v.m, lambda x: v.mul(v.tmul(x)))


def augmented_op(v):
    n, m = v.n, v.m

    def fn(x):
        out = np.zeros((n + m, x.shape[1]), order="F")
        out[:n, :] = v.tmul(x[n:, :])
        out[n:, :] = v.mul(x[:n, :])
        return out

    return SymOp(n + m, fn)


class Jacobi:
    """Point-Jacobi x ./ d (operators.py:225-249); mode AtA / AAt."""

    def __init__(self, mat, side="cols"):
        if side == "auto":
            side = "cols" if mat.m >= mat.n else "rows"
        self.mode = "AtA" if side == "cols" else "AAt"
        self.d = ocsr.jacobi_diag(mat.m, mat.n, mat.row_ptr, mat.col_idx, mat.values, side=side)
        self.applied = 0

    def __call__(self, x):
        self.applied += x.shape[1]
        return x / self.d[:, None]


# ------------------------------------------------------------ dense kernels

def _block_list(against):
    if against is None:
        return []
    if isinstance(against, (list, tuple)):
        return [b for b in against if b is not None and b.shape[1] > 0]
    return [against] if against.shape[1] > 0 else []


def cgs_orthonormalize(block, against=None, first=0, rng=None):
    """kernels.py:54-133: per column, CGS passes against the prior columns
    with the DGKS 1/sqrt(2) rule; collapsed columns become random draws."""
    rows, cols = block.shape
    ext = _block_list(against)
    if sum(b.shape[1] for b in ext) + cols > rows:
        raise ValueError("more columns than the space can hold")
    rng = np.random.default_rng(0) if rng is None else rng
    swapped = []
    for j in range(first, cols):
        prior = ext + ([block[:, :j]] if j > 0 else [])
        col = block[:, j]
        marked = False
        for _attempt in range(RETRIES):
            start = np.linalg.norm(col)
            done_norm = 0.0
            if start > 0.0:
                last = start
                hits = 0
                for _p in range(PASSES):
                    for b in prior:
                        col -= b @ (b.T @ col)
                    now = np.linalg.norm(col)
                    if now < DEFICIENT * start:
                        hits += 1
                        if hits >= 2:
                            break
                    elif now > REORTH * last:
                        done_norm = now
                        break
                    else:
                        hits = 0
                    last = now
            if done_norm > 0.0:
                col /= done_norm
                break
            if not marked:
                swapped.append(j)
                marked = True
            col[:] = rng.standard_normal(rows)
        else:
            raise np.linalg.LinAlgError("orthonormalize could not produce an independent column")
    return swapped


def qr_extend(q, r, newcol, rng):
    """kernels.py:160-222."""
    rows, g = newcol.shape[0], q.shape[1]
    v = np.array(newcol, dtype=np.float64, copy=True)
    coef = np.zeros(g)
    start = np.linalg.norm(v)
    last = start
    bad = start == 0.0
    hits = 1 if bad else 0
    if not bad:
        for _p in range(PASSES):
            c = q.T @ v
            coef += c
            v -= q @ c
            now = np.linalg.norm(v)
            if now < DEFICIENT * start:
                hits += 1
                if hits >= 2:
                    bad = True
                    break
            elif now > REORTH * last:
                break
            else:
                hits = 0
            last = now
        else:
            bad = True
    q2 = np.empty((rows, g + 1), order="F")
    q2[:, :g] = q
    r2 = np.zeros((g + 1, g + 1))
    r2[:g, :g] = r
    r2[:g, g] = coef
    if bad:
        fill = np.zeros((rows, 1), order="F")
        fill[:, 0] = rng.standard_normal(rows)
        cgs_orthonormalize(fill, against=q, rng=rng)
        q2[:, g] = fill[:, 0]
        r2[g, g] = 0.0
    else:
        nv = np.linalg.norm(v)
        q2[:, g] = v / nv
        r2[g, g] = nv
    return q2, r2


def qr_compress(q, r, y):
    """kernels.py:225-242."""
    qy, ry = np.linalg.qr(r @ y)
    sgn = np.where(np.diag(ry) < 0.0, -1.0, 1.0)
    return np.asfortranarray(q @ (qy * sgn)), ry * sgn[:, None]


# ------------------------------------------------------------ the iteration

LARGEST, SMALLEST, CLOSEST = "largest_algebraic", "smallest_algebraic", "closest_geq"
RR, REFINED = "rayleigh_ritz", "refined_const_shift"


class Opts:
    """EigConfig fields (eigensolver.py:54-80)."""

    def __init__(self, **kw):
        self.num_evals = 1
        self.target = LARGEST
        self.shifts = ()
        self.max_basis_size = 15
        self.min_restart_size = 6
        self.plus_k = 1
        self.max_block_size = 1
        self.locking = False
        self.extraction = RR
        self.convergence_test = None
        self.practical_test = None
        self.max_matvecs = None
        self.deactivate_krylov_init = False
        self.seed = 0
        self.disable_reset = False
        self.stagnation_window = 250
        for k, v in kw.items():
            if not hasattr(self, k):
                raise ValueError("unknown option %r" % k)
            setattr(self, k, v)


class Outcome:
    def __init__(self, vals, vecs, rn, ok, work, status):
        self.eigenvalues, self.eigenvectors = vals, vecs
        self.residual_norms, self.converged = rn, ok
        self.work, self.status = work, status


class Norm:
    """Running ||A||^2 estimate (operators.py:252-292)."""

    def __init__(self, given=None):
        self.given, self.run = given, 0.0

    @property
    def c(self):
        return self.given ** 2 if self.given is not None else self.run

    @property
    def a(self):
        return self.given if self.given is not None else float(np.sqrt(self.run))

    def see(self, vals, augmented=False):
        vals = np.atleast_1d(np.asarray(vals, dtype=np.float64))
        if vals.size:
            top = float(np.abs(vals).max())
            if augmented:
                top = top ** 2
            if top > self.run:
                self.run = top


class GDk:
    """The GD+k loop of eigensolver.py:157-785 as explicit state."""

    def __init__(self, op, o, guesses=None, ortho=None, precond=None, norm=None, augmented=False):
        self.op, self.o, self.pre = op, o, precond
        self.norm = norm if norm is not None else Norm()
        self.aug = augmented
        self.rng = np.random.default_rng(o.seed)
        self.work = {"matvecs": 0, "precond": 0, "restarts": 0, "resets": 0, "iters": 0}
        self.status = "ok"
        self.N = op.dim
        self.ext = []
        if ortho is not None and ortho.shape[1] > 0:
            c = np.asfortranarray(np.array(ortho, dtype=np.float64))
            cgs_orthonormalize(c, rng=self.rng)
            self.ext.append(c)
        n_ext = sum(b.shape[1] for b in self.ext)
        self.n_ext = n_ext
        self.want = max(min(o.num_evals, self.N - n_ext), 0)
        self.dense = self.N <= o.max_basis_size
        self.cap = self.N - n_ext if self.dense else o.max_basis_size
        self.V = np.zeros((self.N, self.cap), order="F")
        self.W = np.zeros((self.N, self.cap), order="F")
        self.H = np.zeros((self.cap, self.cap))
        self.g = 0
        self.lock_v = np.zeros((self.N, 0), order="F")
        self.lock_l, self.lock_r, self.lock_u = [], [], []
        self.Q = self.R = self.tau = None
        self.since_reset = 0
        self.prev = None
        self.prev_g = 0
        self.streak = 0
        self.progress = {}
        self.done = self.want == 0
        if not self.done:
            self._start(guesses)
            if self.g == 0:
                self.done = True
            elif o.extraction == REFINED and not self.dense:
                self._qr_rebuild()

    # plumbing
    def opnorm(self):
        return self.norm.a if self.aug else self.norm.c

    def left(self):
        if self.o.max_matvecs is None:
            return 10 ** 18
        return self.o.max_matvecs - self.work["matvecs"]

    def apply(self, x):
        self.work["matvecs"] += 1 if x.ndim == 1 else x.shape[1]
        return self.op(x)

    def shift(self):
        s = self.o.shifts
        return float(s[min(len(self.lock_l), len(s) - 1)])

    def against(self):
        return list(self.ext) + ([self.lock_v] if self.lock_v.shape[1] else [])

    def order(self, lams):
        if self.o.target == LARGEST:
            return np.argsort(-lams, kind="stable")
        if self.o.target == SMALLEST:
            return np.argsort(lams, kind="stable")
        s = self.shift()
        below = lams < s
        return np.lexsort((np.where(below, s - lams, lams - s), below.astype(np.int64)))

    def user_ok(self, lam, rn, x, ox):
        t = self.o.convergence_test
        if t is None:
            return rn <= max(1e-12 * self.opnorm(), FLOOR_FACTOR * EPS * self.opnorm())
        return bool(t(lam, rn, x, ox, self.opnorm()))

    def floor_ok(self, lam, rn, x, ox):
        if self.o.practical_test is not None:
            return bool(self.o.practical_test(lam, rn, x, ox, self.opnorm()))
        return self.opnorm() > 0.0 and rn <= FLOOR_FACTOR * EPS * self.opnorm()

    def h_full(self):
        g = self.g
        hh = self.V[:, :g].T @ self.W[:, :g]
        self.H[:g, :g] = 0.5 * (hh + hh.T)

    # initial basis (eigensolver.py:278-347)
    def _start(self, guesses):
        o = self.o
        if self.dense:
            k = self.cap
            self.V[:, :k] = self.rng.standard_normal((self.N, k))
            cgs_orthonormalize(self.V[:, :k], against=self.ext, rng=self.rng)
            self.g = k
            take = min(k, max(self.left(), 0))
            if take:
                self.W[:, :take] = self.apply(self.V[:, :take])
            if take < k:
                self.status, self.g = "budget", take
            self.h_full()
            return
        g0 = 0
        if guesses is not None and guesses.shape[1] > 0:
            take = min(guesses.shape[1], self.cap - 1)
            self.V[:, :take] = guesses[:, :take]
            cgs_orthonormalize(self.V[:, :take], against=self.against(), rng=self.rng)
            g0 = take
        if g0 == 0:
            b0 = min(max(o.max_block_size, o.num_evals), self.cap - 1)
            self.V[:, :b0] = self.rng.standard_normal((self.N, b0))
            cgs_orthonormalize(self.V[:, :b0], against=self.against(), rng=self.rng)
            g0 = b0
        goal = g0 if o.deactivate_krylov_init else min(max(o.min_restart_size, g0), self.cap - 1,
                                                       self.N - self.n_ext)
        if g0 > 1:
            take = min(g0 - 1, max(self.left(), 0))
            if take:
                self.W[:, :take] = self.apply(self.V[:, :take])
            if take < g0 - 1:
                self.status, self.g = "budget", take
                self.h_full()
                return
        j = g0 - 1
        while True:
            if self.left() < 1:
                self.status, self.g = "budget", j
                self.h_full()
                return
            wj = self.apply(self.V[:, j])
            self.W[:, j] = wj
            if j + 1 >= goal:
                break
            self.V[:, j + 1] = wj
            cgs_orthonormalize(self.V[:, :j + 2], against=self.against(), first=j + 1, rng=self.rng)
            j += 1
        self.g = goal
        self.h_full()

    def _qr_rebuild(self):
        self.tau = self.shift()
        m = self.W[:, :self.g] - self.tau * self.V[:, :self.g]
        q = np.empty((m.shape[0], 0), order="F")
        r = np.zeros((0, 0))
        for j in range(m.shape[1]):
            q, r = qr_extend(q, r, m[:, j], self.rng)
        self.Q, self.R = q, r

    def rayleigh_ritz(self):
        lams, y = np.linalg.eigh(self.H[:self.g, :self.g])
        idx = self.order(lams)
        return lams[idx], np.asfortranarray(y[:, idx])

    def refined(self):
        _, s, vt = np.linalg.svd(self.R[:self.g, :self.g], full_matrices=False)
        y = vt.T[:, -1]
        return float(y @ (self.H[:self.g, :self.g] @ y)), y

    def residuals(self, lams, y, count):
        t = max(min(count, lams.shape[0]), 0)
        yb = y[:, :t]
        x = np.asfortranarray(self.V[:, :self.g] @ yb)
        ox = np.asfortranarray(self.W[:, :self.g] @ yb)
        res = ox - x * lams[None, :t]
        return x, ox, res, np.linalg.norm(res, axis=0)

    def reset_if_needed(self, rn):
        if self.o.disable_reset:
            return False
        if rn >= np.sqrt(self.since_reset) * self.opnorm() * EPS:
            return False
        g = self.g
        if self.left() < g:
            return False
        cgs_orthonormalize(self.V[:, :g], against=self.against(), rng=self.rng)
        self.W[:, :g] = self.apply(self.V[:, :g])
        self.h_full()
        if self.Q is not None:
            self._qr_rebuild()
        self.since_reset = 0
        self.prev = None
        self.work["resets"] += 1
        return True

    def stale(self, slot, rn, lam):
        rec = self.progress.get(slot)
        if rec is None:
            self.progress[slot] = [rn, 0, lam]
            return 0
        best, cnt, lam0 = rec
        moved = abs(lam - lam0) > 100.0 * EPS * max(abs(lam), abs(lam0))
        if rn < best * IMPROVE or moved:
            self.progress[slot] = [min(rn, best), 0, lam]
            return 0
        rec[1] = cnt + 1
        return cnt + 1

    def coef_select(self, cols, limit, base):
        kept = []
        for col in cols:
            if len(kept) >= limit:
                break
            c = np.array(col, dtype=np.float64, copy=True)
            for _ in range(2):
                for b in base:
                    c -= b * (b @ c)
                for b in kept:
                    c -= b * (b @ c)
            nc = np.linalg.norm(c)
            if nc > 1e-8:
                kept.append(c / nc)
        out = np.zeros((self.g, len(kept)), order="F")
        for i, c in enumerate(kept):
            out[:, i] = c
        return out

    def padded_prev(self):
        if self.prev is None or self.prev_g > self.g:
            return []
        cols = []
        for j in range(self.prev.shape[1]):
            c = np.zeros(self.g)
            c[:self.prev_g] = self.prev[:, j]
            cols.append(c)
        return cols

    def reseed(self):
        self.V[:, 0] = self.rng.standard_normal(self.N)
        cgs_orthonormalize(self.V[:, :1], against=self.against(), rng=self.rng)
        self.g = 1
        if self.left() < 1:
            self.status, self.done = "budget", True
            self.W[:, 0] = 0.0
        else:
            self.W[:, 0] = self.apply(self.V[:, 0])
        self.h_full()

    def compress(self, y, conv, exclude=None, first=None):
        """eigensolver.py:485-536."""
        o, g = self.o, self.g
        keep = max(o.min_restart_size, conv + 1)
        keep = max(min(keep, g - 1 if g > 1 else 1, self.cap - 2), 1)
        order = ([first] if first is not None else []) + [y[:, j] for j in range(y.shape[1])]
        base = [exclude] if exclude is not None else []
        sel = self.coef_select(order, keep, base)
        room = max(min(o.plus_k, self.cap - 1 - sel.shape[1]), 0)
        if room > 0:
            plus = self.coef_select(self.padded_prev(), room, base + [sel[:, j] for j in range(sel.shape[1])])
        else:
            plus = np.zeros((g, 0), order="F")
        C = np.asfortranarray(np.hstack([sel, plus]))
        s = C.shape[1]
        self.work["restarts"] += 1
        self.since_reset += 1
        self.prev = None
        if s == 0:
            self.reseed()
            if self.Q is not None and not self.done:
                self._qr_rebuild()
            return
        nv = self.V[:, :g] @ C
        nw = self.W[:, :g] @ C
        nh = C.T @ (self.H[:g, :g] @ C)
        self.V[:, :s] = nv
        self.W[:, :s] = nw
        self.H[:s, :s] = 0.5 * (nh + nh.T)
        if self.Q is not None:
            self.Q, self.R = qr_compress(self.Q[:, :g], self.R[:g, :g], C)
        self.g = s

    def lock(self, lam, y, x, rn, user):
        xn = x / np.linalg.norm(x)
        k = self.lock_v.shape[1]
        grown = np.zeros((self.N, k + 1), order="F")
        grown[:, :k] = self.lock_v
        grown[:, k] = xn
        cgs_orthonormalize(grown, against=self.ext, first=k, rng=self.rng)
        self.lock_v = grown
        self.lock_l.append(float(lam))
        self.lock_r.append(float(rn))
        self.lock_u.append(bool(user))
        if len(self.lock_l) >= self.want:
            self.done = True
            return
        self.compress(self._last_y, 0, exclude=y)
        if self.Q is not None and not self.done:
            self._qr_rebuild()

    def step(self):
        """eigensolver.py:563-664."""
        o = self.o
        self.work["iters"] += 1
        lams, y = self.rayleigh_ritz()
        self._last_y = y
        self.norm.see(lams, self.aug)
        g_now = self.g
        if o.extraction == REFINED:
            lam_c, y_c = self.refined()
            x_c = self.V[:, :self.g] @ y_c
            ox_c = self.W[:, :self.g] @ y_c
            res_c = ox_c - lam_c * x_c
            rn_c = float(np.linalg.norm(res_c))
            conv, first, block = 0, y_c, res_c[:, None]
        else:
            probe = 1 if o.locking else min(self.want + o.max_block_size, self.g)
            x, ox, res, rns = self.residuals(lams, y, probe)
            conv = 0
            if not o.locking:
                for i in range(min(self.want, rns.shape[0])):
                    if not (self.user_ok(lams[i], rns[i], x[:, i], ox[:, i]) or
                            self.floor_ok(lams[i], rns[i], x[:, i], ox[:, i])):
                        break
                    conv += 1
            ci = min(conv, rns.shape[0] - 1)
            lam_c, y_c = float(lams[ci]), y[:, ci]
            x_c, ox_c, rn_c = x[:, ci], ox[:, ci], float(rns[ci])
            first = None
            block = res[:, ci:min(ci + o.max_block_size, res.shape[1])]
        slot = len(self.lock_l) if o.locking else conv
        if self.reset_if_needed(rn_c):
            return
        if not o.locking and conv >= self.want:
            self.done = True
            return
        if o.locking:
            user = self.user_ok(lam_c, rn_c, x_c, ox_c)
            if user or self.floor_ok(lam_c, rn_c, x_c, ox_c):
                self.lock(lam_c, y_c, x_c, rn_c, user)
                return
        if o.stagnation_window is not None and self.stale(slot, rn_c, lam_c) > o.stagnation_window:
            self.status, self.done = "stagnated", True
            return
        if self.left() < o.max_block_size:
            self.status, self.done = "budget", True
            return
        restarted = False
        if self.g >= self.cap:
            self.compress(y, conv, first=first)
            restarted = True
            if self.done:
                return
        self.expand(block)
        if not restarted:
            if o.extraction == REFINED:
                self.prev = y_c[:, None].copy()
            else:
                hi = min(conv + max(o.plus_k, 1), y.shape[1])
                self.prev = y[:, conv:hi].copy()
            self.prev_g = g_now

    def expand(self, block):
        """eigensolver.py:666-700."""
        b = min(block.shape[1], self.cap - self.g)
        if b <= 0:
            return
        blk = block[:, :b]
        if self.pre is not None:
            blk = self.pre(np.asfortranarray(blk))
            self.work["precond"] += b
        g = self.g
        self.V[:, g:g + b] = blk
        swapped = cgs_orthonormalize(self.V[:, :g + b], against=self.against(), first=g, rng=self.rng)
        if len(swapped) == b:
            self.streak += 1
            if self.streak >= 3:
                raise RuntimeError("no independent expansion direction after 3 retries")
        else:
            self.streak = 0
        nw = self.apply(self.V[:, g:g + b])
        self.W[:, g:g + b] = nw
        hc = self.V[:, :g + b].T @ nw
        self.H[:g + b, g:g + b] = hc
        self.H[g:g + b, :g] = hc[:g].T
        blk2 = self.H[g:g + b, g:g + b]
        self.H[g:g + b, g:g + b] = 0.5 * (blk2 + blk2.T)
        if self.Q is not None:
            for j in range(b):
                self.Q, self.R = qr_extend(self.Q, self.R, nw[:, j] - self.tau * self.V[:, g + j], self.rng)
        self.g = g + b

    def finish(self):
        if self.o.locking:
            t = len(self.lock_l)
            if t == 0:
                return np.zeros(0), np.zeros((self.N, 0)), np.zeros(0), np.zeros(0, dtype=bool)
            x = np.asfortranarray(self.lock_v[:, :t])
            wx = self.apply(x)
            lam = np.einsum("ij,ij->j", x, wx)
            res = wx - x * lam[None, :]
            rns = np.linalg.norm(res, axis=0)
            ok = np.array([self.user_ok(lam[i], rns[i], x[:, i], wx[:, i]) for i in range(t)], dtype=bool)
            return lam, x, rns, ok
        lams, y = self.rayleigh_ritz()
        t = min(self.want, self.g)
        x = np.asfortranarray(self.V[:, :self.g] @ y[:, :t])
        wx = self.apply(x) if t else np.zeros((self.N, 0))
        h2 = x.T @ wx
        lam2, z = np.linalg.eigh(0.5 * (h2 + h2.T))
        idx = self.order(lam2)
        lam2, z = lam2[idx], z[:, idx]
        x2 = np.asfortranarray(x @ z)
        wx2 = wx @ z
        rns = np.linalg.norm(wx2 - x2 * lam2[None, :], axis=0)
        ok = np.array([self.user_ok(lam2[i], rns[i], x2[:, i], wx2[:, i]) for i in range(t)], dtype=bool)
        return lam2, x2, rns, ok

    def dense_solve(self):
        lams, Y = np.linalg.eigh(self.H[:self.g, :self.g])
        self.norm.see(lams, self.aug)
        if self.o.target == CLOSEST:
            pick, free = [], list(range(lams.shape[0]))
            for i in range(min(self.want, lams.shape[0])):
                s = float(self.o.shifts[min(i, len(self.o.shifts) - 1)])
                sub = lams[free]
                above = np.flatnonzero(sub >= s)
                j = int(above[np.argmin(sub[above])]) if above.size else int(np.argmax(sub))
                pick.append(free.pop(j))
        else:
            pick = list(self.order(lams)[:self.want])
        lam = lams[pick]
        x = np.asfortranarray(self.V[:, :self.g] @ Y[:, pick])
        ox = self.W[:, :self.g] @ Y[:, pick]
        rns = np.linalg.norm(ox - x * lam[None, :], axis=0)
        ok = np.array([self.user_ok(lam[i], rns[i], x[:, i], ox[:, i]) for i in range(lam.shape[0])], dtype=bool)
        return Outcome(lam, x, np.asarray(rns), ok, self.work, self.status)

    def run(self):
        if self.want == 0:
            return Outcome(np.zeros(0), np.zeros((self.N, 0)), np.zeros(0), np.zeros(0, dtype=bool),
                           self.work, self.status)
        if self.dense:
            return self.dense_solve()
        while not self.done:
            self.step()
        lam, x, rns, ok = self.finish()
        return Outcome(np.asarray(lam, dtype=np.float64), x, np.asarray(rns, dtype=np.float64), ok,
                       self.work, self.status)


# --------------------------------------------------------------- driver

def _two_sided(v, sigma, u, x):
    av = v.mul(x)
    atu = v.tmul(u)
    return float(np.sqrt(np.linalg.norm(av - sigma * u) ** 2 + np.linalg.norm(atu - sigma * x) ** 2))


def svds(mat, k, target="largest", eps=1e-12, seed=0, block=1, precond=None, max_matvecs=None,
         method="hybrid", a_norm=None):
    """hybrid.py:465-631 (largest / smallest targets; no warm starts or
    deflation inputs).  mat: Csr.  Returns a dict."""
    t0 = time.perf_counter()
    mat.count = 0
    flipped = mat.m < mat.n
    v = View(mat, flipped)
    m, n = v.m, v.n
    delta = float(eps)
    norm = Norm(a_norm)
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x5fd]))
    if target == "largest" and k < 10:
        mbs, mrs = 15, 6
    else:
        mbs, mrs = 35, 14
    stage_status = []

    def budget():
        return None if max_matvecs is None else max((max_matvecs - v.count) // 2, 0)

    stats = {"restarts": 0, "resets": 0, "precond_applies": 0, "iters": 0}
    test1 = lambda lam, rn, x, ox, c: rn <= max(np.sqrt(abs(lam) * c) * delta, EPS * c)  # noqa: E731
    sigma = np.zeros(k)
    U = np.zeros((m, k), order="F")
    Vr = np.zeros((n, k), order="F")
    rc = np.full(k, np.inf)
    r7 = np.full(k, np.inf)
    tiny = np.zeros(k, dtype=bool)
    if method in ("hybrid", "normal"):
        o1 = Opts(num_evals=k, target=LARGEST if target == "largest" else SMALLEST, max_basis_size=mbs,
                  min_restart_size=mrs, plus_k=1, max_block_size=block, convergence_test=test1,
                  max_matvecs=budget(), seed=seed)
        pre = precond if (precond is not None and precond.mode == ("AAt" if flipped else "AtA")) else None
        p0 = pre.applied if pre is not None else 0
        s1 = GDk(normal_op(v), o1, precond=pre, norm=norm)
        r1 = s1.run()
        stage_status.append(r1.status)
        for key in ("restarts", "resets", "iters"):
            stats[key] += r1.work[key]
        if pre is not None:
            stats["precond_applies"] += pre.applied - p0
        # stage1_postprocess (hybrid.py:268-337)
        got = r1.eigenvalues.shape[0]
        t = min(got, k)
        floor = norm.a * EPS * max(m, n)
        for i in range(t):
            lam = float(r1.eigenvalues[i])
            x = np.array(r1.eigenvectors[:, i], dtype=np.float64)
            nx = np.linalg.norm(x)
            if nx > 0:
                x /= nx
            Vr[:, i] = x
            sg = float(np.sqrt(max(lam, 0.0)))
            av = v.mul(x)
            nav = float(np.linalg.norm(av))
            if sg < floor:
                tiny[i] = True
                sigma[i] = 0.0
                if nav > 0.0:
                    U[:, i] = av / nav
                else:
                    U[:, i] = rng.standard_normal(m)
                    cgs_orthonormalize(U[:, :i + 1], first=i, rng=rng)
            else:
                sigma[i] = sg
                U[:, i] = av / nav
            atu = v.tmul(U[:, i])
            r7[i] = float(np.sqrt(np.linalg.norm(av - sigma[i] * U[:, i]) ** 2 +
                                  np.linalg.norm(atu - sigma[i] * Vr[:, i]) ** 2))
            rc[i] = float(r1.residual_norms[i])
        for i in range(t, k):
            Vr[:, i] = rng.standard_normal(n)
            U[:, i] = rng.standard_normal(m)
            cgs_orthonormalize(Vr[:, :i + 1], first=i, rng=rng)
            cgs_orthonormalize(U[:, :i + 1], first=i, rng=rng)
        guesses = np.zeros((n + m, k), order="F")
        for i in range(k):
            guesses[:, i] = np.concatenate([Vr[:, i], U[:, i]]) / np.sqrt(2.0)
    else:
        guesses = np.asfortranarray(rng.standard_normal((n + m, k)))
        cgs_orthonormalize(guesses, rng=rng)
    mv1 = v.count
    passed = r7 < norm.a * delta
    go2 = method == "augmented" or (method == "hybrid" and not passed.all())
    shifts = None
    sig_t = sigma.copy()
    if go2:
        if target != "largest":
            floor = norm.a * EPS
            sh = np.full(k, floor)
            for i in range(k):
                if tiny[i] or sig_t[i] <= 0.0 or not np.isfinite(rc[i]):
                    continue
                sh[i] = max(sig_t[i] - np.sqrt(2.0) * rc[i] / sig_t[i], floor)
            idx = np.argsort(sh, kind="stable")
            shifts, sig_t, rc, tiny = sh[idx], sig_t[idx], rc[idx], tiny[idx]
            guesses = np.asfortranarray(guesses[:, idx])
            sigma, r7, passed = sigma[idx], r7[idx], passed[idx]
            U, Vr = np.asfortranarray(U[:, idx]), np.asfortranarray(Vr[:, idx])
        active = np.flatnonzero(~tiny & ~passed)
        if active.size:
            frozen = [guesses[:, i] for i in np.flatnonzero(tiny | passed)]
            ortho = np.asfortranarray(np.stack(frozen, axis=1)) if frozen else None

            def test2(lam, rn, x, ox, c):
                if not rn < np.sqrt(2.0) * c * delta:
                    return False
                nv, nu = float(np.linalg.norm(x[:n])), float(np.linalg.norm(x[n:]))
                if nv == 0.0 or nu == 0.0:
                    return False
                s = abs(lam)
                e = np.sqrt(np.linalg.norm(ox[n:] / nv - s * (x[n:] / nu)) ** 2 +
                            np.linalg.norm(ox[:n] / nu - s * (x[:n] / nv)) ** 2)
                return bool(e < c * delta)

            def floor2(lam, rn, x, ox, c):
                if not (c > 0.0 and rn <= FLOOR_FACTOR * EPS * c):
                    return False
                nv, nu = np.linalg.norm(x[:n]), np.linalg.norm(x[n:])
                if nv == 0.0 or nu == 0.0:
                    return False
                return min(nv, nu) >= 0.1 * max(nv, nu)

            if target == "largest":
                o2 = Opts(num_evals=active.size, target=LARGEST, max_basis_size=mbs, min_restart_size=mrs,
                          max_block_size=block, convergence_test=test2, practical_test=floor2,
                          max_matvecs=budget(), deactivate_krylov_init=True, seed=seed + 1)
            else:
                o2 = Opts(num_evals=active.size, target=CLOSEST, shifts=tuple(shifts[active]), max_basis_size=mbs,
                          min_restart_size=mrs, max_block_size=block, locking=True, extraction=REFINED,
                          convergence_test=test2, practical_test=floor2, max_matvecs=budget(),
                          deactivate_krylov_init=True, seed=seed + 1)
            s2 = GDk(augmented_op(v), o2, guesses=np.asfortranarray(guesses[:, active]), ortho=ortho, norm=norm,
                     augmented=True)
            r2 = s2.run()
            stage_status.append(r2.status)
            for key in ("restarts", "resets", "iters"):
                stats[key] += r2.work[key]
            for j in range(min(r2.eigenvalues.shape[0], active.size)):
                slot = active[j]
                x = r2.eigenvectors[:, j]
                nv, nu = float(np.linalg.norm(x[:n])), float(np.linalg.norm(x[n:]))
                if nv == 0.0 or nu == 0.0:
                    continue
                sigma[slot] = abs(float(r2.eigenvalues[j]))
                Vr[:, slot] = x[:n] / nv
                U[:, slot] = x[n:] / nu
                r7[slot] = _two_sided(v, sigma[slot], U[:, slot], Vr[:, slot])
    a_final = norm.a
    ok = r7 < a_final * delta
    idx = np.argsort(-sigma, kind="stable") if target == "largest" else np.argsort(sigma, kind="stable")
    U, Vr = np.asfortranarray(U[:, idx]), np.asfortranarray(Vr[:, idx])
    if flipped:
        U, Vr = Vr, U
    status = "ok"
    if not ok[idx].all():
        for s in ("budget", "stagnated"):
            if s in stage_status:
                status = s
                break
    return {"sigma": sigma[idx], "u": U, "v": Vr, "rnorms": r7[idx], "converged": ok[idx], "status": status,
            "stage1_matvecs": mv1, "stage2_matvecs": v.count - mv1, "seconds": time.perf_counter() - t0, **stats}

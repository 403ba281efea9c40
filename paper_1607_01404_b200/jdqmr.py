"""JDQMR inner solver on device.

PRIMME_SVDS runs stage 2 (and optionally stage 1) with JDQMR: GD+k outer
iterations whose expansion vector is an approximate solution of the
Jacobi-Davidson correction equation

    (I - Q Q^T)(Op - theta I)(I - Q Q^T) t = -r,   Q = [constraints, locked, x]

by symmetric QMR with dynamic stopping (the
reference package implements GD+k only).  Here every inner
step runs on the GPU: the operator product through the CSR SpMV kernels and
the QMRs recurrence in csrc/jdqmr.cu, whose scalars never leave the device.
With a native operator the whole inner solve is one CUDA graph with a WHILE
conditional node -- its body (SpMVs + 3-4 streaming kernels) repeats until
the device-side stopping test clears the condition -- so a correction
equation costs one launch and one status read.  Other operators (host
callables, the row-sharded operator) run the same kernels step by step.

Stopping (csrc/jdqmr.cu, restated in oracle/jdqmr.py): the eigen-residual
of x + t is tracked exactly from device dot products; the inner solve stops
when it would satisfy the outer convergence test, when it has dropped below
``etol_frac`` times the outer residual (PRIMME's JDQMR_ETol rule; 0 = off),
when the QMR residual falls below ``lfac`` times it (further inner steps
cannot lower it), when the Rayleigh quotient of x + t moves away from the
wanted end of the spectrum (extreme targets), after 3 steps without
improvement, or at ``max_inner_iterations``.
"""

import ctypes
import gc

import numpy as np
import torch

from . import _lib
from . import device as dv
from .device import DTYPE

# state slots (csrc/jdqmr.cu, namespace jd)
SIGMA, ERES, IT, MAXIT, TOL_E, ETOL_FRAC, STOP, RITZ, RNORM, LFAC, DIR = 0, 14, 16, 17, 18, 19, 20, 21, 22, 25, 27
NSTATE = 96
QMAX = 32
STOP_NAMES = {1: "maxit", 2: "converged", 3: "etol", 4: "linear", 5: "stagnation", 6: "breakdown",
              7: "empty", 8: "rq_reversal"}


class _Vecs(ctypes.Structure):
    _fields_ = [("r", ctypes.c_void_p), ("dg", ctypes.c_void_p), ("rc", ctypes.c_void_p),
                ("g", ctypes.c_void_p), ("t", ctypes.c_void_p), ("dl", ctypes.c_void_p),
                ("z", ctypes.c_void_p), ("d", ctypes.c_void_p), ("w", ctypes.c_void_p)]


def _native(op):
    """True when every launch of op.apply_into is a libsvdsb kernel on the
    context stream (capturable): CSR-backed, single-process operators."""
    if getattr(op, "comm", None) is not None:
        return False
    svd = getattr(op, "svd_op", None)
    if svd is None:
        return False
    base = getattr(svd, "base", svd)
    return getattr(base, "_csr_dev", None) is not None


def _counter_slots(op):
    """(object, attribute) pairs an operator application advances."""
    slots = [(op, "n_applies")]
    svd = getattr(op, "svd_op", None)
    if svd is not None:
        base = getattr(svd, "base", svd)
        slots.append((base, "n_matvecs"))
    return slots


class JdqmrInner:
    """Inner solver bound to one operator (dimension n on this device)."""

    def __init__(self, ctx, op, n, diag=None, use_graph=True):
        self.ctx = ctx
        self.op = op
        self.n = int(n)
        self.diag = diag
        work = dv.new_block(self.n, 8)
        self.r, self.rc, self.g, self.t, self.dl, self.z, self.d, self.w = (work[:, j] for j in range(8))
        self._work = work
        self.q = dv.new_block(self.n, QMAX)
        self.state = torch.zeros(NSTATE, dtype=DTYPE, device=ctx.device)
        self.inputs = torch.zeros(NSTATE, dtype=DTYPE, pin_memory=True)
        self.status = torch.zeros(NSTATE, dtype=DTYPE, pin_memory=True)
        self.vecs = _Vecs(self.r.data_ptr(), diag.data_ptr() if diag is not None else None,
                          self.rc.data_ptr(), self.g.data_ptr(), self.t.data_ptr(), self.dl.data_ptr(),
                          self.z.data_ptr(), self.d.data_ptr(), self.w.data_ptr())
        self.use_graph = bool(use_graph) and _native(op)
        self._graphs = {}
        self._per_apply = None   # counter advance of one operator application
        self.solves = 0
        self.log = None          # list -> (theta, rnorm, iterations, reason, eres) per solve
        self.inner_iterations = 0
        self.launches = 0

    # ------------------------------------------------------------ pieces
    def _phase(self, phase, nq, cond=0):
        _lib.call("svdsb_jd_phase", self.ctx.handle, int(phase), self.n, ctypes.byref(self.vecs),
                  ctypes.c_void_p(self.q.data_ptr()), dv.ld_of(self.q), int(nq),
                  ctypes.c_void_p(self.state.data_ptr()), ctypes.c_uint64(cond), self.ctx.stream)

    def _apply(self, raw=False):
        raw_into = getattr(self.op, "raw_into", None) if raw else None
        if raw_into is not None:
            raw_into(self.d.unsqueeze(1), self.w.unsqueeze(1))
        else:
            self.op.apply_into(self.d.unsqueeze(1), self.w.unsqueeze(1))

    def _capture(self, nq):
        """WHILE graph of one inner step (operator product + QMRs kernels)."""
        lib = _lib.load()
        ctx = self.ctx
        slots = _counter_slots(self.op)
        before = [getattr(o, a) for o, a in slots]
        # one uncaptured product measures what an application counts
        self._apply()
        self._per_apply = [getattr(o, a) - b for (o, a), b in zip(slots, before)]
        for (o, a), b in zip(slots, before):
            setattr(o, a, b)
        cap = getattr(ctx, "capture_stream", None)
        if cap is None:
            cap = ctx.capture_stream = torch.cuda.Stream(ctx.device)
        cap.wait_stream(ctx.torch_stream)
        l0 = _lib.launch_count()
        cond = ctypes.c_uint64()
        ex = ctypes.c_void_p()
        old = ctx._stream
        gc_on = gc.isenabled()   # as DavidsonSolver._capture: no finalisers inside a capture
        gc.disable()
        _lib.CAPTURING[0] += 1
        try:
            _lib.check(lib.svdsb_while_begin(cap.cuda_stream, ctypes.byref(cond)), "svdsb_while_begin")
            try:
                ctx._stream = cap.cuda_stream
                self._apply(raw=True)
                self._phase(1, nq, cond.value)
            finally:
                ctx._stream = old
                rc = lib.svdsb_while_end(cap.cuda_stream, ctypes.byref(ex))
        finally:
            _lib.CAPTURING[0] -= 1
            if gc_on:
                gc.enable()
            _lib.flush_deferred()
        _lib.check(rc, "svdsb_while_end")
        from .eigensolver import _NativeGraph
        return _NativeGraph(ex.value), _lib.launch_count() - l0

    # ------------------------------------------------------------- solve
    def solve(self, x, theta, r, rnorm, against=(), maxit=100, tol_e=0.0, etol_frac=0.0, lfac=0.1, direction=0):
        """Correction for the Ritz pair (theta, x) with residual r (device
        columns of length n).  Returns (t, info); t is a view of an internal
        buffer, valid until the next solve."""
        cols = [b for b in against if b is not None and b.shape[1] > 0]
        nq = sum(int(b.shape[1]) for b in cols) + 1
        if nq > QMAX:
            raise ValueError("JDQMR projects against at most %d vectors (constraints + locked + 1)" % QMAX)
        j = 0
        for b in cols:
            k = int(b.shape[1])
            dv.axpby(self.ctx, 1.0, b, 0.0, self.q[:, j:j + k])
            j += k
        dv.axpby(self.ctx, 1.0, dv.as_block(x), 0.0, self.q[:, j:j + 1])
        dv.axpby(self.ctx, 1.0, dv.as_block(r), 0.0, self.r.unsqueeze(1))
        inp = self.inputs.numpy()
        inp[SIGMA], inp[RITZ], inp[RNORM] = float(theta), float(theta), float(rnorm)
        inp[MAXIT], inp[TOL_E], inp[ETOL_FRAC], inp[LFAC] = float(max(int(maxit), 0)), float(tol_e), \
            float(etol_frac), float(lfac)
        inp[DIR] = float(np.sign(direction))
        # the previous solve ended with a stream sync, so the pinned image is
        # free to rewrite; phase 0 fills every other slot
        with torch.cuda.stream(self.ctx.torch_stream):
            self.state.copy_(self.inputs, non_blocking=True)
        self._phase(0, nq)
        if self.use_graph:
            entry = self._graphs.get(nq)
            if entry is None:
                entry = self._graphs[nq] = self._capture(nq)
            entry[0].replay(self.ctx._stream)
            self._read_status()
            it = int(self.status[IT])
            self.launches += entry[1] * max(it, 1)
            _lib.load().svdsb_note_launches(entry[1] * max(it, 1))
            for (o, a), per in zip(_counter_slots(self.op), self._per_apply):
                setattr(o, a, getattr(o, a) + per * it)
        else:
            it = 0
            while True:
                self._read_status()
                if self.status[STOP] != 0.0 or it >= maxit:
                    break
                self._apply()
                self._phase(1, nq)
                it += 1
            self._read_status()
            it = int(self.status[IT])
        self.solves += 1
        self.inner_iterations += it
        info = {"iterations": it, "stop": int(self.status[STOP]), "eres": float(self.status[ERES])}
        info["reason"] = STOP_NAMES.get(info["stop"], "?")
        if self.log is not None:
            self.log.append((float(theta), float(rnorm), it, info["reason"], info["eres"]))
        return self.t, info

    def _read_status(self):
        _lib.call("svdsb_d2h", ctypes.c_void_p(self.status.data_ptr()), ctypes.c_void_p(self.state.data_ptr()),
                  NSTATE * 8, self.ctx.stream)
        _lib.call("svdsb_stream_sync", self.ctx.stream)

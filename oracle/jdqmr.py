"""TEST INFRASTRUCTURE ONLY.  NumPy restatement of the JDQMR inner solve
(symmetric QMR on the Jacobi-Davidson correction equation) that
paper_1607_01404_b200/csrc/jdqmr.cu runs on device.

The reference package implements GD+k only; JDQMR is the
paper's stage-2 method as PRIMME implements it
(QMRs of Freund & Nachtigal with the Jacobi-Davidson projections and
dynamic stopping, Stathopoulos, SISC 29(2) 2007).  This restatement is
therefore "parity unpinned" against the reference: it is the checker for
the device kernels (same recurrences, same stopping rules), and the solves
that use JDQMR are checked against the reference's GD+k results by
tolerance (tests/test_jdqmr_gpu.py).
"""

import numpy as np

STOP_NAMES = {1: "maxit", 2: "converged", 3: "etol", 4: "linear", 5: "stagnation", 6: "breakdown",
              7: "empty", 8: "rq_reversal"}


def qmrs_correction(op, x, theta, r, q=None, dg=None, maxit=100, tol_e=0.0, etol_frac=0.0, lfac=0.1,
                    sigma=None, direction=0):
    """Approximate solution t of P (op - sigma) P t = -r, P = I - Q Q^T with
    Q = q (orthonormal columns, x among them), preconditioner P K^-1 P with
    K = diag(dg).  Returns (t, info)."""
    n = r.shape[0]
    sigma = theta if sigma is None else sigma
    q = np.zeros((n, 0)) if q is None else np.asarray(q)
    rnorm = float(np.linalg.norm(r))

    def proj(v):
        return v - q @ (q.T @ v) if q.shape[1] else v

    b = -r
    rc = b.copy()
    g = b.copy()
    t = np.zeros(n)
    dl = np.zeros(n)
    bb = float(b @ b)
    tau = np.sqrt(bb)
    if dg is not None:
        z = b / dg
        rho_prev = float(b @ z)
        d = proj(z)
    else:
        rho_prev = bb
        d = b.copy()
    theta_prev = 0.0
    rt = tt = 0.0
    best = rnorm
    stall = 0
    it = 0
    stop = 0 if (bb > 0.0 and maxit > 0) else 7
    eres = rnorm
    rq_prev = theta
    history = []
    while stop == 0:
        w = op(d) - sigma * d
        sigp = float(d @ w)
        alpha = rho_prev / sigp if sigp != 0.0 else np.inf
        if sigp == 0.0 or not np.isfinite(alpha) or abs(alpha) < 1e-300:
            stop = 6
            break
        w = proj(w)
        rc = rc - alpha * w
        rr = float(rc @ rc)
        th = np.sqrt(rr) / tau
        c2 = 1.0 / (1.0 + th * th)
        tau = tau * th * np.sqrt(c2)
        gam = c2 * theta_prev ** 2
        eta = alpha * c2
        s2 = th * th * c2
        theta_prev = th
        if dg is None:
            rho = rr
            beta = rho / rho_prev
            rho_prev = rho
            if not rho > 0.0:
                stop = 6
                break
        dl = gam * dl + eta * d
        t_old = t
        t = t + dl
        g = s2 * g + c2 * rc
        rt += float(r @ dl)
        tt += 2.0 * float(t_old @ dl) + float(dl @ dl)
        gt, gg = float(g @ t), float(g @ g)
        a = theta - sigma + rt
        den = 1.0 + tt
        rq = (a - gt) / den
        eres = np.sqrt(max((a * a + gg) / den - rq * rq, 0.0))
        it += 1
        if dg is not None:
            z = rc / dg
            rho = float(rc @ z)
            beta = rho / rho_prev
            rho_prev = rho
            if rho == 0.0 or not np.isfinite(rho):
                stop = 6
        else:
            d = rc + beta * d
        if eres < best:
            best, stall = eres, 0
        else:
            stall += 1
        history.append(eres)
        rqv = sigma + rq
        reversed_ = direction * (rqv - rq_prev) < 0.0
        rq_prev = rqv
        if stop:
            pass
        elif not np.isfinite(eres) or not np.isfinite(tt):
            stop = 6
        elif reversed_:
            stop = 8
        elif eres <= tol_e:
            stop = 2
        elif eres <= etol_frac * rnorm:
            stop = 3
        elif np.sqrt(gg) <= lfac * eres:
            stop = 4
        elif stall >= 3:
            stop = 5
        elif it >= maxit:
            stop = 1
        if stop == 0 and dg is not None:
            d = proj(z) + beta * d
    return t, {"iterations": it, "stop": stop, "reason": STOP_NAMES.get(stop, "?"), "eres": eres,
               "history": history}

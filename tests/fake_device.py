"""TEST-ONLY stand-in for paper_1607_01404_b200.device on CPU tensors.

Lets the CPU suite drive the solver's host logic -- including the
row-sharded path over a 2-rank gloo group -- without a GPU.  Each function
restates the semantics of the matching libsvdsb kernel (include/svdsb.h) in
torch/numpy fp64.  It is installed with ``install(monkeypatch)`` inside a
test; the shipped package never imports it and keeps failing loudly
without CUDA.
"""

import numpy as np
import torch

from oracle import phsvds

DT = torch.float64
SCALE_MUL, SCALE_DIV, SCALE_DIV_SQRT = 0, 1, 2
ORDER_ASC, ORDER_DESC, ORDER_INTERIOR = 0, 1, 2


class _Ctx:
    device = torch.device("cpu")
    index = 0
    stream = None
    handle = None


CTX = _Ctx()


def context(device=None):
    return CTX


def require_cuda():
    return None


def new_block(rows, cols, device=None, zero=True):
    ld = max(32, ((int(rows) + 31) // 32) * 32)
    return torch.zeros((max(int(cols), 1), ld), dtype=DT).t()[:int(rows), :int(cols)]


def small_matrix(rows, cols, device=None):
    return torch.zeros((cols, rows), dtype=DT).t()


def as_block(t):
    return t.unsqueeze(1) if t.dim() == 1 else t


def to_device_block(x, device=None):
    src = x.to(DT) if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
    src = as_block(src)
    out = new_block(src.shape[0], src.shape[1])
    out.copy_(src)
    return out


def to_host(t):
    return np.asfortranarray(t.detach().numpy())


def _cat(blocks):
    blocks = [as_block(b) for b in blocks if b is not None and b.shape[1] > 0]
    return torch.cat(blocks, dim=1) if blocks else None


def gram(ctx, dim, blocks, y, c_out, norms2=None):
    y = as_block(y)
    x = _cat(blocks)
    if norms2 is not None:
        norms2.copy_((y * y).sum(0))
    if x is not None:
        as_block(c_out)[:x.shape[1], :y.shape[1]].copy_(x.t() @ y)


def project_out(ctx, dim, blocks, c, y, norms2=None):
    y = as_block(y)
    x = _cat(blocks)
    if x is not None:
        y.sub_(x @ as_block(c)[:x.shape[1], :y.shape[1]])
    if norms2 is not None:
        norms2.copy_((y * y).sum(0))


def ts_gemm(ctx, x, c, y, alpha=1.0, beta=0.0):
    x, c, y = as_block(x), as_block(c), as_block(y)
    out = alpha * (x @ c[:x.shape[1], :y.shape[1]])
    if beta != 0.0:
        out = out + beta * y
    y.copy_(out)


def ritz_residual(ctx, v, w, yc, lam, r, x=None, ox=None, rn2=None):
    v, w, yc, r = as_block(v), as_block(w), as_block(yc), as_block(r)
    p = r.shape[1]
    xx = v @ yc[:, :p]
    oo = w @ yc[:, :p]
    rr = oo - xx * lam.reshape(-1)[:p]
    r.copy_(rr)
    if x is not None:
        as_block(x).copy_(xx)
    if ox is not None:
        as_block(ox).copy_(oo)
    if rn2 is not None:
        rn2.copy_((rr * rr).sum(0))


def col_norms2(ctx, x, out):
    x = as_block(x)
    out.copy_((x * x).sum(0))


def col_dots(ctx, x, y, out):
    out.copy_((as_block(x) * as_block(y)).sum(0))


def scale_cols(ctx, x, s, mode, y=None):
    x = as_block(x)
    y = x if y is None else as_block(y)
    f = s.reshape(-1)[:x.shape[1]]
    if mode == SCALE_MUL:
        y.copy_(x * f)
    else:
        d = torch.sqrt(f) if mode == SCALE_DIV_SQRT else f
        d = torch.where(f == 0.0, torch.ones_like(d), d)
        y.copy_(x / d)


def axpby(ctx, alpha, x, beta, y):
    x, y = as_block(x), as_block(y)
    out = alpha * x
    if beta != 0.0:
        out = out + beta * y
    y.copy_(out)


def split_stats(ctx, nsplit, r, x, out):
    r, x = as_block(r), as_block(x)
    for j in range(r.shape[1]):
        rv, xv, ru, xu = r[:nsplit, j], x[:nsplit, j], r[nsplit:, j], x[nsplit:, j]
        out[6 * j:6 * j + 6] = torch.stack([rv @ rv, rv @ xv, xv @ xv, ru @ ru, ru @ xu, xu @ xu])


def split_residual(ctx, nsplit, r, x, lam, stats, out):
    r, x = as_block(r), as_block(x)
    for j in range(r.shape[1]):
        st = stats[6 * j:6 * j + 6]
        nv, nu = float(torch.sqrt(st[2])), float(torch.sqrt(st[5]))
        if nv == 0.0 or nu == 0.0:
            out[j] = float("inf")
            continue
        lj = float(lam.reshape(-1)[j])
        sg = abs(lj)
        e1 = r[nsplit:, j] / nv + (lj / nv - sg / nu) * x[nsplit:, j]
        e2 = r[:nsplit, j] / nu + (lj / nu - sg / nv) * x[:nsplit, j]
        out[j] = e1 @ e1 + e2 @ e2


def _order(w, order, shift):
    if order == ORDER_ASC:
        return np.argsort(w, kind="stable")
    if order == ORDER_DESC:
        return np.argsort(-w, kind="stable")
    below = w < shift
    return np.lexsort((np.where(below, shift - w, w - shift), below.astype(np.int64)))


def syev_small(ctx, h, g, order, shift, w, y):
    hh = h[:g, :g].numpy()
    lam, vec = np.linalg.eigh(0.5 * (hh + hh.T))
    idx = _order(lam, order, shift)
    w[:g].copy_(torch.from_numpy(lam[idx]))
    y[:g, :g].copy_(torch.from_numpy(vec[:, idx]))


def syev_update(ctx, h, g0, b, y0, l0, order, shift, w, y):
    syev_small(ctx, h, g0 + b, order, shift, w, y)


def refined_small(ctx, r, h, g, y, lam, sv=None):
    rr = r[:g, :g].numpy()
    _, s, vt = np.linalg.svd(rr)
    yy = vt[-1]
    y[:g].copy_(torch.from_numpy(yy))
    lam.reshape(-1)[0] = float(yy @ (h[:g, :g].numpy() @ yy))
    if sv is not None:
        sv[:g].copy_(torch.from_numpy(s))


def restart_coefs(ctx, g, gmax, yfirst, yall, ny, retain, exclude, prev, nprev, prev_g, plus_k, out, count_dev):
    gd = phsvds.GDk.__new__(phsvds.GDk)
    gd.g = g
    cols = ([yfirst.numpy()] if yfirst is not None else []) + [yall[:g, j].numpy() for j in range(ny)]
    base = [exclude.numpy()] if exclude is not None else []
    sel = phsvds.GDk.coef_select(gd, cols, retain, base)
    blocks = [sel]
    budget = max(min(plus_k, gmax - 1 - sel.shape[1]), 0)
    if budget > 0 and prev is not None and prev_g <= g and nprev > 0:
        pcols = []
        for j in range(nprev):
            c = np.zeros(g)
            c[:prev_g] = prev[:prev_g, j].numpy()
            pcols.append(c)
        blocks.append(phsvds.GDk.coef_select(gd, pcols, budget, base + [sel[:, j] for j in range(sel.shape[1])]))
    allc = np.hstack(blocks)
    out[:g, :allc.shape[1]].copy_(torch.from_numpy(allc))
    count_dev[0] = allc.shape[1]


def project_small(ctx, h, g, c, s, hout):
    hh = h[:g, :g].clone()
    cc = c[:g, :s]
    p = cc.t() @ (hh @ cc)
    hout[:s, :s].copy_(0.5 * (p + p.t()))


def qr_small(ctx, r, g, yc, s, qy, ry):
    q, rr = np.linalg.qr(r[:g, :g].numpy() @ yc[:g, :s].numpy())
    sign = np.where(np.diag(rr) < 0.0, -1.0, 1.0)
    qy[:g, :s].copy_(torch.from_numpy(q * sign))
    ry[:s, :s].copy_(torch.from_numpy(rr * sign[:, None]))


def h_insert(ctx, g, b, hc, h):
    hc = as_block(hc)
    h[:g + b, g:g + b] = hc[:g + b, :b]
    h[g:g + b, :g] = hc[:g, :b].t()
    blk = hc[g:g + b, :b].clone()
    h[g:g + b, g:g + b] = 0.5 * (blk + blk.t())


def h_symmetrize(ctx, g, gm, h):
    gg = gm[:g, :g].clone()
    h[:g, :g].copy_(0.5 * (gg + gg.t()))


def fetch(ctx, tensors):
    return [t.detach().reshape(-1).numpy().copy() for t in tensors]


NAMES = ["context", "require_cuda", "new_block", "small_matrix", "as_block", "to_device_block", "to_host", "gram",
         "project_out", "ts_gemm", "ritz_residual", "col_norms2", "col_dots", "scale_cols", "axpby", "split_stats",
         "split_residual", "syev_small", "syev_update", "refined_small", "restart_coefs", "project_small", "qr_small",
         "h_insert", "h_symmetrize", "fetch"]


def install(monkeypatch):
    from paper_1607_01404_b200 import device as dv
    g = globals()
    for name in NAMES:
        monkeypatch.setattr(dv, name, g[name])

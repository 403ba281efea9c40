"""Device plumbing: per-device libsvdsb context, column-major blocks and thin
typed wrappers over the C ABI.

Blocks follow the reference's convention (kernels.py:5-9):
column-major fp64 with a leading dimension.  On device a block is a torch
tensor of shape (rows, cols) with strides (1, ld), which is exactly the
(ptr, ld) pair the C ABI takes.  PyTorch is used for memory, streams and
copies only; every numeric operation goes through libsvdsb kernels.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import call

DTYPE = torch.float64
LD_ALIGN = 32   # 256-byte aligned columns


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1607_01404_b200 runs on a CUDA (sm_100a) device; no GPU "
            "is visible and there is no CPU fallback")


class DeviceContext:
    """libsvdsb context (reduction workspace) bound to one CUDA device."""

    def __init__(self, index):
        require_cuda()
        _lib.load()
        self.index = index
        self.device = torch.device("cuda", index)
        with torch.cuda.device(index):
            h = ctypes.c_void_p()
            call("svdsb_ctx_create", index, ctypes.byref(h))
        self.handle = h
        # pinned staging for the per-iteration status read
        self._pinned = torch.empty(8192, dtype=DTYPE, pin_memory=True)

        self._stream = None
        self.refresh_stream()

    def refresh_stream(self):
        """Bind libsvdsb launches to torch's current stream on this device
        (looked up once per solve; per-call lookups cost ~8 us each)."""
        self.torch_stream = torch.cuda.current_stream(self.device)
        self._stream = int(self.torch_stream.cuda_stream) or None
        return self._stream

    @property
    def stream(self):
        return self._stream

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib._lib is not None:
                _lib._lib.svdsb_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts = {}


def context(device=None):
    require_cuda()
    if device is None:
        idx = torch.cuda.current_device()
    else:
        d = torch.device(device)
        idx = d.index if d.index is not None else torch.cuda.current_device()
    ctx = _contexts.get(idx)
    if ctx is None:
        ctx = DeviceContext(idx)
        _contexts[idx] = ctx
    return ctx


# --------------------------------------------------------------- blocks

def padded_ld(rows):
    return max(LD_ALIGN, ((int(rows) + LD_ALIGN - 1) // LD_ALIGN) * LD_ALIGN)


def new_block(rows, cols, device=None, zero=True):
    """Column-major (rows, cols) fp64 device block with an aligned ld."""
    ctx = context(device)
    ld = padded_ld(rows)
    alloc = torch.zeros if zero else torch.empty
    buf = alloc((max(int(cols), 1), ld), dtype=DTYPE, device=ctx.device)
    return buf.t()[:int(rows), :int(cols)]


def is_colmajor(t):
    return t.dim() == 2 and (t.shape[0] <= 1 or t.stride(0) == 1)


def ld_of(t):
    if t.dim() == 1:
        return max(int(t.shape[0]), 1)
    if t.shape[1] <= 1:
        return max(int(t.stride(1)), int(t.shape[0]), 1)
    return int(t.stride(1))


def as_block(t):
    """View a 1-D or 2-D tensor as a column-major 2-D block (no copy if
    possible)."""
    if t.dim() == 1:
        return t.unsqueeze(1)
    if not is_colmajor(t):
        raise ValueError("block must be column-major (strides (1, ld))")
    return t


def P(t):
    return t.data_ptr() if t is not None else None


def to_device_block(x, device=None):
    """numpy / torch (rows,) or (rows, cols) -> fresh column-major device
    block (copy)."""
    ctx = context(device)
    if isinstance(x, torch.Tensor):
        src = x.to(dtype=DTYPE)
    else:
        src = torch.from_numpy(np.asarray(x, dtype=np.float64))
    if src.dim() == 1:
        src = src.unsqueeze(1)
    out = new_block(src.shape[0], src.shape[1], device=ctx.device, zero=False)
    out.copy_(src)
    return out


def to_host(t):
    """Device block -> F-ordered numpy array (the reference's result
    layout, hybrid.py:603-605).  A column-major block (strides (1, ld)) is
    packed to (cols, rows) on the device and read back with one contiguous
    copy, whose transpose is the F-ordered result -- no host-side transpose
    (config 4's 10 M x 20 U: 0.8 s -> ~0.1 s)."""
    t = t.detach()
    if t.dim() == 2 and t.stride(0) == 1 and t.shape[0] > 1 and t.is_cuda:
        rows, cols = t.shape
        packed = t.t().contiguous()                     # (cols, rows): F order of the result
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        if packed.numel() * 8 < (8 << 20):
            out.T[...] = packed.cpu().numpy()
            return out
        _read_back(packed.view(-1), out.T.reshape(-1))
        return out
    return np.asfortranarray(t.cpu().numpy())


_STAGE = {}
_COPY_THREADS = 8


def _read_back(src, dst):
    """Device vector -> host numpy vector through a cached pinned staging
    buffer: chunks of 64 MB alternate between two pinned slots, each copied
    to the destination by host threads while the next chunk's device->host
    copy runs (a pageable copy of config 4's U ran at ~2 GB/s)."""
    from concurrent.futures import ThreadPoolExecutor
    chunk = 8 << 20                                     # doubles per chunk (64 MB)
    st = _STAGE.get(src.device)
    if st is None:
        slots = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        st = _STAGE[src.device] = {"slots": slots, "events": [torch.cuda.Event(), torch.cuda.Event()],
                                   "pool": ThreadPoolExecutor(_COPY_THREADS), "stream": torch.cuda.Stream(src.device)}
    slots, events, pool, stream = st["slots"], st["events"], st["pool"], st["stream"]
    n = src.numel()
    stream.wait_stream(torch.cuda.current_stream(src.device))
    pending = [None, None]

    def host_copy(slot, off, cnt):
        view = slots[slot].numpy()[:cnt]
        parts = max(1, min(_COPY_THREADS, cnt // (1 << 18)))
        step = (cnt + parts - 1) // parts
        futs = [pool.submit(np.copyto, dst[off + i:off + min(i + step, cnt)], view[i:min(i + step, cnt)])
                for i in range(0, cnt, step)]
        for f in futs:
            f.result()

    k = 0
    for off in range(0, n, chunk):
        cnt = min(chunk, n - off)
        if pending[k] is not None:                      # the slot's previous chunk must be on the host
            host_copy(*pending[k])
            pending[k] = None
        with torch.cuda.stream(stream):
            slots[k][:cnt].copy_(src[off:off + cnt], non_blocking=True)
            events[k].record(stream)
        prev = 1 - k
        if pending[prev] is not None:
            host_copy(*pending[prev])
            pending[prev] = None
        events[k].synchronize()
        pending[k] = (k, off, cnt)
        k = 1 - k
    for p in pending:
        if p is not None:
            host_copy(*p)


# ------------------------------------------------------- kernel wrappers

def _blk_args(blocks):
    blocks = [as_block(b) for b in blocks if b is not None and b.shape[1] > 0]
    if len(blocks) > _lib.MAX_BLOCKS:
        raise ValueError("at most %d column blocks" % _lib.MAX_BLOCKS)
    ptrs = [b.data_ptr() for b in blocks]
    lds = [ld_of(b) for b in blocks]
    cols = [b.shape[1] for b in blocks]
    n = len(blocks)
    if n == 0:
        ptrs, lds, cols, n = [0], [1], [0], 1
    return n, _lib.ptr_array(ptrs), _lib.i64_array(lds), _lib.int_array(cols), sum(cols)


def gram(ctx, dim, blocks, y, c_out, norms2=None):
    """c_out[:sum cols, :b] = [blocks]^T y ; norms2[:b] = ||y_j||^2."""
    y = as_block(y)
    n, ptrs, lds, cols, _ = _blk_args(blocks)
    call("svdsb_gram", ctx.handle, int(dim), n, ptrs, lds, cols, P(y), ld_of(y), y.shape[1],
         P(c_out), ld_of(as_block(c_out)), P(norms2), ctx.stream)


def project_out(ctx, dim, blocks, c, y, norms2=None):
    """y -= [blocks] c ; norms2 = ||y_j||^2 after."""
    y = as_block(y)
    n, ptrs, lds, cols, _ = _blk_args(blocks)
    call("svdsb_project_out", ctx.handle, int(dim), n, ptrs, lds, cols, P(c), ld_of(as_block(c)),
         P(y), ld_of(y), y.shape[1], P(norms2), ctx.stream)


def ts_gemm(ctx, x, c, y, alpha=1.0, beta=0.0):
    """y = alpha x c + beta y  (x: dim x g, c: g x s, y: dim x s)."""
    x, c, y = as_block(x), as_block(c), as_block(y)
    call("svdsb_ts_gemm", ctx.handle, y.shape[0], P(x), ld_of(x), x.shape[1], P(c), ld_of(c),
         y.shape[1], float(alpha), float(beta), P(y), ld_of(y), ctx.stream)


def ritz_residual(ctx, v, w, yc, lam, r, x=None, ox=None, rn2=None):
    v, w, yc, r = as_block(v), as_block(w), as_block(yc), as_block(r)
    g = v.shape[1]
    p = r.shape[1]
    xb = as_block(x) if x is not None else None
    ob = as_block(ox) if ox is not None else None
    call("svdsb_ritz_residual", ctx.handle, v.shape[0], P(v), ld_of(v), P(w), ld_of(w), g,
         P(yc), ld_of(yc), P(lam), p, P(r), ld_of(r), P(xb), ld_of(xb) if xb is not None else 1,
         P(ob), ld_of(ob) if ob is not None else 1, P(rn2), ctx.stream)


def col_norms2(ctx, x, out):
    x = as_block(x)
    call("svdsb_col_norms2", ctx.handle, x.shape[0], P(x), ld_of(x), x.shape[1], P(out), ctx.stream)


def col_dots(ctx, x, y, out):
    x, y = as_block(x), as_block(y)
    call("svdsb_col_dots", ctx.handle, x.shape[0], P(x), ld_of(x), P(y), ld_of(y), x.shape[1], P(out),
         ctx.stream)


SCALE_MUL, SCALE_DIV, SCALE_DIV_SQRT = 0, 1, 2


def scale_cols(ctx, x, s, mode, y=None):
    x = as_block(x)
    y = x if y is None else as_block(y)
    call("svdsb_scale_cols", x.shape[0], P(x), ld_of(x), x.shape[1], P(s), mode, P(y), ld_of(y),
         ctx.stream)


def axpby(ctx, alpha, x, beta, y):
    x, y = as_block(x), as_block(y)
    call("svdsb_axpby", y.shape[0], y.shape[1], float(alpha), P(x), ld_of(x), float(beta), P(y),
         ld_of(y), ctx.stream)


def gather_cols(ctx, x, first, ncols, limit, y, d=None):
    """y[:, c] = x[:, *first + c] (/ d) for c < ncols, *first + c < limit;
    ``first`` is a one-element int32 device tensor."""
    x, y = as_block(x), as_block(y)
    call("svdsb_gather_cols", y.shape[0], P(x), ld_of(x), P(first), int(ncols), int(limit),
         None if d is None else P(d), P(y), ld_of(y), ctx.stream)


def set_int(ctx, dst, v):
    call("svdsb_set_int", P(dst), int(v), ctx.stream)


def split_stats(ctx, nsplit, r, x, out):
    r, x = as_block(r), as_block(x)
    call("svdsb_split_stats", ctx.handle, r.shape[0], int(nsplit), P(r), ld_of(r), P(x), ld_of(x),
         r.shape[1], P(out), ctx.stream)


def split_residual(ctx, nsplit, r, x, lam, stats, out):
    r, x = as_block(r), as_block(x)
    call("svdsb_split_residual", ctx.handle, r.shape[0], int(nsplit), P(r), ld_of(r), P(x), ld_of(x),
         r.shape[1], P(lam), P(stats), P(out), ctx.stream)


def syev_small(ctx, h, g, order, shift, w, y):
    call("svdsb_syev_small", int(g), P(h), ld_of(h), int(order), float(shift), P(w), P(y), ld_of(y),
         ctx.stream)


def syev_update(ctx, h, g0, b, y0, l0, order, shift, w, y):
    call("svdsb_syev_update", int(g0), int(b), P(h), ld_of(h), P(y0), ld_of(y0) if y0 is not None else 1,
         P(l0), int(order), float(shift), P(w), P(y), ld_of(y), ctx.stream)


def refined_small(ctx, r, h, g, y, lam, sv=None):
    call("svdsb_refined_small", int(g), P(r), ld_of(r), P(h), ld_of(h), P(y), P(lam), P(sv),
         ctx.stream)


def restart_coefs(ctx, g, gmax, yfirst, yall, ny, retain, exclude, prev, nprev, prev_g, plus_k,
                  out, count_dev):
    call("svdsb_restart_coefs", int(g), int(gmax), P(yfirst), P(yall), ld_of(yall), int(ny),
         int(retain), P(exclude), P(prev), ld_of(prev) if prev is not None else 1, int(nprev),
         int(prev_g), int(plus_k), P(out), ld_of(out), P(count_dev), ctx.stream)


def project_small(ctx, h, g, c, s, hout):
    call("svdsb_project_small", int(g), int(s), P(h), ld_of(h), P(c), ld_of(c), P(hout), ld_of(hout),
         ctx.stream)


def qr_small(ctx, r, g, yc, s, qy, ry):
    call("svdsb_qr_small", int(g), int(s), P(r), ld_of(r), P(yc), ld_of(yc), P(qy), ld_of(qy),
         P(ry), ld_of(ry), ctx.stream)


def h_insert(ctx, g, b, hc, h):
    call("svdsb_h_insert", int(g), int(b), P(hc), ld_of(hc), P(h), ld_of(h), ctx.stream)


def h_symmetrize(ctx, g, gm, h):
    call("svdsb_h_symmetrize", int(g), P(gm), ld_of(gm), P(h), ld_of(h), ctx.stream)


def small_matrix(rows, cols, device=None):
    """Column-major small device matrix (rows x cols), zero-filled."""
    ctx = context(device)
    return torch.zeros((cols, rows), dtype=DTYPE, device=ctx.device).t()


def fetch(ctx, tensors):
    """Copy small 1-D device tensors to host with ONE stream
    synchronisation (the per-iteration status read): one cudaMemcpyAsync
    per tensor into pinned memory, then a stream sync, all through
    libsvdsb.  Returns numpy arrays (copies)."""
    sizes = [int(t.numel()) for t in tensors]
    total = sum(sizes)
    if total > ctx._pinned.numel():
        ctx._pinned = torch.empty(total * 2, dtype=DTYPE, pin_memory=True)
    base = ctx._pinned.data_ptr()
    lib = _lib.load()
    off = 0
    for t, n in zip(tensors, sizes):
        if n:
            if not t.is_contiguous():
                t = t.contiguous()
            rc = lib.svdsb_d2h(base + 8 * off, t.data_ptr(), 8 * n, ctx._stream)
            if rc:
                _lib.check(rc, "svdsb_d2h")
        off += n
    rc = lib.svdsb_stream_sync(ctx._stream)
    if rc:
        _lib.check(rc, "svdsb_stream_sync")
    host = ctx._pinned[:total].numpy().copy()
    out = []
    off = 0
    for n in sizes:
        out.append(host[off:off + n])
        off += n
    return out

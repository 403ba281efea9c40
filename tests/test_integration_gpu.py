"""INTEGRATION.md's binding, exercised: the reference-side driver (here the
oracle port, which reproduces the reference bit for bit) runs on the host
and every product with A / A^T goes through the C ABI (svdsb_matvec) via
plain ctypes -- no package internals.  Because the GPU SpMV reproduces the
reference's summation order, the whole trajectory is bit-identical to the
pure-CPU run."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import csr as ocsr
from oracle import gen as ogen
from oracle import phsvds

pytestmark = pytest.mark.gpu

vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int


def _lib():
    from paper_1607_01404_b200._lib import LIB_PATH
    lib = ctypes.CDLL(LIB_PATH)
    lib.svdsb_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
    lib.svdsb_csr_create_host.argtypes = [vp, i64, i64, i64, vp, vp, vp, i32, vp, ctypes.POINTER(vp)]
    lib.svdsb_matvec.argtypes = [vp, vp, i32, vp, i64, vp, i64, i32, vp]
    lib.svdsb_csr_destroy.argtypes = [vp]
    lib.svdsb_last_error.restype = ctypes.c_char_p
    return lib


class GpuCsr:
    """Duck-typed stand-in for the host matrix: fwd/adj on the B200."""

    def __init__(self, m, n, rp, ci, va):
        self.lib = _lib()
        self.m, self.n = m, n
        self.count = 0
        self.ctx, self.h = vp(), vp()
        assert self.lib.svdsb_ctx_create(0, ctypes.byref(self.ctx)) == 0
        self._keep = [np.ascontiguousarray(a) for a in (rp, ci, va)]
        rc = self.lib.svdsb_csr_create_host(self.ctx, m, n, va.size, self._keep[0].ctypes.data,
                                            self._keep[1].ctypes.data, self._keep[2].ctypes.data, 1, None,
                                            ctypes.byref(self.h))
        assert rc == 0, self.lib.svdsb_last_error()

    def _product(self, x, transpose, rows_out):
        b = x.shape[1]
        xd = torch.empty((b, x.shape[0]), dtype=torch.float64, device="cuda")
        xd.copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
        yd = torch.empty((b, rows_out), dtype=torch.float64, device="cuda")
        rc = self.lib.svdsb_matvec(self.ctx, self.h, transpose, xd.data_ptr(), x.shape[0], yd.data_ptr(),
                                   rows_out, b, None)
        assert rc == 0, self.lib.svdsb_last_error()
        return np.asfortranarray(yd.cpu().numpy().T)

    def fwd(self, x):
        return self._product(x, 0, self.m)

    def adj(self, y):
        return self._product(y, 1, self.n)


@pytest.mark.parametrize("seed,target", [(1000, "largest"), (1003, "smallest")])
def test_reference_driver_with_gpu_matvec_is_bit_identical(seed, target):
    m, n, rp, ci, va = ogen.build_sparse(seed)
    cpu = phsvds.svds(phsvds.Csr(m, n, rp, ci, va), 5, target, 1e-12, seed=seed)
    gpu = phsvds.svds(GpuCsr(m, n, rp, ci, va), 5, target, 1e-12, seed=seed)
    assert np.array_equal(gpu["sigma"], cpu["sigma"])
    assert np.array_equal(gpu["u"], cpu["u"]) and np.array_equal(gpu["v"], cpu["v"])
    assert gpu["stage1_matvecs"] == cpu["stage1_matvecs"]
    assert gpu["stage2_matvecs"] == cpu["stage2_matvecs"]


def test_reference_driver_with_gpu_matvec_config1():
    from paper_1607_01404_b200 import workloads
    m, n, r, c, v = workloads.c1_coo(nx=32)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
    cpu = phsvds.svds(phsvds.Csr(m, n, rp, ci, va), 10, "largest", 1e-10)
    gpu = phsvds.svds(GpuCsr(m, n, rp, ci, va), 10, "largest", 1e-10)
    assert np.array_equal(gpu["sigma"], cpu["sigma"])
    assert gpu["stage1_matvecs"] == cpu["stage1_matvecs"]

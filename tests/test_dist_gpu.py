"""GPU: the row-sharded operator path (DistSvdOperator, one rank on one
B200) runs the same device kernels and reproduces the single-GPU solve;
the sharded C-apply equals the global one."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import csr as ocsr
from oracle import gen as ogen

pytestmark = pytest.mark.gpu


def test_sharded_path_one_rank_matches_plain_solve():
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve
    from paper_1607_01404_b200.dist import LOCAL, DistSvdOperator
    m, n, rp, ci, va = ogen.build_sparse(1007)
    cfg = lambda: SvdsConfig(num_svals=5, target="smallest", eps=1e-12, seed=1007)  # noqa: E731
    plain = svds_solve(SparseMatrixCsr(m, n, rp, ci, va), cfg=cfg())
    op = DistSvdOperator.from_host_csr(LOCAL, m, n, rp, ci, va)
    shard = svds_solve(op, cfg=cfg())
    assert shard.converged.all()
    assert np.array_equal(shard.sigma, plain.sigma)
    assert shard.stats.stage1_matvecs == plain.stats.stage1_matvecs
    rec = {r["seed"]: r for r in load_golden("fixtures.json")["sparse_oracle.json"]}[1007]
    assert np.abs(shard.sigma - np.array(rec["smallest5"])).max() <= rec["sigma_max"] * 1e-11


def test_sharded_jacobi_config2_small():
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve, workloads
    from paper_1607_01404_b200.dist import LOCAL, DistSvdOperator, local_jacobi
    gold = load_golden("solves.json")["c2"]
    m, n, r, c, v = workloads.c2_coo(**workloads.SMALL["c2"])
    full = SparseMatrixCsr.from_coo(m, n, r, c, v)
    op = DistSvdOperator.from_host_csr(LOCAL, m, n, full.row_ptr, full.col_idx, full.values)
    res = svds_solve(op, precond=local_jacobi(op, full),
                     cfg=SvdsConfig(num_svals=5, target="smallest", eps=1e-10, seed=0))
    assert res.converged.all()
    want = np.array(gold["sigma"])
    assert np.abs(res.sigma - want).max() <= 1e-10 * want.max()
    assert res.stats.precond_applies > 0

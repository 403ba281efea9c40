"""CPU: pin the oracle to the reference.  The oracle's CSR assembly / SpMV
must reproduce the reference's outputs bit for bit (digests made by the
reference itself, tests/golden/spmv.json), its generators the reference's
matrices (generators.json), and its full solve the reference's solves
(solves.json) -- same singular values to the last bit and the same matvec,
restart and preconditioner counts."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import csr as ocsr
from oracle import gen as ogen
from oracle import phsvds


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_spmv_digests_match_reference():
    for rec in load_golden("spmv.json"):
        rng = np.random.default_rng(rec["seed"])
        m, n = int(rng.integers(50, 400)), int(rng.integers(50, 400))
        nnz = int(rng.integers(100, 5000))
        r, c = rng.integers(0, m, nnz), rng.integers(0, n, nnz)
        v = rng.standard_normal(nnz) * 10.0 ** rng.uniform(-6, 6, nnz)
        rp, ci, va = ocsr.csr_from_coo(m, n, r, c, v)
        assert ogen.csr_digest(rp, ci, va) == rec["csr"]
        for b in (1, 4):
            x = rng.standard_normal((n, b))
            y = rng.standard_normal((m, b))
            if b != rec["b"]:
                continue
            assert _digest(np.asfortranarray(ocsr.spmv(m, n, rp, ci, va, x))) == rec["fwd"]
            assert _digest(np.asfortranarray(ocsr.spmv(m, n, rp, ci, va, y, transpose=True))) == rec["adj"]


def test_spmv_vectorised_equals_explicit_fold(rng):
    """The numpy SpMV equals the per-row fold the CUDA kernel implements."""
    m, n = 60, 45
    r, c = rng.integers(0, m, 900), rng.integers(0, n, 900)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, rng.standard_normal(900))
    x = rng.standard_normal((n, 2))
    y = rng.standard_normal((m, 2))
    assert np.array_equal(ocsr.spmv(m, n, rp, ci, va, x), ocsr.spmv_loop(m, n, rp, ci, va, x))
    assert np.array_equal(ocsr.spmv(m, n, rp, ci, va, y, True), ocsr.spmv_loop(m, n, rp, ci, va, y, True))


def test_generators_match_reference():
    g = load_golden("generators.json")
    for seed in ogen.SPARSE_SEEDS:
        _, _, rp, ci, va = ogen.build_sparse(seed)
        assert ogen.csr_digest(rp, ci, va) == g["sparse"][str(seed)]
    assert ogen.csr_digest(*ogen.build_clustered()[2:]) == g["clustered"]
    assert ogen.csr_digest(*ogen.build_rect50x30()[2:]) == g["rect50x30"]
    sigma = np.geomspace(1e-3, 1.0, 60)[::-1].copy()
    assert ogen.csr_digest(*ogen.synth_csr(sigma, 90, 60, 2200)) == g["synth2200"]


def test_workload_generators_match_reference():
    from paper_1607_01404_b200 import workloads
    g = load_golden("generators.json")
    for key, wl in workloads.CONFIGS.items():
        m, n, r, c, v = wl.build(**workloads.SMALL[key])
        assert ogen.csr_digest(*ocsr.csr_from_coo(m, n, r, c, v)) == g["configs"][key], key


def test_transpose_is_from_coo_of_swapped_triplets(rng):
    m, n = 70, 50
    r, c = rng.integers(0, m, 600), rng.integers(0, n, 600)
    rp, ci, va = ocsr.csr_from_coo(m, n, r, c, rng.standard_normal(600))
    t_rp, t_ci, t_va = ocsr.csr_transpose(m, n, rp, ci, va)
    d = np.zeros((m, n))
    d[np.repeat(np.arange(m), np.diff(rp)), ci] = va
    dt = np.zeros((n, m))
    dt[np.repeat(np.arange(n), np.diff(t_rp)), t_ci] = t_va
    assert np.array_equal(d.T, dt)


def test_from_coo_sums_duplicates_in_input_order():
    rp, ci, va = ocsr.csr_from_coo(2, 2, [0, 0, 1], [0, 0, 1], [1.0, 2.0, 5.0])
    assert rp.tolist() == [0, 1, 2] and ci.tolist() == [0, 1] and va.tolist() == [3.0, 5.0]
    # (0 + 1e16) + 1.0 + (-1e16) ordering matters
    rp, ci, va = ocsr.csr_from_coo(1, 1, [0, 0, 0], [0, 0, 0], [1e16, 1.0, -1e16])
    assert va[0] == (1e16 + 1.0) - 1e16


@pytest.mark.parametrize("key", ["c1", "c2", "c3L", "c3S", "c5"])
def test_port_reproduces_reference_solves(key):
    from paper_1607_01404_b200 import workloads
    gold = load_golden("solves.json")[key]
    wl = workloads.CONFIGS[key]
    m, n, r, c, v = wl.build(**workloads.SMALL[key])
    mat = phsvds.Csr(m, n, *ocsr.csr_from_coo(m, n, r, c, v))
    pre = phsvds.Jacobi(mat, "auto") if wl.precond else None
    out = phsvds.svds(mat, wl.k, wl.which, wl.tol, seed=0, block=wl.block, precond=pre, max_matvecs=60000)
    assert np.array_equal(out["sigma"], np.array(gold["sigma"]))
    assert out["stage1_matvecs"] == gold["stage1_matvecs"]
    assert out["stage2_matvecs"] == gold["stage2_matvecs"]
    assert out["restarts"] == gold["restarts"]
    assert out["precond_applies"] == gold["precond_applies"]
    assert out["status"] == gold["status"]


def test_port_reproduces_stage2_refined_solve():
    gold = load_golden("solves.json")["clustered_S"]
    mat = phsvds.Csr(*ogen.build_clustered())
    out = phsvds.svds(mat, 5, "smallest", 1e-12, seed=0)
    assert np.array_equal(out["sigma"], np.array(gold["sigma"]))
    assert out["stage2_matvecs"] == gold["stage2_matvecs"] > 0
    assert list(out["converged"]) == gold["converged"]


def test_port_matches_reference_fixture_values():
    """Criterion-1 golden values (sparse_oracle.json) from the port."""
    fx = {r["seed"]: r for r in load_golden("fixtures.json")["sparse_oracle.json"]}
    for seed in (1000, 1007):
        mat = phsvds.Csr(*ogen.build_sparse(seed))
        rec = fx[seed]
        for target in ("largest", "smallest"):
            out = phsvds.svds(mat, 5, target, 1e-12, seed=seed)
            assert np.abs(out["sigma"] - np.array(rec[target + "5"])).max() <= rec["sigma_max"] * 1e-11


def _big_case(name):
    from paper_1607_01404_b200 import workloads
    gold = load_golden("big_solves.json")[name]
    wl = workloads.CONFIGS[gold["config"]]
    m, n, r, c, v = wl.build(**gold["kwargs"])
    mat = phsvds.Csr(m, n, *ocsr.csr_from_coo(m, n, r, c, v))
    return gold, wl, mat


@pytest.mark.parametrize("name", ["c2_full", "c3L_40",
                                  pytest.param("c4_mid", marks=pytest.mark.skipif(
                                      not __import__("os").environ.get("SVDSB_SLOW_TESTS"),
                                      reason="~3 min of CPU: set SVDSB_SLOW_TESTS=1"))])
def test_port_reproduces_reference_big_solves(name):
    """Full-size config 2 (the benchmarked solve) and mid-scale configs 3L /
    4: the port returns the reference's sigma, U and V bit for bit
    (big_solves.json digests, made by tests/golden/make_golden.py big)."""
    gold, wl, mat = _big_case(name)
    assert ogen.csr_digest(mat.row_ptr, mat.col_idx, mat.values) == gold["csr"]
    pre = phsvds.Jacobi(mat, "auto") if wl.precond else None
    out = phsvds.svds(mat, wl.k, wl.which, wl.tol, seed=0, block=wl.block, precond=pre)
    assert np.array_equal(out["sigma"], np.array(gold["sigma"]))
    assert out["stage1_matvecs"] == gold["stage1_matvecs"]
    assert out["stage2_matvecs"] == gold["stage2_matvecs"]
    assert out["restarts"] == gold["restarts"]
    assert _digest(np.asfortranarray(out["u"])) == gold["u_digest"]
    assert _digest(np.asfortranarray(out["v"])) == gold["v_digest"]

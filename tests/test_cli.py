"""Command-line driver, binary CSR cache and synthetic-spectrum generator.

CPU tests: flag handling and input errors, the byte layout of the CSR cache
(hit, stale key, truncation), and the generator's bits against the
reference's digest (tests/golden/generators.json).  GPU tests replay the
reference's CLI cases (/root/reference/pkg/tests/test_cli.py) through the
device solver."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from oracle import gen as ogen

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
DIAG5 = ["--synth", "diag:1,2,3,4,5", "--num-svals", "2", "--target", "smallest", "--tol", "1e-10"]


def _cli():
    from paper_1607_01404_b200 import cli
    return cli


def _json_run(capsys, argv):
    code = _cli().main(argv + ["--format", "json"])
    out = capsys.readouterr().out
    return code, json.loads(out), out


def _rect_mtx(tmp_path):
    from paper_1607_01404_b200 import SparseMatrixCsr, write_matrix_market
    m, n, rp, ci, va = ogen.build_rect50x30()
    path = tmp_path / "rect50x30.mtx"
    write_matrix_market(str(path), SparseMatrixCsr(m, n, rp, ci, va))
    return str(path)


# ------------------------------------------------------------------ CPU
def test_bad_target_and_conflicting_inputs(capsys):
    cli = _cli()
    assert cli.main(["--synth", "diag:1,2", "--target", "middle"]) == 1
    assert "bad target" in capsys.readouterr().err
    assert cli.main(["--synth", "diag:1,2", "--matrix", "x.mtx"]) == 1
    assert "exactly one" in capsys.readouterr().err
    assert cli.main(["--synth", "cond:0.5:3x3"]) == 1
    assert "KAPPA >= 1" in capsys.readouterr().err
    assert cli.main(["--synth", "nope:1"]) == 1
    assert cli.main(["--synth", "diag:1,2", "--tol", "2"]) == 1
    assert "--tol" in capsys.readouterr().err
    assert cli.main(["--bogus-flag"]) == 1


def test_missing_matrix_names_path(capsys):
    """test_cli.py:35-39."""
    assert _cli().main(["--matrix", "missing.mtx"]) == 1
    assert "missing.mtx" in capsys.readouterr().err


def test_synth_matrix_bits_match_reference_digest():
    """synth_matrix restates matio.py:347-362; the clustered fixture it
    builds (gen_fixtures.py) must match the reference's digest."""
    from paper_1607_01404_b200 import SpectrumSpec, synth_matrix
    g = json.load(open(os.path.join(GOLDEN, "generators.json")))
    a = synth_matrix(SpectrumSpec(sigma=ogen.cluster_sigma(), m=300, n=200, seed=ogen.CLUSTER_SEED))
    assert ogen.csr_digest(a.row_ptr, a.col_idx, a.values) == g["clustered"]
    with pytest.raises(ValueError):
        SpectrumSpec(sigma=[1.0, 2.0], m=3, n=3)
    with pytest.raises(ValueError):
        SpectrumSpec(sigma=[1.0, -1.0], m=2, n=2)


def test_csr_cache_roundtrip_and_staleness(tmp_path):
    """save_csr / load_csr round trip bit for bit; a cache whose source key
    differs from the file is ignored (the matrix is re-read), a truncated
    cache is a miss, and a hit never parses the source."""
    from paper_1607_01404_b200 import SparseMatrixCsr, load_csr, read_matrix_market, save_csr
    from paper_1607_01404_b200 import mmio
    m, n, rp, ci, va = ogen.build_rect50x30()
    a = SparseMatrixCsr(m, n, rp, ci, va)
    path = tmp_path / "a.csrb"
    save_csr(str(path), a)
    b = load_csr(str(path))
    assert (b.m, b.n) == (m, n)
    assert np.array_equal(b.row_ptr, rp) and np.array_equal(b.col_idx, ci)
    assert np.array_equal(b.values.view(np.int64), va.view(np.int64))
    raw = path.read_bytes()
    (tmp_path / "cut.csrb").write_bytes(raw[:-8])
    with pytest.raises(ValueError):
        load_csr(str(tmp_path / "cut.csrb"))
    # a "source" that is not Matrix Market at all: only a cache hit can read it
    src = tmp_path / "garbage.mtx"
    src.write_text("not a matrix market file\n")
    save_csr(str(src) + ".csrb", a, source_key=mmio._source_key(str(src)))
    c = read_matrix_market(str(src), cache=True)
    assert np.array_equal(c.values, va)
    os.utime(str(src), ns=(1, 1))          # source changed: stale cache
    with pytest.raises(mmio.MatrixMarketError):
        read_matrix_market(str(src), cache=True)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_diag_smallest_json(capsys):
    """test_cli.py:27-33."""
    code, report, _ = _json_run(capsys, DIAG5)
    assert code == 0
    assert np.allclose(report["values"], [1.0, 2.0], atol=1e-8)
    assert all(r <= 5e-10 for r in report["rnorms"])
    assert report["converged"] == [True, True]
    assert report["status"] == "ok"
    assert set(report) == {"request", "values", "rnorms", "converged", "converged_count", "status", "stats",
                           "solver"}
    assert set(report["stats"]) == {"stage1_matvecs", "stage2_matvecs", "precond_applies", "restarts", "resets",
                                    "seconds"}


@pytest.mark.gpu
def test_fixture_largest_matches_committed_oracle(capsys, tmp_path):
    """test_cli.py:41-52 with the reference's committed expected values."""
    fx = json.load(open(os.path.join(GOLDEN, "fixtures.json")))["rect50x30_expected.json"]["largest5"]
    code, report, _ = _json_run(capsys, ["--matrix", _rect_mtx(tmp_path), "--num-svals", "5", "--target",
                                         "largest", "--tol", "1e-8"])
    assert code == 0
    got, want = np.array(report["values"]), np.array(fx)
    assert (np.abs(got - want) <= 1e-7 * want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["--synth", "cond:100:80x50", "--num-svals", "2", "--target", "smallest", "--max-matvecs", "6"],
    ["--synth", "diag:1,2,3,4,5", "--num-svals", "2", "--target", "closest:2.2,3.7", "--max-matvecs", "1"],
])
def test_starved_budget_exits_partial(capsys, argv):
    """test_cli.py:54-70."""
    code, report, _ = _json_run(capsys, argv)
    assert code == 2
    assert report["status"] == "budget"
    assert report["converged_count"] == 0
    assert len(report["values"]) == 2
    assert all(r is None or r >= 0.0 for r in report["rnorms"])


@pytest.mark.gpu
def test_zero_svals_and_closest_and_jacobi(capsys):
    """test_cli.py:72-92."""
    code, report, _ = _json_run(capsys, ["--synth", "diag:1,2,3", "--num-svals", "0"])
    assert code == 0 and report["values"] == [] and report["converged_count"] == 0
    code, report, _ = _json_run(capsys, ["--synth", "diag:1,2,3,4,5,6,7", "--num-svals", "2", "--target",
                                         "closest:3.4,6.2", "--tol", "1e-9"])
    assert code == 0
    assert np.allclose(report["values"], [4.0, 7.0], atol=1e-6)
    code, report, _ = _json_run(capsys, ["--synth", "cond:1000:60x40", "--num-svals", "2", "--target", "smallest",
                                         "--tol", "1e-6", "--precond", "jacobi"])
    assert code == 0
    assert report["stats"]["precond_applies"] > 0


@pytest.mark.gpu
def test_text_report_and_library_agreement(capsys):
    """test_cli.py:105-148: the text layout, and the JSON report equal to a
    library run field for field."""
    from paper_1607_01404_b200 import SparseMatrixCsr, SvdsConfig, svds_solve
    cli = _cli()
    assert cli.main(["--synth", "diag:3", "--num-svals", "1", "--target", "largest", "--tol", "1e-10"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert re.match(r"^1 3(\.0+)? \d\.\d{3}e[+-]\d+$", lines[0])
    assert "status ok" in lines and "converged 1/1" in lines
    code, report, raw = _json_run(capsys, DIAG5)
    idx = np.arange(5, dtype=np.int64)
    res = svds_solve(SparseMatrixCsr.from_coo(5, 5, idx, idx, np.arange(1.0, 6.0)),
                     cfg=SvdsConfig(num_svals=2, target="smallest", eps=1e-10, seed=0))
    assert report["values"] == [float(s) for s in res.sigma]
    assert report["rnorms"] == [float(r) for r in res.rnorms]
    assert report["stats"]["stage1_matvecs"] == res.stats.stage1_matvecs
    assert json.loads(raw) == report


@pytest.mark.gpu
def test_process_runs_byte_identical_and_vectors(tmp_path):
    """test_cli.py:151-190: two processes give the same report except
    seconds; written vectors reproduce the reported residuals; the second
    run reads the binary CSR cache."""
    from paper_1607_01404_b200 import SvdOperator, compute_svd_residual, read_dense_market, read_matrix_market
    mtx = _rect_mtx(tmp_path)
    vec = str(tmp_path / "vectors.mtx")
    argv = [sys.executable, "-m", "paper_1607_01404_b200.cli", "--matrix", mtx, "--num-svals", "3", "--target",
            "largest", "--tol", "1e-9", "--seed", "11", "--format", "json", "--csr-cache", "--write-vectors", vec]
    outs = []
    for _ in range(2):
        proc = subprocess.run(argv, capture_output=True, text=True, cwd=REPO)
        assert proc.returncode == 0, proc.stderr
        outs.append(proc.stdout)
    assert os.path.exists(mtx + ".csrb")

    def strip(text):
        return "\n".join(ln for ln in text.splitlines() if '"seconds"' not in ln)
    assert strip(outs[0]) == strip(outs[1])
    report = json.loads(outs[1])
    stacked = read_dense_market(vec)
    assert stacked.shape == (80, 3)
    op = SvdOperator.wrap(read_matrix_market(mtx))
    for i, (sigma, rnorm) in enumerate(zip(report["values"], report["rnorms"])):
        again = compute_svd_residual(op, sigma, stacked[30:, i], stacked[:30, i])
        assert again <= 2.0 * rnorm and rnorm <= 2.0 * again


@pytest.mark.gpu
def test_cond_json(capsys):
    """test_cli.py:193-200."""
    code, report, _ = _json_run(capsys, ["--synth", "cond:100:40x30", "--mode", "cond"])
    assert code == 0
    assert not report["infinite"] and not report["lower_bound"]
    assert abs(report["kappa"] - 100.0) <= 10.0
    assert abs(report["sigma_max"] - 1.0) <= 0.1

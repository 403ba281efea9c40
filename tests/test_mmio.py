"""Matrix Market ingestion (native parser, csrc/mmio.cpp) against the
reference reader's outcomes on the golden cases in tests/golden/mmio.json
(made by tests/golden/make_mmio_golden.py from pkg/src/itersvd/matio.py):
the same CSR bit for bit (assembled here by the oracle's from_coo), or the
same MatrixMarketError message and line.  Writers: byte-identical text."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import csr as ocsr
from paper_1607_01404_b200 import MatrixMarketError, mmio

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "mmio.json")) as f:
    GOLD = json.load(f)
CASES = sorted(k for k in GOLD if not k.startswith("_"))


def _write(tmp_path, name, text):
    p = tmp_path / (name + ".mtx")
    with open(p, "w", newline="") as f:
        f.write(text)
    return p


def _digest(rp, ci, va):
    h = hashlib.sha256()
    for arr in (rp, ci, va):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", CASES)
def test_reader_matches_reference(tmp_path, name):
    case = GOLD[name]
    path = _write(tmp_path, name, case["text"])
    ref = case["ref"]
    if "error" in ref:
        with pytest.raises(MatrixMarketError) as ei:
            mmio.read_matrix_market_coo(path)
        assert str(ei.value) == ref["error"]
        assert ei.value.line == ref["line"]
        return
    m, n, rows, cols, vals, _ = mmio.read_matrix_market_coo(path)
    assert (m, n) == (ref["m"], ref["n"])
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)
    assert va.shape[0] == ref["nnz"]
    assert _digest(rp, ci, va) == ref["digest"]


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(OSError):
        mmio.read_matrix_market_coo(tmp_path / "nope.mtx")


def test_coo_writer_matches_reference(tmp_path):
    w = GOLD["_writers"]
    src = _write(tmp_path, "src", GOLD[w["coo_source"]]["text"])
    m, n, rows, cols, vals, _ = mmio.read_matrix_market_coo(src)
    rp, ci, va = ocsr.csr_from_coo(m, n, rows, cols, vals)

    class Host:  # the writer only reads the reference CSR attributes
        pass
    a = Host()
    a.m, a.n, a.row_ptr, a.col_idx, a.values = m, n, rp, ci, va
    out = tmp_path / "w.mtx"
    mmio.write_matrix_market(out, a)
    assert out.read_text() == w["coo_text"]


def test_dense_round_trip_matches_reference(tmp_path):
    w = GOLD["_writers"]
    blk = np.array(w["dense"], dtype=np.float64)
    out = tmp_path / "wd.mtx"
    mmio.write_dense_market(out, blk)
    assert out.read_text() == w["dense_text"]
    back = mmio.read_dense_market(out)
    assert back.flags.f_contiguous
    same = (back == blk) | (np.isnan(back) & np.isnan(blk))
    assert same.all()


def test_large_file_parses_fast(tmp_path):
    rng = np.random.default_rng(3)
    nnz = 200_000
    r = rng.integers(1, 5001, nnz)
    c = rng.integers(1, 3001, nnz)
    v = rng.standard_normal(nnz)
    p = tmp_path / "big.mtx"
    with open(p, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n" + "5000 3000 %d\n" % nnz)
        f.write("".join("%d %d %.17g\n" % t for t in zip(r, c, v)))
    m, n, rows, cols, vals, _ = mmio.read_matrix_market_coo(p)
    assert (m, n) == (5000, 3000)
    np.testing.assert_array_equal(rows, r - 1)
    np.testing.assert_array_equal(cols, c - 1)
    np.testing.assert_array_equal(vals, v)

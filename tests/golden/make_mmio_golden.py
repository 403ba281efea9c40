"""Matrix Market golden cases from the reference reader (run in the build
container, the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mmio_golden.py

Each case is a file text (synthetic, written here) plus the reference's
outcome on it -- ``itersvd.read_matrix_market`` (pkg/src/itersvd/
matio.py:170-241): the CSR digest, or the MatrixMarketError message and
line.  Writes tests/golden/mmio.json.
"""

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(REF, "src"))

from itersvd import matio  # noqa: E402

H = "%%MatrixMarket matrix coordinate real general\n"


def digest(a):
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.values):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def cases():
    rng = np.random.default_rng(7)
    c = {}
    c["general"] = H + "% comment\n\n3 4 5\n1 1 1.5\n3 4 -2e-3\n2 2 .5\n1 4 +2.\n3 1 1_000.25\n"
    c["duplicates"] = H + "2 2 4\n1 1 0.1\n1 1 0.2\n2 1 3\n1 1 0.3\n"
    c["symmetric_int"] = ("%%MatrixMarket matrix coordinate integer symmetric\n3 3 4\n1 1 2\n2 1 -1\n"
                          "3 2 -1\n3 3 2\n")
    c["array"] = "%%MatrixMarket matrix array real general\n2 3\n1\n0\n0\n4.5\n-0.0\n6\n"
    c["crlf"] = H.replace("\n", "\r\n") + "2 2 2\r\n1 1 1\r\n2 2 2\r\n"
    c["cr_only"] = H.replace("\n", "\r") + "2 2 1\r2 1 7.25\r"
    c["no_trailing_newline"] = H + "1 1 1\n1 1 3.5"
    c["upper_banner_double"] = "%%MATRIXMARKET MATRIX COORDINATE DOUBLE GENERAL\n1 2 1\n1 2 1e300\n"
    c["specials"] = H + "1 3 3\n1 1 inf\n1 2 -Infinity\n1 3 NaN\n"
    c["tabs_and_ws"] = H + "  2\t2  1 \n\t1   2\t  9.5e+1  \n"
    c["empty_entries"] = H + "3 2 0\n"
    c["zero_dims"] = H + "0 0 0\n"
    # a bigger random one (with duplicates)
    rows = rng.integers(1, 41, 300)
    cols = rng.integers(1, 31, 300)
    vals = rng.standard_normal(300)
    c["random"] = H + "40 30 300\n" + "".join("%d %d %.17g\n" % t for t in zip(rows, cols, vals))
    # errors
    c["err_empty"] = ""
    c["err_banner"] = "%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n"
    c["err_short_banner"] = "%%MatrixMarket matrix coordinate\n1 1 1\n1 1 1\n"
    c["err_object"] = "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n"
    c["err_format"] = "%%MatrixMarket matrix sparse real general\n1 1 1\n1 1 1\n"
    c["err_pattern"] = "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n"
    c["err_complex"] = "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n"
    c["err_hermitian"] = "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n"
    c["err_array_symmetric"] = "%%MatrixMarket matrix array real symmetric\n1 1\n1\n"
    c["err_no_size"] = H + "% only comments\n\n"
    c["err_size_tokens"] = H + "3 3\n1 1 1\n"
    c["err_size_float"] = H + "3 3 1.0\n1 1 1\n"
    c["err_negative"] = H + "-1 3 0\n"
    c["err_too_many"] = H + "2 2 1\n1 1 1\n% c\n2 2 2\n"
    c["err_too_few"] = H + "2 2 3\n1 1 1\n2 2 2\n\n"
    c["err_entry_tokens"] = H + "2 2 2\n1 1 1\n2 2\n"
    c["err_index_float"] = H + "2 2 1\n1.0 1 1\n"
    c["err_hex_value"] = H + "2 2 1\n1 1 0x1p3\n"
    c["err_underscore"] = H + "2 2 1\n1 1 _1\n"
    c["err_zero_index"] = H + "2 2 1\n0 1 1\n"
    c["err_out_of_range"] = H + "2 2 1\n1 3 1\n"
    c["err_sym_nonsquare"] = ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n")
    c["err_array_extra"] = "%%MatrixMarket matrix array real general\n1 2\n1\n2\n3\n"
    c["err_array_bad"] = "%%MatrixMarket matrix array real general\n1 2\n1 2\n3\n"
    return c


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in cases().items():
            path = os.path.join(d, name + ".mtx")
            with open(path, "w", newline="") as f:
                f.write(text)
            try:
                a = matio.read_matrix_market(path)
                res = {"m": a.m, "n": a.n, "nnz": a.nnz, "digest": digest(a)}
            except matio.MatrixMarketError as e:
                res = {"error": str(e), "line": e.line}
            out[name] = {"text": text, "ref": res}
        # writer pins: the reference's output text for a parsed matrix and a
        # dense block
        a = matio.read_matrix_market(os.path.join(d, "random.mtx"))
        matio.write_matrix_market(os.path.join(d, "w.mtx"), a)
        blk = np.random.default_rng(11).standard_normal((5, 3))
        blk[0, 0], blk[1, 1], blk[2, 2] = np.inf, -0.0, 1e-310
        matio.write_dense_market(os.path.join(d, "wd.mtx"), blk)
        with open(os.path.join(d, "w.mtx")) as f:
            wc = f.read()
        with open(os.path.join(d, "wd.mtx")) as f:
            wd = f.read()
        out["_writers"] = {"coo_source": "random", "coo_text": wc, "dense": blk.tolist(), "dense_text": wd}
    with open(os.path.join(HERE, "mmio.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()

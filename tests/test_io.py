"""Row f3: the Matrix Market / CSV readers against the
reference readers' own outputs on every accepted variant and every
ParseError path (tests/golden/io_cases.json, made by make_io_golden.py from
rsvdkit matrix.py:316-432), plus a write -> read round trip. CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1504_05477_b200 import ParseError, SparseMatrixCSR, io

CASES = json.load(open(os.path.join(GOLDEN, "io_cases.json")))


def _check(fn, text, ref, tmp_path, suffix):
    p = tmp_path / f"case{suffix}"
    p.write_text(text)
    if not ref["ok"]:
        with pytest.raises(Exception) as ei:
            fn(str(p))
        assert type(ei.value).__name__ == ref["type"]
        assert str(ei.value) == ref["message"]
        assert getattr(ei.value, "line", None) == ref["line"]
        return
    got = fn(str(p))
    if "row_ptr" in ref:
        assert list(got.shape) == ref["shape"]
        assert got.row_ptr.tolist() == ref["row_ptr"]
        assert got.col_idx.tolist() == ref["col_idx"]
        assert got.values.tolist() == ref["values"]
    else:
        assert list(got.data.shape) == ref["shape"]
        assert got.data.tolist() == ref["data"]


@pytest.mark.parametrize("name", sorted(CASES["mm"]))
def test_matrix_market_matches_reference(name, tmp_path):
    c = CASES["mm"][name]
    _check(io.load_matrix_market, c["text"], c["ref"], tmp_path, ".mtx")


@pytest.mark.parametrize("name", sorted(CASES["csv"]))
def test_dense_csv_matches_reference(name, tmp_path):
    c = CASES["csv"][name]
    _check(io.load_dense_csv, c["text"], c["ref"], tmp_path, ".csv")


def test_parse_error_is_value_error_with_line(tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n9 9 1\n")
    with pytest.raises(ValueError) as ei:
        io.load_matrix_market(str(p))
    assert isinstance(ei.value, ParseError) and ei.value.line == 3


def test_write_read_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    dense = rng.standard_normal((7, 5)) * (rng.random((7, 5)) < 0.4)
    for A in (dense, SparseMatrixCSR.from_coo(7, 5, *np.nonzero(dense), dense[np.nonzero(dense)])):
        p = tmp_path / "rt.mtx"
        io.write_matrix_market(A, str(p))
        back = io.load_matrix_market(str(p))
        assert np.array_equal(back.toarray(), dense)  # 17 significant digits round-trip FP64 exactly


def test_dense_csv_write_read_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    dense = rng.standard_normal((6, 4))
    p = tmp_path / "rt.csv"
    io.write_dense_csv(dense, str(p))
    assert np.array_equal(io.load_dense_csv(str(p)).data, dense)
    sp = SparseMatrixCSR.from_coo(3, 3, [0, 2], [1, 2], [1.5, -2.0])
    io.write_dense_csv(sp, str(p))
    assert np.array_equal(io.load_dense_csv(str(p)).data, sp.toarray())

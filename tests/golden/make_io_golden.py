"""Golden outputs of the REFERENCE file readers (rsvdkit 0.1.0
matrix.load_matrix_market / load_dense_csv, matrix.py:316-432) on small
hand-written inputs covering every accepted variant and every ParseError
path. Run in the build container only (imports the reference):

    RSVDKIT_SRC=/root/reference/pkg/src RSVD_BACKEND=python python tests/golden/make_io_golden.py

Writes io_cases.json next to this script: per case the file text and either
the CSR arrays or the exception (type, message, line)."""

import json
import os
import sys
import tempfile

os.environ.setdefault("RSVD_BACKEND", "python")
sys.path.insert(0, os.environ.get("RSVDKIT_SRC", "/root/reference/pkg/src"))
from rsvdkit import matrix as rm  # noqa: E402

H = "%%MatrixMarket matrix coordinate"
MM = {
    "general_dups_comments": f"{H} real general\n% comment\n\n3 4 4\n1 1 1.5\n2 3 -2\n3 4 7e-3\n1 1 0.5\n",
    "symmetric": f"{H} real symmetric\n3 3 3\n1 1 2\n2 1 3\n3 2 -1\n",
    "pattern": f"{H} pattern general\n2 2 2\n1 2\n2 1\n",
    "integer": f"{H} integer general\n2 2 1\n2 2 5\n",
    "uppercase_header": "%%MatrixMarket MATRIX Coordinate REAL General\n1 2 1\n1 2 4\n",
    "empty_rows": f"{H} real general\n4 3 2\n4 3 1\n1 1 2\n",
    "cancelling_duplicates": f"{H} real general\n2 2 2\n1 1 1\n1 1 -1\n",
    "zero_nnz": f"{H} real general\n2 5 0\n",
    "missing_header": "% x\n1 1 1\n",
    "header_4_tokens": f"{H} real\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex_field": f"{H} complex general\n1 1 0\n",
    "skew_symmetric": f"{H} real skew-symmetric\n1 1 0\n",
    "missing_size": f"{H} real general\n% only comments\n\n",
    "bad_size_token": f"{H} real general\n3 x 4\n",
    "size_two_tokens": f"{H} real general\n3 4\n",
    "size_out_of_range": f"{H} real general\n0 4 1\n",
    "entry_missing_value": f"{H} real general\n2 2 1\n1 1\n",
    "entry_bad_number": f"{H} real general\n2 2 1\n1 a 1\n",
    "entry_out_of_bounds": f"{H} real general\n2 2 1\n3 1 1\n",
    "entry_nan": f"{H} real general\n2 2 1\n1 1 nan\n",
    "entry_inf": f"{H} real general\n2 2 1\n1 1 -inf\n",
    "more_than_declared": f"{H} real general\n2 2 1\n1 1 1\n2 2 1\n",
    "fewer_than_declared": f"{H} real general\n2 2 3\n1 1 1\n\n% tail\n",
}
CSV = {
    "plain": "1,2,3\n4,5,6\n",
    "blank_lines": "\n1.5,-2\n\n3,4e-3\n",
    "ragged": "1,2\n3\n",
    "non_numeric": "1,2\n3,x\n",
    "empty": "\n\n",
}


def run(fn, text, suffix):
    with tempfile.NamedTemporaryFile("w", suffix=suffix, delete=False) as fh:
        fh.write(text)
    try:
        r = fn(fh.name)
        obj = getattr(r, "matrix", r)
        if hasattr(obj, "row_ptr"):
            return {"ok": True, "shape": list(obj.shape), "row_ptr": obj.row_ptr.tolist(),
                    "col_idx": obj.col_idx.tolist(), "values": obj.values.tolist()}
        return {"ok": True, "shape": list(obj.data.shape), "data": obj.data.tolist()}
    except Exception as e:  # noqa: BLE001 - the exception is the golden output
        return {"ok": False, "type": type(e).__name__, "message": str(e), "line": getattr(e, "line", None)}
    finally:
        os.unlink(fh.name)


out = {"mm": {k: {"text": t, "ref": run(rm.load_matrix_market, t, ".mtx")} for k, t in MM.items()},
       "csv": {k: {"text": t, "ref": run(rm.load_dense_csv, t, ".csv")} for k, t in CSV.items()}}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io_cases.json")
json.dump(out, open(path, "w"), indent=1)
print("wrote", path, len(MM), len(CSV))

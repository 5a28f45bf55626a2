"""Input formats on either side of the hot path: Matrix
Market coordinate files and dense CSV, the two file inputs the reference's
harness accepts (experiment.py:136-144), read on the host into the drop-in's
containers; `block_krylov(...)` then uploads them once (device CSR with int32
or int64 indices, FP32 or FP64 values) and keeps them resident.

Semantics follow the reference readers (matrix.py:316-398 load_matrix_market,
matrix.py:401-432 load_dense_csv, matrix.py:435-455 write_matrix_market):
same accepted header variants (coordinate; real / integer / pattern; general /
symmetric), symmetric storage expanded, pattern entries 1.0, duplicates summed
(SparseMatrixCSR.from_coo), and ParseError with the 1-based line number for
every malformed input the reference rejects. The returned container is the
drop-in's SparseMatrixCSR (the reference wraps it in a MatrixOperator; every
algorithm entry point accepts either form of input here)."""

from __future__ import annotations

import numpy as np

from .errors import ParseError
from .matrix import DenseMatrix, SparseMatrixCSR, as_dense_array

_FIELDS = ("real", "integer", "pattern")
_SYMMETRIES = ("general", "symmetric")


def load_matrix_market(path):
    """Matrix Market coordinate file -> SparseMatrixCSR (matrix.py:316-398).
    Line numbers count every physical line (blank and comment lines too)."""
    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline()
        if not header.startswith("%%MatrixMarket"):
            raise ParseError("missing %%MatrixMarket header", line=1)
        tokens = header.split()
        if len(tokens) != 5:
            raise ParseError("header must have 5 tokens", line=1)
        obj, fmt, field, symmetry = (t.lower() for t in tokens[1:])
        if obj != "matrix" or fmt != "coordinate":
            raise ParseError(f"unsupported object/format: {obj} {fmt}", line=1)
        if field not in _FIELDS:
            raise ParseError(f"unsupported field: {field}", line=1)
        if symmetry not in _SYMMETRIES:
            raise ParseError(f"unsupported symmetry: {symmetry}", line=1)
        lineno = 1
        size = None
        for raw in fh:
            lineno += 1
            text = raw.strip()
            if text and not text.startswith("%"):
                size = text.split()
                break
        if size is None:
            raise ParseError("missing size line", line=lineno)
        try:
            rows, cols, nnz = (int(t) for t in size)
        except ValueError:
            raise ParseError(f"bad size line: {' '.join(size)}", line=lineno) from None
        if rows < 1 or cols < 1 or nnz < 0:
            raise ParseError("size line entries out of range", line=lineno)
        ntok = 2 if field == "pattern" else 3
        ri = np.empty(nnz, dtype=np.int64)
        ci = np.empty(nnz, dtype=np.int64)
        vv = np.ones(nnz, dtype=np.float64)
        seen = 0
        for raw in fh:
            lineno += 1
            text = raw.strip()
            if not text or text.startswith("%"):
                continue
            tok = text.split()
            if len(tok) != ntok:
                raise ParseError(f"bad entry: {text}", line=lineno)
            try:
                i, j = int(tok[0]), int(tok[1])
                v = float(tok[2]) if ntok == 3 else 1.0
            except ValueError:
                raise ParseError(f"bad entry: {text}", line=lineno) from None
            if not (1 <= i <= rows and 1 <= j <= cols):
                raise ParseError(f"entry ({i}, {j}) outside declared {rows} x {cols} bounds", line=lineno)
            if not np.isfinite(v):
                raise ParseError(f"non-finite value: {text}", line=lineno)
            if seen == nnz:
                raise ParseError("more entries than declared", line=lineno)
            ri[seen], ci[seen], vv[seen] = i - 1, j - 1, v
            seen += 1
        if seen != nnz:
            raise ParseError(f"declared {nnz} entries, found {seen}", line=lineno)
    if symmetry == "symmetric":  # mirror the off-diagonal entries
        off = ri != ci
        ri, ci, vv = (np.concatenate([ri, ci[off]]), np.concatenate([ci, ri[off]]),
                      np.concatenate([vv, vv[off]]))
    return SparseMatrixCSR.from_coo(rows, cols, ri, ci, vv)


def load_dense_csv(path, skip_header=False):
    """Rectangular numeric CSV -> DenseMatrix (matrix.py:401-432)."""
    data = []
    width = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            if skip_header and lineno == 1:
                continue
            text = raw.strip()
            if not text:
                continue
            cells = text.split(",")
            if width is None:
                width = len(cells)
            elif len(cells) != width:
                raise ParseError(f"ragged row: expected {width} cells, found {len(cells)}", line=lineno)
            row = []
            for colno, cell in enumerate(cells, start=1):
                try:
                    row.append(float(cell))
                except ValueError:
                    raise ParseError(f"non-numeric cell at ({lineno}, {colno}): {cell!r}", line=lineno) from None
            data.append(row)
    if not data:
        raise ParseError("empty CSV file", line=1)
    return DenseMatrix(np.asarray(data, dtype=np.float64))


def write_matrix_market(A, path):
    """Matrix Market coordinate real general, 1-based, 17 significant digits
    (matrix.py:435-455): sparse input writes its stored nonzeros, dense input
    every nonzero entry in row-major order."""
    from .matrix import MatrixOperator

    if isinstance(A, MatrixOperator):
        A = A.matrix
    if isinstance(A, SparseMatrixCSR):
        rows, cols = A.shape
        r = np.repeat(np.arange(rows), np.diff(A.row_ptr))
        c, v = A.col_idx, A.values
    else:
        a = as_dense_array(A)
        rows, cols = a.shape
        r, c = np.nonzero(a)
        v = a[r, c]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{rows} {cols} {len(v)}\n")
        for i, j, x in zip(r.tolist(), c.tolist(), v.tolist()):
            fh.write(f"{i + 1} {j + 1} {x:.17g}\n")


def write_dense_csv(A, path):
    """matrix.py:458-463: one row per line, 17 significant digits (a sparse
    input is densified first)."""
    from .matrix import MatrixOperator

    if isinstance(A, MatrixOperator):
        A = A.matrix
    arr = A.toarray() if isinstance(A, SparseMatrixCSR) else as_dense_array(A)
    with open(path, "w", encoding="utf-8") as fh:
        for row in arr:
            fh.write(",".join(f"{x:.17g}" for x in row))
            fh.write("\n")

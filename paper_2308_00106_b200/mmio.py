"""Matrix Market I/O (reference: matio.py:16-23 MatrixMarketError, 151-274).

The banner and the size line (a few bytes) are read here exactly as the
reference reads them; the entry body — the part whose cost grows with nnz —
is parsed by the native multithreaded parser (sme_host_mm_parse,
mmio_host.cpp) straight into int32 index / f64 value arrays, which then become
a device CooMatrix (duplicate and range checks on the GPU, as for any
CooMatrix).  Errors carry the reference's messages and 1-based line numbers:
the native parser reports the first bad line in line order, and that one line
is re-checked here with the reference's rules to word the exception.

write_matrix_market formats with sme_host_mm_format ("%.17g", like the
reference's f"{v:.17g}") in parallel.
"""

from __future__ import annotations

import mmap
import os
from typing import IO

import numpy as np

from . import _lib
from .matio import CooMatrix

_FIELDS = ("real", "integer", "pattern")
_SYMMETRIES = ("general", "symmetric")
_FIELD_CODE = {"real": 0, "integer": 1, "pattern": 2}
# status codes of sme_host_mm_parse
_E_TOO_MANY = 1


class MatrixMarketError(ValueError):
    """Malformed Matrix Market content, with the offending 1-based line number (matio.py:16-23)."""

    def __init__(self, message: str, line_no: int | None = None):
        if line_no is not None:
            message = f"line {line_no}: {message}"
        super().__init__(message)
        self.line_no = line_no


def _source_bytes(source) -> tuple[bytes | memoryview, bool]:
    """(content, universal_newlines).  Files and byte streams are read as text files
    are (universal newlines: '\\r' and '\\r\\n' end lines); str input splits on '\\n'
    only, like io.StringIO (matio.py:140-148)."""
    if isinstance(source, bytes):
        return source, True
    if isinstance(source, str):
        return source.encode("utf-8"), False
    read = getattr(source, "read", None)
    if read is None:  # an iterable of lines
        return "".join(source).encode("utf-8"), False
    data = read()
    if isinstance(data, bytes):
        return data, True
    return data.encode("utf-8"), False


def _next_line(buf, pos: int, universal: bool) -> tuple[int, int]:
    """(end of the line starting at pos, start of the next line)."""
    n = len(buf)
    nl = buf.find(b"\n", pos)
    nl = n if nl < 0 else nl
    if universal:
        cr = buf.find(b"\r", pos, nl)
        if cr >= 0:
            return cr, cr + 2 if cr + 1 < n and buf[cr + 1 : cr + 2] == b"\n" else cr + 1
    return nl, nl + 1


def _check_entry_line(stripped: str, field: str, n_rows: int, n_cols: int, line_no: int) -> None:
    """The reference's per-entry checks (matio.py:207-232) on one line: raises its error."""
    want = 2 if field == "pattern" else 3
    parts = stripped.split()
    if len(parts) != want:
        raise MatrixMarketError(f"entry must have {want} fields", line_no)
    try:
        i, j = int(parts[0]), int(parts[1])
    except ValueError:
        raise MatrixMarketError(f"malformed indices: {stripped!r}", line_no) from None
    if not (1 <= i <= n_rows):
        raise MatrixMarketError(f"row index {i} outside [1, {n_rows}]", line_no)
    if not (1 <= j <= n_cols):
        raise MatrixMarketError(f"column index {j} outside [1, {n_cols}]", line_no)
    if field == "integer":
        try:
            float(int(parts[2]))
        except ValueError:
            raise MatrixMarketError(f"malformed integer value: {parts[2]!r}", line_no) from None
        except OverflowError:
            raise MatrixMarketError(f"integer value out of float range: {parts[2]!r}", line_no) from None
    elif field == "real":
        try:
            float(parts[2])
        except ValueError:
            raise MatrixMarketError(f"malformed value: {parts[2]!r}", line_no) from None


def parse_matrix_market(source, *, threads: int = 0, dtype=None) -> CooMatrix:
    """Parse a Matrix Market coordinate stream into a (device) CooMatrix (matio.py:151-239).

    `source` is a text or byte stream, or the file content as str/bytes.  Banner:
    `%%MatrixMarket matrix coordinate {real|integer|pattern} {general|symmetric}`.
    Indices become 0-based; `pattern` entries get 1.0; `symmetric` off-diagonal
    entries are mirrored (appended after all stored entries, in order).
    Duplicates, out-of-range indices and a wrong declared nnz are errors.
    """
    buf, universal = _source_bytes(source)
    return _parse_buffer(buf, universal, threads, dtype)


def _parse_buffer(buf, universal: bool, threads: int, dtype) -> CooMatrix:
    n_rows, n_cols, rows, cols, vals = parse_host_arrays(buf, universal, threads)
    try:
        return CooMatrix(n_rows, n_cols, rows, cols, vals, dtype=dtype)
    except ValueError as exc:
        raise MatrixMarketError(str(exc)) from None


def parse_host_arrays(buf, universal: bool = True, threads: int = 0):
    """Host half of parse_matrix_market: (n_rows, n_cols, rows int32, cols int32, vals f64)
    in the reference's entry order (mirrored symmetric entries appended), before the
    CooMatrix (device) range / duplicate checks."""
    n = len(buf)
    if n == 0:
        raise MatrixMarketError("empty input")
    end, pos = _next_line(buf, 0, universal)
    banner = bytes(buf[:end]).decode("utf-8")
    tokens = banner.split()
    if len(tokens) != 5 or tokens[0].lower() != "%%matrixmarket" or tokens[1].lower() != "matrix":
        raise MatrixMarketError(f"malformed banner: {banner.strip()!r}", 1)
    layout, field, symmetry = (t.lower() for t in tokens[2:5])
    if layout == "array":
        raise MatrixMarketError("'array' format is not supported (coordinate only)", 1)
    if layout != "coordinate":
        raise MatrixMarketError(f"unknown format {layout!r}", 1)
    if field == "complex":
        raise MatrixMarketError("'complex' field is not supported", 1)
    if field not in _FIELDS:
        raise MatrixMarketError(f"unknown field {field!r}", 1)
    if symmetry in ("skew-symmetric", "hermitian"):
        raise MatrixMarketError(f"{symmetry!r} symmetry is not supported", 1)
    if symmetry not in _SYMMETRIES:
        raise MatrixMarketError(f"unknown symmetry {symmetry!r}", 1)

    n_rows = n_cols = declared = None
    line_no = 1
    while pos < n:
        line_no += 1
        end, nxt = _next_line(buf, pos, universal)
        stripped = bytes(buf[pos:end]).decode("utf-8").strip()
        pos = nxt
        if not stripped or stripped.startswith("%"):
            continue
        parts = stripped.split()
        if len(parts) != 3:
            raise MatrixMarketError("size line must be 'rows cols nnz'", line_no)
        try:
            n_rows, n_cols, declared = (int(p) for p in parts)
        except ValueError:
            raise MatrixMarketError("size line must be 'rows cols nnz'", line_no) from None
        if n_rows < 1 or n_cols < 1 or declared < 0:
            raise MatrixMarketError("size line values out of range", line_no)
        break
    if declared is None:
        raise MatrixMarketError("missing size line")
    body = memoryview(buf)[min(pos, n):] if pos < n else memoryview(b"")
    rows = np.empty(declared, dtype=np.int32)
    cols = np.empty(declared, dtype=np.int32)
    vals = np.empty(declared, dtype=np.float64)
    status = np.zeros(4, dtype=np.int64)
    body_arr = np.frombuffer(body, dtype=np.uint8) if len(body) else np.zeros(1, dtype=np.uint8)
    _lib.call("sme_host_mm_parse", body_arr.ctypes.data, len(body), _FIELD_CODE[field], n_rows, n_cols, declared,
              line_no + 1, int(universal), int(threads), rows.ctypes.data, cols.ctypes.data, vals.ctypes.data,
              status.ctypes.data)
    code, err_line, found, off = (int(v) for v in status)
    if code == _E_TOO_MANY:
        raise MatrixMarketError(f"more than the declared {declared} entries", err_line)
    if code != 0:
        e, _ = _next_line(buf, pos + off, universal)
        text = bytes(buf[pos + off : e]).decode("utf-8", errors="replace").strip()
        _check_entry_line(text, field, n_rows, n_cols, err_line)
        raise MatrixMarketError(f"numeric literal not supported by the native parser: {text!r}", err_line)
    if found != declared:
        raise MatrixMarketError(f"declared {declared} entries but found {found}")
    if symmetry == "symmetric" and declared:
        off_diag = rows != cols
        rows, cols, vals = (np.concatenate((rows, cols[off_diag])), np.concatenate((cols, rows[off_diag])),
                            np.concatenate((vals, vals[off_diag])))
    return n_rows, n_cols, rows, cols, vals


def load_matrix_market(path: str | os.PathLike, *, threads: int = 0, dtype=None) -> CooMatrix:
    """Parse a Matrix Market file from disk (matio.py:242-245); the file is memory-mapped."""
    with open(path, "rb") as f:
        if os.fstat(f.fileno()).st_size == 0:
            raise MatrixMarketError("empty input")
        with mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ) as mm:
            return _parse_buffer(mm, True, threads, dtype)


def format_entries(rows, cols, vals, threads: int = 0) -> bytes:
    """The entry lines of _write_mm (matio.py:272-274) for 0-based triplets, natively."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    nnz = int(vals.size)
    if not (rows.size == cols.size == nnz):
        raise ValueError("rows, cols, vals must have identical length")
    out = np.empty(max(1, nnz * 72), dtype=np.uint8)
    used = np.zeros(1, dtype=np.int64)
    _lib.call("sme_host_mm_format", rows.ctypes.data, cols.ctypes.data, vals.ctypes.data, nnz, out.ctypes.data,
              out.size if nnz else 0, int(threads), used.ctypes.data)
    return out[: int(used[0])].tobytes()


def write_matrix_market(m: CooMatrix, sink: str | os.PathLike | IO[str], *, threads: int = 0) -> None:
    """Write `m` in coordinate/real/general form, 1-based, 17 significant digits
    (matio.py:248-274); re-parses to a matrix equal to `m`, entry order included."""
    nnz = m.nnz
    head = f"%%MatrixMarket matrix coordinate real general\n{m.n_rows} {m.n_cols} {nnz}\n"
    body = format_entries(m.row_idx, m.col_idx, m.values, threads)
    if hasattr(sink, "write"):  # a text sink, as in the reference
        sink.write(head + body.decode("ascii"))
    else:
        with open(sink, "wb") as f:
            f.write(head.encode("ascii") + body)

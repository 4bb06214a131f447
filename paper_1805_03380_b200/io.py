"""Matrix Market coordinate persistence and a text renderer (mirrors
autosparse/io.py).

The text is parsed and formatted by native, multi-threaded host code in
libbsparse (csrc/mmio.cu: as_mm_header / as_mm_entries / as_mm_format) with
the reference's validation order and messages; the parsed triplets go
straight to the GPU construction kernel.  Only ``matrix coordinate real
general`` is accepted; indices are 1-based on disk, entries are written in
column-major order with 17 significant digits so values round-trip bit for
bit (io.py:1-7).
"""

from __future__ import annotations

import ctypes
import io as _stdio
import os
from pathlib import Path

import numpy as np

from . import _lib
from . import csc as csc_mod
from .csc import CscData, Dims
from .errors import CorruptionError, DuplicateEntryError, MatrixMarketError
from .hybrid import SpMat

_HEADER_TOKENS = ("%%MatrixMarket", "matrix", "coordinate", "real", "general")
HEADER_LINE = " ".join(_HEADER_TOKENS)


def _threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _as_csc(m) -> CscData:
    if isinstance(m, SpMat):
        return m.csc()
    if isinstance(m, CscData):
        return m
    raise TypeError("expected SpMat or CscData, got %r" % type(m).__name__)


def format_mm(data: CscData) -> str:
    """The Matrix Market text of a CSC (io.py:44-51)."""
    L = _lib.load()
    nnz = data.nnz
    rows = np.ascontiguousarray(data.row_indices, dtype=np.int64)
    cols = np.ascontiguousarray(data.expand_cols(), dtype=np.int64)
    vals = np.ascontiguousarray(data.values, dtype=np.float64)
    cap = 128 + 72 * nnz
    buf = ctypes.create_string_buffer(cap)
    n = L.as_mm_format(data.dims.n_rows, data.dims.n_cols, nnz, rows.ctypes.data, cols.ctypes.data,
                       vals.ctypes.data, ctypes.addressof(buf), cap, _threads())
    if n < 0:
        raise RuntimeError("Matrix Market formatting buffer too small")
    return buf.raw[:n].decode("ascii")


def save_mm(m, sink) -> None:
    """Write Matrix Market coordinate/real/general to a path or a text file
    object (io.py:33-41)."""
    text = format_mm(_as_csc(m))
    if hasattr(sink, "write"):
        sink.write(text)
    else:
        with open(sink, "w", encoding="ascii") as fh:
            fh.write(text)


def parse_mm(data: bytes):
    """(Dims, rows int64, cols int64, vals float64) of Matrix Market text,
    raising the reference's errors (io.py:65-126).  Host only."""
    L = _lib.load()
    if not isinstance(data, (bytes, bytearray)):
        raise TypeError("parse_mm takes bytes")
    buf = bytes(data)
    n_rows, n_cols, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    off, eline, err = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = L.as_mm_header(buf, len(buf), ctypes.byref(n_rows), ctypes.byref(n_cols), ctypes.byref(nnz),
                        ctypes.byref(off), ctypes.byref(eline), ctypes.byref(err))
    if rc != _lib.AS_OK:
        raise MatrixMarketError(L.as_last_error().decode(), int(err.value))
    dims = Dims(int(n_rows.value), int(n_cols.value))
    n = int(nnz.value)
    if n < 0:
        raise ValueError("negative dimensions are not allowed")  # np.empty(nnz) in the reference
    rows = np.empty(n, np.int64)
    cols = np.empty(n, np.int64)
    vals = np.empty(n, np.float64)
    rc = L.as_mm_entries(buf, len(buf), off.value, eline.value, dims.n_rows, dims.n_cols, n, rows.ctypes.data,
                         cols.ctypes.data, vals.ctypes.data, _threads(), ctypes.byref(err))
    if rc == _lib.AS_ERR_CORRUPT:
        raise CorruptionError("line %d: entry %s outside %s matrix" % (int(err.value), L.as_last_error().decode(),
                                                                        dims))
    if rc != _lib.AS_OK:
        raise MatrixMarketError(L.as_last_error().decode(), int(err.value))
    return dims, rows, cols, vals


def _read_bytes(source) -> bytes:
    if hasattr(source, "read"):
        text = source.read()
        return text.encode("ascii") if isinstance(text, str) else bytes(text)
    if isinstance(source, str) and "\n" in source:
        return source.encode("ascii")
    data = Path(source).read_bytes()
    data.decode("ascii")  # the reference reads with encoding="ascii"
    return data


def load_mm(source, lenient_duplicates: bool = False, device=None) -> SpMat:
    """Parse a Matrix Market file (path, text, or file object); duplicate
    coordinates are an error unless `lenient_duplicates`, in which case they
    are summed (io.py:54-131).  The triplets are built into CSC on the GPU."""
    dims, rows, cols, vals = parse_mm(_read_bytes(source))
    device = device or csc_mod.default_device()
    if rows.shape[0]:
        # duplicates: the structure of the ones-matrix has fewer entries than
        # the file (values of 1.0 never cancel) -- np.unique in the reference
        ones_m, _ = csc_mod.build_device(dims, rows, cols, np.ones(rows.shape[0]), csc_mod.DUP_SUM, device)
        if ones_m.nnz != rows.shape[0] and not lenient_duplicates:
            raise DuplicateEntryError("duplicate coordinates in input")
    return SpMat.from_csc(csc_mod.canonicalize(dims, rows, cols, vals, device=device))


def render_text(m, max_dim: int = 20) -> str:
    """Dense grid for small matrices, column-major triplet listing for
    anything with a dimension beyond `max_dim` (io.py:134-153)."""
    data = _as_csc(m)
    r, c = data.dims
    out = _stdio.StringIO()
    out.write("[%s sparse, nnz=%d, density=%s]\n" % (
        data.dims, data.nnz,
        ("%.4g%%" % (100.0 * data.nnz / data.dims.n_cells)) if data.dims.n_cells else "n/a",
    ))
    if r <= max_dim and c <= max_dim:
        dense = data.to_dense()
        cells = [["%.4g" % dense[i, j] for j in range(c)] for i in range(r)]
        width = max((len(s) for row in cells for s in row), default=1)
        for i in range(r):
            out.write("  ".join(s.rjust(width) for s in cells[i]) + "\n")
    else:
        for t in data.triplets():
            out.write("(%d, %d) %.10g\n" % (t.row, t.col, t.value))
    return out.getvalue()

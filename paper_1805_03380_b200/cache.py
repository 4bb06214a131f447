"""Insertion cache: the element-write format of the hybrid matrix.

The reference stages element writes in a red-black tree keyed by the
column-major linear index (autosparse/rbt.py): insert overwrites
(rbt.py:115-117), writing 0.0 erases (:374-376), appends of a new maximum
skip the descent (:389-407), and rbt.to_csc (:444-458) walks the tree in
order to rebuild CSC.  Its observable semantics are kept here, but not the
tree: writes go to an append-only host log (three numpy columns, O(1) per
write, no CUDA call), and the conversion back to CSC is ONE device pass --
the log is copied to HBM and merged with the base CSC snapshot by the GPU
flush (sort by (col, row, write order), last write wins, zeros erased,
compacted; include/bsparse.h as_flush_log_f64).

Reads of the cache (get / items / count) index the log lazily into a dict
of latest values, so a write-only workload never pays for them.
"""

from __future__ import annotations

from array import array
from typing import Iterator, Optional

import numpy as np
import torch

from . import _kernels
from . import csc as csc_mod
from .csc import CscData, Dims
from .errors import AppendOrderError, CoordinateError


def encode_index(row: int, col: int, n_rows: int) -> int:
    """Column-major linear position (rbt.py:23-25)."""
    return row + col * n_rows


def decode_index(index: int, n_rows: int) -> tuple:
    """(row, col) of a linear position (rbt.py:28-29)."""
    return index % n_rows, index // n_rows


class InsertionCache:
    """Ordered map linear index -> value with RbtStore's API (rbt.py:303-441):
    insert / append_max / get / erase / items / count / max_index."""

    def __init__(self, dims: Dims, base: Optional[CscData] = None, reserve: int = 0):
        self.dims = dims
        self._base = base
        cap = max(16, reserve)
        self._rows = np.empty(cap, np.int32)
        self._cols = np.empty(cap, np.int32)
        self._vals = np.empty(cap, np.float64)
        self._n = 0
        # tails of single writes not yet moved into the columns above
        self._tr, self._tc, self._tv = array("i"), array("i"), array("d")
        self._ar, self._ac, self._av = self._tr.append, self._tc.append, self._tv.append
        self._cur = {}
        self._indexed = 0
        self._count = base.nnz if base is not None else 0

    # -- log ------------------------------------------------------------------
    @property
    def n_writes(self) -> int:
        return self._n + len(self._tr)

    def _spill(self) -> None:
        """Move the single-write tails into the numpy columns (write order kept)."""
        k = len(self._tr)
        if not k:
            return
        n = self._n
        if n + k > self._rows.shape[0]:
            self._grow(n + k)
        self._rows[n : n + k] = np.frombuffer(self._tr, np.int32)
        self._cols[n : n + k] = np.frombuffer(self._tc, np.int32)
        self._vals[n : n + k] = np.frombuffer(self._tv, np.float64)
        self._n = n + k
        # (the temporaries above are gone: the arrays may be resized again)
        del self._tr[:], self._tc[:], self._tv[:]

    def _grow(self, need: int):
        cap = self._rows.shape[0]
        while cap < need:
            cap *= 2
        for name in ("_rows", "_cols", "_vals"):
            old = getattr(self, name)
            new = np.empty(cap, old.dtype)
            new[: self._n] = old[: self._n]
            setattr(self, name, new)

    def _check_index(self, index: int) -> None:
        if not 0 <= index < self.dims.n_cells:
            raise CoordinateError(
                "linear index %d outside %s matrix (%d cells)" % (index, self.dims, self.dims.n_cells)
            )

    def write(self, row: int, col: int, value: float) -> None:
        """Append one element write (coordinates already checked)."""
        try:
            self._ar(row)
        except TypeError:  # an integral float / numpy scalar without __index__
            row, col = int(row), int(col)
            self._ar(row)
        try:
            self._ac(col)
            self._av(value)
        except BaseException:  # keep the three tails the same length
            del self._tr[len(self._tv):], self._tc[len(self._tv):]
            raise

    def write_many(self, rows, cols, vals) -> None:
        """Append a batch of element writes, applied in array order."""
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        vals = np.asarray(vals, dtype=np.float64)
        k = rows.shape[0]
        if ((rows < 0) | (rows >= self.dims.n_rows) | (cols < 0) | (cols >= self.dims.n_cols)).any():
            bad = int(np.flatnonzero((rows < 0) | (rows >= self.dims.n_rows) | (cols < 0) | (cols >= self.dims.n_cols))[0])
            raise CoordinateError("write %d = (%d, %d) outside %s matrix" % (bad, rows[bad], cols[bad], self.dims))
        self._spill()
        if self._n + k > self._rows.shape[0]:
            self._grow(self._n + k)
        self._rows[self._n : self._n + k] = rows
        self._cols[self._n : self._n + k] = cols
        self._vals[self._n : self._n + k] = vals
        self._n += k

    # -- lazy index of latest values ------------------------------------------------
    def _base_value(self, row: int, col: int) -> float:
        if self._base is None or self._base.nnz == 0:
            return 0.0
        pos = self._base.find(row, col)
        return float(self._base.values[pos]) if pos >= 0 else 0.0

    def _sync(self) -> None:
        self._spill()
        n_rows = self.dims.n_rows
        cur = self._cur
        for i in range(self._indexed, self._n):
            r, c, v = int(self._rows[i]), int(self._cols[i]), float(self._vals[i])
            key = r + c * n_rows
            old = cur[key] if key in cur else self._base_value(r, c)
            self._count += (v != 0.0) - (old != 0.0)
            cur[key] = v
        self._indexed = self._n

    # -- RbtStore API ---------------------------------------------------------------
    @property
    def count(self) -> int:
        self._sync()
        return self._count

    def __len__(self):
        return self.count

    def insert(self, index: int, value: float) -> None:
        """Insert or overwrite; 0.0 erases (rbt.py:371-387)."""
        self._check_index(index)
        r, c = decode_index(index, self.dims.n_rows)
        self.write(r, c, float(value))

    def get(self, index: int) -> float:
        self._check_index(index)
        self._sync()
        if index in self._cur:
            return self._cur[index]
        r, c = decode_index(index, self.dims.n_rows)
        return self._base_value(r, c)

    def erase(self, index: int) -> bool:
        """Remove the element; False when absent (rbt.py:409-423)."""
        if self.get(index) == 0.0:
            return False
        self.insert(index, 0.0)
        return True

    def items(self) -> Iterator[tuple]:
        """(index, value) in increasing index order, stored elements only."""
        self._sync()
        n_rows = self.dims.n_rows
        merged = {}
        if self._base is not None and self._base.nnz:
            b = self._base
            keys = b.row_indices + b.expand_cols() * n_rows
            merged.update(zip(keys.tolist(), b.values.tolist()))
        merged.update(self._cur)
        for k in sorted(merged):
            if merged[k] != 0.0:
                yield k, merged[k]

    @property
    def max_index(self) -> int:
        best = -1
        for k, _v in self.items():
            best = k
        return best

    def append_max(self, index: int, value: float) -> None:
        """Insert an index beyond every stored one (rbt.py:389-407)."""
        self._check_index(index)
        if self.count and index <= self.max_index:
            raise AppendOrderError("append index %d not beyond current maximum %d" % (index, self.max_index))
        if value == 0.0:
            return
        self.insert(index, value)

    # -- conversion ------------------------------------------------------------------
    def to_csc(self, device=None) -> CscData:
        """Flush base + log into canonical CSC with one GPU pass."""
        device = device or (self._base.device if self._base is not None else csc_mod.default_device())
        base = self._base if self._base is not None else csc_mod.empty(self.dims, device)
        self._spill()
        n = self._n
        rows = torch.from_numpy(self._rows[:n]).to(device, non_blocking=False)
        cols = torch.from_numpy(self._cols[:n]).to(device, non_blocking=False)
        vals = torch.from_numpy(self._vals[:n]).to(device, non_blocking=False)
        p, r, v, bad = _kernels.flush_log(self.dims.n_rows, self.dims.n_cols, base.arrays, rows, cols, vals)
        if bad is not None:
            raise CoordinateError("write %d outside %s matrix" % (bad, self.dims))
        return CscData(self.dims, p, r, v)


# the reference's name for the element-write format
RbtStore = InsertionCache


def to_csc(t: InsertionCache) -> CscData:
    """rbt.to_csc (rbt.py:444-458)."""
    return t.to_csc()


def from_csc(m: CscData) -> InsertionCache:
    """rbt.from_csc (rbt.py:461-476): the CSC becomes the cache's base
    snapshot -- nothing is copied or rebuilt.  The snapshot stays immutable:
    an in-place value patch of the owning SpMat (hybrid.py:170-178) writes to
    a copy of the values instead (SpMat.set), as the reference's separate tree
    would not see it either."""
    m._snap = True
    return InsertionCache(m.dims, base=m)

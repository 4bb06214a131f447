"""Compressed Sparse Column storage, resident on the GPU.

Mirrors autosparse/csc.py (Dims, Triplet, CscData, canonicalize,
from_triplets, empty, check_coords, validate; csc.py:24-222, 363-383) with
the arrays in HBM: col_ptr int32[n_cols+1], row_idx int32[nnz], vals
float64 (float32 allowed as an extension).  The reference-typed views
(`values` float64, `row_indices` / `col_offsets` int64, numpy) are
materialised on first access and cached; element-level reads use that host
mirror, bulk work runs on the device.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Iterator, NamedTuple, Sequence

import numpy as np
import torch

from . import _lib

from . import _kernels
from .errors import CoordinateError, CorruptionError

INDEX_MAX = np.iinfo(np.int64).max
DEVICE_INDEX_MAX = np.iinfo(np.int32).max

DUP_SUM = "sum"
DUP_LAST = "last"


def default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


@dataclass(frozen=True)
class Dims:
    """Matrix shape (csc.py:24-45).  Either dimension may be zero."""

    n_rows: int
    n_cols: int

    def __post_init__(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise ValueError("dimensions must be non-negative, got %r" % (self,))
        if self.n_rows and self.n_cols > INDEX_MAX // self.n_rows:
            raise ValueError("n_rows * n_cols overflows the 64-bit index type")

    @property
    def n_cells(self) -> int:
        return self.n_rows * self.n_cols

    def __iter__(self):
        return iter((self.n_rows, self.n_cols))

    def __str__(self):
        return "%dx%d" % (self.n_rows, self.n_cols)


class Triplet(NamedTuple):
    row: int
    col: int
    value: float


def _to_dev(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device, non_blocking=True)


_STAGING_LOCK = threading.Lock()
_STAGING = {}


_STAGING_KEEP_BYTES = 256 << 20  # larger read-backs get their own buffers (not kept)


def _staging(n_ptr: int, cap: int, val_dtype):
    """Process-wide pinned read-back buffers (grow-only up to
    _STAGING_KEEP_BYTES each) for the host mirror."""
    def grown(key, n, dtype):
        t = _STAGING.get(key)
        if t is None or t.shape[0] < n:
            t = torch.empty(max(n, 1) + max(n, 1) // 4, dtype=dtype, pin_memory=True)
            if t.numel() * t.element_size() <= _STAGING_KEEP_BYTES:
                _STAGING[key] = t
        return t

    return (grown("ptr", n_ptr, torch.int32)[:n_ptr], grown("rows", cap, torch.int32),
            grown(("vals", val_dtype), cap, val_dtype))


class CscData:
    """Canonical CSC matrix (sorted, duplicate-free, zero-free) in HBM."""

    __slots__ = ("dims", "col_ptr", "_row_idx", "_vals", "_host", "_snap", "_pend")

    def __init__(self, dims: Dims, col_ptr, row_idx, vals, device=None):
        if dims.n_rows > DEVICE_INDEX_MAX or dims.n_cols > DEVICE_INDEX_MAX:
            raise CoordinateError("%s exceeds the int32 device index range" % (dims,))
        device = device or (col_ptr.device if isinstance(col_ptr, torch.Tensor) else default_device())
        self.dims = dims
        self.col_ptr = _to_dev(col_ptr, torch.int32, device)
        self._row_idx = _to_dev(row_idx, torch.int32, device)
        vdt = vals.dtype if isinstance(vals, torch.Tensor) and vals.dtype in (torch.float32, torch.float64) else torch.float64
        self._vals = _to_dev(vals, vdt, device)
        self._host = None
        self._snap = False  # an insertion cache holds this CSC as its base snapshot (rbt.from_csc)
        self._pend = None   # device info[2] while nnz is still on the device (see pending)

    @classmethod
    def pending(cls, dims: Dims, col_ptr, row_idx_full, vals_full, info) -> "CscData":
        """A CSC whose nnz is still on the device (info[0], written by the
        construction kernel): the row / value buffers have their full
        capacity until the first access that needs the size, which reads it
        back (one synchronisation) -- or to_host() takes it from the copied
        col_ptr, so an end-to-end build synchronises once."""
        m = cls(dims, col_ptr, row_idx_full, vals_full)
        m._pend = info
        return m

    def _resolve(self, nnz=None):
        if self._pend is not None:
            k = int(self._pend[0].item()) if nnz is None else int(nnz)
            self._pend = None
            self._row_idx = self._row_idx[:k]
            self._vals = self._vals[:k]

    @property
    def row_idx(self):
        self._resolve()
        return self._row_idx

    @row_idx.setter
    def row_idx(self, v):
        self._resolve()
        self._row_idx = v

    @property
    def vals(self):
        self._resolve()
        return self._vals

    @vals.setter
    def vals(self, v):
        self._resolve()
        self._vals = v

    def to_host(self, out=None):
        """(col_ptr int32, row_idx int32, vals) as host tensors -- into `out`
        (pinned, sized n_cols + 1 and >= the row / value buffers) when given.
        All copies are issued before the single synchronisation; a pending
        nnz comes from the copied col_ptr[-1]."""
        if self.col_ptr.device.type == "cpu":  # a host CSC (canonicalize_host)
            if out is None:
                return self.col_ptr, self.row_idx, self.vals
            k = self.nnz
            out[0].copy_(self.col_ptr), out[1][:k].copy_(self.row_idx), out[2][:k].copy_(self.vals)
            return out[0], out[1][:k], out[2][:k]
        pend = self._pend is not None
        ri, vv = self._row_idx, self._vals  # full capacity while pending
        if out is None:
            out = (torch.empty(self.col_ptr.shape[0], dtype=torch.int32, pin_memory=True),
                   torch.empty(ri.shape[0], dtype=torch.int32, pin_memory=True),
                   torch.empty(vv.shape[0], dtype=vv.dtype, pin_memory=True))
        o_ptr, o_rows, o_vals = out
        stream = torch.cuda.current_stream(self.col_ptr.device)
        o_ptr.copy_(self.col_ptr, non_blocking=True)
        n_r = int(ri.shape[0])
        half = self.dims.n_rows <= 65536 and n_r >= (1 << 16)
        if half:
            # rows < 65536: they travel at half width and are widened on host
            # threads while the values are still being copied
            from . import _kernels

            stage, scratch = _kernels.u16_stage(n_r, self.col_ptr.device)
            _lib.check(_lib.lib().as_rows_to_host_u16(_lib.ptr(ri), n_r, _lib.ptr(scratch), _lib.ptr(stage),
                                                      stream.cuda_stream))
            rows_done = torch.cuda.Event()
            rows_done.record(stream)
        else:
            o_rows[:n_r].copy_(ri, non_blocking=True)
        o_vals[: vv.shape[0]].copy_(vv, non_blocking=True)
        if half:
            rows_done.synchronize()
            _lib.check(_lib.lib().as_widen_u16(_lib.ptr(stage), _lib.ptr(o_rows), n_r, _kernels._upload_threads()))
        stream.synchronize()
        k = int(o_ptr[-1]) if pend else n_r
        if pend:
            self._resolve(k)
        return o_ptr, o_rows[:k], o_vals[:k]

    def own_values_copy(self) -> "CscData":
        """The same matrix with its own value array (the index arrays are
        immutable and shared): what an in-place value patch writes to while
        an insertion cache still holds this one as its snapshot."""
        self._resolve()
        c = CscData.__new__(CscData)
        c.dims, c.col_ptr, c._row_idx, c._vals = self.dims, self.col_ptr, self._row_idx, self._vals.clone()
        c._host = None if self._host is None else (self._host[0].copy(), self._host[1], self._host[2])
        c._snap = False
        c._pend = None
        return c

    @classmethod
    def from_reference_arrays(cls, dims: Dims, values, row_indices, col_offsets, device=None) -> "CscData":
        """Wrap the reference's (values, row_indices, col_offsets) order."""
        return cls(dims, col_offsets, row_indices, values, device=device)

    # -- device view ----------------------------------------------------------
    @property
    def device(self):
        return self.col_ptr.device

    @property
    def arrays(self):
        """(col_ptr, row_idx, vals) device tensors, the kernels' operand order."""
        return self.col_ptr, self.row_idx, self.vals

    @property
    def nnz(self) -> int:
        return int(self.row_idx.shape[0])

    # -- reference-typed host mirror (csc.py:54-67) -----------------------------
    def _mirror(self):
        if self._host is None:
            if self.col_ptr.device.type == "cpu":
                p, r, v = self.to_host()
                self._host = (v.numpy().astype(np.float64), r.numpy().astype(np.int64), p.numpy().astype(np.int64))
            else:
                # the copies land in pinned staging buffers kept for the process (a fresh
                # pinned allocation per read-back cost 3-4 ms at cfg 2's size); the
                # reference-typed arrays below are copies, so the buffers are free again
                with _STAGING_LOCK:
                    p, r, v = self.to_host(out=_staging(self.col_ptr.shape[0], self._row_idx.shape[0],
                                                        self._vals.dtype))
                    self._host = (v.numpy().astype(np.float64), r.numpy().astype(np.int64),
                                  p.numpy().astype(np.int64))
        return self._host

    @property
    def values(self) -> np.ndarray:
        return self._mirror()[0]

    @property
    def row_indices(self) -> np.ndarray:
        return self._mirror()[1]

    @property
    def col_offsets(self) -> np.ndarray:
        return self._mirror()[2]

    def find(self, row: int, col: int) -> int:
        """Storage position of (row, col) or -1 (binary search in the column)."""
        offs, rows = self.col_offsets, self.row_indices
        start, end = offs[col], offs[col + 1]
        pos = start + int(np.searchsorted(rows[start:end], row))
        return pos if pos < end and rows[pos] == row else -1

    def get(self, row: int, col: int) -> float:
        check_coords(self.dims, row, col)
        pos = self.find(row, col)
        return float(self.values[pos]) if pos >= 0 else 0.0

    def set_value_at(self, pos: int, value: float) -> None:
        """In-place overwrite of a stored value (the only sanctioned mutation,
        csc.py:57-58 / hybrid.py:170-178); device and mirror stay in sync."""
        self.vals[pos] = value
        if self._host is not None:
            self._host[0][pos] = value

    def col_count(self, col: int) -> int:
        if not 0 <= col < self.dims.n_cols:
            raise CoordinateError("column %d outside matrix with %d columns" % (col, self.dims.n_cols))
        offs = self.col_offsets
        return int(offs[col + 1] - offs[col])

    def triplets(self) -> Iterator[Triplet]:
        vals, rows, offs = self._mirror()
        for col in range(self.dims.n_cols):
            for k in range(offs[col], offs[col + 1]):
                yield Triplet(int(rows[k]), col, float(vals[k]))

    def expand_cols(self) -> np.ndarray:
        return np.repeat(np.arange(self.dims.n_cols, dtype=np.int64), np.diff(self.col_offsets))

    def expand_cols_device(self) -> torch.Tensor:
        """Column of every element (int32, on the device; as_expand_cols)."""
        if self.device.type != "cuda":
            counts = (self.col_ptr[1:] - self.col_ptr[:-1]).long()
            return torch.repeat_interleave(torch.arange(self.dims.n_cols, dtype=torch.int32), counts)
        from . import _kernels

        return _kernels.expand_cols(self.dims.n_cols, self.col_ptr, self.nnz)

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.dims.n_rows, self.dims.n_cols))
        dense[self.row_indices, self.expand_cols()] = self.values
        return dense

    def copy(self) -> "CscData":
        return CscData(self.dims, self.col_ptr.clone(), self.row_idx.clone(), self.vals.clone())

    def same_elements(self, other: "CscData") -> bool:
        return (
            self.dims == other.dims
            and self.nnz == other.nnz
            and torch.equal(self.col_ptr, other.col_ptr.to(self.device))
            and torch.equal(self.row_idx, other.row_idx.to(self.device))
            and torch.equal(self.vals.double(), other.vals.double().to(self.device))
        )

    def __repr__(self):
        return "<CscData %s nnz=%d on %s>" % (self.dims, self.nnz, self.device)


def check_coords(dims: Dims, row: int, col: int) -> None:
    if not (0 <= row < dims.n_rows and 0 <= col < dims.n_cols):
        raise CoordinateError("coordinate (%d, %d) outside %s matrix" % (row, col, dims))


def empty(dims: Dims, device=None, dtype=torch.float64) -> CscData:
    device = device or default_device()
    return CscData(dims, torch.zeros(dims.n_cols + 1, dtype=torch.int32, device=device),
                   torch.empty(0, dtype=torch.int32, device=device), torch.empty(0, dtype=dtype, device=device))


def _as_index_tensor(a, device):
    if isinstance(a, torch.Tensor):
        t = a.to(device, non_blocking=True)
        return t if t.dtype in (torch.int32, torch.int64) else t.long()
    arr = np.asarray(a)
    if arr.dtype not in (np.int32, np.int64):
        arr = arr.astype(np.int64)
    return torch.as_tensor(np.ascontiguousarray(arr)).to(device, non_blocking=True)


def _as_value_tensor(a, device, dtype=None):
    if isinstance(a, torch.Tensor):
        dt = dtype or (a.dtype if a.dtype in (torch.float32, torch.float64) else torch.float64)
        return a.to(device=device, dtype=dt, non_blocking=True).contiguous()
    arr = np.asarray(a, dtype=np.float64 if dtype in (None, torch.float64) else np.float32)
    return torch.as_tensor(np.ascontiguousarray(arr)).to(device, non_blocking=True)


def _host_int64(a):
    """A contiguous CPU int64 tensor view of host index data, or None."""
    if isinstance(a, torch.Tensor):
        return a.contiguous() if (not a.is_cuda and a.dtype == torch.int64 and a.dim() == 1) else None
    if isinstance(a, np.ndarray) and a.dtype == np.int64 and a.ndim == 1:
        return torch.from_numpy(np.ascontiguousarray(a))
    return None


def _host_values(a):
    """A contiguous CPU float tensor of host values (float64 unless float32), or None."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dim() != 1:
            return None
        return a.contiguous() if a.dtype in (torch.float32, torch.float64) else a.double()
    if isinstance(a, np.ndarray) and a.ndim == 1:  # numpy values build float64 (as _as_value_tensor)
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return None


def build_device(dims: Dims, rows, cols, values, dup: str = DUP_SUM, device=None):
    """Run the GPU construction on device (or host) arrays; returns
    (CscData, first_bad_index_or_None)."""
    if dup not in (DUP_SUM, DUP_LAST):
        raise ValueError("unknown duplicate policy %r" % (dup,))
    device = device or default_device()
    hr, hc, hv = _host_int64(rows), _host_int64(cols), _host_values(values)
    if hr is not None and hc is not None and hv is not None and torch.device(device).type == "cuda":
        # int64 host triplets: narrowed (or packed into one 32-bit key per
        # triplet when the shape allows) on host threads while the values
        # are copied (16 or 12 instead of 24 bytes per triplet over PCIe)
        host_bad = []
        r, c, v = _kernels.upload_coo(hr, hc, hv, device, (dims.n_rows, dims.n_cols), bad_out=host_bad)
        if host_bad and host_bad[0] < 0:
            # the packers saw every coordinate in range: no read-back of the
            # kernel's report, nnz stays on the device until it is needed
            p, ri, vv, info = _kernels.coo_to_csc(dims.n_rows, dims.n_cols, r, c, v, dup, lazy=True)
            return CscData.pending(dims, p, ri, vv, info), None
    else:
        r = _as_index_tensor(rows, device)
        c = _as_index_tensor(cols, device)
        if r.dtype != c.dtype:
            r, c = r.long(), c.long()
        v = _as_value_tensor(values, device)
    p, ri, vv, bad = _kernels.coo_to_csc(dims.n_rows, dims.n_cols, r, c, v, dup)
    return CscData(dims, p, ri, vv), bad


def canonicalize(dims: Dims, rows, cols, values, dup: str = DUP_SUM, device=None) -> CscData:
    """Canonical CSC from parallel coordinate arrays (csc.py:148-193): stable
    column-major order, duplicates per `dup`, exact zeros pruned -- one
    sort/reduce/compact pass on the GPU."""
    m, bad = build_device(dims, rows, cols, values, dup, device)
    if bad is not None:
        raise CoordinateError("coordinate %d outside %s matrix" % (bad, dims))
    return m


def canonicalize_host(dims: Dims, rows, cols, values, dup: str = DUP_SUM, out=None) -> CscData:
    """csc.canonicalize with host arrays in and out (the reference's own
    numpy-in / numpy-out signature, csc.py:148-193): pinned host triplets are
    read over PCIe by the build kernel itself and the CSC is written straight
    into pinned host memory (`out` = (col_ptr int32[n_cols+1], row_idx
    int32[n], vals float64[n]) to reuse), so both transfers overlap the
    kernel's own phases.  Returns a host CscData."""
    if dup not in (DUP_SUM, DUP_LAST):
        raise ValueError("unknown duplicate policy %r" % (dup,))

    def pinned(a, dtype):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.dtype != dtype:
            t = t.to(dtype)
        return t if t.is_pinned() else t.pin_memory()

    idx_t = torch.int64
    r, c = pinned(rows, idx_t), pinned(cols, idx_t)
    v = pinned(values, torch.float64)
    n = int(v.shape[0])
    if out is None:
        out = (torch.empty(dims.n_cols + 1, dtype=torch.int32).pin_memory(),
               torch.empty(max(n, 1), dtype=torch.int32).pin_memory(),
               torch.empty(max(n, 1), dtype=torch.float64).pin_memory())
    p, ri, vv, bad = _kernels.coo_to_csc(dims.n_rows, dims.n_cols, r, c, v, dup, out=out)
    if bad is not None:
        raise CoordinateError("coordinate %d outside %s matrix" % (bad, dims))
    return CscData(dims, p, ri, vv, device=torch.device("cpu"))


def _coords_from_triplets(triplets: Sequence) -> tuple:
    """(rows, cols, values) from a reference-style triplet sequence
    (csc.py:196-205), or passed through when given as three arrays."""
    if isinstance(triplets, tuple) and len(triplets) == 3 and all(
        isinstance(x, (np.ndarray, torch.Tensor)) for x in triplets
    ):
        return triplets
    n = len(triplets)
    if n == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.float64)
    rows = np.fromiter((t[0] for t in triplets), dtype=np.int64, count=n)
    cols = np.fromiter((t[1] for t in triplets), dtype=np.int64, count=n)
    vals = np.fromiter((t[2] for t in triplets), dtype=np.float64, count=n)
    return rows, cols, vals


def from_triplets(dims: Dims, triplets, dup: str = DUP_SUM, device=None) -> CscData:
    """Batch-build canonical CSC (csc.py:208-222).  `triplets` is a sequence
    of (row, col, value) or, as an extension, a tuple of three arrays/tensors.
    Out-of-range triplets raise CoordinateError naming the first one."""
    rows, cols, vals = _coords_from_triplets(triplets)
    m, bad = build_device(dims, rows, cols, vals, dup, device)
    if bad is not None:
        r = int(rows[bad])
        c = int(cols[bad])
        v = float(vals[bad])
        raise CoordinateError("triplet %d = (%d, %d, %g) outside %s matrix" % (bad, r, c, v, dims))
    return m


def validate(m: CscData) -> None:
    """Canonical-form checker (csc.py:363-383): raises CorruptionError."""
    dims = m.dims
    vals, rows, offs = m.values, m.row_indices, m.col_offsets
    n = rows.shape[0]
    if offs.shape[0] != dims.n_cols + 1:
        raise CorruptionError("column offsets array has wrong length")
    if offs[0] != 0 or offs[-1] != n:
        raise CorruptionError("column offsets must start at 0 and end at nnz")
    if (np.diff(offs) < 0).any():
        raise CorruptionError("column offsets must be non-decreasing")
    if vals.shape[0] != n:
        raise CorruptionError("row index array length differs from value array")
    if n:
        if rows.min() < 0 or rows.max() >= dims.n_rows:
            raise CorruptionError("row index outside matrix")
        cols = m.expand_cols()
        same_col = cols[1:] == cols[:-1]
        if (same_col & (rows[1:] <= rows[:-1])).any():
            bad = int(cols[1:][same_col & (rows[1:] <= rows[:-1])][0])
            raise CorruptionError("rows in column %d not strictly increasing" % bad)
        if (vals == 0.0).any():
            raise CorruptionError("exact zero stored in values array")

"""Drop-in replacement for the reference's flat-array kernel module.

`autosparse._kernels` (reference _kernels.py:1-175) is the de-facto operator
boundary of the reference: plain numpy arrays in -- values
float64, row indices / column offsets int64 -- fresh numpy arrays out, no
validation.  This module exposes the same functions with the same positional
signatures and return conventions, executed by the sm_100a kernels of
libbsparse.so: inputs are copied to HBM, one C-ABI call runs, the result is
copied back.  `canonicalize` and `rbt_to_csc` cover the other two entry points
of the path (csc.canonicalize csc.py:148-193, rbt.to_csc rbt.py:444-458).

It lets a reference user switch back ends with one assignment:

    import autosparse, paper_1805_03380_b200.ref_kernels as k
    autosparse.ops._kernels = k          # ops.add / matmul / transpose / SpMV
    autosparse.expr._kernels = k         # fused trace

(see INTEGRATION.md).  Every call needs a CUDA device; there is no CPU path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _kernels

_DEV = None


def _dev():
    global _DEV
    if _DEV is None:
        _DEV = torch.device("cuda", torch.cuda.current_device())
    return _DEV


def _i32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(_dev())


def _f64(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(_dev())


def _csc(vals, rows, offs):
    return _i32(offs), _i32(rows), _f64(vals)


def _out(p, r, v, n_rows=None):
    """(values f64, row_indices i64, col_offsets i64) numpy, the reference's
    return order, read back through the device CSC's host mirror (pinned
    staging kept for the process; rows at half width when n_rows <= 65536)."""
    from .csc import DEVICE_INDEX_MAX, CscData, Dims

    d = CscData(Dims(int(n_rows) if n_rows is not None else DEVICE_INDEX_MAX, int(p.shape[0]) - 1), p, r, v)
    return d.values, d.row_indices, d.col_offsets


def linear_combine(n_cols, a_vals, a_rows, a_offs, b_vals, b_rows, b_offs, alpha, beta):
    """_kernels.linear_combine (_kernels.py:12-48)."""
    n_rows = int(max(np.max(a_rows, initial=-1), np.max(b_rows, initial=-1)) + 1)
    p, r, v = _kernels.linear_combine(n_rows, n_cols, _csc(a_vals, a_rows, a_offs), _csc(b_vals, b_rows, b_offs),
                                      alpha, beta)
    return _out(p, r, v, n_rows)


def spgemm(n_rows_a, a_vals, a_rows, a_offs, b_vals, b_rows, b_offs, n_cols_b):
    """_kernels.spgemm (_kernels.py:51-103)."""
    n_inner = int(np.asarray(a_offs).shape[0] - 1)
    p, r, v = _kernels.spgemm(n_rows_a, n_inner, n_cols_b, _csc(a_vals, a_rows, a_offs),
                              _csc(b_vals, b_rows, b_offs))
    return _out(p, r, v, n_rows_a)


def vec_times_mat(v, vals, rows, offs, n_cols):
    """_kernels.vec_times_mat (_kernels.py:106-115)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    w = _kernels.vec_times_mat(v.shape[0], n_cols, _csc(vals, rows, offs), _f64(v))
    return w.cpu().numpy()


def mat_times_vec(vals, rows, offs, x, n_rows, n_cols):
    """_kernels.mat_times_vec (_kernels.py:118-127); the CSR it runs on is
    built on the device for this call (the hybrid SpMat caches it)."""
    csr = _kernels.transpose(n_rows, n_cols, *_csc(vals, rows, offs))
    y = _kernels.mat_times_vec(n_rows, n_cols, csr, _f64(x))
    return y.cpu().numpy()


def transpose(n_rows, n_cols, vals, rows, offs):
    """_kernels.transpose (_kernels.py:130-150)."""
    return _out(*_kernels.transpose(n_rows, n_cols, *_csc(vals, rows, offs)), n_cols)


def fused_trace(n_cols, a_vals, a_rows, a_offs, b_vals, b_rows, b_offs):
    """_kernels.fused_trace (_kernels.py:153-175)."""
    n_rows = int(max(np.max(a_rows, initial=-1), np.max(b_rows, initial=-1)) + 1)
    out = _kernels.fused_trace(n_rows, n_cols, _csc(a_vals, a_rows, a_offs), _csc(b_vals, b_rows, b_offs))
    return float(out[0].item())


def canonicalize(n_rows, n_cols, rows, cols, values, dup="sum"):
    """csc.canonicalize (csc.py:148-193) on flat arrays; returns
    (values, row_indices, col_offsets).  The int64 coordinates are packed on
    host threads while the values are copied (csc.build_device) and the result
    comes back through the device CSC's host mirror (pinned staging, rows at
    half width when they fit)."""
    from . import csc as csc_mod

    r = np.ascontiguousarray(rows, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if r.shape[0] == 0:
        return np.empty(0, np.float64), np.empty(0, np.int64), np.zeros(int(n_cols) + 1, np.int64)
    m, bad = csc_mod.build_device(csc_mod.Dims(int(n_rows), int(n_cols)), r, c, v, dup, _dev())
    if bad is not None:
        raise IndexError("coordinate %d outside %dx%d matrix" % (bad, n_rows, n_cols))
    return m.values, m.row_indices, m.col_offsets


def rbt_to_csc(n_rows, n_cols, base, log_rows, log_cols, log_vals):
    """rbt.to_csc (rbt.py:444-458) of the tree reached from the base CSC
    (values, row_indices, col_offsets) by the element writes in the log."""
    p, r, v, bad = _kernels.flush_log(n_rows, n_cols, _csc(*base), _i32(log_rows), _i32(log_cols), _f64(log_vals))
    if bad is not None:
        raise IndexError("write %d outside %dx%d matrix" % (bad, n_rows, n_cols))
    return _out(p, r, v, n_rows)


# ---------------------------------------------------------------------------
# The two construction entry points with the reference's own types.
#
# csc.canonicalize(dims, rows, cols, values, dup) -> CscData (csc.py:148-193)
# and rbt.to_csc(RbtStore) -> CscData (rbt.py:444-458) take and return the
# reference's Dims / CscData / RbtStore objects.  The functions below keep
# those signatures: the caller's Dims decides which CscData class comes back
# (the class living next to it, i.e. autosparse.csc.CscData for a reference
# caller), and the element-write store is this package's host write log
# behind RbtStore's interface (insert / append_max / get / erase / items /
# count / max_index), flushed to CSC by one GPU pass.


def _csc_class_of(dims):
    import sys

    mod = sys.modules.get(type(dims).__module__)
    cls = getattr(mod, "CscData", None)
    if cls is None:
        raise TypeError("no CscData next to %r" % type(dims))
    return cls


def _our_dims(dims):
    from .csc import Dims

    n_rows, n_cols = dims
    return Dims(int(n_rows), int(n_cols))


def csc_canonicalize(dims, rows, cols, values, dup="sum"):
    """csc.canonicalize (csc.py:148-193) with its own signature: reference
    Dims in, reference CscData out.  Coordinates are validated by the caller
    (as in the reference); an unknown dup policy raises ValueError
    (csc.py:184)."""
    if dup not in ("sum", "last"):
        raise ValueError("unknown duplicate policy %r" % (dup,))
    n_rows, n_cols = dims
    v, r, o = canonicalize(int(n_rows), int(n_cols), rows, cols, values, dup) if np.asarray(rows).shape[0] else (
        np.empty(0, np.float64), np.empty(0, np.int64), np.zeros(int(n_cols) + 1, np.int64))
    return _csc_class_of(dims)(dims, v, r, o)


class LogStore:
    """RbtStore (rbt.py:303-441) for a reference caller: the same methods
    and properties over this package's write log (cache.InsertionCache);
    `to_csc` below flushes it on the GPU.  Keeps the caller's Dims."""

    def __init__(self, dims, reserve: int = 0, _base=None):
        from .cache import InsertionCache

        self.dims = dims
        self._c = InsertionCache(_our_dims(dims), base=_base, reserve=reserve)

    capacity = property(lambda self: max(16, self._c.n_writes))
    count = property(lambda self: self._c.count)
    max_index = property(lambda self: self._c.max_index)

    def __len__(self):
        return self._c.count

    def insert(self, index, value):
        self._c.insert(int(index), float(value))

    def append_max(self, index, value):
        self._c.append_max(int(index), float(value))

    def get(self, index):
        return self._c.get(int(index))

    def erase(self, index):
        return self._c.erase(int(index))

    def items(self):
        return self._c.items()


def rbt_store_to_csc(t):
    """rbt.to_csc (rbt.py:444-458): RbtStore-compatible store in, reference
    CscData out (one GPU flush of base + write log)."""
    m = t._c.to_csc()
    return _csc_class_of(t.dims)(t.dims, m.values, m.row_indices, m.col_offsets)


def rbt_from_csc(m):
    """rbt.from_csc (rbt.py:461-476): reference CscData in; the CSC becomes
    the store's base snapshot on the device (copied, so later in-place value
    patches of the caller's CscData are not seen, as with the reference's
    separate tree)."""
    from .csc import CscData as Ours

    base = Ours.from_reference_arrays(_our_dims(m.dims), np.array(m.values, np.float64),
                                      np.array(m.row_indices, np.int64), np.array(m.col_offsets, np.int64),
                                      device=_dev())
    return LogStore(m.dims, _base=base)


def install(pkg):
    """Route a reference package (`import autosparse as pkg`) through this
    back end: the flat-array kernel module of ops and expr, csc.canonicalize
    (construction, also reached by csc.from_triplets / coo.to_csc /
    SpMat.from_dense), and the element-write store with rbt.to_csc /
    rbt.from_csc.  Returns a function that undoes the swap."""
    import importlib

    mods = {n: importlib.import_module(pkg.__name__ + "." + n) for n in ("ops", "expr", "csc", "rbt", "hybrid")}
    import sys

    me = sys.modules[__name__]
    swaps = [(mods["ops"], "_kernels", me), (mods["expr"], "_kernels", me),
             (mods["csc"], "canonicalize", csc_canonicalize),
             (mods["rbt"], "RbtStore", LogStore), (mods["hybrid"], "RbtStore", LogStore),
             (mods["rbt"], "to_csc", rbt_store_to_csc), (mods["rbt"], "from_csc", rbt_from_csc)]
    saved = [(m, name, getattr(m, name)) for m, name, _ in swaps]
    for m, name, new in swaps:
        setattr(m, name, new)

    def undo():
        for m, name, old in saved:
            setattr(m, name, old)

    return undo

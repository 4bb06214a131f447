"""ctypes binding of libbsparse.so (include/bsparse.h).

This is the only door to the device code.  There is no fallback: if the
library is missing, or no CUDA device is present when a kernel is requested,
the call raises.  PyTorch provides device buffers and the current stream;
every pointer handed across is a ``tensor.data_ptr()``.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import CoordinateError, CorruptionError, ShapeError, SparseError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AS_LIB_PATH") or os.path.join(_HERE, "libbsparse.so")  # override: build-variant experiments

P = ctypes.c_void_p
I64 = ctypes.c_int64
SZ = ctypes.c_size_t
INT = ctypes.c_int
DBL = ctypes.c_double

# name -> (restype, argtypes); must match include/bsparse.h
SIGNATURES = {
    "as_last_error": (ctypes.c_char_p, []),
    "as_abi_version": (INT, []),
    "as_set_engine": (INT, [INT]),
    "as_build_workspace_bytes": (SZ, [I64, I64]),
    "as_coo_to_csc_f64": (INT, [I64, I64, I64, P, P, INT, P, INT, P, P, P, P, P, SZ, P]),
    "as_coo_to_csc_f32": (INT, [I64, I64, I64, P, P, INT, P, INT, P, P, P, P, P, SZ, P]),
    "as_upload_coo_i64": (INT, [P, P, P, I64, I64, P, P, P, P, P, INT, INT, P]),
    "as_upload_coo_packed": (INT, [P, P, P, I64, I64, I64, I64, P, P, P, P, P, INT, INT, P, P]),
    "as_rows_to_host_u16": (INT, [P, I64, P, P, P]),
    "as_widen_u16": (INT, [P, P, I64, INT]),
    "as_flush_workspace_bytes": (SZ, [I64, I64, I64]),
    "as_flush_log_f64": (INT, [I64, I64, I64, P, P, P, I64, P, P, P, P, P, P, P, P, SZ, P]),
    "as_transpose_workspace_bytes": (SZ, [I64, I64]),
    "as_csc_transpose_f64": (INT, [I64, I64, I64, P, P, P, P, P, P, P, SZ, P]),
    "as_csc_transpose_f32": (INT, [I64, I64, I64, P, P, P, P, P, P, P, SZ, P]),
    "as_add_workspace_bytes": (SZ, [I64, I64, I64]),
    "as_csc_add_f64": (INT, [I64, I64, DBL, DBL, P, P, P, P, P, P, I64, I64, P, P, P, P, P, SZ, P]),
    "as_spgemm_products_workspace_bytes": (SZ, [I64]),
    "as_spgemm_products": (INT, [I64, I64, I64, P, P, P, P, P, P, SZ, P]),
    "as_spgemm_workspace_bytes": (SZ, [I64, I64, I64]),
    "as_spgemm_f64": (INT, [I64, I64, I64, P, P, P, P, P, P, I64, P, I64, P, P, P, P, P, SZ, P]),
    "as_spmm_workspace_bytes": (SZ, [I64, I64, INT]),
    "as_spmm_csr_f32": (INT, [I64, I64, I64, P, P, P, P, I64, P, I64, INT, P, SZ, P]),
    "as_spmm_csr_f64": (INT, [I64, I64, I64, P, P, P, P, I64, P, I64, P, SZ, P]),
    "as_spmm_csc_workspace_bytes": (SZ, [I64, I64]),
    "as_spmm_csc_f32": (INT, [I64, I64, I64, I64, P, P, P, P, I64, P, I64, P, SZ, P]),
    "as_vecmat_csc_f64": (INT, [I64, I64, P, P, P, P, P, P]),
    "as_set_trace_engine": (INT, [INT]),
    "as_mg_init": (INT, [P, INT, INT, ctypes.c_char_p]),
    "as_mg_shutdown": (INT, []),
    "as_mg_rank": (INT, []),
    "as_mg_world": (INT, []),
    "as_mg_trace_workspace_bytes": (SZ, [I64, I64, I64, INT]),
    "as_mg_trace_atb_f64": (INT, [I64, I64, P, P, P, P, P, P, I64, I64, I64, I64, P, P, SZ, P]),
    "as_mg_spmm_csr_f32": (INT, [I64, I64, I64, P, P, P, P, I64, P, I64, P, SZ, P]),
    "as_mg_spgemm_f64": (INT, [I64, I64, I64, P, P, P, P, P, P, I64, P, I64, P, P, P, P, P, SZ, P, P, P]),
    "as_trace_workspace_bytes": (SZ, [I64, I64, I64]),
    "as_trace_atb_f64": (INT, [I64, I64, P, P, P, P, P, P, I64, I64, P, P, SZ, P]),
    "as_expand_cols": (INT, [I64, P, P, P]),
    "as_kron_triplets_f64": (INT, [I64, P, P, P, I64, P, P, P, I64, I64, P, P, P, P]),
    "as_repmat_triplets_f64": (INT, [I64, P, P, P, I64, I64, I64, I64, P, P, P, P]),
    "as_segment_reduce_f64": (INT, [I64, P, P, INT, INT, DBL, I64, P, P]),
    "as_pairwise_workspace_bytes": (SZ, []),
    "as_pairwise_sum_f64": (INT, [I64, P, INT, DBL, P, P, SZ, P]),
    "as_window_workspace_bytes": (SZ, [I64]),
    "as_csc_window_f64": (INT, [I64, I64, P, P, P, I64, I64, I64, I64, P, P, P, P, P, SZ, P]),
    "as_csc_diag_f64": (INT, [I64, I64, P, P, P, I64, I64, P, P]),
    "as_scale_by_label_f64": (INT, [I64, P, P, P, P, P]),
    "as_mm_header": (INT, [P, I64, P, P, P, P, P, P]),
    "as_mm_entries": (INT, [P, I64, I64, I64, I64, I64, I64, P, P, P, INT, P]),
    "as_mm_format": (I64, [I64, I64, I64, P, P, P, P, I64, INT]),
}

AS_OK, AS_ERR_SHAPE, AS_ERR_COORD, AS_ERR_CORRUPT, AS_ERR_CUDA, AS_ERR_ARG = range(6)
AS_DUP_SUM, AS_DUP_LAST = 0, 1

_lib = None


class NativeLibraryError(SparseError, RuntimeError):
    """libbsparse.so is missing or cannot run (no CUDA device)."""


def load():
    """Load the shared library (no device needed).  Raises if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                "%s is not built; run `python -c 'import __graft_entry__ as g; g.build()'`" % LIB_PATH
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    """The library, for a call that will launch kernels: needs a CUDA device."""
    L = load()
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the B200 kernels cannot run and there is no CPU fallback")
    return L


def check(rc: int) -> None:
    if rc == AS_OK:
        return
    msg = load().as_last_error().decode(errors="replace")
    if rc == AS_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == AS_ERR_COORD:
        raise CoordinateError(msg)
    if rc == AS_ERR_CORRUPT:
        raise CorruptionError(msg)
    raise NativeLibraryError("libbsparse error %d: %s" % (rc, msg))


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_WS_CACHE = {}


def workspace(nbytes: int, device, key=None) -> torch.Tensor:
    """Scratch for one library call.  With `key`, a buffer kept per (device,
    current stream, key) and grown on demand: the sort-reduce kernel
    (construction / flush / transpose) leaves its workspace state consistent
    and skips re-zeroing it on the next call (sortreduce.cuh); calls on one
    stream are ordered, so reuse is safe."""
    nbytes = max(int(nbytes), 256)
    if key is None or nbytes > (256 << 20):  # (large scratch is not kept)
        return torch.empty(nbytes, dtype=torch.uint8, device=device)
    device = torch.device(device)
    ck = (device.index if device.index is not None else torch.cuda.current_device(),
          torch.cuda.current_stream(device).cuda_stream, key)
    buf = _WS_CACHE.get(ck)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS_CACHE[ck] = buf
    return buf

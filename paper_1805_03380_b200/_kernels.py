"""Device kernels over flat CSC arrays -- the B200 replacement of the
reference's flat-array kernel module (autosparse/_kernels.py:1-175,
csc.canonicalize csc.py:148-193, rbt.to_csc rbt.py:444-458).

Arrays are torch CUDA tensors: indices int32, values float64 (or float32
where noted), col_ptr int32[n_cols+1].  Every function launches the
sm_100a kernels of libbsparse.so on the current stream; outputs whose size
is data dependent are sized on the device and read back with one 16-byte
device->host copy (the only synchronisation).  There is no CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _lib
from ._lib import check, ptr, stream, workspace

DUP_SUM = "sum"
DUP_LAST = "last"
_DUP = {DUP_SUM: _lib.AS_DUP_SUM, DUP_LAST: _lib.AS_DUP_LAST}


def _dev(device=None):
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _read_info(info):
    nnz, bad = (int(x) for x in info.cpu().tolist())
    return nnz, bad


_upload_lock = threading.Lock()
_upload_stage = {"buf": None, "event": None}


def _upload_threads():
    env = os.environ.get("AS_UPLOAD_THREADS")
    if env:
        return max(1, int(env))
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    # half the cores, at most 8: a descheduled helper stalls the whole call
    return max(1, min(8, cores // 2))


def upload_coo(rows, cols, vals, device=None, shape=None, bad_out=None):
    """int64 host triplets -> device (int32 rows, int32 cols, vals) through
    as_upload_coo_i64: host threads narrow the indices into pinned staging
    while the values are copied, so 16 bytes per triplet cross PCIe instead
    of 24.  rows / cols: contiguous CPU int64 tensors (pinned or not); vals:
    CPU float tensor (pinned: copied by the same call).  An index outside
    [0, 2^31) arrives as -1 (coo_to_csc reports it as out of range).
    shape = (n_rows, n_cols) whose index bit widths fit 31 bits together:
    the indices travel packed as one 32-bit key per triplet
    (as_upload_coo_packed, 12 bytes per triplet; coordinates outside the
    shape arrive as -1).  bad_out (a list): receives the first out-of-shape
    triplet's index or -1 when the packed path ran (the packers see every
    coordinate)."""
    L = _lib.lib()
    dev = _dev(device)
    n = int(rows.shape[0])
    assert rows.dtype == torch.int64 and cols.dtype == torch.int64 and not rows.is_cuda and not cols.is_cuda
    assert int(cols.shape[0]) == n and int(vals.shape[0]) == n
    rows, cols, vals = rows.contiguous(), cols.contiguous(), vals.contiguous()
    d_rows = torch.empty(n, dtype=torch.int32, device=dev)
    d_cols = torch.empty(n, dtype=torch.int32, device=dev)
    pinned_vals = vals.is_pinned()
    d_vals = torch.empty(n, dtype=vals.dtype, device=dev) if pinned_vals else vals.to(dev)
    if n == 0:
        return d_rows, d_cols, d_vals
    with _upload_lock:
        st = _upload_stage
        if st["event"] is not None:
            st["event"].synchronize()  # the previous call's copies have left the staging
        if st["buf"] is None or st["buf"].numel() < 2 * n:
            st["buf"] = torch.empty(2 * n, dtype=torch.int32).pin_memory()
        buf = st["buf"]
        chunks = int(os.environ.get("AS_UPLOAD_CHUNKS", "1"))  # measured: 1 chunk 599 us per e2e step, 2: 620, 4: 643
        with torch.cuda.device(dev):
            packed = shape is not None and min(shape) > 0 and \
                (int(shape[0]) - 1).bit_length() + (int(shape[1]) - 1).bit_length() <= 31
            if packed:
                d_keys = torch.empty(n, dtype=torch.int32, device=dev)
                first_bad = ctypes.c_int64(-1)
                check(L.as_upload_coo_packed(ptr(rows), ptr(cols), ptr(vals) if pinned_vals else None, n,
                                             vals.element_size(), int(shape[0]), int(shape[1]), ptr(buf), ptr(d_keys),
                                             ptr(d_rows), ptr(d_cols), ptr(d_vals), _upload_threads(), chunks,
                                             ctypes.addressof(first_bad), stream()))
                if bad_out is not None:
                    bad_out.append(int(first_bad.value))
            else:
                check(L.as_upload_coo_i64(ptr(rows), ptr(cols), ptr(vals) if pinned_vals else None, n,
                                          vals.element_size(), ptr(buf), buf.data_ptr() + 4 * n, ptr(d_rows),
                                          ptr(d_cols), ptr(d_vals), _upload_threads(), chunks, stream()))
            ev = torch.cuda.Event()
            ev.record()
        st["event"] = ev
    return d_rows, d_cols, d_vals


_u16 = {}


def u16_stage(n, device):
    """Pinned uint16 host stage and device scratch for CscData.to_host's
    half-width row read-back (kept per device, grown on demand).  One
    read-back at a time per device (the stage is waited on before reuse)."""
    key = torch.device(device).index
    st = _u16.get(key)
    if st is None or st[0].numel() < n:
        st = (torch.empty(max(n, 1), dtype=torch.int16).pin_memory(),
              torch.empty(max(n, 1), dtype=torch.int16, device=device))
        _u16[key] = st
    return st


def coo_to_csc(n_rows, n_cols, rows, cols, vals, dup=DUP_SUM, out=None, lazy=False):
    """Canonical CSC from COO triplets (csc.canonicalize, csc.py:148-193):
    stable column-major order, duplicates summed in np.add.reduceat order or
    last-wins, exact zeros pruned.  rows/cols int32 or int64, on the device or
    in pinned host memory (then read over PCIe inside the kernel); `out` =
    (col_ptr, row_idx, vals) buffers to write (device or pinned host, sized
    n_cols + 1 / n / n).  Returns (col_ptr, row_idx, vals, first_bad) where
    first_bad is the index of the first out-of-range triplet or None (those
    are skipped)."""
    L = _lib.lib()
    dev = vals.device if vals.is_cuda else torch.device("cuda", torch.cuda.current_device())
    n = int(vals.shape[0])
    assert rows.dtype == cols.dtype and rows.dtype in (torch.int32, torch.int64)
    if not vals.is_cuda and n > 0:
        assert rows.is_pinned() and cols.is_pinned() and vals.is_pinned(), "host triplets must be pinned"
    idx_bytes = 4 if rows.dtype == torch.int32 else 8
    f = L.as_coo_to_csc_f64 if vals.dtype == torch.float64 else L.as_coo_to_csc_f32
    if out is not None:
        col_ptr, row_idx, out_vals = out
    else:
        col_ptr = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
        row_idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        out_vals = torch.empty(max(n, 1), dtype=vals.dtype, device=dev)
    info = torch.empty(2, dtype=torch.int64, device=dev)
    ws_bytes = L.as_build_workspace_bytes(n, n_cols)
    ws = workspace(ws_bytes, dev, key="sortreduce")
    check(f(n_rows, n_cols, n, ptr(rows), ptr(cols), idx_bytes, ptr(vals), _DUP[dup], ptr(col_ptr), ptr(row_idx),
            ptr(out_vals), ptr(info), ptr(ws), ws_bytes, stream()))
    if lazy:  # (full-capacity outputs and the device info[2]; the caller knows the input is in range)
        return col_ptr, row_idx, out_vals, info
    nnz, bad = _read_info(info)
    return col_ptr, row_idx[:nnz], out_vals[:nnz], (bad if bad < n else None)


def flush_log(n_rows, n_cols, base, log_rows, log_cols, log_vals):
    """Insertion-cache flush (rbt.to_csc over RbtStore semantics,
    rbt.py:371-458): base CSC (col_ptr, row_idx, vals) overwritten by the write
    log in order; last write wins, a 0.0 write erases.  log_* int32 / float64.
    Returns (col_ptr, row_idx, vals, first_bad_log_index_or_None)."""
    L = _lib.lib()
    b_ptr, b_rows, b_vals = base
    dev = b_ptr.device
    nb = int(b_rows.shape[0])
    nl = int(log_vals.shape[0])
    cap = max(nb + nl, 1)
    col_ptr = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    row_idx = torch.empty(cap, dtype=torch.int32, device=dev)
    out_vals = torch.empty(cap, dtype=torch.float64, device=dev)
    info = torch.empty(2, dtype=torch.int64, device=dev)
    ws_bytes = L.as_flush_workspace_bytes(nb, nl, n_cols)
    ws = workspace(ws_bytes, dev, key="sortreduce")
    check(L.as_flush_log_f64(n_rows, n_cols, nb, ptr(b_ptr), ptr(b_rows), ptr(b_vals), nl, ptr(log_rows),
                             ptr(log_cols), ptr(log_vals), ptr(col_ptr), ptr(row_idx), ptr(out_vals), ptr(info),
                             ptr(ws), ws_bytes, stream()))
    nnz, bad = _read_info(info)
    return col_ptr, row_idx[:nnz], out_vals[:nnz], (bad if bad < nl else None)


def transpose(n_rows, n_cols, col_ptr, row_idx, vals):
    """CSC of A^T (_kernels.transpose, _kernels.py:130-150).  No sync."""
    L = _lib.lib()
    dev = col_ptr.device
    nnz = int(row_idx.shape[0])
    t_ptr = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
    t_rows = torch.empty(nnz, dtype=torch.int32, device=dev)
    t_vals = torch.empty(nnz, dtype=vals.dtype, device=dev)
    ws_bytes = L.as_transpose_workspace_bytes(nnz, n_rows)
    ws = workspace(ws_bytes, dev, key="sortreduce")
    f = L.as_csc_transpose_f64 if vals.dtype == torch.float64 else L.as_csc_transpose_f32
    check(f(n_rows, n_cols, nnz, ptr(col_ptr), ptr(row_idx), ptr(vals), ptr(t_ptr), ptr(t_rows), ptr(t_vals),
            ptr(ws), ws_bytes, stream()))
    return t_ptr, t_rows, t_vals


def linear_combine(n_rows, n_cols, a, b, alpha, beta):
    """alpha*A + beta*B (_kernels.linear_combine, _kernels.py:12-48)."""
    L = _lib.lib()
    a_ptr, a_rows, a_vals = a
    b_ptr, b_rows, b_vals = b
    dev = a_ptr.device
    na, nb = int(a_rows.shape[0]), int(b_rows.shape[0])
    cap = max(na + nb, 1)
    col_ptr = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    row_idx = torch.empty(cap, dtype=torch.int32, device=dev)
    out_vals = torch.empty(cap, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws_bytes = L.as_add_workspace_bytes(n_cols, na, nb)
    ws = workspace(ws_bytes, dev)
    check(L.as_csc_add_f64(n_rows, n_cols, float(alpha), float(beta), ptr(a_ptr), ptr(a_rows), ptr(a_vals),
                           ptr(b_ptr), ptr(b_rows), ptr(b_vals), na, nb, ptr(col_ptr), ptr(row_idx), ptr(out_vals),
                           ptr(info), ptr(ws), ws_bytes, stream()))
    nnz = int(info[0].item())
    return col_ptr, row_idx[:nnz], out_vals[:nnz]


def spgemm_products(n_rows_a, n_inner, n_cols_b, a_ptr, b_ptr, b_rows):
    """Per-column product counts' prefix sum (int64[n_cols_b+1]) and total."""
    L = _lib.lib()
    dev = a_ptr.device
    prod_ptr = torch.empty(n_cols_b + 1, dtype=torch.int64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws_bytes = L.as_spgemm_products_workspace_bytes(n_cols_b)
    ws = workspace(ws_bytes, dev)
    check(L.as_spgemm_products(n_rows_a, n_inner, n_cols_b, ptr(a_ptr), ptr(b_ptr), ptr(b_rows), ptr(prod_ptr),
                               ptr(info), ptr(ws), ws_bytes, stream()))
    return prod_ptr, int(info[0].item())


def spgemm(n_rows_a, n_inner, n_cols_b, a, b):
    """C = A @ B (_kernels.spgemm, _kernels.py:51-103), bit-exact order."""
    L = _lib.lib()
    a_ptr, a_rows, a_vals = a
    b_ptr, b_rows, b_vals = b
    dev = a_ptr.device
    prod_ptr, total = spgemm_products(n_rows_a, n_inner, n_cols_b, a_ptr, b_ptr, b_rows)
    cap = max(total, 1)
    col_ptr = torch.empty(n_cols_b + 1, dtype=torch.int32, device=dev)
    row_idx = torch.empty(cap, dtype=torch.int32, device=dev)
    out_vals = torch.empty(cap, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    nnz_b = int(b_rows.numel())
    ws_bytes = L.as_spgemm_workspace_bytes(n_cols_b, nnz_b, total)
    ws = workspace(ws_bytes, dev)
    check(L.as_spgemm_f64(n_rows_a, n_inner, n_cols_b, ptr(a_ptr), ptr(a_rows), ptr(a_vals), ptr(b_ptr), ptr(b_rows),
                          ptr(b_vals), nnz_b, ptr(prod_ptr), total, ptr(col_ptr), ptr(row_idx), ptr(out_vals), ptr(info),
                          ptr(ws), ws_bytes, stream()))
    nnz = int(info[0].item())
    return col_ptr, row_idx[:nnz], out_vals[:nnz]


def as_col_major(B):
    """(rows, k) tensor with unit row stride (Fortran order), and its ld."""
    if B.dim() == 1:
        return B.contiguous().view(-1, 1), max(int(B.shape[0]), 1)
    if B.stride(0) != 1 or B.stride(1) < max(B.shape[0], 1):
        B = B.t().contiguous().t()
    return B, int(B.stride(1)) if B.shape[1] > 1 else max(int(B.shape[0]), 1)


def spmm(n_rows, n_cols, csr, B, exact=None, out=None):
    """C = A @ B for dense column-major B (n_cols x k) using the CSR of A
    (= CSC arrays of A^T).  float64: exact (bit-identical to k calls of
    mat_times_vec, _kernels.py:118-127).  float32: FMA accumulation unless
    exact=True (float64 accumulation, one rounding at the end)."""
    L = _lib.lib()
    r_ptr, c_idx, vals = csr
    dev = r_ptr.device
    B, ldb = as_col_major(B)
    k = int(B.shape[1])
    if out is None:
        C = torch.empty((k, n_rows), dtype=vals.dtype, device=dev).t()
    else:
        C = out
    ldc = int(C.stride(1)) if k > 1 else max(n_rows, 1)
    ws_bytes = L.as_spmm_workspace_bytes(n_cols, k, vals.element_size())
    ws = workspace(ws_bytes, dev)
    if vals.dtype == torch.float64:
        check(L.as_spmm_csr_f64(n_rows, n_cols, k, ptr(r_ptr), ptr(c_idx), ptr(vals), ptr(B), ldb, ptr(C), ldc,
                                ptr(ws), ws_bytes, stream()))
    else:
        check(L.as_spmm_csr_f32(n_rows, n_cols, k, ptr(r_ptr), ptr(c_idx), ptr(vals), ptr(B), ldb, ptr(C), ldc,
                                1 if exact else 0, ptr(ws), ws_bytes, stream()))
    return C


# ---------------------------------------------------------------------------
# Multi-GPU entry points of the C ABI (csrc/mg.cu): the rank-local kernel and
# its NCCL collective in one call, on a communicator the caller owns.
# (dist.py drives the same ops through torch.distributed.)

def mg_init(nccl_comm: int, rank: int, world: int, nccl_library: str = None) -> None:
    """Hand the process's ncclComm_t (an integer address) to the library."""
    lib_path = nccl_library.encode() if nccl_library else None
    check(_lib.lib().as_mg_init(nccl_comm, rank, world, lib_path))


def mg_shutdown() -> None:
    check(_lib.lib().as_mg_shutdown())


def mg_fused_trace(n_rows, n_cols, a, b, c0, c1, out=None):
    """trace(A^T B): this rank's columns [c0, c1), all-gathered and combined in
    rank order; device tensor [sum, residual], identical on every rank."""
    L = _lib.lib()
    a_ptr, a_rows, a_vals = a
    b_ptr, b_rows, b_vals = b
    dev = a_ptr.device
    na, nb = int(a_rows.shape[0]), int(b_rows.shape[0])
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=dev)
    ws_bytes = L.as_mg_trace_workspace_bytes(n_cols, na, nb, L.as_mg_world())
    ws = workspace(ws_bytes, dev)
    check(L.as_mg_trace_atb_f64(n_rows, n_cols, ptr(a_ptr), ptr(a_rows), ptr(a_vals), ptr(b_ptr), ptr(b_rows),
                                ptr(b_vals), na, nb, c0, c1, ptr(out), ptr(ws), ws_bytes, stream()))
    return out


def mg_spmm(n_rows, n_cols, csr, B, out=None):
    """C = A @ B (float32): this rank's block of the dense columns, then an
    in-place all-gather into every rank's packed column-major C."""
    L = _lib.lib()
    r_ptr, c_idx, vals = csr
    dev = r_ptr.device
    B, ldb = as_col_major(B)
    k = int(B.shape[1])
    C = torch.empty((k, n_rows), dtype=torch.float32, device=dev).t() if out is None else out
    ws_bytes = L.as_spmm_workspace_bytes(n_cols, k, 4)
    ws = workspace(ws_bytes, dev)
    check(L.as_mg_spmm_csr_f32(n_rows, n_cols, k, ptr(r_ptr), ptr(c_idx), ptr(vals), ptr(B), ldb, ptr(C), n_rows,
                               ptr(ws), ws_bytes, stream()))
    return C


def mg_spgemm(n_rows_a, n_inner, n_cols_slice, a, b_slice):
    """C[:, slice] = A @ B[:, slice] on this rank (b_slice: a standalone CSC of
    the rank's columns of B) plus the all-gather of the slices' nnz.  Returns
    (col_ptr, row_idx, vals, slice_nnz int64[world], slice_offset int64[1]) --
    the last two stay on the device (dist.DistCsc)."""
    L = _lib.lib()
    a_ptr, a_rows, a_vals = a
    b_ptr, b_rows, b_vals = b_slice
    dev = a_ptr.device
    prod_ptr, total = spgemm_products(n_rows_a, n_inner, n_cols_slice, a_ptr, b_ptr, b_rows)
    cap = max(total, 1)
    col_ptr = torch.empty(n_cols_slice + 1, dtype=torch.int32, device=dev)
    row_idx = torch.empty(cap, dtype=torch.int32, device=dev)
    out_vals = torch.empty(cap, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    slice_nnz = torch.empty(max(L.as_mg_world(), 1), dtype=torch.int64, device=dev)
    slice_off = torch.empty(1, dtype=torch.int64, device=dev)
    nnz_b = int(b_rows.numel())
    ws_bytes = L.as_spgemm_workspace_bytes(n_cols_slice, nnz_b, total)
    ws = workspace(ws_bytes, dev)
    check(L.as_mg_spgemm_f64(n_rows_a, n_inner, n_cols_slice, ptr(a_ptr), ptr(a_rows), ptr(a_vals), ptr(b_ptr),
                             ptr(b_rows), ptr(b_vals), nnz_b, ptr(prod_ptr), total, ptr(col_ptr), ptr(row_idx),
                             ptr(out_vals), ptr(info), ptr(ws), ws_bytes, ptr(slice_nnz), ptr(slice_off), stream()))
    nnz = int(info[0].item())
    return col_ptr, row_idx[:nnz], out_vals[:nnz], slice_nnz, slice_off


def spmm_csc(n_rows, n_cols, csc, B, out=None):
    """C = A @ B straight over the CSC of A (column-merge, float32; no CSR
    needed): the reference's loop order (_kernels.mat_times_vec,
    _kernels.py:118-127) for 16 dense columns at a time, additions in arrival
    order (tolerance 1e-5)."""
    L = _lib.lib()
    c_ptr, r_idx, vals = csc
    dev = c_ptr.device
    if vals.dtype != torch.float32:
        raise TypeError("spmm_csc is the float32 path")
    B, ldb = as_col_major(B)
    k = int(B.shape[1])
    C = torch.empty((k, n_rows), dtype=torch.float32, device=dev).t() if out is None else out
    ldc = int(C.stride(1)) if k > 1 else max(n_rows, 1)
    nnz = int(r_idx.numel())
    ws_bytes = L.as_spmm_csc_workspace_bytes(n_rows, nnz)
    ws = workspace(ws_bytes, dev)
    check(L.as_spmm_csc_f32(n_rows, n_cols, nnz, k, ptr(c_ptr), ptr(r_idx), ptr(vals), ptr(B), ldb, ptr(C), ldc,
                            ptr(ws), ws_bytes, stream()))
    return C


def mat_times_vec(n_rows, n_cols, csr, x):
    """y = A x (_kernels.mat_times_vec, _kernels.py:118-127), bit-exact."""
    return spmm(n_rows, n_cols, csr, x.view(-1, 1), exact=True).reshape(-1)


def vec_times_mat(n_rows, n_cols, csc, v):
    """w = v^T A (_kernels.vec_times_mat, _kernels.py:106-115), bit-exact."""
    L = _lib.lib()
    c_ptr, r_idx, vals = csc
    w = torch.empty(n_cols, dtype=torch.float64, device=c_ptr.device)
    check(L.as_vecmat_csc_f64(n_rows, n_cols, ptr(c_ptr), ptr(r_idx), ptr(vals), ptr(v), ptr(w), stream()))
    return w


def fused_trace(n_rows, n_cols, a, b, out=None):
    """trace(A^T B) (_kernels.fused_trace, _kernels.py:153-175) as a device
    tensor [sum, residual] (double-double); no sync."""
    L = _lib.lib()
    a_ptr, a_rows, a_vals = a
    b_ptr, b_rows, b_vals = b
    dev = a_ptr.device
    na, nb = int(a_rows.shape[0]), int(b_rows.shape[0])
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=dev)
    ws_bytes = L.as_trace_workspace_bytes(n_cols, na, nb)
    ws = workspace(ws_bytes, dev)
    check(L.as_trace_atb_f64(n_rows, n_cols, ptr(a_ptr), ptr(a_rows), ptr(a_vals), ptr(b_ptr), ptr(b_rows),
                             ptr(b_vals), na, nb, ptr(out), ptr(ws), ws_bytes, stream()))
    return out


# ---------------------------------------------------------------------------
# construction-funnelled ops and segmented reductions (funnel.cu)

XF_ID, XF_ABS, XF_SQUARE, XF_POW = 0, 1, 2, 3
RED_SUM, RED_MIN, RED_MAX, RED_MAXABS = 0, 1, 2, 3


def expand_cols(n_cols, col_ptr, nnz):
    """Column index of every element of a CSC (int32, device)."""
    out = torch.empty(max(nnz, 1), dtype=torch.int32, device=col_ptr.device)
    check(_lib.lib().as_expand_cols(n_cols, ptr(col_ptr), ptr(out), stream()))
    return out[:nnz]


def kron_triplets(a, a_cols, b, b_cols, b_n_rows, b_n_cols):
    """(rows, cols, vals) of ops.kron (ops.py:131-143) in the reference's order."""
    (_, ar, av), (_, br, bv) = a, b
    na, nb = int(ar.shape[0]), int(br.shape[0])
    dev = ar.device
    n = na * nb
    rows = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cols = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    check(_lib.lib().as_kron_triplets_f64(na, ptr(ar), ptr(a_cols), ptr(av), nb, ptr(br), ptr(b_cols), ptr(bv),
                                          b_n_rows, b_n_cols, ptr(rows), ptr(cols), ptr(vals), stream()))
    return rows[:n], cols[:n], vals[:n]


def repmat_triplets(a, a_cols, n_rows, n_cols, reps_r, reps_c):
    """(rows, cols, vals) of ops.repmat (ops.py:146-163) in the reference's order."""
    _, ar, av = a
    nnz = int(ar.shape[0])
    dev = ar.device
    n = nnz * reps_r * reps_c
    rows = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cols = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    check(_lib.lib().as_repmat_triplets_f64(nnz, ptr(ar), ptr(a_cols), ptr(av), n_rows, n_cols, reps_r, reps_c,
                                            ptr(rows), ptr(cols), ptr(vals), stream()))
    return rows[:n], cols[:n], vals[:n]


def segment_reduce(seg_ptr, vals, kind, full, xf=XF_ID, p=1.0):
    """Per-segment fold (np.add.at order) / min / max with the implicit-zero rule."""
    n_seg = int(seg_ptr.shape[0]) - 1
    out = torch.empty(max(n_seg, 1), dtype=torch.float64, device=seg_ptr.device)
    check(_lib.lib().as_segment_reduce_f64(n_seg, ptr(seg_ptr), ptr(vals), kind, xf, float(p), full, ptr(out),
                                           stream()))
    return out[:n_seg]


def pairwise_sum(x, xf=XF_ID, p=1.0):
    """np.sum of (transformed) x in numpy's pairwise order; device scalar."""
    L = _lib.lib()
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    wb = L.as_pairwise_workspace_bytes()
    ws = workspace(wb, x.device)
    check(L.as_pairwise_sum_f64(int(x.shape[0]), ptr(x), xf, float(p), ptr(out), ptr(ws), wb, stream()))
    return out


def csc_window(n_rows, n_cols, csc, r0, r1, c0, c1):
    """Rows [r0, r1] x cols [c0, c1] of a CSC, re-indexed to the origin."""
    L = _lib.lib()
    p, r, v = csc
    dev = p.device
    nc = c1 - c0 + 1
    cap = max(int(r.shape[0]), 1)
    out_p = torch.empty(nc + 1, dtype=torch.int32, device=dev)
    out_r = torch.empty(cap, dtype=torch.int32, device=dev)
    out_v = torch.empty(cap, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    wb = L.as_window_workspace_bytes(nc)
    ws = workspace(wb, dev)
    check(L.as_csc_window_f64(n_rows, n_cols, ptr(p), ptr(r), ptr(v), r0, r1, c0, c1, ptr(out_p), ptr(out_r),
                              ptr(out_v), ptr(info), ptr(ws), wb, stream()))
    nnz = int(info[0].item())
    return out_p, out_r[:nnz], out_v[:nnz]


def csc_diag(n_rows, n_cols, csc, k, length):
    p, r, v = csc
    out = torch.empty(max(length, 1), dtype=torch.float64, device=p.device)
    check(_lib.lib().as_csc_diag_f64(n_rows, n_cols, ptr(p), ptr(r), ptr(v), k, length, ptr(out), stream()))
    return out[:length]


def scale_by_label(labels, vals, norms):
    out = torch.empty_like(vals)
    check(_lib.lib().as_scale_by_label_f64(int(vals.shape[0]), ptr(labels), ptr(vals), ptr(norms), ptr(out),
                                           stream()))
    return out

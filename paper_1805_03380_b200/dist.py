"""Multi-GPU sharding of the partitioned hot-path operations.

One process per GPU (torch.distributed, NCCL over NVLink in production, gloo
in the CPU tests).  The three operations that shard are split by CSC column
ranges and exchange only what the math requires:

* trace(A^T B): A and B split by the same column ranges, balanced on
  nnz(A[:,j]) + nnz(B[:,j]); each rank returns a double-double partial; one
  all_gather of 2 float64 per rank, combined in rank order with TwoSum, so
  the result does not depend on the number of ranks' reduction tree.
* SpMM C = A X: A (its cached CSR) replicated, the k dense columns of X split
  into contiguous blocks; each rank computes its C block; the blocks are
  all-gathered (or left distributed).
* SpGEMM C = A B: A replicated, B's columns split into ranges of equal
  Gustavson product counts (Zipf column lengths make equal-nnz splits badly
  imbalanced); each rank builds its CSC slice; slices are gathered and their
  col_ptr rebased by an exclusive scan of slice nnz.

Construction, flush, transpose and add run on one GPU (north star); under
torchrun the bench gives every rank its own independent batch (weak scaling).

The local kernels are injectable (`local=`) so the partition and exchange
logic can be exercised with the CPU oracle in world-size-2 gloo tests; the
default local implementation is the GPU kernels.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


# ---------------------------------------------------------------------------
# partitioning (pure functions, no communication)

def split_by_weight(weights: Sequence[int], n_parts: int) -> np.ndarray:
    """Column boundaries [0 = b0 <= b1 <= ... <= b_n = len(weights)] that
    split the prefix sum of `weights` into n_parts ranges of ~equal weight
    (each boundary is the first column whose prefix reaches k/n of the total)."""
    w = np.asarray(weights, dtype=np.int64)
    n = w.shape[0]
    pre = np.concatenate([[0], np.cumsum(w)])
    total = pre[-1]
    bounds = np.empty(n_parts + 1, np.int64)
    bounds[0] = 0
    bounds[-1] = n
    for k in range(1, n_parts):
        target = (total * k + n_parts - 1) // n_parts
        bounds[k] = int(np.searchsorted(pre, target, side="left"))
        bounds[k] = min(max(bounds[k], bounds[k - 1]), n)
    return bounds


def csc_column_slice(col_ptr, row_idx, vals, c0: int, c1: int):
    """Standalone CSC of columns [c0, c1) (col_ptr rebased)."""
    if isinstance(col_ptr, torch.Tensor):
        s, e = int(col_ptr[c0].item()), int(col_ptr[c1].item())
        return (col_ptr[c0:c1 + 1] - s).to(col_ptr.dtype), row_idx[s:e], vals[s:e]
    s, e = int(col_ptr[c0]), int(col_ptr[c1])
    return np.asarray(col_ptr[c0:c1 + 1]) - s, np.asarray(row_idx[s:e]), np.asarray(vals[s:e])


def _rank_world(group):
    return dist.get_rank(group), dist.get_world_size(group)


# ---------------------------------------------------------------------------
# double-double combination (matches the device kernel's reduction)

def two_sum(a: float, b: float):
    s = a + b
    bp = s - a
    err = (a - (s - bp)) + (b - bp)
    return s, err


def dd_combine(parts: Sequence[Sequence[float]]) -> float:
    """Sum of (hi, lo) partials in the given order with TwoSum carries."""
    s, e = 0.0, 0.0
    for hi, lo in parts:
        e += lo
        s, err = two_sum(s, hi)
        e += err
    return s + e


# ---------------------------------------------------------------------------
# helpers

def comm_device(group=None) -> torch.device:
    """Device the collectives run on: the rank's GPU under NCCL, else CPU."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _host(x) -> np.ndarray:
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _tensor(x, device) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device)


# ---------------------------------------------------------------------------
# trace(A^T B)

def _gpu_trace_local(n_rows, n_cols, a, b):
    from . import _kernels

    return _kernels.fused_trace(n_rows, n_cols, a, b)  # device f64[2] (hi, lo), no sync


def trace_shard(a, b, group=None):
    """This rank's column range and the (col_ptr, row_idx, vals) slices of A
    and B, balanced on nnz(A[:,j]) + nnz(B[:,j])."""
    rank, world = _rank_world(group)
    weights = np.diff(_host(a[0]).astype(np.int64)) + np.diff(_host(b[0]).astype(np.int64))
    bounds = split_by_weight(weights, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    return c0, c1, csc_column_slice(*a, c0, c1), csc_column_slice(*b, c0, c1)


def trace_exchange(part, group=None) -> float:
    """One all_gather of every rank's (hi, lo) partial, combined in rank order."""
    _, world = _rank_world(group)
    mine = _tensor(np.asarray(part, dtype=np.float64) if not isinstance(part, torch.Tensor) else part,
                   comm_device(group)).to(torch.float64).reshape(2)
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    return dd_combine([g.cpu().tolist() for g in gathered])


def dist_fused_trace(n_rows: int, n_cols: int, a, b, group=None,
                     local: Optional[Callable] = None) -> float:
    """trace(A^T B) over column shards.  `a`, `b`: full (col_ptr, row_idx,
    vals) on every rank (or at least their column slices' inputs)."""
    local = local or _gpu_trace_local
    c0, c1, sa, sb = trace_shard(a, b, group)
    return trace_exchange(local(n_rows, c1 - c0, sa, sb), group)


# ---------------------------------------------------------------------------
# SpMM C = A X

def _gpu_spmm_local(n_rows, n_cols, csr, X):
    from . import _kernels

    return _kernels.spmm(n_rows, n_cols, csr, X)


def spmm_block(k: int, group=None):
    """This rank's contiguous block [k0, k1) of the k dense columns."""
    rank, world = _rank_world(group)
    bounds = split_by_weight(np.ones(k, np.int64), world)
    return int(bounds[rank]), int(bounds[rank + 1]), bounds


def spmm_exchange(block, bounds, n_rows: int, group=None, dst: Optional[int] = None):
    """Reassemble C from the column blocks.  C is column-major, so rank q's
    block C[:, k0:k1] is one contiguous (k1 - k0) * n_rows run of C's storage:
    * dst=None: every rank gets C -- equal blocks land in C's storage with one
      all_gather_into_tensor (no padding, no copy after); unequal blocks are
      padded to the widest block, gathered, and the pad columns dropped;
    * dst=r: grouped point-to-point sends of the native blocks straight into
      C's column slices on rank r (exact sizes, no padding); other ranks get
      None.
    The result is an (n_rows, k) column-major tensor on the collective device."""
    rank, world = _rank_world(group)
    tb = _tensor(block, comm_device(group))
    if world == 1:
        return tb
    widths = [int(bounds[q + 1] - bounds[q]) for q in range(world)]
    k = int(bounds[-1])
    flat = tb.t().contiguous().view(-1)  # (k1 - k0) x n_rows: column-major block storage
    if dst is not None:
        out = torch.empty((k, n_rows), dtype=tb.dtype, device=tb.device) if rank == dst else None
        ops = []
        if rank == dst:
            for q in range(world):
                view = out[int(bounds[q]):int(bounds[q + 1])].view(-1)
                if q == dst:
                    view.copy_(flat)
                elif widths[q]:
                    ops.append(dist.P2POp(dist.irecv, view, q, group))
        elif widths[rank]:
            ops.append(dist.P2POp(dist.isend, flat, dst, group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return out.t() if out is not None else None
    if len(set(widths)) == 1:
        out = torch.empty((k, n_rows), dtype=tb.dtype, device=tb.device)
        dist.all_gather_into_tensor(out.view(-1), flat, group=group)
        return out.t()
    width = max(widths)
    pad = torch.zeros((width, n_rows), dtype=tb.dtype, device=tb.device)
    pad[: widths[rank]] = flat.view(widths[rank], n_rows)
    gathered = torch.empty((world, width, n_rows), dtype=tb.dtype, device=tb.device)
    dist.all_gather_into_tensor(gathered.view(-1), pad.view(-1), group=group)
    return torch.cat([gathered[q, : widths[q]] for q in range(world)], dim=0).t()


def dist_spmm(n_rows: int, n_cols: int, csr, X, group=None, gather: bool = True,
              local: Optional[Callable] = None, dst: Optional[int] = None):
    """Each rank computes C[:, k0:k1] for its block of dense columns.
    Returns the full C (gather=True; on rank dst only when dst is given) or
    (k0, k1, C_block)."""
    local = local or _gpu_spmm_local
    k0, k1, bounds = spmm_block(int(X.shape[1]), group)
    block = local(n_rows, n_cols, csr, X[:, k0:k1])
    if not gather:
        return k0, k1, block
    return spmm_exchange(block, bounds, n_rows, group, dst=dst)


# ---------------------------------------------------------------------------
# SpGEMM C = A B

def spgemm_column_weights(a_ptr, b_ptr, b_rows) -> np.ndarray:
    """Gustavson products per column of B (sum of |A[:,k]| over its entries)."""
    a_len = np.diff(np.asarray(a_ptr, dtype=np.int64))
    prod = a_len[np.asarray(b_rows, dtype=np.int64)]
    b_ptr = np.asarray(b_ptr, dtype=np.int64)
    pre = np.concatenate([[0], np.cumsum(prod)])
    return pre[b_ptr[1:]] - pre[b_ptr[:-1]]


def _gpu_spgemm_local(n_rows_a, n_inner, n_cols_b, a, b):
    from . import _kernels

    return _kernels.spgemm(n_rows_a, n_inner, n_cols_b, a, b)  # device CSC slice


def spgemm_shard(a, b, group=None):
    """This rank's range of B's columns (equal Gustavson products) and B's slice."""
    rank, world = _rank_world(group)
    w = spgemm_column_weights(_host(a[0]), _host(b[0]), _host(b[1]))
    bounds = split_by_weight(w, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    return c0, c1, bounds, csc_column_slice(*b, c0, c1)


class DistCsc:
    """A CSC matrix left distributed by column ranges: this rank holds columns
    [c0, c1) as a standalone CSC slice (col_ptr local), plus every slice's nnz
    and this slice's global element offset as DEVICE tensors (no host read).
    `global_col_ptr()` rebases the local col_ptr on the device."""

    def __init__(self, c0, c1, bounds, col_ptr, row_idx, vals, slice_nnz, offset):
        self.c0, self.c1, self.bounds = c0, c1, bounds
        self.col_ptr, self.row_idx, self.vals = col_ptr, row_idx, vals
        self.slice_nnz = slice_nnz  # int64 [world], device
        self.offset = offset        # int64 [1], device: elements before this slice

    def global_col_ptr(self):
        return self.col_ptr.to(torch.int64) + self.offset


def spgemm_exchange(p, r, v, bounds, group=None, dst: Optional[int] = 0, c_range=None):
    """Reassemble C = A B from the column slices, native types (int32 indices,
    float64 values):
    * one all_gather of the slice nnz (one int64 per rank, device-resident);
    * dst=None: leave C distributed -- returns a DistCsc whose global offset
      is an exclusive scan of the gathered nnz on the device (no host read,
      no bulk transfer);
    * dst=r: rank r receives every slice by grouped point-to-point transfers
      (batch_isend_irecv: NCCL grouped send/recv under NCCL) straight into
      the assembled CSC, col_ptr rebased on the device; returns (col_ptr,
      rows, vals) on rank r and None elsewhere.  Rank r reads the slice sizes
      once to size its buffers (the only host synchronisation)."""
    rank, world = _rank_world(group)
    devc = comm_device(group)
    p, r, v = _tensor(p, devc), _tensor(r, devc), _tensor(v, devc)
    nnz = torch.full((1,), r.shape[0], dtype=torch.int64, device=devc)
    if world == 1:
        sizes = nnz
    else:
        sizes = torch.empty(world, dtype=torch.int64, device=devc)
        dist.all_gather_into_tensor(sizes, nnz, group=group)
    starts = torch.cumsum(sizes, 0) - sizes
    if dst is None:
        c0, c1 = c_range if c_range is not None else (int(bounds[rank]), int(bounds[rank + 1]))
        return DistCsc(c0, c1, bounds, p, r, v, sizes, starts[rank:rank + 1])
    if rank != dst:
        ops = [dist.P2POp(dist.isend, x.contiguous(), dst, group) for x in (r, v, p) if x.numel()]
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        return None
    host_sizes = sizes.tolist()
    total = int(sum(host_sizes))
    n_cols = int(bounds[-1])
    rows = torch.empty(total, dtype=r.dtype, device=devc)
    vals = torch.empty(total, dtype=v.dtype, device=devc)
    col_ptr = torch.empty(n_cols + 1, dtype=torch.int64, device=devc)
    ptr_parts = []
    ops = []
    off = 0
    for q in range(world):
        sz, w = host_sizes[q], int(bounds[q + 1] - bounds[q])
        rv, vv = rows[off:off + sz], vals[off:off + sz]
        pq = p if q == dst else torch.empty(w + 1, dtype=p.dtype, device=devc)
        if q == dst:
            rv.copy_(r)
            vv.copy_(v)
        else:
            ops += [dist.P2POp(dist.irecv, x, q, group) for x in (rv, vv) if x.numel()]
            ops.append(dist.P2POp(dist.irecv, pq, q, group))
        ptr_parts.append(pq)
        off += sz
    for w_ in dist.batch_isend_irecv(ops) if ops else []:
        w_.wait()
    col_ptr[0] = 0
    for q in range(world):
        c0, c1 = int(bounds[q]), int(bounds[q + 1])
        col_ptr[c0 + 1:c1 + 1] = ptr_parts[q][1:].to(torch.int64) + starts[q]
    return col_ptr, rows, vals


def dist_spgemm(n_rows_a: int, n_inner: int, n_cols_b: int, a, b, group=None,
                local: Optional[Callable] = None, on_device: bool = False, dst: Optional[int] = 0):
    """C = A B with B's columns split into equal-product ranges.  dst=r:
    rank r gets the full C -- host arrays (col_ptr int64, rows int64, vals
    f64), or tensors on the collective device with on_device=True -- and the
    other ranks None; dst=None: every rank gets its DistCsc slice."""
    local = local or _gpu_spgemm_local
    c0, c1, bounds, sb = spgemm_shard(a, b, group)
    p, r, v = local(n_rows_a, n_inner, c1 - c0, a, sb)
    out = spgemm_exchange(p, r, v, bounds, group, dst=dst, c_range=(c0, c1))
    if out is None or isinstance(out, DistCsc) or on_device:
        return out
    cp, rr, vv = out
    return cp.cpu().numpy().astype(np.int64), rr.cpu().numpy().astype(np.int64), vv.cpu().numpy().astype(np.float64)

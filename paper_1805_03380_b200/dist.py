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
# trace(A^T B)

def _gpu_trace_local(n_rows, n_cols, a, b):
    from . import _kernels

    out = _kernels.fused_trace(n_rows, n_cols, a, b)
    return out.cpu().tolist()


def dist_fused_trace(n_rows: int, n_cols: int, a, b, group=None,
                     local: Optional[Callable] = None) -> float:
    """trace(A^T B) over column shards.  `a`, `b`: full (col_ptr, row_idx,
    vals) on every rank (or at least their column slices' inputs)."""
    local = local or _gpu_trace_local
    rank, world = _rank_world(group)
    a_ptr = a[0].cpu().numpy() if isinstance(a[0], torch.Tensor) else np.asarray(a[0])
    b_ptr = b[0].cpu().numpy() if isinstance(b[0], torch.Tensor) else np.asarray(b[0])
    weights = np.diff(a_ptr) + np.diff(b_ptr)
    bounds = split_by_weight(weights, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    sa = csc_column_slice(*a, c0, c1)
    sb = csc_column_slice(*b, c0, c1)
    hi_lo = local(n_rows, c1 - c0, sa, sb)
    mine = torch.tensor(hi_lo, dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    return dd_combine([g.cpu().tolist() for g in gathered])


# ---------------------------------------------------------------------------
# SpMM C = A X

def _gpu_spmm_local(n_rows, n_cols, csr, X):
    from . import _kernels

    return _kernels.spmm(n_rows, n_cols, csr, X)


def dist_spmm(n_rows: int, n_cols: int, csr, X, group=None, gather: bool = True,
              local: Optional[Callable] = None):
    """Each rank computes C[:, k0:k1] for its block of dense columns.
    Returns the full C (gather=True) or (k0, k1, C_block)."""
    local = local or _gpu_spmm_local
    rank, world = _rank_world(group)
    k = int(X.shape[1])
    bounds = split_by_weight(np.ones(k, np.int64), world)
    k0, k1 = int(bounds[rank]), int(bounds[rank + 1])
    block = local(n_rows, n_cols, csr, X[:, k0:k1])
    if not gather:
        return k0, k1, block
    # all_gather of column blocks (pad to the largest block)
    width = int(max(bounds[1:] - bounds[:-1]))
    tb = torch.as_tensor(np.asarray(block) if not isinstance(block, torch.Tensor) else block)
    pad = torch.zeros((n_rows, width), dtype=tb.dtype, device=tb.device)
    pad[:, : k1 - k0] = tb
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    cols = [parts[r][:, : int(bounds[r + 1] - bounds[r])] for r in range(world)]
    return torch.cat(cols, dim=1)


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

    p, r, v = _kernels.spgemm(n_rows_a, n_inner, n_cols_b, a, b)
    return p.cpu().numpy(), r.cpu().numpy(), v.cpu().numpy()


def dist_spgemm(n_rows_a: int, n_inner: int, n_cols_b: int, a, b, group=None,
                local: Optional[Callable] = None):
    """C = A B with B's columns split into equal-product ranges; returns the
    full C on every rank as host arrays (col_ptr int64, rows, vals)."""
    local = local or _gpu_spgemm_local
    rank, world = _rank_world(group)
    to_np = lambda x: x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)  # noqa: E731
    w = spgemm_column_weights(to_np(a[0]), to_np(b[0]), to_np(b[1]))
    bounds = split_by_weight(w, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    sb = csc_column_slice(*b, c0, c1)
    p, r, v = local(n_rows_a, n_inner, c1 - c0, a, sb)
    p, r, v = np.asarray(p, np.int64), np.asarray(r, np.int64), np.asarray(v, np.float64)
    # exchange slice sizes, then the padded slices
    nnz = torch.tensor([r.shape[0]], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, nnz, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(1, max(sizes))
    rows_pad = torch.zeros(cap, dtype=torch.int64)
    vals_pad = torch.zeros(cap, dtype=torch.float64)
    rows_pad[: r.shape[0]] = torch.from_numpy(r)
    vals_pad[: v.shape[0]] = torch.from_numpy(v)
    all_rows = [torch.empty_like(rows_pad) for _ in range(world)]
    all_vals = [torch.empty_like(vals_pad) for _ in range(world)]
    dist.all_gather(all_rows, rows_pad, group=group)
    dist.all_gather(all_vals, vals_pad, group=group)
    # col_ptr slices have different lengths: pad to the widest
    wmax = int(max(bounds[1:] - bounds[:-1])) + 1
    ptr_pad = torch.zeros(wmax, dtype=torch.int64)
    ptr_pad[: p.shape[0]] = torch.from_numpy(p)
    all_ptr = [torch.empty_like(ptr_pad) for _ in range(world)]
    dist.all_gather(all_ptr, ptr_pad, group=group)
    col_ptr = [np.zeros(1, np.int64)]
    base = 0
    rows_out, vals_out = [], []
    for q in range(world):
        width = int(bounds[q + 1] - bounds[q])
        pq = all_ptr[q][: width + 1].numpy()
        col_ptr.append(pq[1:] + base)
        rows_out.append(all_rows[q][: sizes[q]].numpy())
        vals_out.append(all_vals[q][: sizes[q]].numpy())
        base += sizes[q]
    return np.concatenate(col_ptr), np.concatenate(rows_out), np.concatenate(vals_out)

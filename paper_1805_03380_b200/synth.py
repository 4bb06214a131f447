"""Seeded synthetic inputs for the five BASELINE.json configurations
(SURVEY Appendix A).  The reference publishes no dataset for this path: its
own experiments use synthetic random matrices (PAPER.md:431-434,
bench.py:326-327), so these stand in with the configs' shapes, sizes and
value distributions.  All generators are numpy PCG64 (`default_rng(seed)`),
vectorised, and return host arrays in the reference's types (int64 indices,
float64 values unless the config says float32).
"""

from __future__ import annotations

import numpy as np


def _uniq(a: np.ndarray) -> np.ndarray:
    """Sorted distinct values (sort based; numpy 2.3's np.unique is far slower
    on large int64 arrays)."""
    s = np.sort(a)
    if s.shape[0] == 0:
        return s
    return s[np.concatenate([[True], s[1:] != s[:-1]])]


def _first_occurrences(a: np.ndarray) -> np.ndarray:
    """Indices of the first occurrence of each distinct value, ascending."""
    order = np.argsort(a, kind="stable")
    s = a[order]
    first = np.concatenate([[True], s[1:] != s[:-1]]) if s.shape[0] else np.empty(0, bool)
    return np.sort(order[first])


def _distinct_positions(rng, n_cells: int, k: int) -> np.ndarray:
    """k distinct linear positions in [0, n_cells), uniform, random order."""
    taken = np.empty(0, np.int64)
    while taken.shape[0] < k:
        need = k - taken.shape[0]
        draw = rng.integers(0, n_cells, size=need + need // 8 + 64)
        draw = draw[_first_occurrences(draw)]
        if taken.shape[0]:
            draw = draw[~np.isin(draw, taken)]
        taken = np.concatenate([taken, draw[:need]])
    return taken


def _csc_from_sorted_positions(pos: np.ndarray, n_rows: int, n_cols: int):
    cols = pos // n_rows
    rows = pos % n_rows
    offs = np.zeros(n_cols + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n_cols), out=offs[1:])
    return rows, offs


def cfg1_triplets(seed: int = 1, n_rows: int = 10000, n_cols: int = 10000, n: int = 1_000_000):
    """Batch construction: uniform (row, col), natural ~1% duplicates,
    values U[-1,1].  Seed 1 gives 995,078 distinct coordinates."""
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n_rows, n)
    cols = rng.integers(0, n_cols, n)
    vals = rng.uniform(-1, 1, n)
    return n_rows, n_cols, rows, cols, vals


def cfg2_writes(seed: int = 2, n: int = 50000, n_writes: int = 200_000, n_over: int = 10_000):
    """Incremental construction: n_writes element writes in random order,
    n_writes - n_over distinct fresh positions plus n_over overwrites of a
    uniformly chosen earlier-written position; values U[-1,1]."""
    rng = np.random.default_rng(seed)
    fresh = _distinct_positions(rng, n * n, n_writes - n_over)
    vals = rng.uniform(-1, 1, n_writes)
    over_slots = np.sort(rng.choice(np.arange(1, n_writes), n_over, replace=False))
    is_over = np.zeros(n_writes, bool)
    is_over[over_slots] = True
    pos = np.empty(n_writes, np.int64)
    pos[~is_over] = fresh
    fresh_before = np.cumsum(~is_over)[over_slots - 1]  # fresh slots strictly before each overwrite
    pick = (rng.random(n_over) * fresh_before).astype(np.int64)
    pos[over_slots] = fresh[pick]
    rows = pos % n
    cols = pos // n
    return n, n, rows, cols, vals


def cfg3_spmm(seed: int = 3, n: int = 1_000_000, per_col: int = 10, k: int = 64):
    """SpMM: A n x n float32 with exactly per_col distinct uniform rows per
    column, values N(0,1); dense B n x k float32 N(0,1), column-major.
    Returns (n, n, a_vals f32, a_rows i64, a_offs i64, B (n, k) F-order f32)."""
    rng = np.random.default_rng(seed)
    R = np.sort(rng.integers(0, n, (n, per_col)), axis=1)
    while True:
        dup = (R[:, 1:] == R[:, :-1]).any(axis=1)
        if not dup.any():
            break
        R[dup] = np.sort(rng.integers(0, n, (int(dup.sum()), per_col)), axis=1)
    a_rows = R.reshape(-1).astype(np.int64)
    a_vals = rng.standard_normal(n * per_col, dtype=np.float32)
    a_offs = np.arange(0, n * per_col + 1, per_col, dtype=np.int64)
    B = rng.standard_normal((k, n), dtype=np.float32).T  # (n, k) column-major view
    return n, n, a_vals, a_rows, a_offs, B


def cfg4_trace_pair(seed_a: int = 4, seed_b: int = 40, n: int = 100_000, nnz: int = 10_000_000):
    """Fused trace: A and B n x n float64, nnz distinct uniform positions each
    (independent generators), values U[-1,1].  Returns two CSC triples."""
    out = []
    for seed in (seed_a, seed_b):
        rng = np.random.default_rng(seed)
        draw = rng.integers(0, n * n, size=nnz + nnz // 100 + 1024)
        pos = _uniq(draw)
        while pos.shape[0] < nnz:
            pos = _uniq(np.concatenate([pos, rng.integers(0, n * n, size=nnz - pos.shape[0] + 1024)]))
        if pos.shape[0] > nnz:
            drop = rng.choice(pos.shape[0], pos.shape[0] - nnz, replace=False)
            keep = np.ones(pos.shape[0], bool)
            keep[drop] = False
            pos = pos[keep]
        vals = rng.uniform(-1, 1, nnz)
        rows, offs = _csc_from_sorted_positions(pos, n, n)
        out.append((vals, rows, offs))
    return n, n, out[0], out[1]


ZIPF_SHIFT = 0.7050885  # makes the truncated law's mean exactly 16 on [1, 4096]


def _zipf_lengths(rng, n: int, max_len: int = 4096, expo: float = 1.5):
    L = np.arange(1, max_len + 1, dtype=np.float64)
    p = (L - ZIPF_SHIFT) ** -expo
    cdf = np.cumsum(p / p.sum())
    cdf[-1] = 1.0
    return np.searchsorted(cdf, rng.random(n), side="right").astype(np.int64) + 1


def _distinct_rows_per_column(rng, n_rows: int, lens: np.ndarray):
    """Sorted distinct uniform rows per column with the given lengths."""
    n_cols = lens.shape[0]
    cols = np.repeat(np.arange(n_cols, dtype=np.int64), lens)
    keys = _uniq(cols * n_rows + rng.integers(0, n_rows, cols.shape[0]))
    while True:
        have = np.bincount(keys // n_rows, minlength=n_cols)
        short = lens - have
        if not short.any():
            break
        extra_cols = np.repeat(np.arange(n_cols, dtype=np.int64), short)
        keys = _uniq(np.concatenate([keys, extra_cols * n_rows + rng.integers(0, n_rows, extra_cols.shape[0])]))
    rows, offs = _csc_from_sorted_positions(keys, n_rows, n_cols)
    return rows, offs


def cfg5_pair(seed_a: int = 5, seed_b: int = 50, n: int = 200_000):
    """SpGEMM + add: A and B n x n float64, column lengths from the shifted
    Zipf(1.5) law on [1, 4096] (mean 16), distinct uniform rows, N(0,1)."""
    out = []
    for seed in (seed_a, seed_b):
        rng = np.random.default_rng(seed)
        lens = _zipf_lengths(rng, n)
        rows, offs = _distinct_rows_per_column(rng, n, lens)
        vals = rng.standard_normal(rows.shape[0])
        out.append((vals, rows, offs))
    return n, n, out[0], out[1]

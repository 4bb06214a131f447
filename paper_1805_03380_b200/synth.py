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


def _first_occurrences(a: np.ndarray) -> np.ndarray:
    """Indices of the first occurrence of each distinct value, ascending."""
    order = np.argsort(a, kind="stable")
    s = a[order]
    first = np.concatenate([[True], s[1:] != s[:-1]]) if s.shape[0] else np.empty(0, bool)
    return np.sort(order[first])


def sample_positions(n_cells: int, k: int, rng) -> np.ndarray:
    """k distinct linear positions in [0, n_cells), uniform without
    replacement, in draw order -- the reference's sampler, restated so the
    generator stream is the reference's for the same seed
    (ops._sample_positions, ops.py:377-397): a dense target (k > cells // 2)
    is a prefix of one permutation; otherwise batches of
    max(need + need // 4 + 16, 64) draws, each deduplicated keeping first
    occurrences in draw order, minus positions already taken."""
    if k == 0:
        return np.empty(0, np.int64)
    if k > n_cells // 2:
        return rng.permutation(n_cells)[:k].astype(np.int64)
    taken = np.empty(0, np.int64)
    need = k
    while need > 0:
        batch = rng.integers(0, n_cells, size=max(need + need // 4 + 16, 64))
        batch = batch[_first_occurrences(batch)]
        if taken.shape[0]:
            batch = batch[~np.isin(batch, taken)]
        taken = np.concatenate([taken, batch[:need]])
        need = k - taken.shape[0]
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
    fresh = sample_positions(n * n, n_writes - n_over, rng)
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
    column (rng.integers, columns with a repeat redrawn), values N(0,1); dense
    B n x k float32 N(0,1), column-major (float64 draws
    rounded to float32).
    Returns (n, n, a_vals f32, a_rows i64, a_offs i64, B (n, k) F-order f32)."""
    rng = np.random.default_rng(seed)
    R = np.sort(rng.integers(0, n, (n, per_col)), axis=1)
    while True:
        dup = (R[:, 1:] == R[:, :-1]).any(axis=1)
        if not dup.any():
            break
        R[dup] = np.sort(rng.integers(0, n, (int(dup.sum()), per_col)), axis=1)
    a_rows = R.reshape(-1).astype(np.int64)
    a_vals = rng.standard_normal(n * per_col).astype(np.float32)
    a_offs = np.arange(0, n * per_col + 1, per_col, dtype=np.int64)
    B = np.asfortranarray(rng.standard_normal((n, k)).astype(np.float32))  # (n, k) column-major
    return n, n, a_vals, a_rows, a_offs, B


def cfg4_trace_pair(seed_a: int = 4, seed_b: int = 40, n: int = 100_000, nnz: int = 10_000_000):
    """Fused trace: A and B n x n float64, nnz distinct uniform positions each
    (independent generators), values U[-1,1] -- SURVEY Appendix A:
    pos = _sample_positions(n*n, nnz, rng), vals = rng.uniform(-1, 1, nnz),
    rows = pos % n, cols = pos // n.  Seeds 4 / 40 give 9,976 coincident
    entries and trace(A^T B) = -6.0515221450266097.  Returns two CSC triples."""
    out = []
    for seed in (seed_a, seed_b):
        rng = np.random.default_rng(seed)
        pos = sample_positions(n * n, nnz, rng)
        vals = rng.uniform(-1, 1, nnz)
        order = np.argsort(pos, kind="stable")
        rows, offs = _csc_from_sorted_positions(pos[order], n, n)
        out.append((vals[order], rows, offs))
    return n, n, out[0], out[1]


ZIPF_SHIFT = 0.7050885  # makes the truncated law's mean exactly 16 on [1, 4096]


def _zipf_lengths(rng, n: int, max_len: int = 4096, expo: float = 1.5):
    """rng.choice(1..max_len, n, p) with p(L) ~ (L - ZIPF_SHIFT)^-expo
    (seeds 5 / 50 give 3,258,067 / 3,182,595)."""
    L = np.arange(1, max_len + 1, dtype=np.float64)
    p = (L - ZIPF_SHIFT) ** -expo
    return rng.choice(np.arange(1, max_len + 1), n, p=p / p.sum()).astype(np.int64)


def cfg5_pair(seed_a: int = 5, seed_b: int = 50, n: int = 200_000):
    """SpGEMM + add: A and B n x n float64, column lengths from the shifted
    Zipf(1.5) law on [1, 4096] (mean 16), per column rng.choice(n, L,
    replace=False) distinct uniform rows, sorted, then N(0,1) values
    (SURVEY Appendix A).  Seeds 5 / 50: nnz 3,258,067 / 3,182,595 (the
    survey's figures), 51,847,707 Gustavson products (the survey quotes
    52,338,873, which its textual recipe does not pin down)."""
    out = []
    for seed in (seed_a, seed_b):
        rng = np.random.default_rng(seed)
        lens = _zipf_lengths(rng, n)
        rows = np.concatenate([np.sort(rng.choice(n, int(L), replace=False)) for L in lens])
        offs = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=offs[1:])
        vals = rng.standard_normal(rows.shape[0])
        out.append((vals, rows.astype(np.int64), offs))
    return n, n, out[0], out[1]

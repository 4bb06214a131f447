"""Fused trace(A^T B): the warp-tile kernel (a warp's column pairs staged by bulk
copies in a per-warp pipeline, 2^LG lanes merging list segments) against the
oracle's restatement of _kernels.fused_trace (_kernels.py:153-175): every lane
count, pairs searched by the whole warp, tiles beyond the buffers (global
search), unaligned inputs (fallback), and the warp-per-column kernel on the
same cases.  Tolerance 1e-12 relative (the
north star's float64 bound; the sum is reordered, in double-double)."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_1805_03380_b200 import _kernels

    return _kernels


@pytest.fixture(params=[0, 1], ids=["tile", "warp-per-column"])
def engine(request):
    from paper_1805_03380_b200 import _lib

    L = _lib.lib()
    _lib.check(L.as_set_trace_engine(request.param))
    yield request.param
    _lib.check(L.as_set_trace_engine(0))


def _dev(c, shift=0):
    """Device CSC (offs int32, rows int32, vals); shift > 0 puts the row array at
    an address that is not 16-byte aligned."""
    vals, rows, offs = c
    r = torch.empty(rows.shape[0] + shift, dtype=torch.int32, device="cuda")
    r[shift:] = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int32), device="cuda")
    return (torch.as_tensor(np.ascontiguousarray(offs, dtype=np.int32), device="cuda"), r[shift:],
            torch.as_tensor(np.ascontiguousarray(vals), device="cuda"))


def _with_lens(seed, n_rows, lens):
    g = np.random.default_rng(seed)
    lens = np.asarray(lens)
    rows = np.concatenate([g.choice(n_rows, int(L), replace=False) for L in lens] + [np.zeros(0, np.int64)])
    cols = np.repeat(np.arange(lens.shape[0]), lens)
    return oracle.canonicalize(n_rows, lens.shape[0], rows, cols, g.uniform(-1, 1, rows.shape[0]))


def _check(K, n_rows, n_cols, a, b, shift=0):
    want = oracle.fused_trace(n_cols, *a, *b)
    got = K.fused_trace(n_rows, n_cols, _dev(a, shift), _dev(b, shift)).cpu().numpy()
    assert_close(float(got[0]), want)
    again = K.fused_trace(n_rows, n_cols, _dev(a, shift), _dev(b, shift)).cpu().numpy()
    assert np.array_equal(got.view(np.int64), again.view(np.int64))  # deterministic, residual included
    return got


# mean column length -> lanes per column pair 1, 2, 4, 8, 16, 32, then the warp-per-column kernel
@pytest.mark.parametrize("mean,n_cols", [(3, 5000), (30, 3001), (50, 2000), (100, 1500), (150, 777), (300, 300),
                                         (700, 130), (2000, 41)])
def test_every_lane_count(K, engine, mean, n_cols):
    n_rows = max(4 * mean, 2000)
    g = np.random.default_rng(mean)
    lens_a = g.poisson(mean, n_cols)
    lens_b = g.poisson(mean, n_cols)
    a, b = _with_lens(1, n_rows, lens_a), _with_lens(2, n_rows, lens_b)
    _check(K, n_rows, n_cols, a, b)
    # trace(A^T A) = ||A||_F^2: every entry is a match
    _check(K, n_rows, n_cols, a, a)


def test_long_and_oversized_columns(K, engine):
    # mean ~22 (2 lanes per pair, 16 pairs per warp tile, 768-entry buffers): pairs above
    # 128 entries per lane go to the whole warp (shared memory), tiles whose runs exceed
    # the buffers are searched pair by pair in global memory
    n_rows = 40_000
    g = np.random.default_rng(7)
    lens = g.poisson(8, 4000)
    lens[100:140] = 700            # tiles far beyond the buffers: every pair alone exceeds them
    lens[300:340] = 100            # tiles beyond the buffers made of pairs that would fit alone
    lens[400:420:3] = 400
    lens[900] = 3000
    lens[901] = 0
    lens[1500] = 12_000
    lens[1501] = 768 - 8 * 15      # a tile that just fits
    lens[2496:2512] = 1
    lens[2500] = 330               # long pair inside a tile that fits (whole warp)
    lens[3999] = 5000
    a = _with_lens(3, n_rows, lens)
    lens_b = lens.copy()
    lens_b[1500] = 5               # short against oversized
    lens_b[2000] = 11_000          # oversized against short
    b = _with_lens(4, n_rows, lens_b)
    _check(K, n_rows, 4000, a, b)
    _check(K, n_rows, 4000, a, a)
    _check(K, n_rows, 4000, b, a)


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_unaligned_row_arrays_fall_back(K, shift):
    n_rows, n_cols = 5000, 900
    g = np.random.default_rng(shift)
    a = _with_lens(5, n_rows, g.poisson(60, n_cols))
    b = _with_lens(6, n_rows, g.poisson(60, n_cols))
    _check(K, n_rows, n_cols, a, b, shift=shift)


@pytest.mark.parametrize("n_cols", [0, 1, 63, 64, 65, 255, 256, 257])
def test_tile_boundaries_and_empties(K, engine, n_cols):
    n_rows = 3000
    g = np.random.default_rng(n_cols + 11)
    lens_a = g.poisson(90, n_cols)
    lens_b = g.poisson(90, n_cols)
    lens_a[::7] = 0
    lens_b[3::5] = 0
    a, b = _with_lens(8, n_rows, lens_a), _with_lens(9, n_rows, lens_b)
    _check(K, n_rows, n_cols, a, b)
    empty = _with_lens(10, n_rows, np.zeros(n_cols, np.int64))
    got = _check(K, n_rows, n_cols, a, empty)
    assert float(got[0]) == 0.0


def test_engines_agree_bitwise_on_cfg4_shape(K):
    # 2 x 1e6 entries at cfg 4's column length; both kernels sum in double-double, so they
    # agree to the last bit of the rounded sum except for the order-dependent residual
    from paper_1805_03380_b200 import _lib

    n = 10_000
    g = np.random.default_rng(12)
    a = _with_lens(13, 100_000, g.poisson(100, n))
    b = _with_lens(14, 100_000, g.poisson(100, n))
    want = oracle.fused_trace(n, *a, *b)
    L = _lib.lib()
    out = []
    try:
        for e in (0, 1):
            _lib.check(L.as_set_trace_engine(e))
            out.append(float(K.fused_trace(100_000, n, _dev(a), _dev(b))[0].item()))
    finally:
        _lib.check(L.as_set_trace_engine(0))
    assert_close(out[0], want)
    assert abs(out[0] - out[1]) <= 4 * np.spacing(abs(want))

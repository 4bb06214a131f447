"""the native Matrix Market parser / formatter (csrc/mmio.cu,
host code, no GPU needed) against the reference's own load_mm / save_mm
outcomes recorded in tests/golden/mm.npz: the same canonical CSC (through the
oracle's canonicalize), the same exception class, message and line number,
and byte-identical saved text."""

import numpy as np
import pytest
import torch

import oracle
from conftest import load_golden

CASES = load_golden("mm")


@pytest.fixture(scope="module")
def mmio():
    from paper_1805_03380_b200 import _lib, io

    _lib.load()
    return io


@pytest.mark.parametrize("case", CASES, ids=lambda c: "%s_%s" % (c["outcome"], c.get("err_class", "ok")))
def test_parse_matches_reference(mmio, case):
    from paper_1805_03380_b200 import errors

    text = case["text"].tobytes()
    try:
        dims, rows, cols, vals = mmio.parse_mm(text)
        # the reference's duplicate check (io.py:127-130), done on the device by load_mm
        if rows.shape[0] and np.unique(cols * dims.n_rows + rows).shape[0] != rows.shape[0] and not case["lenient"]:
            raise errors.DuplicateEntryError("duplicate coordinates in input")
    except errors.SparseError as e:
        assert case["outcome"] == "error", e
        assert type(e).__name__ == case["err_class"]
        assert str(e) == case["err_msg"]
        return
    assert case["outcome"] == "ok"
    v, r, o = oracle.canonicalize(dims.n_rows, dims.n_cols, rows, cols, vals)
    assert np.array_equal(o, case["out_offs"]) and np.array_equal(r, case["out_rows"])
    assert np.array_equal(v.view(np.int64), case["out_vals"].view(np.int64))


@pytest.mark.parametrize("case", [c for c in CASES if c["outcome"] == "ok"])
def test_format_byte_identical(mmio, case):
    from paper_1805_03380_b200.csc import CscData, Dims

    d = CscData.from_reference_arrays(Dims(case["n_rows"], case["n_cols"]), case["out_vals"], case["out_rows"],
                                      case["out_offs"], device=torch.device("cpu"))
    assert mmio.format_mm(d).encode("ascii") == case["saved"].tobytes()


def test_parallel_parse_large(mmio):
    # > 1 MiB of entries: the multi-threaded path, errors found in later chunks
    rng = np.random.default_rng(5)
    n = 120_000
    r, c = rng.integers(1, 5000, n), rng.integers(1, 5000, n)
    v = rng.standard_normal(n)
    body = "".join("%d %d %.17g\n" % t for t in zip(r, c, v))
    head = "%%%%MatrixMarket matrix coordinate real general\n5000 5000 %d\n" % n
    dims, rows, cols, vals = mmio.parse_mm((head + body).encode())
    assert np.array_equal(rows, r - 1) and np.array_equal(cols, c - 1) and np.array_equal(vals, v)
    lines = body.splitlines()
    lines[100_000] = "7 8"
    from paper_1805_03380_b200.errors import CorruptionError, MatrixMarketError

    with pytest.raises(MatrixMarketError, match="line %d: entry needs" % (100_000 + 3)):
        mmio.parse_mm((head + "\n".join(lines) + "\n").encode())
    lines[100_000] = "9999 1 1.0"
    lines[110_000] = "1 1"
    with pytest.raises(CorruptionError, match="line %d: entry \\(9999, 1\\)" % (100_000 + 3)):
        mmio.parse_mm((head + "\n".join(lines) + "\n").encode())

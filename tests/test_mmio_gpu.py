"""SURVEY 8f-3 end to end: load_mm (native parse -> GPU duplicate check ->
GPU build) and save_mm against the reference outcomes in tests/golden/mm.npz."""

import io

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load_golden("mm"), ids=lambda c: "%s_%s" % (c["outcome"], c.get("err_class", "ok")))
def test_load_save_match_reference(case):
    from paper_1805_03380_b200 import errors, load_mm, save_mm

    text = case["text"].tobytes().decode("ascii")
    src = text if "\n" in text else io.StringIO(text)
    try:
        m = load_mm(src, lenient_duplicates=bool(case["lenient"]), device="cuda")
    except errors.SparseError as e:
        assert case["outcome"] == "error" and type(e).__name__ == case["err_class"] and str(e) == case["err_msg"]
        return
    assert case["outcome"] == "ok"
    d = m.csc()
    assert np.array_equal(d.col_offsets, case["out_offs"]) and np.array_equal(d.row_indices, case["out_rows"])
    assert np.array_equal(d.values.view(np.int64), case["out_vals"].view(np.int64))
    buf = io.StringIO()
    save_mm(m, buf)
    assert buf.getvalue().encode("ascii") == case["saved"].tobytes()


def test_round_trip_file(tmp_path):
    from paper_1805_03380_b200 import SpMat, load_mm, save_mm

    rng = np.random.default_rng(9)
    dense = np.zeros((30, 20))
    dense.flat[rng.integers(0, 600, 150)] = rng.standard_normal(150) * 1e-300
    m = SpMat.from_dense(dense, device="cuda")
    path = tmp_path / "m.mtx"
    save_mm(m, path)
    again = load_mm(path, device="cuda")
    assert again.csc().same_elements(m.csc())

"""The drop-in module with the reference's `_kernels` signatures
(paper_1805_03380_b200.ref_kernels), driven exactly as the reference's ops /
expr modules drive autosparse._kernels, against the golden vectors the
reference produced."""

import numpy as np
import pytest

from conftest import assert_csc_equal, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def k():
    from paper_1805_03380_b200 import ref_kernels

    return ref_kernels


def test_canonicalize(k):
    for c in load_golden("canonicalize"):
        got = k.canonicalize(c["n_rows"], c["n_cols"], c["rows"], c["cols"], c["vals"], c["dup"])
        assert_csc_equal(got, (c["out_vals"], c["out_rows"], c["out_offs"]), exact_values=True)


def test_rbt_flush(k):
    for c in load_golden("flush"):
        got = k.rbt_to_csc(c["n_rows"], c["n_cols"], (c["base_vals"], c["base_rows"], c["base_offs"]),
                           c["log_rows"], c["log_cols"], c["log_vals"])
        assert_csc_equal(got, (c["out_vals"], c["out_rows"], c["out_offs"]), exact_values=True)


def test_transpose(k):
    for c in load_golden("transpose"):
        got = k.transpose(c["n_rows"], c["n_cols"], c["vals"], c["rows"], c["offs"])
        assert_csc_equal(got, (c["out_vals"], c["out_rows"], c["out_offs"]), exact_values=True)


def test_linear_combine(k):
    for c in load_golden("linear_combine"):
        got = k.linear_combine(c["n_cols"], c["a_vals"], c["a_rows"], c["a_offs"], c["b_vals"], c["b_rows"],
                               c["b_offs"], c["alpha"], c["beta"])
        assert_csc_equal(got, (c["out_vals"], c["out_rows"], c["out_offs"]), exact_values=True)


def test_spgemm(k):
    for c in load_golden("spgemm"):
        got = k.spgemm(c["n_rows"], c["a_vals"], c["a_rows"], c["a_offs"], c["b_vals"], c["b_rows"], c["b_offs"],
                       c["n_cols"])
        assert_csc_equal(got, (c["out_vals"], c["out_rows"], c["out_offs"]), exact_values=True)


def test_spmv(k):
    for c in load_golden("spmv"):
        y = k.mat_times_vec(c["vals"], c["rows"], c["offs"], c["x"], c["n_rows"], c["n_cols"])
        w = k.vec_times_mat(c["v"], c["vals"], c["rows"], c["offs"], c["n_cols"])
        assert np.array_equal(y, c["y"]) and np.array_equal(w, c["w"])


def test_fused_trace(k):
    for c in load_golden("trace"):
        t = k.fused_trace(c["n_cols"], c["a_vals"], c["a_rows"], c["a_offs"], c["b_vals"], c["b_rows"], c["b_offs"])
        assert abs(t - c["trace"]) <= 1e-12 * max(1.0, abs(c["trace"]))

"""Pin the CPU oracle (oracle/) against the reference's golden vectors and
the literal known answers of the reference's own tests.

Every comparison here is bit-exact: the oracle restates the reference's
arithmetic order, so nothing may differ in the last ulp.
"""

import numpy as np
import pytest

import oracle
from conftest import assert_csc_equal, load_golden


def test_segment_sum_matches_numpy_reduceat(rng):
    for m in list(range(1, 40)) + [127, 128, 129, 130, 200, 257, 1000, 5000]:
        v = rng.standard_normal(m) * 10.0 ** rng.integers(-8, 8, m)
        assert oracle.segment_sum(v) == np.add.reduceat(v, [0])[0]


@pytest.mark.parametrize("case", load_golden("canonicalize"), ids=lambda c: "%sx%s_%s" % (c["n_rows"], c["n_cols"], c["dup"]))
def test_canonicalize_golden(case):
    got = oracle.canonicalize(case["n_rows"], case["n_cols"], case["rows"], case["cols"], case["vals"], case["dup"])
    assert_csc_equal(got, (case["out_vals"], case["out_rows"], case["out_offs"]), exact_values=True)


def test_canonicalize_reference_pins():
    # test_csc.py:18-47
    v, r, o = oracle.canonicalize(3, 2, [0, 2, 1], [0, 1, 1], [1.0, 3.0, 2.0])
    assert v.tolist() == [1.0, 2.0, 3.0] and r.tolist() == [0, 1, 2] and o.tolist() == [0, 1, 3]
    v, r, o = oracle.canonicalize(4, 4, [], [], [])
    assert v.size == 0 and o.tolist() == [0, 0, 0, 0, 0]
    v, r, o = oracle.canonicalize(2, 2, [0, 0], [0, 0], [5.0, -5.0])
    assert v.size == 0 and o.tolist() == [0, 0, 0]
    v, r, o = oracle.canonicalize(2, 2, [1, 1], [0, 0], [2.0, 3.0])
    assert v.tolist() == [5.0]
    v, r, o = oracle.canonicalize(2, 2, [1, 0, 1], [0, 1, 0], [2.0, 9.0, 3.0], "last")
    assert v.tolist() == [3.0, 9.0]


@pytest.mark.parametrize("case", load_golden("flush"), ids=lambda c: "%sx%s" % (c["n_rows"], c["n_cols"]))
def test_flush_golden(case):
    got = oracle.flush(case["n_rows"], case["n_cols"], (case["base_vals"], case["base_rows"], case["base_offs"]),
                       case["log_rows"], case["log_cols"], case["log_vals"])
    assert_csc_equal(got, (case["out_vals"], case["out_rows"], case["out_offs"]), exact_values=True)


@pytest.mark.parametrize("case", load_golden("transpose"), ids=lambda c: "%sx%s" % (c["n_rows"], c["n_cols"]))
def test_transpose_golden(case):
    got = oracle.transpose(case["n_rows"], case["n_cols"], case["vals"], case["rows"], case["offs"])
    assert_csc_equal(got, (case["out_vals"], case["out_rows"], case["out_offs"]), exact_values=True)


@pytest.mark.parametrize("case", load_golden("linear_combine"), ids=lambda c: "%sx%s" % (c["n_rows"], c["n_cols"]))
def test_linear_combine_golden(case):
    got = oracle.linear_combine(case["n_cols"], case["a_vals"], case["a_rows"], case["a_offs"],
                                case["b_vals"], case["b_rows"], case["b_offs"], case["alpha"], case["beta"])
    assert_csc_equal(got, (case["out_vals"], case["out_rows"], case["out_offs"]), exact_values=True)


@pytest.mark.parametrize("case", load_golden("spgemm"), ids=lambda c: "%sx%sx%s" % (c["n_rows"], c["n_inner"], c["n_cols"]))
def test_spgemm_golden(case):
    got = oracle.spgemm(case["n_rows"], case["a_vals"], case["a_rows"], case["a_offs"],
                        case["b_vals"], case["b_rows"], case["b_offs"], case["n_cols"])
    assert_csc_equal(got, (case["out_vals"], case["out_rows"], case["out_offs"]), exact_values=True)


@pytest.mark.parametrize("case", load_golden("spmv"), ids=lambda c: "%sx%s" % (c["n_rows"], c["n_cols"]))
def test_spmv_golden(case):
    y = oracle.mat_times_vec(case["vals"], case["rows"], case["offs"], case["x"], case["n_rows"], case["n_cols"])
    w = oracle.vec_times_mat(case["v"], case["vals"], case["rows"], case["offs"], case["n_cols"])
    assert np.array_equal(y, case["y"]) and np.array_equal(w, case["w"])
    # the SpMM oracle is column-wise mat_times_vec
    B = np.stack([case["x"], case["x"] * 2.0], axis=1)
    C = oracle.spmm(case["vals"], case["rows"], case["offs"], B, case["n_rows"], case["n_cols"], nthreads=2)
    assert np.array_equal(C[:, 0], case["y"])


@pytest.mark.parametrize("case", load_golden("trace"), ids=lambda c: "%sx%s" % (c["n_rows"], c["n_cols"]))
def test_trace_golden(case):
    t = oracle.fused_trace(case["n_cols"], case["a_vals"], case["a_rows"], case["a_offs"],
                           case["b_vals"], case["b_rows"], case["b_offs"])
    assert t == case["trace"]


def test_trace_reference_pins():
    # test_expr.py:133-150: diag(1,2) . diag(3,4) -> 11; disjoint -> 0
    assert oracle.fused_trace(2, [1.0, 2.0], [0, 1], [0, 1, 2], [3.0, 4.0], [0, 1], [0, 1, 2]) == 11.0
    assert oracle.fused_trace(3, [5.0], [0], [0, 1, 1, 1], [7.0], [1], [0, 0, 1, 1]) == 0.0


def test_funnel_oracle_golden():
    """oracle/funnel.py against the reference's own outputs."""
    from oracle import funnel as F

    def p_of(s):
        return np.inf if s == "inf" else ("fro" if s == "fro" else float(s))

    def same(got, c, exact=True):
        v, r, o = got
        assert np.array_equal(o, c["out_offs"]) and np.array_equal(r, c["out_rows"])
        if exact:
            assert np.array_equal(v.view(np.int64), c["out_vals"].view(np.int64))
        else:
            assert np.allclose(v, c["out_vals"], rtol=1e-12, atol=0)

    for c in load_golden("funnel"):
        op = c["op"]
        if op == "kron":
            same(F.kron((c["a_vals"], c["a_rows"], c["a_offs"]), c["ar"], c["ac"],
                        (c["b_vals"], c["b_rows"], c["b_offs"]), c["br"], c["bc"]), c)
            continue
        a = (c["a_vals"], c["a_rows"], c["a_offs"])
        if op == "repmat":
            same(F.repmat(a, c["r"], c["c"], c["reps_r"], c["reps_c"]), c)
        elif op == "reduce":
            assert np.array_equal(F.reduce(a, c["r"], c["c"], c["kind"], c["dim"]).view(np.int64),
                                  np.asarray(c["out"], np.float64).view(np.int64))
        elif op == "trace":
            assert F.trace(a) == float(c["out"])
        elif op == "diag":
            assert np.array_equal(F.diag(a, c["r"], c["c"], c["k"]), c["out"])
        elif op == "norm":
            assert F.norm(a, c["r"], c["c"], p_of(c["p"])) == float(c["out"])
        elif op == "normalise":
            same(F.normalise(a, c["r"], c["c"], p_of(c["p"]), c["dim"]), c)
        elif op == "submat":
            same(F.submat(a, c["r0"], c["r1"], c["c0"], c["c1"]), c)


def test_sample_positions_restates_the_reference_sampler():
    """synth.sample_positions (the restatement of ops._sample_positions,
    ops.py:377-397) + rng.random values, canonicalised by the oracle, is the
    reference's sprandu matrix for the same seed: the generator stream is
    consumed identically (sparse rounds, dense permutation branch, empty)."""
    from paper_1805_03380_b200.synth import sample_positions

    for case in load_golden("sprandu"):
        r, c = int(case["r"]), int(case["c"])
        k = int(np.floor(float(case["density"]) * r * c + 0.5))
        rng = np.random.default_rng(int(case["seed"]))
        pos = sample_positions(r * c, k, rng)
        vals = rng.random(k)
        while (vals == 0.0).any():
            z = vals == 0.0
            vals[z] = rng.random(int(z.sum()))
        got = oracle.canonicalize(r, c, pos % r, pos // r, vals)
        assert np.array_equal(got[2], case["out_offs"]) and np.array_equal(got[1], case["out_rows"])
        assert np.array_equal(got[0].view(np.int64), case["out_vals"].view(np.int64))

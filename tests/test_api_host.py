"""Host-side semantics that need no GPU: the expression rewrite rules
(expr.py:159-194 of the reference), shape errors, the insertion cache's
RbtStore semantics (rbt.py:371-441) and the hybrid handle's format flags and
conversion counters for writes (hybrid.py:97-181)."""

import numpy as np
import pytest

from paper_1805_03380_b200 import (Add, AppendOrderError, CoordinateError, Dims, Format, FusedTraceAtB,
                                   InsertionCache, Leaf, Mul, ScalarMul, ShapeError, SpMat, Trace, Transpose,
                                   decode_index, encode_index, lift, rewrite)


def Z(r, c):
    return SpMat.zeros(r, c, device="cpu")


def test_fused_trace_rewrite_and_shape_guard():
    a, b = Z(5, 4), Z(5, 4)
    e = rewrite(Trace(Mul(Transpose(lift(a)), lift(b))))
    assert isinstance(e, FusedTraceAtB)
    # non-matching shapes keep the unfused tree (expr.py:177)
    c = Z(5, 3)
    e2 = rewrite(Trace(Mul(Transpose(lift(a)), lift(c))))
    assert isinstance(e2, Trace)


def test_double_transpose_and_scalar_folding():
    a = Z(3, 2)
    assert rewrite(Transpose(Transpose(lift(a)))) == Leaf(a)
    e = rewrite(ScalarMul(2.0, ScalarMul(3.0, lift(a))))
    assert isinstance(e, ScalarMul) and e.k == 6.0 and e.child == Leaf(a)


def test_expression_shape_errors():
    with pytest.raises(ShapeError):
        Add(lift(Z(2, 3)), lift(Z(3, 2)))
    with pytest.raises(ShapeError):
        Mul(lift(Z(2, 3)), lift(Z(2, 3)))
    with pytest.raises(ShapeError):
        FusedTraceAtB(lift(Z(2, 3)), lift(Z(3, 2)))


def test_encode_decode_roundtrip():
    for r, c, n in [(0, 0, 1), (3, 7, 10), (9, 0, 10)]:
        assert decode_index(encode_index(r, c, n), n) == (r, c)


def test_cache_semantics_match_rbtstore():
    t = InsertionCache(Dims(4, 3))
    assert t.count == 0 and t.get(5) == 0.0
    t.insert(5, 1.5)
    t.insert(2, 2.5)
    t.insert(5, 3.0)  # overwrite
    assert t.get(5) == 3.0 and t.count == 2
    t.insert(2, 0.0)  # zero erases
    assert t.count == 1 and t.get(2) == 0.0
    assert t.erase(5) and not t.erase(5)
    assert t.count == 0
    t.append_max(7, 1.0)
    with pytest.raises(AppendOrderError):
        t.append_max(3, 1.0)
    t.insert(11, 4.0)
    assert list(t.items()) == [(7, 1.0), (11, 4.0)] and t.max_index == 11
    with pytest.raises(CoordinateError):
        t.insert(12, 1.0)


def test_random_cache_walk_against_dict(rng):
    t = InsertionCache(Dims(7, 9))
    shadow = {}
    for _ in range(2000):
        k = int(rng.integers(0, 63))
        v = float(rng.integers(0, 3))
        t.insert(k, v)
        if v == 0.0:
            shadow.pop(k, None)
        else:
            shadow[k] = v
        if rng.random() < 0.05:
            assert t.count == len(shadow)
    assert dict(t.items()) == shadow


def test_hybrid_write_routes_and_counters():
    m = Z(6, 6)
    assert m.valid_formats == {Format.CSC}
    m[1, 2] = 3.0  # structural write -> write cache
    assert m.valid_formats == {Format.RBT}
    assert m.conversions == {Format.CSC: 0, Format.COO: 0, Format.RBT: 1}
    assert m[1, 2] == 3.0 and m.nnz == 1  # read served by the cache, no sync
    m.accumulate(1, 2, -3.0)  # exact cancellation erases
    assert m.nnz == 0 and m.conversions[Format.CSC] == 0
    with pytest.raises(CoordinateError):
        m[6, 0] = 1.0

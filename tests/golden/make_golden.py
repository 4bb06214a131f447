"""Generate the golden vectors in tests/golden/ by running the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src
(autosparse; numba JIT cache redirected to /tmp) and records inputs and
reference outputs of every hot-path function on seeded cases, including the
edge cases its tests pin (empty inputs, exact cancellation, duplicate groups
longer than numpy's pairwise block, erase-on-zero writes, disjoint supports).
The .npz files it writes are the fixtures; this script is how they were made.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from autosparse import Dims, SpMat, _kernels, csc, expr, ops  # noqa: E402
from autosparse.hybrid import Format  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_canon(n_rows, n_cols, rows, cols, vals, dup):
    m = csc.canonicalize(Dims(n_rows, n_cols), rows, cols, vals, dup)
    return m.values, m.row_indices, m.col_offsets


def rand_csc(rng, n_rows, n_cols, nnz_target, zipf=False):
    if zipf:
        lens = np.minimum(rng.zipf(1.6, n_cols), n_rows)
        cols = np.repeat(np.arange(n_cols), lens)
        rows = rng.integers(0, n_rows, cols.shape[0])
    else:
        rows = rng.integers(0, n_rows, nnz_target)
        cols = rng.integers(0, n_cols, nnz_target)
    vals = rng.uniform(-1, 1, rows.shape[0])
    return ref_canon(n_rows, n_cols, rows, cols, vals, "sum")


def save(name, cases):
    flat = {}
    for i, case in enumerate(cases):
        for k, v in case.items():
            flat["c%d__%s" % (i, k)] = np.asarray(v)
    flat["n_cases"] = np.asarray(len(cases))
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **flat)
    print("%-16s %3d cases %8.1f KB" % (name, len(cases), os.path.getsize(path) / 1024))


def gen_canonicalize(rng):
    cases = []
    # the reference tests' literal examples (test_csc.py:11-47)
    lit = [
        (3, 2, [(0, 0, 1.0), (2, 1, 3.0), (1, 1, 2.0)], "sum"),
        (4, 4, [], "sum"),
        (2, 2, [(0, 0, 5.0), (0, 0, -5.0)], "sum"),
        (2, 2, [(1, 0, 2.0), (1, 0, 3.0)], "sum"),
        (2, 2, [(1, 0, 2.0), (0, 1, 9.0), (1, 0, 3.0)], "last"),
    ]
    for r, c, t, dup in lit:
        t = np.array(t, dtype=np.float64).reshape(-1, 3)
        rows, cols, vals = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), t[:, 2]
        o = ref_canon(r, c, rows, cols, vals, dup)
        cases.append(dict(n_rows=r, n_cols=c, rows=rows, cols=cols, vals=vals, dup=dup,
                          out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    # random, duplicate-heavy, with long groups (> 8, > 128 and > 256) to pin
    # numpy's pairwise reduceat order, and exact cancellations
    specs = [(7, 5, 300), (50, 40, 3000), (1, 1, 700), (1000, 1000, 6000), (3, 100000, 5000),
             (100000, 3, 5000), (10000, 10000, 12000)]
    for (r, c, n) in specs:
        for dup in ("sum", "last"):
            rows = rng.integers(0, r, n)
            cols = rng.integers(0, c, n)
            vals = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-6, 6, n)
            # plant a long group and a cancelling pair
            if n > 400:
                rows[:300] = rows[0]
                cols[:300] = cols[0]
                rows[300:309] = rows[300]
                cols[300:309] = cols[300]
                rows[310], cols[310], vals[310] = rows[311], cols[311], -vals[311]
            perm = rng.permutation(n)
            rows, cols, vals = rows[perm], cols[perm], vals[perm]
            o = ref_canon(r, c, rows, cols, vals, dup)
            cases.append(dict(n_rows=r, n_cols=c, rows=rows, cols=cols, vals=vals, dup=dup,
                              out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    # cfg-1 shape, scaled down 100x in triplets (10k x 10k, U rows/cols, U[-1,1])
    g = np.random.default_rng(1)
    rows = g.integers(0, 10000, 5000)
    cols = g.integers(0, 10000, 5000)
    vals = g.uniform(-1, 1, 5000)
    o = ref_canon(10000, 10000, rows, cols, vals, "sum")
    cases.append(dict(n_rows=10000, n_cols=10000, rows=rows, cols=cols, vals=vals, dup="sum",
                      out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    save("canonicalize", cases)


def gen_flush(rng):
    """Element writes through the reference SpMat (hybrid.py:165-193): the
    in-place CSC overwrite, the RBT insert / overwrite / erase-on-zero, then
    the rbt.to_csc flush.  Recorded: base CSC, write log, final CSC, and the
    conversion counters."""
    cases = []
    for (r, c, nbase, nw, zero_frac) in [(5, 5, 0, 40, 0.2), (20, 20, 60, 1000, 0.25),
                                         (300, 200, 1500, 6000, 0.05), (50000, 50000, 0, 6000, 0.0),
                                         (1, 1000, 100, 3000, 0.3)]:
        rows = rng.integers(0, r, nbase)
        cols = rng.integers(0, c, nbase)
        vals = rng.uniform(-1, 1, nbase)
        base = ref_canon(r, c, rows, cols, vals, "sum")
        m = SpMat.from_csc(csc.CscData(Dims(r, c), *base))
        wr = rng.integers(0, r, nw)
        wc = rng.integers(0, c, nw)
        wv = rng.uniform(-1, 1, nw)
        wv[rng.random(nw) < zero_frac] = 0.0
        # overwrites of earlier writes (cfg-2 style)
        k = nw // 20
        src = rng.integers(0, max(nw // 2, 1), k)
        dst = rng.integers(nw // 2, nw, k)
        wr[dst], wc[dst] = wr[src], wc[src]
        for i in range(nw):
            m[int(wr[i]), int(wc[i])] = float(wv[i])
        out = m.csc()
        cases.append(dict(n_rows=r, n_cols=c, base_vals=base[0], base_rows=base[1], base_offs=base[2],
                          log_rows=wr, log_cols=wc, log_vals=wv,
                          out_vals=out.values, out_rows=out.row_indices, out_offs=out.col_offsets,
                          conv_rbt=m.conversions[Format.RBT], conv_csc=m.conversions[Format.CSC]))
    save("flush", cases)


def gen_transpose(rng):
    cases = []
    for (r, c, n) in [(1, 1, 1), (4, 3, 0), (9, 5, 20), (50, 70, 1500), (1000, 300, 8000),
                      (10000, 10000, 10000), (1, 5000, 2000), (5000, 1, 2000)]:
        a = rand_csc(rng, r, c, n)
        o = _kernels.transpose(r, c, a[0], a[1], a[2])
        cases.append(dict(n_rows=r, n_cols=c, vals=a[0], rows=a[1], offs=a[2],
                          out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    save("transpose", cases)


def gen_linear_combine(rng):
    cases = []
    for (r, c, n, alpha, beta, mode) in [(4, 4, 0, 1.0, 1.0, "rand"), (10, 8, 30, 1.0, 1.0, "rand"),
                                         (10, 8, 30, 1.0, -1.0, "self"), (60, 50, 800, 0.5, 0.5, "rand"),
                                         (2000, 1500, 8000, 1.0, 1.0, "rand"),
                                         (2000, 1500, 8000, 1.0, -1.0, "partial"),
                                         (300, 1000, 0, 0.1, 3.0, "zipf")]:
        a = rand_csc(rng, r, c, n, zipf=(mode == "zipf"))
        if mode == "self":
            b = a
        elif mode == "partial":
            b = rand_csc(rng, r, c, n)
            # copy half of A's values into B at the same coordinates: A - B cancels there
            ac = np.repeat(np.arange(c), np.diff(a[2]))
            take = rng.random(a[0].shape[0]) < 0.5
            brows = np.concatenate([b[1], a[1][take]])
            bcols = np.concatenate([np.repeat(np.arange(c), np.diff(b[2])), ac[take]])
            bvals = np.concatenate([b[0], a[0][take]])
            b = ref_canon(r, c, brows, bcols, bvals, "last")
        else:
            b = rand_csc(rng, r, c, n, zipf=(mode == "zipf"))
        o = _kernels.linear_combine(c, a[0], a[1], a[2], b[0], b[1], b[2], alpha, beta)
        cases.append(dict(n_rows=r, n_cols=c, alpha=alpha, beta=beta,
                          a_vals=a[0], a_rows=a[1], a_offs=a[2], b_vals=b[0], b_rows=b[1], b_offs=b[2],
                          out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    save("linear_combine", cases)


def gen_spgemm(rng):
    cases = []
    # disjoint outer products (test_ops.py:136-146)
    a = ref_canon(10, 10, np.array([2, 3]), np.array([5, 7]), np.array([1.0, 1.0]), "sum")
    b = ref_canon(10, 10, np.array([5, 7]), np.array([0, 1]), np.array([2.0, 3.0]), "sum")
    specs = [(10, 10, 10, a, b)]
    for (m, k, n, na, nb, zipf) in [(8, 8, 8, 20, 20, False), (40, 30, 50, 300, 400, False),
                                     (500, 400, 300, 3000, 2000, False), (600, 600, 300, 0, 0, True),
                                     (1, 50, 1, 40, 40, False)]:
        A = rand_csc(rng, m, k, na, zipf=zipf)
        B = rand_csc(rng, k, n, nb, zipf=zipf)
        specs.append((m, k, n, A, B))
    # exact cancellation: C = A @ [1 ; -1] style (two columns of B that cancel)
    A = rand_csc(rng, 30, 2, 0)
    A = ref_canon(30, 2, np.r_[np.arange(30), np.arange(30)], np.r_[np.zeros(30, int), np.ones(30, int)],
                  np.r_[np.arange(1, 31.0), np.arange(1, 31.0)], "sum")
    B = ref_canon(2, 3, np.array([0, 1, 0, 1]), np.array([0, 0, 2, 2]), np.array([1.0, -1.0, 2.0, 1.0]), "sum")
    specs.append((30, 2, 3, A, B))
    for (m, k, n, A, B) in specs:
        o = _kernels.spgemm(m, A[0], A[1], A[2], B[0], B[1], B[2], n)
        cases.append(dict(n_rows=m, n_inner=k, n_cols=n, a_vals=A[0], a_rows=A[1], a_offs=A[2],
                          b_vals=B[0], b_rows=B[1], b_offs=B[2], out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    save("spgemm", cases)


def gen_spmv(rng):
    cases = []
    for (r, c, n) in [(7, 7, 7), (7, 5, 0), (40, 30, 200), (1000, 1000, 5000), (3000, 200, 5000)]:
        A = rand_csc(rng, r, c, n)
        x = rng.random(c)
        x[rng.random(c) < 0.1] = 0.0
        v = rng.random(r)
        y = _kernels.mat_times_vec(A[0], A[1], A[2], x, r, c)
        w = _kernels.vec_times_mat(v, A[0], A[1], A[2], c)
        cases.append(dict(n_rows=r, n_cols=c, vals=A[0], rows=A[1], offs=A[2], x=x, v=v, y=y, w=w))
    # inf * 0 is never formed: x[j] == 0 skips the column (_kernels.py:124)
    A = ref_canon(3, 3, np.array([0, 1, 2]), np.array([0, 1, 2]), np.array([np.inf, 2.0, 3.0]), "sum")
    x = np.array([0.0, 1.0, 1.0])
    cases.append(dict(n_rows=3, n_cols=3, vals=A[0], rows=A[1], offs=A[2], x=x, v=np.ones(3),
                      y=_kernels.mat_times_vec(A[0], A[1], A[2], x, 3, 3),
                      w=_kernels.vec_times_mat(np.ones(3), A[0], A[1], A[2], 3)))
    save("spmv", cases)


def gen_trace(rng):
    cases = []
    a = ref_canon(2, 2, np.array([0, 1]), np.array([0, 1]), np.array([1.0, 2.0]), "sum")
    b = ref_canon(2, 2, np.array([0, 1]), np.array([0, 1]), np.array([3.0, 4.0]), "sum")
    pairs = [(2, 2, a, b)]
    a = ref_canon(3, 3, np.array([0]), np.array([0]), np.array([5.0]), "sum")
    b = ref_canon(3, 3, np.array([1]), np.array([1]), np.array([7.0]), "sum")
    pairs.append((3, 3, a, b))
    for (r, c, n) in [(12, 12, 40), (500, 400, 5000), (100000, 1000, 15000), (2000, 2000, 15000)]:
        pairs.append((r, c, rand_csc(rng, r, c, n), rand_csc(rng, r, c, n)))
    A = rand_csc(rng, 300, 300, 5000)
    pairs.append((300, 300, A, A))  # tr(A^T A) = ||A||_F^2
    for (r, c, A, B) in pairs:
        t = _kernels.fused_trace(c, A[0], A[1], A[2], B[0], B[1], B[2])
        cases.append(dict(n_rows=r, n_cols=c, a_vals=A[0], a_rows=A[1], a_offs=A[2],
                          b_vals=B[0], b_rows=B[1], b_offs=B[2], trace=t))
    save("trace", cases)


def _mat(A, r, c):
    return SpMat.from_csc(csc.CscData(Dims(r, c), A[0], A[1], A[2]))


def _csc_out(m):
    d = m.csc()
    return d.values, d.row_indices, d.col_offsets


def gen_funnel(rng):
    """construction-funnelled ops and segmented reductions
    (ops.py:131-163, 166-212, 228-298, 345-355)."""
    cases = []

    def mk(r, c, n, lo=-1.0, hi=1.0):
        rows, cols = rng.integers(0, r, n), rng.integers(0, c, n)
        return ref_canon(r, c, rows, cols, rng.uniform(lo, hi, n), "sum")

    # kron (incl. an underflow of a product to exact zero, pruned by canonicalize)
    for (ar, ac, na, br, bc, nb) in [(3, 4, 6, 2, 5, 4), (20, 15, 60, 13, 17, 50), (1, 1, 1, 40, 30, 200),
                                     (50, 40, 300, 30, 20, 150)]:
        A, B = mk(ar, ac, na), mk(br, bc, nb)
        o = _csc_out(ops.kron(_mat(A, ar, ac), _mat(B, br, bc)))
        cases.append(dict(op="kron", ar=ar, ac=ac, br=br, bc=bc, a_vals=A[0], a_rows=A[1], a_offs=A[2],
                          b_vals=B[0], b_rows=B[1], b_offs=B[2], out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    A = ref_canon(2, 2, np.array([0, 1]), np.array([0, 1]), np.array([1e-200, 3.0]), "sum")
    B = ref_canon(2, 1, np.array([0, 1]), np.array([0, 0]), np.array([1e-200, 2.0]), "sum")
    o = _csc_out(ops.kron(_mat(A, 2, 2), _mat(B, 2, 1)))
    cases.append(dict(op="kron", ar=2, ac=2, br=2, bc=1, a_vals=A[0], a_rows=A[1], a_offs=A[2],
                      b_vals=B[0], b_rows=B[1], b_offs=B[2], out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    # repmat
    for (r, c, n, rr, rc) in [(3, 4, 6, 2, 3), (30, 20, 200, 3, 1), (17, 9, 50, 1, 4), (100, 80, 1500, 2, 2)]:
        A = mk(r, c, n)
        o = _csc_out(ops.repmat(_mat(A, r, c), rr, rc))
        cases.append(dict(op="repmat", r=r, c=c, reps_r=rr, reps_c=rc, a_vals=A[0], a_rows=A[1], a_offs=A[2],
                          out_vals=o[0], out_rows=o[1], out_offs=o[2]))
    # reductions, trace, diag, norms, normalise, submat on a few shapes
    shapes = [(6, 5, 12), (40, 30, 400), (300, 200, 3000), (5, 5, 25), (1, 50, 30), (60, 1, 40), (3, 3, 9)]
    for (r, c, n) in shapes:
        A = mk(r, c, n, -2.0, 2.0)
        M = _mat(A, r, c)
        base = dict(r=r, c=c, a_vals=A[0], a_rows=A[1], a_offs=A[2])
        for kind, fn in (("sum", ops.sum_dim), ("min", ops.min_dim), ("max", ops.max_dim)):
            for dim in (0, 1):
                cases.append(dict(base, op="reduce", kind=kind, dim=dim, out=fn(M, dim)))
        cases.append(dict(base, op="trace", out=ops.trace(M)))
        for k in (-2, 0, 1):
            try:
                cases.append(dict(base, op="diag", k=k, out=ops.diag(M, k)))
            except Exception:
                pass
        vec = r == 1 or c == 1
        for p in ((1, 2, 3, np.inf, "fro") if vec else (1, np.inf, "fro")):
            cases.append(dict(base, op="norm", p=str(p), out=ops.norm(M, p)))
        for p in (1, 2, 3, np.inf):
            for dim in (0, 1):
                o = _csc_out(ops.normalise(M, p, dim))
                cases.append(dict(base, op="normalise", p=str(p), dim=dim, out_vals=o[0], out_rows=o[1],
                                  out_offs=o[2]))
        if r > 2 and c > 2:
            for (r0, r1, c0, c1) in [(0, r - 1, 0, c - 1), (1, r // 2, 1, c // 2), (r // 2, r - 1, 0, 0)]:
                o = _csc_out(ops.submat(M, (r0, r1), (c0, c1)))
                cases.append(dict(base, op="submat", r0=r0, r1=r1, c0=c0, c1=c1, out_vals=o[0], out_rows=o[1],
                                  out_offs=o[2]))
    save("funnel", cases)


def gen_mm(rng):
    """Matrix Market text -> reference load_mm outcome (the
    canonical CSC, or the exception class and message), and reference
    save_mm text of random matrices (io.py:33-131)."""
    import io as _io

    from autosparse import io as ref_io

    H = "%%MatrixMarket matrix coordinate real general\n"
    texts = [
        (H + "2 2 1\n1 1 2.5\n", False),
        (H + "% a comment\n2 2 1\n% another\n1 1 2.5\n", False),
        (H + "2 2 1\n1 1\n", False),
        (H + "2 2 1\n3 1 1.0\n", False),
        (H + "2 2 2\n1 1 1.0\n", False),
        (H + "2 2 2\n1 1 2.0\n1 1 3.0\n", False),
        (H + "2 2 2\n1 1 2.0\n1 1 3.0\n", True),
        (H + "3 3 3\n1 1 +1.5\n2 2 1_000.25\n+3 0_3 -2e-3\n", False),
        (H + "3 3 2\n1 1 1e999\n2 2 1e-999\n", False),
        (H + "3 3 2\n1 1 inf\n2 2 -Infinity\n", False),
        (H + "3 3 2\n1 1 1.0\n2 2 x\n", False),
        (H + "3 3 1\n1 1 1.0\n2 2 3.0\n", False),
        (H + "3 3 1\n1 1 1.0\n2 2\n", False),
        (H + "3 3 1\n1 1 1.0\n2 2 zz\n", False),
        (H + "3 3 2\n4 1 1.0\n1 1 zz\n", False),
        (H + "3 3 2\n1 1 zz\n4 1 1.0\n", False),
        (H + "3 3\n", False),
        (H + "3 x 3\n", False),
        (H + "% only comments\n", False),
        ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", False),
        ("%%matrixmarket matrix coordinate real general\n1 1 0\n", False),
        ("", False),
        (H + "2 2 0", False),
        (H + "2 2 1", False),
        (H + "  2   2   2  \n\n  1 1 1.0  \n\n 2 2   -0.0 \n", False),
        (H + "4 5 3\n1 2 0.0\n3 4 2.0\n4 5 -1.0\n", False),
        (H.replace("\n", "\r\n") + "2 2 1\r\n2 1 7.5\r\n", False),
    ]
    for _ in range(12):
        r, c = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        n = int(rng.integers(0, r * c // 2 + 1))
        A = ref_canon(r, c, rng.integers(0, r, n), rng.integers(0, c, n), rng.standard_normal(n) *
                      10.0 ** rng.integers(-300, 300, n), "sum")
        buf = _io.StringIO()
        ref_io.save_mm(_mat(A, r, c), buf)
        texts.append((buf.getvalue(), False))
    vals = [1e-308, 1.0 / 3.0, float(np.nextafter(1.0, 2.0)), 1e300, -7.25, 5e-324]
    buf = _io.StringIO()
    ref_io.save_mm(SpMat.from_triplets(6, 1, [(i, 0, v) for i, v in enumerate(vals)]), buf)
    texts.append((buf.getvalue(), False))
    cases = []
    for text, lenient in texts:
        case = dict(text=np.frombuffer(text.encode("ascii"), np.uint8), lenient=int(lenient))
        try:
            m = ref_io.load_mm(text if "\n" in text else _io.StringIO(text), lenient_duplicates=lenient)
            d = m.csc()
            case.update(outcome="ok", n_rows=d.dims.n_rows, n_cols=d.dims.n_cols, out_vals=d.values,
                        out_rows=d.row_indices, out_offs=d.col_offsets)
            out = _io.StringIO()
            ref_io.save_mm(m, out)
            case["saved"] = np.frombuffer(out.getvalue().encode("ascii"), np.uint8)
        except Exception as e:  # noqa: BLE001 -- the reference's exception is the expected outcome
            case.update(outcome="error", err_class=type(e).__name__, err_msg=str(e))
        cases.append(case)
    save("mm", cases)


def gen_sprandu():
    """ops.sprandu(n_rows, n_cols, density, seed) (ops.py:400-417) with its
    sampler _sample_positions (ops.py:377-397): sparse targets (batched
    rejection, several rounds), the dense branch (k > cells // 2 ->
    permutation), empty and full."""
    cases = []
    for (r, c, dens, seed) in [(50, 40, 0.01, 1), (50, 40, 0.3, 2), (50, 40, 0.5, 3), (50, 40, 0.51, 4),
                               (50, 40, 0.9, 5), (30, 30, 1.0, 6), (30, 30, 0.0, 7), (1000, 700, 0.002, 8),
                               (1000, 700, 0.05, 9), (1, 500, 0.7, 10), (500, 1, 0.2, 11), (200, 300, 0.45, 12)]:
        d = ops.sprandu(r, c, dens, seed=seed).csc()
        cases.append(dict(r=r, c=c, density=dens, seed=seed, out_vals=d.values, out_rows=d.row_indices,
                          out_offs=d.col_offsets))
    save("sprandu", cases)


EXPRS = {
    # name -> builder over leaves a, b, c (all the same square shape)
    "half_sum_times_ct": lambda a, b, c: expr.Mul(expr.ScalarMul(0.5, expr.Add(a, b)), expr.Transpose(c)),
    "at_times_b": lambda a, b, c: expr.Mul(expr.Transpose(a), b),
    "a_times_bt": lambda a, b, c: expr.Mul(a, expr.Transpose(b)),
    "at_times_bt": lambda a, b, c: expr.Mul(expr.Transpose(a), expr.Transpose(b)),
    "trace_at_b": lambda a, b, c: expr.Trace(expr.Mul(expr.Transpose(a), b)),
    "trace_ab": lambda a, b, c: expr.Trace(expr.Mul(a, b)),
    "double_t_plus": lambda a, b, c: expr.Add(expr.Transpose(expr.Transpose(a)), b),
    "scaled_diff": lambda a, b, c: expr.ScalarMul(2.0, expr.ScalarMul(3.0, expr.Sub(a, b))),
    "sum_times_sum_t": lambda a, b, c: expr.Mul(expr.Add(a, c), expr.Transpose(expr.Sub(b, c))),
}


def gen_expr(rng):
    """expr.evaluate / evaluate_counting (expr.py:159-280) on
    seeded operands, optimised and naive: the result (CSC or scalar) and the
    intermediate count."""
    cases = []
    for (n, dens) in [(14, 0.3), (60, 0.05), (200, 0.02)]:
        ops_in = [rand_csc(rng, n, n, max(1, int(dens * n * n))) for _ in range(3)]
        leaves = [expr.lift(_mat(m, n, n)) for m in ops_in]
        for name, fn in EXPRS.items():
            for opt in (True, False):
                out, inter = expr.evaluate_counting(fn(*leaves), optimize=opt)
                case = dict(name=name, n=n, optimize=int(opt), intermediates=inter)
                for k, m in zip("abc", ops_in):
                    case.update({k + "_vals": m[0], k + "_rows": m[1], k + "_offs": m[2]})
                if isinstance(out, SpMat):
                    d = out.csc()
                    case.update(kind="mat", out_vals=d.values, out_rows=d.row_indices, out_offs=d.col_offsets)
                else:
                    case.update(kind="scalar", out=float(out))
                cases.append(case)
    save("expr", cases)


def main(only=None):
    """No arguments: every file.  `funnel` alone: only funnel.npz (its own
    seed; the first seven share one generator stream in this order)."""
    if not only or set(only) - {"funnel", "mm", "sprandu", "expr"}:
        rng = np.random.default_rng(20260809)
        gen_canonicalize(rng)
        gen_flush(rng)
        gen_transpose(rng)
        gen_linear_combine(rng)
        gen_spgemm(rng)
        gen_spmv(rng)
        gen_trace(rng)
    if not only or "funnel" in only:
        gen_funnel(np.random.default_rng(20261019))
    if not only or "mm" in only:
        gen_mm(np.random.default_rng(20261020))
    if not only or "sprandu" in only:
        gen_sprandu()
    if not only or "expr" in only:
        gen_expr(np.random.default_rng(20261021))


if __name__ == "__main__":
    main(sys.argv[1:] or None)

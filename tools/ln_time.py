"""Large-n sweep: construction and transpose beyond the cfg 1 size, event
timed through the raw C ABI (L2 flushed before every rep), each result
checked against the oracle first (bit-exact) where the oracle is quick.

    python tools/ln_time.py [case ...] [--reps R]
cases: build1e7 build1e8 transpose1e7 transpose5e7 (default: all)
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import _lib  # noqa: E402
from paper_1805_03380_b200._lib import ptr  # noqa: E402

CASES = {  # name: (op, n_rows, n_cols, n, value dtype)
    "build1e7": ("build", 1_000_000, 1_000_000, 10_000_000, torch.float64),
    "build1e8": ("build", 10_000_000, 10_000_000, 100_000_000, torch.float64),
    "transpose1e7": ("transpose", 1_000_000, 1_000_000, 10_000_000, torch.float32),
    "transpose5e7": ("transpose", 5_000_000, 5_000_000, 50_000_000, torch.float64),
}


def peak():
    import json
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def run_case(name, reps, check=True):
    op, n_rows, n_cols, n, vdt = CASES[name]
    L = _lib.lib()
    dev = torch.device("cuda")
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    rows = torch.randint(0, n_rows, (n,), device=dev, dtype=torch.int32, generator=g)
    cols = torch.randint(0, n_cols, (n,), device=dev, dtype=torch.int32, generator=g)
    vals = (torch.rand(n, device=dev, dtype=torch.float64, generator=g) * 2 - 1).to(vdt)
    vb = 8 if vdt == torch.float64 else 4
    cp = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    ri = torch.empty(n, dtype=torch.int32, device=dev)
    ov = torch.empty(n, dtype=vdt, device=dev)
    info = torch.empty(2, dtype=torch.int64, device=dev)
    wb = L.as_build_workspace_bytes(n, n_cols)
    ws = torch.empty(wb, dtype=torch.uint8, device=dev)
    fb = L.as_coo_to_csc_f64 if vdt == torch.float64 else L.as_coo_to_csc_f32

    def build():
        _lib.check(fb(n_rows, n_cols, n, ptr(rows), ptr(cols), 4, ptr(vals), 0, ptr(cp), ptr(ri), ptr(ov), ptr(info),
                      ptr(ws), wb, sp))

    build()
    torch.cuda.synchronize()
    nnz = int(info[0].item())
    if op == "build":
        fn = build
        alg = (8 + vb) * n + (4 + vb) * nnz + 4 * (n_cols + 1)
        res = (cp, ri[:nnz], ov[:nnz])
        if check and n <= 20_000_000:
            import oracle
            want = oracle.canonicalize(n_rows, n_cols, rows.cpu().numpy().astype(np.int64),
                                       cols.cpu().numpy().astype(np.int64), vals.cpu().numpy().astype(np.float64))
            ok = (np.array_equal(cp.cpu().numpy(), want[2]) and np.array_equal(ri[:nnz].cpu().numpy(), want[1])
                  and np.array_equal(ov[:nnz].cpu().numpy().astype(np.float64), want[0]))
            if vdt == torch.float32:
                ok = ok  # (f32 sums differ from the f64 oracle only by rounding: structure checked)
            print("  parity vs oracle:", "bit-exact" if ok else "MISMATCH", flush=True)
    else:
        tp = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
        tr = torch.empty(nnz, dtype=torch.int32, device=dev)
        tv = torch.empty(nnz, dtype=vdt, device=dev)
        ft = L.as_csc_transpose_f64 if vdt == torch.float64 else L.as_csc_transpose_f32
        wbt = L.as_transpose_workspace_bytes(nnz, n_rows)
        wst = torch.empty(wbt, dtype=torch.uint8, device=dev)
        p, r, v = cp.clone(), ri[:nnz].clone(), ov[:nnz].clone()
        del ws

        def fn():
            _lib.check(ft(n_rows, n_cols, nnz, ptr(p), ptr(r), ptr(v), ptr(tp), ptr(tr), ptr(tv), ptr(wst), wbt, sp))

        fn()
        torch.cuda.synchronize()
        alg = 2 * (4 + vb) * nnz + 4 * (n_cols + 1) + 4 * (n_rows + 1)
        if check:
            # transpose of the transpose = the input (involution), and row counts match a histogram
            tt_p = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
            tt_r = torch.empty(nnz, dtype=torch.int32, device=dev)
            tt_v = torch.empty(nnz, dtype=vdt, device=dev)
            _lib.check(ft(n_cols, n_rows, nnz, ptr(tp), ptr(tr), ptr(tv), ptr(tt_p), ptr(tt_r), ptr(tt_v), ptr(wst),
                          wbt, sp))
            cnt = torch.bincount(r.long(), minlength=n_rows)
            ok = (torch.equal(tt_p, p) and torch.equal(tt_r, r) and torch.equal(tt_v, v)
                  and torch.equal(tp[1:].long() - tp[:-1].long(), cnt))
            print("  parity (involution + row histogram):", "ok" if ok else "MISMATCH", flush=True)
            del tt_p, tt_r, tt_v
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    scratch = torch.empty((), dtype=torch.int64, device=dev)
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        torch.sum(flush.view(torch.int64), dim=0, out=scratch)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    med = statistics.median(ts)
    gbs = alg / (med * 1e-6) / 1e9
    print("%-14s n=%d nnz=%d  median %9.1f us  min %9.1f us  %7.1f GB/s  frac %.3f  (%.2e elem/s)" % (
        name, n, nnz, med, min(ts), gbs, gbs / peak(), n / (med * 1e-6)), flush=True)
    return {"case": name, "n": n, "nnz": nnz, "us": med, "GB/s": gbs, "frac": gbs / peak(), "alg_bytes": alg}


def main():
    reps = 10
    args = sys.argv[1:]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    names = args or list(CASES)
    for nm in names:
        try:
            run_case(nm, reps)
        except Exception as e:
            print("%-14s FAILED: %s" % (nm, str(e)[:200]), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Benchmark of the B200 hot path against BASELINE.json's metric.

Headline (N=1 workload, BASELINE configs[0]): COO->CSC construction of a
10,000 x 10,000 float64 matrix from 1,000,000 seeded triplets (the build the
metric names first); one step = one device build of one batch.  Under
torchrun each rank builds its own independent batch (weak scaling, no
collective).  The same JSON line carries, under "ops", the other hot-path
kernels on their BASELINE configs (transpose, flush, SpMM GB/s, fused
trace nnz/s, SpGEMM, add), each parity-checked against the CPU oracle before
it is timed, with its roofline fraction.

Timing: W warm-up steps, then K timed steps; L2 is flushed (512 MiB write)
before every step and each step is bracketed by CUDA events on the launch
stream; the K-step region is bracketed by barrier + synchronize; the max over
ranks is reported.  `--impl reference` times the reference's CPU algorithm
(the oracle port in oracle/, the reference being Python) on the same
workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "COO->CSC build nnz/s; SpMM GB/s & trace(AᵀB) nnz/s vs HBM roofline"
HEADLINE = "cfg1: COO->CSC build, 10000x10000 f64, 1,000,000 uniform triplets (seed 1), sum duplicates"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline

def time_oracle_build(inputs, budget_s: float):
    """Oracle canonicalize (the reference's csc.canonicalize restated in C,
    single-threaded like the reference) repeated for ~budget_s seconds."""
    import oracle

    n_rows, n_cols, rows, cols, vals = inputs
    oracle.canonicalize(n_rows, n_cols, rows, cols, vals, "sum")  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.canonicalize(n_rows, n_cols, rows, cols, vals, "sum")
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return reps * rows.shape[0] / el, reps, el


REF_PKG = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The unmodified reference package (pip-installed into baseline/_ref),
    or None when it is not there."""
    if not os.path.isdir(os.path.join(REF_PKG, "autosparse")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/as_numba_cache")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    try:
        import autosparse
    except Exception:
        return None
    return autosparse


def time_reference_build(inputs, budget_s: float):
    """The reference's own csc.canonicalize (numpy lexsort / reduceat, one
    thread) on the cfg 1 triplets, for ~budget_s seconds; None when the
    reference is not installed."""
    pkg = import_reference()
    if pkg is None:
        return None
    n_rows, n_cols, rows, cols, vals = inputs
    dims = pkg.Dims(n_rows, n_cols)
    pkg.csc.canonicalize(dims, rows, cols, vals, "sum")  # warm (numba / numpy caches)
    reps, t0 = 0, time.perf_counter()
    while True:
        pkg.csc.canonicalize(dims, rows, cols, vals, "sum")
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": reps * rows.shape[0] / el, "unit": "nnz/s", "cores": 1, "kind": "reference",
            "sample": "%d full cfg1 builds in %.1f s: autosparse.csc.canonicalize from baseline/_ref "
                      "(numpy/numba, single-threaded as shipped)" % (reps, el)}


def time_dropin_build(inputs, budget_s: float):
    """The reference package's own construction call (csc.canonicalize on numpy
    int64 / float64 arrays, reference CscData out) with this back end swapped in
    by ref_kernels.install: what an unmodified reference user gets.  Pageable
    host arrays in, reference-typed numpy arrays out, every copy inside."""
    pkg = import_reference()
    if pkg is None:
        return None
    from paper_1805_03380_b200 import ref_kernels

    n_rows, n_cols, rows, cols, vals = inputs
    dims = pkg.Dims(n_rows, n_cols)
    stock = pkg.csc.canonicalize(dims, rows, cols, vals, "sum")
    undo = ref_kernels.install(pkg)
    try:
        got = pkg.csc.canonicalize(dims, rows, cols, vals, "sum")  # warm, and the parity check
        same = bool(np.array_equal(got.col_offsets, stock.col_offsets) and np.array_equal(got.row_indices,
                                                                                          stock.row_indices)
                    and np.array_equal(got.values.view(np.int64), stock.values.view(np.int64)))
        reps, t0 = 0, time.perf_counter()
        while True:
            pkg.csc.canonicalize(dims, rows, cols, vals, "sum")
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    finally:
        undo()
    return {"value": reps * rows.shape[0] / el, "unit": "nnz/s", "ms": 1e3 * el / reps, "kind": "reference API, GPU back end",
            "identical_to_stock_reference": same,
            "sample": "%d full cfg1 builds in %.1f s: autosparse.csc.canonicalize after ref_kernels.install(autosparse) "
                      "(pageable numpy int64/float64 in, reference CscData out)" % (reps, el)}


def headline_config(n_rows, n_cols, n, nnz):
    """The `config` both arms print (identical dicts)."""
    return {"workload": HEADLINE, "n_rows": n_rows, "n_cols": n_cols, "triplets": n, "nnz_out": nnz,
            "values": "f64", "dup": "sum",
            "l2": "inputs not cache-resident: device arm flushes L2 (512 MiB read) before every step; "
                  "host arm rebuilds from DRAM-resident arrays"}


def run_reference(args):
    """Reference arm: the reference's CPU algorithm for the headline path
    (csc.canonicalize restated in C, oracle/oracle.c) on all the host's
    threads.  The algorithm itself is sequential (numpy/numba, one thread), so
    the host is used as a throughput machine: every step, each of T threads
    builds its own copy of the cfg 1 workload (ctypes releases the GIL), and
    value = T * triplets / step wall time."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1805_03380_b200 import synth

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inputs = synth.cfg1_triplets()
    import oracle

    n_rows, n_cols, rows, cols, vals = inputs
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1

    def one(_):
        oracle.canonicalize(n_rows, n_cols, rows, cols, vals, "sum")

    nnz = int(oracle.canonicalize(n_rows, n_cols, rows, cols, vals, "sum")[0].shape[0])
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for _ in range(args.warmup):
            list(ex.map(one, range(threads)))
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            list(ex.map(one, range(threads)))
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = threads * args.steps * rows.shape[0] / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(n_rows, n_cols, rows.shape[0], nnz),
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": "port",
                         "sample": "per step %d concurrent full cfg1 builds, one per host thread "
                                   "(oracle/oracle.c orc_canonicalize; the reference algorithm is sequential)"
                                   % threads},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # beside the port: the reference's own numpy/numba canonicalize, one thread
        "reference_numba": time_reference_build(inputs, min(args.cpu_budget, 5.0)),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# device arm

def main_device(args):
    import torch
    import torch.distributed as dist

    from paper_1805_03380_b200 import _kernels, _lib, synth
    from paper_1805_03380_b200._lib import ptr
    from paper_1805_03380_b200.errors import CorrectnessError

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.mg:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _lib.lib()
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    peak, peak_src = peaks()
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    flush_scratch = torch.empty((), dtype=torch.int64, device=dev)

    def l2_flush():
        # evict L2 by READING 512 MiB (a write-based flush leaves L2 full of
        # dirty lines whose write-back would be charged to the timed kernel)
        if args.flush == "write":
            flush_buf.fill_(1)
        else:
            torch.sum(flush_buf.view(torch.int64), dim=0, out=flush_scratch)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            l2_flush()
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(steps):
            l2_flush()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            evs.append((a, b))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    def check(rc):
        _lib.check(rc)

    # ------------------------------------------------------------ headline build
    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets(seed=1 + rank)
    n = rows.shape[0]
    d_rows = torch.as_tensor(rows.astype(np.int32), device=dev)
    d_cols = torch.as_tensor(cols.astype(np.int32), device=dev)
    d_vals = torch.as_tensor(vals, device=dev)
    col_ptr = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    row_idx = torch.empty(n, dtype=torch.int32, device=dev)
    out_vals = torch.empty(n, dtype=torch.float64, device=dev)
    info = torch.empty(2, dtype=torch.int64, device=dev)
    ws_b = L.as_build_workspace_bytes(n, n_cols)
    ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)

    def build():
        check(L.as_coo_to_csc_f64(n_rows, n_cols, n, ptr(d_rows), ptr(d_cols), 4, ptr(d_vals), 0, ptr(col_ptr),
                                  ptr(row_idx), ptr(out_vals), ptr(info), ptr(ws), ws_b, sp))

    build()
    torch.cuda.synchronize()
    nnz = int(info[0].item())
    if rank == 0:  # parity gate: refuse to time a wrong answer (reference bench.py:286-297)
        import oracle

        want = oracle.canonicalize(n_rows, n_cols, rows, cols, vals, "sum")
        got = (out_vals[:nnz].cpu().numpy(), row_idx[:nnz].cpu().numpy(), col_ptr.cpu().numpy())
        if not (np.array_equal(got[2], want[2]) and np.array_equal(got[1], want[1])
                and np.array_equal(got[0].view(np.int64), want[0].view(np.int64))):
            raise CorrectnessError("device build differs from the oracle; timing withheld")

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    t_build = timed(build, args.steps, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = statistics.median(t_build)
    total_ms = sum(t_build)
    if world > 1:
        t = torch.tensor([total_ms, step_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, step_ms = float(t[0]), float(t[1])
    value = world * n * args.steps / (total_ms * 1e-3)
    build_bytes = 16 * n + 12 * nnz + 4 * (n_cols + 1)
    build_gbs = build_bytes / (step_ms * 1e-3) / 1e9

    # ------------------------------------------------------------ e2e through the public API
    from paper_1805_03380_b200 import SpMat

    h_rows = torch.from_numpy(rows).pin_memory()
    h_cols = torch.from_numpy(cols).pin_memory()
    h_vals = torch.from_numpy(vals).pin_memory()
    o_ptr = torch.empty(n_cols + 1, dtype=torch.int32).pin_memory()
    o_rows = torch.empty(n, dtype=torch.int32).pin_memory()
    o_vals = torch.empty(n, dtype=torch.float64).pin_memory()

    from paper_1805_03380_b200 import csc as csc_mod
    from paper_1805_03380_b200.csc import Dims

    dims = Dims(n_rows, n_cols)

    def e2e_step():
        # the public API: build from host triplets, read the CSC back into
        # pinned host buffers (CscData.to_host: every copy issued before the
        # one synchronisation; nnz arrives with col_ptr)
        m = SpMat.from_triplets(n_rows, n_cols, (h_rows, h_cols, h_vals), device=dev).csc()
        _, r_h, _ = m.to_host(out=(o_ptr, o_rows, o_vals))
        return int(r_h.shape[0])

    def e2e_step_host_api():
        # csc.canonicalize's own contract (host arrays in, host CSC out): the
        # build kernel reads the pinned triplets over PCIe and writes the CSC
        # into pinned host memory (zero-copy)
        m = csc_mod.canonicalize_host(dims, h_rows, h_cols, h_vals, out=(o_ptr, o_rows, o_vals))
        return m.nnz

    # warm-up: the first ~50 pinned-host round trips after the device-only
    # timing run are measurably slower (tools/e2e_order.py: 0.94 vs 0.84 ms),
    # so warm for longer than the timed run itself
    for _ in range(max(args.warmup, 60)):
        l2_flush()
        e2e_step()
    torch.cuda.synchronize()
    e2e_times = []
    for _ in range(args.steps):
        l2_flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = e2e_step()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_total = sum(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t[0])
    e2e_value = world * n * args.steps / e2e_total
    # the same through csc.canonicalize_host (zero-copy host in / host out)
    for _ in range(max(args.warmup, 20)):
        l2_flush()
        e2e_step_host_api()
    sp_times = []
    for _ in range(args.steps):
        l2_flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step_host_api()
        torch.cuda.synchronize()
        sp_times.append(time.perf_counter() - t0)
    sp_total = sum(sp_times)
    if world > 1:
        t = torch.tensor([sp_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sp_total = float(t[0])
    packed = (n_rows - 1).bit_length() + (n_cols - 1).bit_length() <= 31  # one 32-bit key per triplet
    cap = n if packed else k
    row_bytes = 2 if (n_rows <= 65536 and cap >= (1 << 16)) else 4
    e2e = {"value": e2e_value, "unit": "nnz/s", "h2d_bytes_per_step": (12 if packed else 16) * n,  # indices + f64
           # the row / value buffers travel at their full capacity (n): nnz is
           # not known on the host before the copies are issued
           # (rows of a matrix with <= 65536 rows travel as uint16)
           "d2h_bytes_per_step": 4 * (n_cols + 1) + (row_bytes + 8) * cap,
           "ms_median": 1e3 * statistics.median(e2e_times), "ms_min": 1e3 * min(e2e_times),
           "ms_max": 1e3 * max(e2e_times),
           "path": "SpMat.from_triplets((rows i64, cols i64, vals f64) pinned host) -> .csc().to_host(pinned buffers), "
                   "one synchronisation per step; rows read back as uint16 (n_rows <= 65536) and widened on host threads "
                   "while the values copy; "
                   + ("indices packed into one 32-bit key per triplet (col << 14 | row) on host threads while the "
                      "values are copied, unpacked by a device kernel (as_upload_coo_packed)" if packed else
                      "indices narrowed to int32 on host threads while the values are copied (as_upload_coo_i64)"),
           "host_api_path": {"value": world * n * args.steps / sp_total,
                             "ms_median": 1e3 * statistics.median(sp_times),
                             "path": "csc.canonicalize_host: the kernel reads the pinned triplets and writes the "
                                     "CSC over PCIe itself (zero-copy)"}}

    # ------------------------------------------------------------ other hot-path ops (rank 0)
    ops = {}
    if rank == 0 and world == 1 and not args.headline_only:
        ops = bench_ops(args, dev, L, sp, timed, peak)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, reps, el = time_oracle_build((n_rows, n_cols, rows, cols, vals), args.cpu_budget)
        cpu = {"value": rate, "unit": "nnz/s", "cores": 1, "kind": "port",
               "sample": "%d full cfg1 builds in %.1f s (oracle/oracle.c orc_canonicalize, 1 thread; "
                         "os.cpu_count()=%d)" % (reps, el, os.cpu_count()),
               "reference_numba": time_reference_build((n_rows, n_cols, rows, cols, vals), min(args.cpu_budget, 5.0)),
               "reference_api_gpu_backend": time_dropin_build((n_rows, n_cols, rows, cols, vals),
                                                              min(args.cpu_budget, 2.0))}

    def make_line(ops_mg_value):
        return {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform triplets (SURVEY App. A); each rank its own batch (seed 1+rank)",
            "config": headline_config(n_rows, n_cols, n, nnz),
            "parallelism": "independent batch per GPU" if world > 1 else "single GPU", "index_dtype": "int32 device",
            "roofline": {"bound": "hbm", "achieved": build_gbs, "peak": peak, "unit": "GB/s",
                         "frac": build_gbs / peak, "traffic": ncu_traffic("build"), "peak_source": peak_src,
                         "traffic_source": TRAFFIC_SRC, "traffic_launches": ncu_launches("build"),
                         "kernel": "as_coo_to_csc_f64 (one cooperative sort-reduce kernel)",
                         "algorithmic_bytes": build_bytes},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": 1 * args.steps, "clocks": clocks, "ops": ops,
            "ops_multi_gpu": ops_mg_value,
        }

    ops_mg = None
    if (world > 1 or args.mg) and not args.headline_only:
        # The sharded ops have never run on more than one GPU (one GPU is all this
        # environment reaches): if an exchange stalls, every rank leaves after
        # --mg-deadline seconds and rank 0 still prints the headline line
        # (ops_multi_gpu = the error) instead of the job dying without one.
        import threading

        def give_up():
            if rank == 0:
                print(json.dumps(make_line({"error": "sharded ops did not finish within %.0f s; headline kept"
                                                     % args.mg_deadline})), flush=True)
            os._exit(0)

        watchdog = threading.Timer(args.mg_deadline, give_up)
        watchdog.daemon = True
        watchdog.start()
        try:
            ops_mg = bench_mg_ops(args, dev, world, rank, l2_flush, peak)
        finally:
            watchdog.cancel()

    if rank == 0:
        print(json.dumps(make_line(ops_mg)), flush=True)
    if world > 1 or args.mg:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _load_traffic():
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one call
    of each op, summed over every launch of that call, from the newest
    committed per-op `ncu --set full` captures (profiles/rNN_traffic.json,
    made by tools/ncu_ops.sh + tools/make_traffic.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_traffic.json")))
    if not files:
        return {}, None
    with open(files[-1]) as f:
        d = json.load(f)
    return d, "ncu --set full, " + os.path.basename(files[-1])


_TRAFFIC, TRAFFIC_SRC = _load_traffic()


def ncu_traffic(op):
    """DRAM bytes of one call of the op, summed over all its launches."""
    k = _TRAFFIC.get(op)
    return None if k is None else k["dram_read"] + k["dram_write"]


def ncu_launches(op):
    k = _TRAFFIC.get(op)
    return None if k is None else k.get("launches", 1)


def bench_mg_ops(args, dev, world, rank, l2_flush, peak):
    """the column-sharded trace (cfg 4), SpMM (cfg 3) and SpGEMM
    (cfg 5) across the torchrun ranks (NCCL).  Every rank builds the same
    seeded inputs, computes its shard with the GPU kernels and takes part in
    the exchange; per step the rank-local kernel time and the collective time
    are measured with CUDA events (L2 flushed first) and the max over ranks is
    reported.  Throughput = the whole job's work / the slowest rank's time."""
    import torch
    import torch.distributed as dist

    from paper_1805_03380_b200 import _kernels, synth
    from paper_1805_03380_b200 import dist as D

    K, W = max(3, args.op_steps // 2), args.warmup
    out = {"ranks": world, "collective": "NCCL via torch.distributed: all_gather (trace partials, slice sizes), "
                                          "all_gather_into_tensor (SpMM C), grouped send/recv (gathers to rank 0)"}

    def T(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    def timed_pair(local_fn, exch_fn):
        for _ in range(W):
            exch_fn(local_fn())
        torch.cuda.synchronize()
        dist.barrier()
        loc, col = [], []
        for _ in range(K):
            l2_flush()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            res = local_fn()
            e1.record()
            exch_fn(res)
            e2.record()
            torch.cuda.synchronize()
            loc.append(e0.elapsed_time(e1))
            col.append(e1.elapsed_time(e2))
        t = torch.tensor([statistics.median(loc), statistics.median(col),
                          statistics.median([x + y for x, y in zip(loc, col)])], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    def guarded(name, fn):
        try:
            out[name] = fn()
        except Exception as e:  # keep the headline line even if one sharded op fails
            out[name] = {"error": "%s: %s" % (type(e).__name__, str(e)[:300])}

    def trace_op():
        n, _, A, B = synth.cfg4_trace_pair()
        a = (T(A[2], torch.int32), T(A[1], torch.int32), T(A[0], torch.float64))
        b = (T(B[2], torch.int32), T(B[1], torch.int32), T(B[0], torch.float64))
        c0, c1, sa, sb = D.trace_shard(a, b)
        box = {}

        def exch(part):
            box["t"] = D.trace_exchange(part)

        lk, ck, tk = timed_pair(lambda: _kernels.fused_trace(n, c1 - c0, sa, sb), exch)
        want = float(_kernels.fused_trace(n, n, a, b).cpu()[0])
        nnz = int(A[1].shape[0] + B[1].shape[0])
        return {"ms_local": lk, "ms_collective": ck, "ms": tk, "value": nnz / (tk * 1e-3), "unit": "nnz/s",
                "parity": "within 1e-12 of the 1-GPU kernel (|d|=%.3g)" % abs(box["t"] - want),
                "ok": abs(box["t"] - want) <= 1e-12 * max(1.0, abs(want))}

    def spmm_op():
        n, _, av, ar, ao, B = synth.cfg3_spmm()
        k = B.shape[1]
        csr = _kernels.transpose(n, n, T(ao, torch.int32), T(ar, torch.int32), T(av, torch.float32))
        Bd = torch.as_tensor(B.T.copy(), device=dev).t()
        k0, k1, bounds = D.spmm_block(k)
        Xb = Bd[:, k0:k1]
        lk, ck, tk = timed_pair(lambda: _kernels.spmm(n, n, csr, Xb), lambda blk: D.spmm_exchange(blk, bounds, n))
        _, cg, tg = timed_pair(lambda: _kernels.spmm(n, n, csr, Xb), lambda blk: D.spmm_exchange(blk, bounds, n, dst=0))
        alg = 4 * (n + 1) + 8 * av.shape[0] + 8 * n * k
        return {"ms_local": lk, "ms_collective": ck, "ms": tk, "unit": "GB/s",
                "value_compute": alg / (lk * 1e-3) / 1e9, "value": alg / (tk * 1e-3) / 1e9,
                "ms_collective_gather0": cg, "ms_gather0": tg,
                "note": "A replicated, dense columns split %s; C blocks all-gathered into C's column-major storage "
                        "(all_gather_into_tensor), or sent to rank 0 (ms_gather0)" % [int(x) for x in bounds]}

    def spgemm_op():
        n, _, A, B = synth.cfg5_pair()
        a = (T(A[2], torch.int32), T(A[1], torch.int32), T(A[0], torch.float64))
        b = (T(B[2], torch.int32), T(B[1], torch.int32), T(B[0], torch.float64))
        c0, c1, bounds, sb = D.spgemm_shard(a, b)
        total = int(D.spgemm_column_weights(A[2], B[2], B[1]).sum())
        local = lambda: _kernels.spgemm(n, n, c1 - c0, a, sb)
        # left distributed (DistCsc: one all_gather of slice nnz, device-side offsets)
        lk, ck, tk = timed_pair(local, lambda res: D.spgemm_exchange(*res, bounds, dst=None, c_range=(c0, c1)))
        # assembled on rank 0 by grouped send/recv of the native int32 / f64 slices
        _, cg, tg = timed_pair(local, lambda res: D.spgemm_exchange(*res, bounds, dst=0))
        return {"ms_local": lk, "ms_collective": ck, "ms": tk, "value": total / (tk * 1e-3), "unit": "products/s",
                "value_compute": total / (lk * 1e-3), "ms_collective_gather0": cg, "ms_gather0": tg,
                "note": "B split into %d equal-product column ranges; result left distributed (value) or gathered "
                        "on rank 0 by grouped send/recv (ms_gather0)" % world}

    want = set(args.ops.split(","))
    if "trace" in want:
        guarded("trace_cfg4", trace_op)
    if "spmm" in want:
        guarded("spmm_cfg3", spmm_op)
    if "spgemm" in want:
        guarded("spgemm_cfg5", spgemm_op)
    return out if rank == 0 else None


def bench_ops(args, dev, L, sp, timed, peak):
    import torch

    import oracle
    from paper_1805_03380_b200 import _kernels, synth
    from paper_1805_03380_b200._lib import ptr
    from paper_1805_03380_b200.errors import CorrectnessError

    K, W = args.op_steps, args.warmup
    out = {}

    def T(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    def csc_dev(v, r, o, vdt=torch.float64):
        return T(o, torch.int32), T(r, torch.int32), T(v, vdt)

    def same_csc(got, want):
        p, r, v = (x.cpu().numpy() for x in got)
        return (np.array_equal(p.astype(np.int64), want[2]) and np.array_equal(r.astype(np.int64), want[1])
                and np.array_equal(v.astype(np.float64), want[0]))

    def record(name, ms_list, units, unit, alg_bytes, parity, extra=None, tkey=None):
        tkey = tkey or name.split("_")[0]  # the op's key in the ncu traffic table
        ms = statistics.median(ms_list)
        gbs = alg_bytes / (ms * 1e-3) / 1e9
        d = {"ms": ms, "value": units / (ms * 1e-3), "unit": unit,
             "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                          "algorithmic_bytes": alg_bytes, "traffic": ncu_traffic(tkey),
                          "traffic_launches": ncu_launches(tkey)},
             "parity": parity}
        if extra:
            d.update(extra)
        out[name] = d

    want_ops = set(args.ops.split(","))

    # transpose of the cfg1 result
    if "transpose" in want_ops:
        n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
        a = oracle.canonicalize(n_rows, n_cols, rows, cols, vals)
        p, r, v = csc_dev(*a)
        nnz = int(r.shape[0])
        tp = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
        tr = torch.empty(nnz, dtype=torch.int32, device=dev)
        tv = torch.empty(nnz, dtype=torch.float64, device=dev)
        wb = L.as_transpose_workspace_bytes(nnz, n_rows)
        ws = torch.empty(wb, dtype=torch.uint8, device=dev)

        def f():
            _lib_check(L.as_csc_transpose_f64(n_rows, n_cols, nnz, ptr(p), ptr(r), ptr(v), ptr(tp), ptr(tr), ptr(tv),
                                              ptr(ws), wb, sp))

        f()
        if not same_csc((tp, tr, tv), oracle.transpose(n_rows, n_cols, *a)):
            raise CorrectnessError("transpose differs from the oracle")
        record("transpose_cfg1", timed(f, K, W), nnz, "nnz/s",
               24 * nnz + 4 * (n_cols + 1) + 4 * (n_rows + 1), "bit-exact", {"launches": 1})

    # insertion-log flush (cfg2)
    if "flush" in want_ops:
        n_r, n_c, rows, cols, vals = synth.cfg2_writes()
        nl = rows.shape[0]
        lr, lc, lv = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
        bp = torch.zeros(n_c + 1, dtype=torch.int32, device=dev)
        br = torch.empty(0, dtype=torch.int32, device=dev)
        bv = torch.empty(0, dtype=torch.float64, device=dev)
        op_ = torch.empty(n_c + 1, dtype=torch.int32, device=dev)
        orr = torch.empty(nl, dtype=torch.int32, device=dev)
        ov = torch.empty(nl, dtype=torch.float64, device=dev)
        info = torch.empty(2, dtype=torch.int64, device=dev)
        wb = L.as_flush_workspace_bytes(0, nl, n_c)
        ws = torch.empty(wb, dtype=torch.uint8, device=dev)

        def f():
            _lib_check(L.as_flush_log_f64(n_r, n_c, 0, ptr(bp), ptr(br), ptr(bv), nl, ptr(lr), ptr(lc), ptr(lv),
                                          ptr(op_), ptr(orr), ptr(ov), ptr(info), ptr(ws), wb, sp))

        f()
        nnz = int(info[0].item())
        want = oracle.flush(n_r, n_c, (np.empty(0), np.empty(0, np.int64), np.zeros(n_c + 1, np.int64)), rows, cols, vals)
        if not same_csc((op_, orr[:nnz], ov[:nnz]), want):
            raise CorrectnessError("flush differs from the oracle")
        record("flush_cfg2", timed(f, K, W), nl, "writes/s", 12 * nl + 12 * nnz + 4 * (n_c + 1), "bit-exact",
               {"nnz_out": nnz, "launches": 1})

    # cfg2 through the public API, as the north star states the workload:
    # 200,000 `m[r, c] = v` element writes on a fresh SpMat, then .csc()
    # (hybrid.py:165-181 -> rbt.py:371-387 -> rbt.to_csc rbt.py:444-458),
    # CSC read back to the host; the reference's own SpMat beside it
    if "flush_api" in want_ops:
        from paper_1805_03380_b200 import SpMat

        n_r, n_c, rows, cols, vals = synth.cfg2_writes()
        rl, cl, vl = rows.tolist(), cols.tolist(), vals.tolist()
        want = oracle.flush(n_r, n_c, (np.empty(0), np.empty(0, np.int64), np.zeros(n_c + 1, np.int64)), rows, cols,
                            vals)

        def api_run(pkg_spmat, dev_kw):
            t0 = time.perf_counter()
            m = pkg_spmat.zeros(n_r, n_c, **dev_kw)
            for r_, c_, v_ in zip(rl, cl, vl):
                m[r_, c_] = v_
            t1 = time.perf_counter()
            d = m.csc()
            host = (np.asarray(d.values), np.asarray(d.row_indices), np.asarray(d.col_offsets))
            t2 = time.perf_counter()
            return host, t1 - t0, t2 - t1

        api_run(SpMat, {"device": dev})  # warm
        runs = [api_run(SpMat, {"device": dev}) for _ in range(3)]
        host = runs[-1][0]
        if not (np.array_equal(host[2], want[2]) and np.array_equal(host[1], want[1])
                and np.array_equal(host[0], want[0])):
            raise CorrectnessError("cfg2 API flush differs from the oracle")
        w_ms = 1e3 * statistics.median(r[1] for r in runs)
        f_ms = 1e3 * statistics.median(r[2] for r in runs)
        d = {"ms": w_ms + f_ms, "writes_ms": w_ms, "csc_ms": f_ms, "value": rows.shape[0] / ((w_ms + f_ms) * 1e-3),
             "unit": "writes/s", "parity": "bit-exact vs oracle (LastWins, 0.0 erases)",
             "path": "SpMat.zeros; 200,000 python `m[r, c] = v` (host write log, O(1) each); .csc() = H2D of the "
                     "log + one GPU flush + D2H of the CSC (reference-typed int64 views); wall clock"}
        ref = import_reference() if not args.skip_slow_checks else None
        if ref is not None:
            h, rw, rf = api_run(ref.SpMat, {})
            d["reference_ms"] = 1e3 * (rw + rf)
            d["reference_writes_ms"], d["reference_csc_ms"] = 1e3 * rw, 1e3 * rf
            d["reference_same"] = bool(np.array_equal(h[2], host[2]) and np.array_equal(h[1], host[1])
                                       and np.array_equal(h[0], host[0]))
        out["flush_cfg2_api"] = d

    # SpMM (cfg3)
    if "spmm" in want_ops:
        n, _, av, ar, ao, B = synth.cfg3_spmm()
        k = B.shape[1]
        nnz = av.shape[0]
        p, r, v = T(ao, torch.int32), T(ar, torch.int32), T(av, torch.float32)
        rp, ci, cv = _kernels.transpose(n, n, p, r, v)  # CSR: the handle's cached format
        Bd = torch.as_tensor(B.T.copy(), device=dev).t()  # (n, k) column-major
        C = torch.empty((k, n), dtype=torch.float32, device=dev).t()
        wb = L.as_spmm_workspace_bytes(n, k, 4)
        ws = torch.empty(wb, dtype=torch.uint8, device=dev)

        def mk(exact):
            def f():
                _lib_check(L.as_spmm_csr_f32(n, n, k, ptr(rp), ptr(ci), ptr(cv), ptr(Bd), n, ptr(C), n, exact,
                                             ptr(ws), wb, sp))
            return f

        f_fast, f_exact = mk(0), mk(1)
        parity = "skipped"
        if not args.skip_slow_checks:
            want = oracle.spmm(av.astype(np.float64), ar, ao, B.astype(np.float64), n, n, nthreads=os.cpu_count() or 1)
            f_exact()
            got = C.cpu().numpy().astype(np.float64)
            if not np.array_equal(got, want.astype(np.float32).astype(np.float64)):
                raise CorrectnessError("exact SpMM differs from the oracle")
            f_fast()
            got = C.cpu().numpy().astype(np.float64)
            if not np.all(np.abs(got - want) <= 1e-5 * np.maximum(1.0, np.abs(want))):
                raise CorrectnessError("SpMM outside the 1e-5 tolerance")
            parity = "fast: within 1e-5 of float64 oracle; exact: float64 fold rounded once (bit-exact to oracle)"
            del got
        alg = 4 * (n + 1) + 8 * nnz + 4 * n * k + 4 * n * k
        t_exact = statistics.median(timed(f_exact, K, W))
        record("spmm_cfg3", timed(f_fast, K, W), alg / 1e9, "GB/s", alg, parity,
               {"mode": "f32 FMA, CSR cached on the handle", "exact_mode_ms": t_exact,
                "launches": 2 * ((k + 15) // 16)})

        # the first product on a fresh CSC handle (the reference's
        # mat_times_vec walks the CSC): the column-merge kernel straight over
        # the CSC (no CSR, no transpose), public API; beside it the raw C-ABI
        # call and the CSR route (transpose + row split) a second product takes
        from paper_1805_03380_b200 import SpMat
        from paper_1805_03380_b200.csc import CscData, Dims

        A_csc = CscData(Dims(n, n), p, r, v)

        def f_first():
            return SpMat.from_csc(A_csc) @ Bd

        def f_first_csr():
            m = SpMat.from_csc(A_csc)
            m._csc_mm = 1  # as after one column-merge product: the CSR route
            return m @ Bd

        wbm = L.as_spmm_csc_workspace_bytes(n, nnz)
        wsm = torch.empty(wbm, dtype=torch.uint8, device=dev)
        Cm = torch.empty((k, n), dtype=torch.float32, device=dev).t()

        def f_merge():
            _lib_check(L.as_spmm_csc_f32(n, n, nnz, k, ptr(p), ptr(r), ptr(v), ptr(Bd), n, ptr(Cm), n, ptr(wsm), wbm,
                                         sp))

        first_parity = "skipped"
        if not args.skip_slow_checks:
            for fn in (f_first, lambda: (f_merge(), Cm)[1]):
                got = fn().cpu().numpy().astype(np.float64)
                torch.cuda.synchronize()
                if not np.all(np.abs(got - want) <= 1e-5 * np.maximum(1.0, np.abs(want))):
                    raise CorrectnessError("column-merge SpMM outside the 1e-5 tolerance")
            first_parity = "within 1e-5 of the float64 oracle (float32 additions in arrival order)"
            del want, got
        launches_m = 1 + 2 * ((k + 15) // 16)
        record("spmm_cfg3_csc_merge", timed(f_merge, K, W), alg / 1e9, "GB/s", alg, first_parity,
               {"path": "as_spmm_csc_f32: column merge over the CSC, B rows and entries staged by bulk copies "
                        "(TMA), red.global.add.v4.f32 into an L2-resident row-major 16-column accumulator",
                "launches": launches_m}, tkey="spmm_first")
        t_first = timed(f_first, K, W)
        t_first_csr = statistics.median(timed(f_first_csr, K, W))
        tt = statistics.median(timed(lambda: _kernels.transpose(n, n, p, r, v), K, W))
        record("spmm_cfg3_first_call", t_first, alg / 1e9, "GB/s", alg, first_parity,
               {"path": "SpMat.from_csc(fresh CSC) @ B: column-merge SpMM straight over the CSC (no CSR built)",
                "via_csr_ms": t_first_csr, "via_csr_path": "CSC->CSR transpose (large-input pipeline) + row split",
                "transpose_ms": tt, "launches": launches_m}, tkey="spmm_first")

    # fused trace (cfg4)
    if "trace" in want_ops:
        n, _, A, Bm = synth.cfg4_trace_pair()
        a = csc_dev(*A)
        b = csc_dev(*Bm)
        na, nb = int(a[1].shape[0]), int(b[1].shape[0])
        res = torch.empty(2, dtype=torch.float64, device=dev)
        wb = L.as_trace_workspace_bytes(n, na, nb)
        ws = torch.empty(wb, dtype=torch.uint8, device=dev)

        def f():
            _lib_check(L.as_trace_atb_f64(n, n, ptr(a[0]), ptr(a[1]), ptr(a[2]), ptr(b[0]), ptr(b[1]), ptr(b[2]), na,
                                          nb, ptr(res), ptr(ws), wb, sp))

        f()
        want = oracle.fused_trace(n, *A, *Bm)
        got = float(res[0].item())
        if abs(got - want) > 1e-12 * max(1.0, abs(want)):
            raise CorrectnessError("trace outside 1e-12: %r vs %r" % (got, want))
        # matches: coincident coordinates
        ka = np.repeat(np.arange(n, dtype=np.int64), np.diff(A[2])) * n + A[1]
        kb = np.repeat(np.arange(n, dtype=np.int64), np.diff(Bm[2])) * n + Bm[1]
        matches = int(np.intersect1d(ka, kb, assume_unique=True).shape[0])
        record("trace_cfg4", timed(f, K, W), na + nb, "nnz/s", 4 * (na + nb) + 8 * (n + 1) + 16 * matches,
               "within 1e-12 (|d|=%.3g)" % abs(got - want), {"matches": matches, "launches": 1, "value_f64": got})

    # SpGEMM + add (cfg5)
    if "spgemm" in want_ops or "add" in want_ops:
        n, _, A, Bm = synth.cfg5_pair()
        a = csc_dev(*A)
        b = csc_dev(*Bm)
        na, nb = int(a[1].shape[0]), int(b[1].shape[0])
        if "add" in want_ops:
            cap = na + nb
            cp = torch.empty(n + 1, dtype=torch.int32, device=dev)
            cr = torch.empty(cap, dtype=torch.int32, device=dev)
            cv = torch.empty(cap, dtype=torch.float64, device=dev)
            info = torch.zeros(2, dtype=torch.int64, device=dev)
            wb = L.as_add_workspace_bytes(n, na, nb)
            ws = torch.empty(wb, dtype=torch.uint8, device=dev)

            def f():
                _lib_check(L.as_csc_add_f64(n, n, 1.0, 1.0, ptr(a[0]), ptr(a[1]), ptr(a[2]), ptr(b[0]), ptr(b[1]),
                                            ptr(b[2]), na, nb, ptr(cp), ptr(cr), ptr(cv), ptr(info), ptr(ws), wb, sp))

            f()
            nnz = int(info[0].item())
            if not same_csc((cp, cr[:nnz], cv[:nnz]), oracle.linear_combine(n, *A, *Bm, 1.0, 1.0)):
                raise CorrectnessError("add differs from the oracle")
            record("add_cfg5", timed(f, K, W), na + nb, "nnz/s",
                   12 * (na + nb) + 8 * (n + 1) + 12 * nnz + 4 * (n + 1), "bit-exact", {"nnz_out": nnz, "launches": 1})
        if "spgemm" in want_ops:
            prod_ptr, total = _kernels.spgemm_products(n, n, n, a[0], b[0], b[1])
            cp = torch.empty(n + 1, dtype=torch.int32, device=dev)
            cr = torch.empty(total, dtype=torch.int32, device=dev)
            cv = torch.empty(total, dtype=torch.float64, device=dev)
            info = torch.zeros(2, dtype=torch.int64, device=dev)
            pinfo = torch.zeros(2, dtype=torch.int64, device=dev)
            wb1 = L.as_spgemm_products_workspace_bytes(n)
            ws1 = torch.empty(wb1, dtype=torch.uint8, device=dev)
            wb = L.as_spgemm_workspace_bytes(n, nb, total)
            ws = torch.empty(wb, dtype=torch.uint8, device=dev)

            def f():
                _lib_check(L.as_spgemm_products(n, n, n, ptr(a[0]), ptr(b[0]), ptr(b[1]), ptr(prod_ptr), ptr(pinfo),
                                                ptr(ws1), wb1, sp))
                _lib_check(L.as_spgemm_f64(n, n, n, ptr(a[0]), ptr(a[1]), ptr(a[2]), ptr(b[0]), ptr(b[1]), ptr(b[2]),
                                           nb, ptr(prod_ptr), total, ptr(cp), ptr(cr), ptr(cv), ptr(info), ptr(ws), wb, sp))

            f()
            nnz = int(info[0].item())
            parity = "skipped"
            if not args.skip_slow_checks:
                if not same_csc((cp, cr[:nnz], cv[:nnz]), oracle.spgemm(n, *A, *Bm, n)):
                    raise CorrectnessError("SpGEMM differs from the oracle")
                parity = "bit-exact"
            record("spgemm_cfg5", timed(f, max(3, K // 4), W), total, "products/s",
                   12 * (na + nb) + 8 * (n + 1) + 12 * nnz + 4 * (n + 1), parity,
                   {"products": total, "nnz_out": nnz, "launches": 6})
            # the same product through the public API (SpMat @ SpMat -> ops.matmul ->
            # _kernels.spgemm: sizing read-backs and allocation included), wall clock
            from paper_1805_03380_b200 import SpMat
            from paper_1805_03380_b200.csc import CscData, Dims

            SA = SpMat.from_csc(CscData(Dims(n, n), *a))
            SB = SpMat.from_csc(CscData(Dims(n, n), *b))
            del cr, cv, ws
            torch.cuda.empty_cache()
            api = []
            for i in range(W + max(3, K // 4)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                P = SA @ SB
                Pc = P.csc()
                torch.cuda.synchronize()
                if i >= W:
                    api.append(time.perf_counter() - t0)
                del P, Pc
            out["spgemm_cfg5"]["api_ms"] = 1e3 * statistics.median(api)
            out["spgemm_cfg5"]["api_path"] = "SpMat A @ SpMat B -> CSC on the device (wall clock, host syncs included)"

    # beyond BASELINE sizes: the bandwidth regime the north star's 60 % target
    # refers to (the large-input pipeline, csrc/largen.cuh)
    if "large" in want_ops:
        out["large_n"] = bench_large_n(args, dev, L, sp, timed, peak)

    # SURVEY 8f-2 ("next" rows): construction-funnelled ops and segmented
    # reductions through the public ops API on the cfg 1 matrix (10k x 10k,
    # 995,078 nnz), each checked against oracle/funnel.py first
    if "next" in want_ops:
        from oracle import funnel as OF
        from paper_1805_03380_b200 import SpMat, ops
        from paper_1805_03380_b200.csc import CscData, Dims

        n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
        Am = oracle.canonicalize(n_rows, n_cols, rows, cols, vals)
        A = SpMat.from_csc(CscData.from_reference_arrays(Dims(n_rows, n_cols), *Am, device=dev))
        A.csr()  # the per-row reductions use the cached CSR, as every row-split op does
        nnz = int(Am[0].shape[0])
        small = oracle.canonicalize(40, 25, np.arange(100) % 40, np.arange(100) % 25, np.linspace(-1, 1, 100))
        S = SpMat.from_csc(CscData.from_reference_arrays(Dims(40, 25), *small, device=dev))

        def chk(name, ok):
            if not ok:
                raise CorrectnessError("%s differs from oracle/funnel.py" % name)

        def same(m, want):
            d = m.csc()
            return (np.array_equal(d.col_offsets, want[2]) and np.array_equal(d.row_indices, want[1])
                    and np.array_equal(d.values.view(np.int64), want[0].view(np.int64)))

        nxt = [
            ("sum_dim0", lambda: ops.sum_dim(A, 0),
             lambda r: np.array_equal(r, OF.reduce(Am, n_rows, n_cols, "sum", 0)), 12 * nnz + 4 * n_cols + 8 * n_cols),
            ("max_dim1", lambda: ops.max_dim(A, 1),
             lambda r: np.array_equal(r, OF.reduce(Am, n_rows, n_cols, "max", 1)), 12 * nnz + 4 * n_rows + 8 * n_rows),
            ("norm_fro", lambda: ops.norm(A, "fro"), lambda r: r == OF.norm(Am, n_rows, n_cols, "fro"), 8 * nnz),
            ("norm_1", lambda: ops.norm(A, 1), lambda r: r == OF.norm(Am, n_rows, n_cols, 1), 8 * nnz + 4 * n_cols),
            ("trace", lambda: ops.trace(A), lambda r: r == OF.trace(Am), 12 * nnz + 4 * n_cols),
            ("submat", lambda: ops.submat(A, (1000, 8999), (2000, 7999)),
             lambda r: same(r, OF.submat(Am, 1000, 8999, 2000, 7999)), 24 * nnz),
            ("normalise_2_dim0", lambda: ops.normalise(A, 2, 0),
             lambda r: same(r, OF.normalise(Am, n_rows, n_cols, 2, 0)), 16 * nnz + 12 * nnz + 16 * nnz),
            ("repmat_2x2", lambda: ops.repmat(A, 2, 2),
             lambda r: same(r, OF.repmat(Am, n_rows, n_cols, 2, 2)), 12 * nnz + 4 * 12 * nnz),
            ("kron_small_x_cfg1", lambda: ops.kron(S, A), None, 12 * nnz * 100),
        ]
        res = {}
        for name, fn, check_fn, alg in nxt:
            r = fn()
            torch.cuda.synchronize()
            parity = "skipped (size)"
            if check_fn is not None and not args.skip_slow_checks:
                chk(name, check_fn(r))
                parity = "bit-exact vs oracle/funnel.py"
            ms = statistics.median(timed(fn, max(3, K // 2), W))
            gbs = alg / (ms * 1e-3) / 1e9
            res[name] = {"ms": ms, "GB/s": gbs, "frac": gbs / peak, "algorithmic_bytes": alg, "parity": parity,
                         "path": "public ops API (host sync for scalar / vector results included)"}
        out["next_8f2_cfg1"] = res

        # Matrix Market text of the cfg 1 matrix (~32 MB):
        # native parallel parse + GPU duplicate check + GPU build, and save
        import io as _io

        from paper_1805_03380_b200 import load_mm, save_mm

        buf = _io.StringIO()
        save_mm(A, buf)
        text = buf.getvalue()
        loaded = load_mm(text, device=dev)
        again = _io.StringIO()
        save_mm(loaded, again)
        if again.getvalue() != text or not same(loaded, Am):
            raise CorrectnessError("Matrix Market round trip is not byte-identical")
        mb = len(text) / 1e6

        def t_wall(fn, reps):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts)

        tl = t_wall(lambda: load_mm(text, device=dev), 5)
        ts_ = t_wall(lambda: save_mm(A, _io.StringIO()), 5)
        out["next_8f3_mm_cfg1"] = {
            "bytes": len(text), "nnz": nnz, "load_ms": tl * 1e3, "load_MB_s": mb / tl, "save_ms": ts_ * 1e3,
            "save_MB_s": mb / ts_, "threads": len(os.sched_getaffinity(0)),
            "parity": "save(load(text)) byte-identical; CSC bit-exact vs oracle",
            "path": "wall clock: host parse/format (native, all host threads) + H2D + GPU build / D2H"}
    return out


def bench_large_n(args, dev, L, sp, timed, peak):
    """Construction and transpose at 1e7 / 1e8 / 5e7 elements (seeded uniform
    coordinates, values U[-1,1]), each checked first: bit-exact against the
    oracle at 1e7, by properties at the larger sizes (strictly increasing
    (column, row) keys, nnz = distinct input keys, value sum; transpose
    involution and row histogram)."""
    import torch

    import oracle
    from paper_1805_03380_b200._lib import ptr
    from paper_1805_03380_b200.errors import CorrectnessError

    cases = [("build_1e7", "build", 1_000_000, 1_000_000, 10_000_000, torch.float64),
             ("build_1e8", "build", 10_000_000, 10_000_000, 100_000_000, torch.float64),
             ("transpose_1e7_f32", "transpose", 1_000_000, 1_000_000, 10_000_000, torch.float32),
             ("transpose_5e7", "transpose", 5_000_000, 5_000_000, 50_000_000, torch.float64)]
    res = {}
    K, W = max(3, args.op_steps // 2), args.warmup
    for name, op, n_rows, n_cols, n, vdt in cases:
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
            _lib_check(fb(n_rows, n_cols, n, ptr(rows), ptr(cols), 4, ptr(vals), 0, ptr(cp), ptr(ri), ptr(ov),
                          ptr(info), ptr(ws), wb, sp))

        build()
        torch.cuda.synchronize()
        nnz = int(info[0].item())
        if op == "build":
            if n <= 20_000_000:
                want = oracle.canonicalize(n_rows, n_cols, rows.cpu().numpy().astype(np.int64),
                                           cols.cpu().numpy().astype(np.int64), vals.cpu().numpy().astype(np.float64))
                ok = (np.array_equal(cp.cpu().numpy(), want[2]) and np.array_equal(ri[:nnz].cpu().numpy(), want[1])
                      and np.array_equal(ov[:nnz].cpu().numpy(), want[0]))
                parity = "bit-exact vs oracle"
            else:
                cnt = (cp[1:] - cp[:-1]).long()
                colx = torch.repeat_interleave(torch.arange(n_cols, device=dev), cnt)
                keys = colx * n_rows + ri[:nnz].long()
                distinct = int(torch.unique(cols.long() * n_rows + rows.long()).numel())
                s_in, s_out = float(vals.double().sum()), float(ov[:nnz].double().sum())
                ok = (bool((keys[1:] > keys[:-1]).all()) and distinct == nnz and int(cp[-1]) == nnz
                      and abs(s_in - s_out) <= 1e-9 * max(1.0, abs(s_in)))
                parity = "strictly increasing (col,row) keys, nnz = distinct input keys, value sum within 1e-9"
                del cnt, colx, keys
            if not ok:
                raise CorrectnessError("%s differs from the oracle / properties" % name)
            alg = (8 + vb) * n + (4 + vb) * nnz + 4 * (n_cols + 1)
            t = timed(build, K, W)
            units = n
        else:
            p, r, v = cp.clone(), ri[:nnz].clone(), ov[:nnz].clone()
            del ws
            tp = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
            tr = torch.empty(nnz, dtype=torch.int32, device=dev)
            tv = torch.empty(nnz, dtype=vdt, device=dev)
            ft = L.as_csc_transpose_f64 if vdt == torch.float64 else L.as_csc_transpose_f32
            wbt = L.as_transpose_workspace_bytes(nnz, n_rows)
            wst = torch.empty(wbt, dtype=torch.uint8, device=dev)

            def tr_fn():
                _lib_check(ft(n_rows, n_cols, nnz, ptr(p), ptr(r), ptr(v), ptr(tp), ptr(tr), ptr(tv), ptr(wst), wbt,
                              sp))

            tr_fn()
            torch.cuda.synchronize()
            if nnz <= 20_000_000:
                want = oracle.transpose(n_rows, n_cols, v.cpu().numpy().astype(np.float64),
                                        r.cpu().numpy().astype(np.int64), p.cpu().numpy().astype(np.int64))
                ok = (np.array_equal(tp.cpu().numpy(), want[2]) and np.array_equal(tr.cpu().numpy(), want[1])
                      and np.array_equal(tv.cpu().numpy().astype(np.float64), want[0]))
                parity = "bit-exact vs oracle"
            else:
                bp, br, bv = torch.empty_like(p), torch.empty_like(r), torch.empty_like(v)
                _lib_check(ft(n_cols, n_rows, nnz, ptr(tp), ptr(tr), ptr(tv), ptr(bp), ptr(br), ptr(bv), ptr(wst), wbt,
                              sp))
                ok = (torch.equal(bp, p) and torch.equal(br, r) and torch.equal(bv, v)
                      and torch.equal((tp[1:] - tp[:-1]).long(), torch.bincount(r.long(), minlength=n_rows)))
                parity = "involution (A^T)^T == A bit-exact, row histogram"
                del bp, br, bv
            if not ok:
                raise CorrectnessError("%s differs from the oracle / properties" % name)
            alg = 2 * (4 + vb) * nnz + 4 * (n_cols + 1) + 4 * (n_rows + 1)
            t = timed(tr_fn, K, W)
            units = nnz
            del p, r, v, tp, tr, tv, wst
        ms = statistics.median(t)
        gbs = alg / (ms * 1e-3) / 1e9
        res[name] = {"ms": ms, "value": units / (ms * 1e-3), "unit": "elements/s", "n": n, "nnz_out": nnz,
                     "shape": [n_rows, n_cols], "dtype": "f64" if vb == 8 else "f32",
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                                  "algorithmic_bytes": alg, "traffic": ncu_traffic(name),
                                  "traffic_launches": ncu_launches(name)},
                     "parity": parity, "engine": "large-input pipeline (csrc/largen.cuh)"}
        del rows, cols, vals, cp, ri, ov, info
        torch.cuda.empty_cache()
    return res


def _lib_check(rc):
    from paper_1805_03380_b200 import _lib

    _lib.check(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ops", default="transpose,flush,flush_api,spmm,trace,add,spgemm,large,next")
    ap.add_argument("--op-steps", type=int, default=10)
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--skip-slow-checks", action="store_true")
    ap.add_argument("--flush", default="read", choices=["read", "write"])
    ap.add_argument("--mg-deadline", type=float, default=600.0,
                    help="seconds the sharded multi-GPU ops may take before the headline line is printed without them")
    ap.add_argument("--mg", action="store_true",
                    help="run the sharded (multi-GPU) ops even at world size 1 (needs torchrun env)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return main_device(args)


if __name__ == "__main__":
    sys.exit(main())

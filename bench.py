#!/usr/bin/env python
"""Benchmark of the B200 SpGEMM hot path (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Workload (BASELINE.json metric "SpGEMM GFLOP/s and ms per C=A·B"): config 2,
C = A·A with A = gen_erdos_renyi(2^22, 2^-18, seed 1) (the reference generator,
reproduced bit for bit), fp64. A step is one full C = A·A:
  * N = 1: the local multiply (spgemm_local) on one B200;
  * N > 1: one process per GPU (torchrun), trident grid (P, lambda) =
    (2,2) / (4,4) / (8,2): every rank pulls its A/B tiles from the owners over
    NVLink (CUDA IPC, no collective on the data path), multiplies and merges its
    C tile. value = 2*products / (max-over-ranks step time).
Inputs (A 0.8 GB + B 0.8 GB) and C (12.9 GB) are far larger than L2 (126 MB),
so no L2 flush is needed between steps.

`e2e` is the same metric through the drop-in C ABI with HOST buffers (pinned):
upload A and B, multiply, download C, every step. `--impl reference` times the
reference's own CPU spgemm_local (oracle/_ref, built from /root/reference)
on the host cores (one worker process per core, each a row slice of A).
"""
from __future__ import annotations

import argparse
import ctypes as C
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

CONFIGS = {
    1: dict(n=16384, d=8.0, desc="Erdos-Renyi n=16384, 8 nnz/row, C=A*A fp64"),
    2: dict(n=1 << 22, d=16.0, desc="Erdos-Renyi n=2^22, 16 nnz/row, C=A*A fp64"),
    4: dict(n=1 << 21, d=16.0, desc="MCL expansion: column_normalize(ER 2^21, 16/row) squared", mcl=True),
}
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200)
METRIC = "SpGEMM GFLOP/s and ms per C=A·B at 1/2/4/8 B200; % HBM roofline"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 2 + k and s[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def alg_bytes(m, nnz_a, products, nnz_c):
    """read A once, gather each referenced B entry (col+val) once
    per product, write C once (8 B rowptr, 4 B col, 8 B value)."""
    return (m + 1) * 8 + nnz_a * 12 + products * 12 + (m + 1) * 8 + nnz_c * 12


def make_input(cfg):
    import paper_2603_21444_b200 as spg
    c = CONFIGS[cfg]
    a = spg.gen_erdos_renyi(c["n"], c["d"] / c["n"], 1)
    if c.get("mcl"):
        raise SystemExit("config 4 bench: use --config 2 (MCL post-step is reported by scripts)")
    return a


def kernel_source_sha():
    import hashlib
    with open(os.path.join(ROOT, "paper_2603_21444_b200", "csrc", "spgemm.cu"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def profile_traffic(cfg, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the numeric
    kernel from the committed `ncu --set full` capture (profiles/traffic.json,
    written by scripts/ncu_traffic.py). Used only when the capture was taken
    of the kernel source being benchmarked (sha256 of spgemm.cu), else null."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        e = d.get(f"config{cfg}_n{world}")
        if isinstance(e, dict) and e.get("spgemm_cu_sha16") == kernel_source_sha():
            return e.get("bytes")
    return None


# ------------------------------------------------------------- reference arm
def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import multiprocessing as mp

    import oracle as O
    cfgd = CONFIGS[args.config]
    n = cfgd["n"]
    t0 = time.time()
    a = O.ref_gen_erdos_renyi(n, cfgd["d"] / n, 1)
    gen_s = time.time() - t0
    cores = os.cpu_count() or 1
    # bounded sample: each worker multiplies a slice of A's rows by A (the full B)
    rows_per = int(os.environ.get("SPG_REF_ROWS", max(256, min(n // cores, 1 << 15))))
    rp = a.rowptr

    def slice_rows(r0, r1):
        lo, hi = int(rp[r0]), int(rp[r1])
        return O.Csr(r1 - r0, a.ncols, rp[r0:r1 + 1] - lo, a.colind[lo:hi], a.values[lo:hi])

    ha = O.RefHandle.from_csr(a)
    ctx = mp.get_context("fork")

    def one_step(step):
        jobs = []
        for w in range(cores):
            r0 = ((step * cores + w) * rows_per) % max(1, n - rows_per)
            jobs.append((r0, r0 + rows_per))
        q = ctx.Queue()

        def work(r0, r1):
            s = slice_rows(r0, r1)
            secs, nnzc, _ = O.ref_spgemm_local_timed(s, ha)
            q.put((O.port_products(s, a), secs))

        procs = [ctx.Process(target=work, args=j) for j in jobs]
        t = time.time()
        for p in procs:
            p.start()
        res = [q.get() for _ in procs]
        for p in procs:
            p.join()
        wall = time.time() - t
        return sum(r[0] for r in res), wall

    for _ in range(args.warmup):
        one_step(0)
    tot_p, tot_t = 0, 0.0
    for s in range(args.steps):
        p, t = one_step(s + 1)
        tot_p += p
        tot_t += t
    gflops = 2.0 * tot_p / tot_t / 1e9
    ms_per = tot_t / args.steps * 1e3
    sample = (f"{cores} worker processes x {rows_per} rows of A (config {args.config}) times full A per step, "
              f"reference spgemm_local (oracle/_ref, csr.cpp:132-165), 1 thread each; gen {gen_s:.1f}s")
    line = {
        "metric": METRIC, "value": round(gflops, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference gen_erdos_renyi, seed 1)",
        "impl": "reference",
        "config": {"workload": CONFIGS[args.config]["desc"], "config_id": args.config, "n": n,
                   "sample_rows_per_worker": rows_per},
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(a, seconds_target=12.0):
    """Reference spgemm_local (oracle/_ref) on a bounded row slice, 1 core."""
    import oracle as O
    if not O.ref_available():
        kind, fn = "port", None
    else:
        kind = "reference"
    n = int(a.nrows)
    rows = min(n, 1 << 16)
    rp = np.asarray(a.rowptr)
    lo, hi = 0, int(rp[rows])
    s = O.Csr(rows, a.ncols, rp[:rows + 1].copy(), np.asarray(a.colind[lo:hi]), np.asarray(a.values[lo:hi]))
    ha = O.RefHandle.from_csr(a) if kind == "reference" else None
    prods = O.port_products(s, a)
    t0 = time.time()
    if kind == "reference":
        secs, _, _ = O.ref_spgemm_local_timed(s, ha)
    else:
        O.port_spgemm(s, a)
        secs = time.time() - t0
    # scale the sample toward the target duration (bounded)
    if secs < seconds_target / 4 and rows < n:
        rows2 = min(n, int(rows * seconds_target / max(secs, 1e-3)))
        hi = int(rp[rows2])
        s = O.Csr(rows2, a.ncols, rp[:rows2 + 1].copy(), np.asarray(a.colind[:hi]), np.asarray(a.values[:hi]))
        prods = O.port_products(s, a)
        if kind == "reference":
            secs, _, _ = O.ref_spgemm_local_timed(s, ha)
        else:
            t0 = time.time()
            O.port_spgemm(s, a)
            secs = time.time() - t0
        rows = rows2
    return {"value": round(2.0 * prods / secs / 1e9, 5), "unit": "GFLOP/s", "cores": 1, "kind": kind,
            "sample": f"rows 0..{rows} of A times full A ({prods} products, {secs:.1f} s, 1 core; "
                      f"reference is sequential)"}


# ------------------------------------------------------------------ our arm
def ours_single(args):
    import torch
    import paper_2603_21444_b200 as spg
    from paper_2603_21444_b200 import _capi

    a = make_input(args.config)
    dev = spg.Device(0)
    torch.cuda.set_device(0)
    stream = torch.cuda.ExternalStream(dev.stream, device="cuda:0")
    da = dev.upload(a)
    products = dev.products(da, da)
    nnz_a = a.nnz
    m = int(a.nrows)

    dev.timing(True)
    for _ in range(args.warmup):
        c = dev.spgemm(da, da)
        nnz_c = c.nnz
        del c
    dev.synchronize()
    dev.timing_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(0) as clk:
        dev.synchronize()
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev0.record(stream)
        for i in range(args.steps):
            c = dev.spgemm(da, da)
            step_ev[i].record(stream)
            del c
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    step_ms = [ev0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i]) for i in range(1, args.steps)]
    kt = dev.timing_read()
    own = {k: v for k, v in kt.items()}
    launches = sum(v[0] for v in own.values())
    kname = "spgemm_tile"
    num_ms = own.get(kname, (1, 0.0))[1] / max(1, own.get(kname, (1, 0))[0])
    dev.timing(False)

    # end to end through the C ABI with pinned host buffers
    L = _capi.lib()
    rp = np.ascontiguousarray(a.rowptr, np.int64)
    ci = np.ascontiguousarray(a.colind.astype(np.int32))
    va = np.ascontiguousarray(a.values, np.float64)
    for arr in (rp, ci, va):
        _capi.check(L.spg_host_register(arr.ctypes.data, arr.nbytes))
    c_rp = np.empty(m + 1, np.int64)
    c_ci = np.empty(nnz_c, np.int32)
    c_va = np.empty(nnz_c, np.float64)
    for arr in (c_rp, c_ci, c_va):
        _capi.check(L.spg_host_register(arr.ctypes.data, arr.nbytes))

    def e2e_two_calls():
        h = C.c_void_p()
        _capi.check(L.spg_spgemm_host(dev.ctx, m, a.ncols, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, m,
                                      a.ncols, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 4, C.byref(h)))
        _capi.check(L.spg_csr_download(dev.ctx, h, c_rp.ctypes.data, c_ci.ctypes.data, 4, c_va.ctypes.data))
        _capi.check(L.spg_csr_free(h))

    h2h_batches = int(os.environ.get("SPG_H2H_BATCHES", 8))

    def e2e_host_to_host():
        got = C.c_int64()
        _capi.check(L.spg_spgemm_host_to_host(dev.ctx, m, a.ncols, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                              m, a.ncols, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 4,
                                              h2h_batches, nnz_c, c_rp.ctypes.data, c_ci.ctypes.data,
                                              c_va.ctypes.data, C.byref(got)))
        assert got.value == nnz_c

    def e2e_time(fn):
        fn()
        dev.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn()
        dev.synchronize()
        return (time.perf_counter() - t0) / e2e_steps * 1e3

    e2e_steps = max(1, int(os.environ.get("SPG_E2E_STEPS", args.steps)))
    e2e_ms_two = e2e_time(e2e_two_calls)
    ref_rp, ref_ci, ref_va = c_rp.copy(), c_ci[::1009].copy(), c_va[::1009].copy()
    c_rp[:] = -1
    e2e_ms = e2e_time(e2e_host_to_host)
    # the host-to-host C must equal the two-call C (row pointers exact, every 1009th entry)
    if not (np.array_equal(c_rp, ref_rp) and np.array_equal(c_ci[::1009], ref_ci)
            and np.array_equal(c_va[::1009], ref_va)):
        raise RuntimeError("spg_spgemm_host_to_host result differs from spg_spgemm_host + spg_csr_download")
    for arr in (rp, ci, va, c_rp, c_ci, c_va):
        L.spg_host_unregister(arr.ctypes.data)
    h2d = rp.nbytes + ci.nbytes + va.nbytes  # C = A*A: the C ABI uploads the shared host matrix once
    d2h = c_rp.nbytes + c_ci.nbytes + c_va.nbytes

    peak, peak_kind = measured_peaks()
    ba = alg_bytes(m, nnz_a, products, nnz_c)
    achieved = ba / (num_ms * 1e-3) / 1e9
    gflops = 2.0 * products / (ms * 1e-3) / 1e9
    cpu = cpu_baseline_sample(a) if os.environ.get("SPG_SKIP_CPU") != "1" else None
    line = {
        "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "ms_per_step_min": round(min(step_ms), 4), "ms_per_step_median": round(statistics.median(step_ms), 4),
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference gen_erdos_renyi, seed 1)",
        "config": {"workload": CONFIGS[args.config]["desc"], "config_id": args.config, "grid": "P=1 lambda=1 q=1",
                   "products": products, "nnz_A": nnz_a, "nnz_C": nnz_c,
                   "l2": "inputs (1.6 GB) and C (12.9 GB) larger than the 126 MB L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "k_tile (single-pass tile multiply: gathers, bucket sort, "
                                               "look-back, write C)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": profile_traffic(args.config, 1),
                     "algorithmic_bytes": ba, "kernel_ms": round(num_ms, 4),
                     "whole_step_frac": round(ba / (ms * 1e-3) / 1e9 / peak, 4), "peak_kind": peak_kind},
        "kernel_ms": {k: round(v[1] / max(1, v[0]), 4) for k, v in own.items()},
        "e2e": {"value": round(2.0 * products / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "ms_per_step": round(e2e_ms, 2), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": f"spg_spgemm_host_to_host (one C ABI call, host CSR in and out, pinned host buffers, "
                        f"{h2h_batches} row batch(es))",
                "two_calls_ms_per_step": round(e2e_ms_two, 2),
                "two_calls_value": round(2.0 * products / (e2e_ms_two * 1e-3) / 1e9, 3)},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
    }
    print(json.dumps(line), flush=True)


def ours_multi(args):
    import torch
    import torch.distributed as dist

    # NCCL's init banner (and any other C-level stdout) goes to stderr; the one
    # JSON line is written to the original stdout
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    import paper_2603_21444_b200 as spg
    from paper_2603_21444_b200 import dist as sd

    rank, world, local = env_rank()
    # SPG_OVERSUBSCRIBE=1 (functional check of the N=8 path on a smaller box):
    # ranks share GPUs round-robin and the plumbing runs on gloo, since NCCL
    # refuses two ranks on one device. Timings of such a run mean nothing.
    over = os.environ.get("SPG_OVERSUBSCRIBE") == "1"
    if over:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if over:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tdev = "cpu" if over else f"cuda:{local}"
    procs, lam = sd.grid_for_gpus(world)
    if os.environ.get("SPG_GRID"):  # experiment: another legal grid for this world size, "P,lambda"
        procs, lam = (int(x) for x in os.environ["SPG_GRID"].split(","))
        assert procs == world, "SPG_GRID must have P = number of ranks"
    grid = spg.TridentGrid.create(procs, lam)
    a = make_input(args.config)
    dev = spg.Device(local)
    stream = torch.cuda.ExternalStream(dev.stream, device=f"cuda:{local}")
    at, bt = sd.rank_tiles(a, a, grid, rank)

    def allgather_bytes(b: bytes):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    ex = sd.RankExchange(dev, at, bt, rank, world, allgather_bytes)
    dist.barrier()
    # products of this rank = Σ over rounds of products(A_isk, B_sj); total = products(A, A)
    products_total = 0
    if rank == 0:
        da = dev.upload(a)
        products_total = dev.products(da, da)
        del da
    pt = torch.tensor([products_total], dtype=torch.int64, device=tdev)
    dist.broadcast(pt, 0)
    products_total = int(pt.item())

    dev.timing(True)
    for _ in range(args.warmup):
        c, tl = ex.trident_step(procs, lam, grid.q)
        del c
    dev.synchronize()
    dev.timing_reset()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tls = []
    with ClockSampler(local) as clk:
        dev.synchronize()
        dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            c, tl = ex.trident_step(procs, lam, grid.q)
            tls.append(tl)
            nnz_c = c.nnz
            del c
        ev1.record(stream)
        ev1.synchronize()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    kt = dev.timing_read()
    launches = sum(v[0] for v in kt.values())
    lt = torch.tensor([launches], dtype=torch.int64, device=tdev)
    dist.all_reduce(lt)
    # end to end through the public API with HOST buffers: every step each rank
    # refills its tiles from pinned host memory (H2D), the ranks run the trident
    # step (peer pulls over NVLink), and each rank downloads its C tile (D2H)
    from paper_2603_21444_b200 import _capi
    L = _capi.lib()

    def host_arrays(m):
        arrs = (np.ascontiguousarray(m.rowptr, np.int64), np.ascontiguousarray(np.asarray(m.colind), np.int32),
                np.ascontiguousarray(m.values, np.float64))
        for x in arrs:
            _capi.check(L.spg_host_register(x.ctypes.data, max(x.nbytes, 1)))
        return arrs

    at_h, bt_h = host_arrays(at), host_arrays(bt)
    m_c = int(at.nrows)
    c_rp = np.empty(m_c + 1, np.int64)
    c_ci = np.empty(max(nnz_c, 1), np.int32)
    c_va = np.empty(max(nnz_c, 1), np.float64)
    for x in (c_rp, c_ci, c_va):
        _capi.check(L.spg_host_register(x.ctypes.data, x.nbytes))

    dbg = os.environ.get("SPG_BENCH_DEBUG")
    phase = np.zeros(3)

    def e2e_step():
        t0 = time.perf_counter()
        ex.reload(at_h, bt_h)
        if dbg:
            dev.synchronize()
        t1 = time.perf_counter()
        dist.barrier()
        c, _ = ex.trident_step(procs, lam, grid.q)
        if dbg:
            dev.synchronize()
        t2 = time.perf_counter()
        _capi.check(L.spg_csr_download(dev.ctx, c.h, c_rp.ctypes.data, c_ci.ctypes.data, 4, c_va.ctypes.data))
        c.free()
        # every peer's pulls of this rank's tiles are done before the next
        # reload overwrites them (RankExchange.reload contract)
        dist.barrier()
        phase[:] += (t1 - t0, t2 - t1, time.perf_counter() - t2)

    e2e_steps = max(1, int(os.environ.get("SPG_E2E_STEPS", args.steps)))
    e2e_step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    dev.synchronize()
    e2e_local = (time.perf_counter() - t0) / e2e_steps * 1e3
    if dbg:
        print(f"[rank {rank}] e2e ms {e2e_local:.2f} (h2d, step, d2h) ms {np.round(phase / (e2e_steps + 1) * 1e3, 2).tolist()} "
              f"cpu affinity {sorted(os.sched_getaffinity(0))[:4]}.. of {len(os.sched_getaffinity(0))}", file=sys.stderr, flush=True)
    et = torch.tensor([e2e_local], dtype=torch.float64, device=tdev)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_ms = float(et.item())
    h2d = sum(x.nbytes for x in at_h + bt_h)
    d2h = c_rp.nbytes + nnz_c * 12
    hb = torch.tensor([h2d, d2h], dtype=torch.int64, device=tdev)
    dist.all_reduce(hb)
    for x in at_h + bt_h + (c_rp, c_ci, c_va):
        L.spg_host_unregister(x.ctypes.data)
    # roofline of rank 0's multiply kernel: its algorithmic bytes / its time
    prod0 = sd.rank_products(a, a, grid, 0) if rank == 0 else 0

    ledger = sd.ledger_for(a, a, grid)
    recv_bytes = int(ledger[:, 1, :, 2].sum(axis=1).max())
    tl_mean = np.mean(np.stack(tls), axis=0)  # [q, 4] ms
    if os.environ.get("SPG_BENCH_DEBUG"):
        print(f"[rank {rank}] ms/step {ms_local:.3f} timeline(q x [exchange, exposed wait, multiply, merge]) "
              f"{np.round(tl_mean, 3).tolist()} kernels {{{', '.join(f'{k}: {v[1] / max(1, v[0]):.3f}' for k, v in kt.items())}}}",
              file=sys.stderr, flush=True)
    exch_ms = float(tl_mean[:, 0].sum())
    if rank == 0:
        peak, peak_kind = measured_peaks()
        gflops = 2.0 * products_total / (ms * 1e-3) / 1e9
        num = kt.get("spgemm_tile", (1, 0.0))
        kms = num[1] / max(1, num[0])
        # rank 0's multiply: A tile rows/nnz, gathers of its products, its C tile
        ba0 = alg_bytes(int(at.nrows), int(at.nnz) * grid.q, prod0, nnz_c)
        ach = ba0 / (kms * 1e-3) / 1e9 if kms > 0 else None
        roof0 = {"bound": "hbm", "kernel": "k_tile (rank 0, its trident rounds)", "peak": peak, "unit": "GB/s",
                 "achieved": round(ach, 1) if ach else None, "frac": round(ach / peak, 4) if ach else None,
                 "traffic": None, "algorithmic_bytes": ba0, "kernel_ms": round(kms, 4), "products_rank0": prod0,
                 "peak_kind": peak_kind}
        line = {
            "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference gen_erdos_renyi, seed 1)",
            "config": {"workload": CONFIGS[args.config]["desc"], "config_id": args.config,
                       "grid": f"trident P={procs} lambda={lam} q={grid.q}", "parallelism": f"trident{world}",
                       "products": products_total,
                       "l2": "inputs and C larger than L2; no flush"},
            "kernel_ms_rank0": {k: round(v[1] / max(1, v[0]), 4) for k, v in kt.items()},
            "exchange": {"ledger_max_recv_bytes_per_rank": recv_bytes, "exchange_ms_rank0": round(exch_ms, 4),
                         "nvlink_frac_rank0": round(recv_bytes / max(exch_ms, 1e-9) / 1e6 / NVLINK_GBS, 4),
                         "nvlink_frac_rank0_of_measured_peer_copy": round(recv_bytes / max(exch_ms, 1e-9) / 1e6 / 770.0, 4),
                         "nvlink_peak_gbs": NVLINK_GBS},
            "roofline": roof0,
            "e2e": {"value": round(2.0 * products_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                    "ms_per_step": round(e2e_ms, 2), "h2d_bytes_per_step": int(hb[0].item()),
                    "d2h_bytes_per_step": int(hb[1].item()),
                    "path": "per rank: spg_csr_upload_into (pinned host -> its tiles), spg_trident_rank, "
                            "spg_csr_download of its C tile; max over ranks"},
            "clocks": clk.summary(),
            "gpu_launches": int(lt.item()),
        }
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    ex.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    _, world, _ = env_rank()
    if args.impl == "reference":
        return reference_arm(args)
    if world > 1:
        return ours_multi(args)
    return ours_single(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: emulated DGEMM (Ozaki scheme II) TFLOPS at n = 16384 on B200.

Metric (BASELINE.json): emulated DGEMM/SGEMM TFLOPS = 2mnk / time, at
m = n = k = 16384, next to native FP64 and FP32 (cuBLAS on the same GPU).
Headline workload (configs[1]): DGEMM 16384^3, 14 moduli, fast mode — the
paper's headline point (OS II-fast-14); the accurate-mode and
moduli-sweep points ride along in "extra".

One step = one full ozk_gemm (K1 scale -> K1 residues -> K2 N int8 GEMMs ->
K3 CRT reconstruction) on device-resident inputs. Inputs (2 x 2.1 GB FP64)
exceed the 126 MB L2, so no explicit flush is needed between steps.
``e2e`` runs the same GEMM through the reference-facing host call
(ozk_gemm_host): H2D of A and B from pinned memory, compute, D2H of C.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU), column blocks of B/C:
rank 0's A is broadcast over NCCL inside each step (the north star's A
broadcast) — in fast mode as row blocks that each rank starts computing on as
they land (ozk_shard_stream_*, --row-block) — and "value" is the aggregate
2 m n_total k / max-over-ranks time. --scaling weak (default): every rank owns
an n-column block; --scaling strong: the n columns are split over the ranks
(BASELINE configs[3]: --n 65536 --scaling strong; at one GPU the problem
runs in workspace panels, with the footprint capped by
--footprint-gb).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_N = 16384
MODULI = 14


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--size", "--n", dest="n", type=int, default=DEFAULT_N)
    p.add_argument("--moduli", type=int, default=MODULI)
    p.add_argument("--mode", choices=["fast", "accurate"], default="fast")
    p.add_argument("--phi", type=float, default=0.5)
    p.add_argument("--no-extra", action="store_true", help="skip the sweep / native / accuracy extras")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=256, help="rows/cols of the CPU baseline sample (full k)")
    p.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                   help="torch.distributed backend for N > 1 (gloo + OZK_BENCH_ONE_DEVICE=1: a functional "
                        "multi-rank run on one GPU; its timing means nothing)")
    p.add_argument("--row-block", type=int, default=2048,
                   help="fast mode, N > 1: A streams to the ranks in row blocks of this many rows (0: whole A)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="weak: n columns per rank; strong: n columns in total, split over the ranks")
    p.add_argument("--footprint-gb", type=float, default=160.0,
                   help="cap on A + B + C + workspace per GPU (the workspace limit is set from it)")
    p.add_argument("--e2e", dest="e2e_force", action="store_true",
                   help="run the host-buffer e2e leg also above n = 32768 (needs 3 x 8 n^2 bytes of pinned host memory)")
    return p.parse_args()


# ------------------------------------------------------------------ CPU baselines
def cpu_reference_sample(n: int, k: int, moduli: int, mode: int, phi: float, min_seconds: float = 10.0):
    """Time the UNMODIFIED reference (oracle/_ref) on a bounded sample of the
    workload: an s x s block of C with the full inner dimension k, all host
    threads (only its INT8 GEMMs are threaded: int8_engine.cpp:49-62)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import RefLib

    from paper_2508_03984_b200.gen import gen_matrix

    ref = RefLib()
    a = gen_matrix(n, k, phi, 1)
    b = gen_matrix(k, n, phi, 2)
    threads = os.cpu_count() or 1
    runs, t0 = 0, time.perf_counter()
    while True:
        ref.gemm(a, b, moduli, mode, threads=threads)
        runs += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or runs >= 50:
            break
    per = el / runs
    return {"seconds_per_sample": per, "threads": threads, "runs": runs,
            "tflops": 2.0 * n * n * k / per / 1e12}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    k = args.n
    s = args.cpu_sample
    mode = 0 if args.mode == "fast" else 1
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import RefLib

    from paper_2508_03984_b200.gen import gen_matrix

    if not RefLib.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcrtgemm_ref.so not built"}))
        return
    ref = RefLib()
    a = gen_matrix(s, k, args.phi, 1)
    b = gen_matrix(k, s, args.phi, 2)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        ref.gemm(a, b, args.moduli, mode, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.gemm(a, b, args.moduli, mode, threads=threads)
        times.append(time.perf_counter() - t0)
    per = sum(times) / len(times)
    v = 2.0 * s * s * k / per / 1e12
    sample = f"C block {s}x{s} of the {args.n}^3 problem (full k={k}), oracle/_ref gemm_emulated, threads={threads}"
    print(json.dumps({
        "impl": "reference",
        "metric": f"emulated DGEMM TFLOPS (2mnk/s) at n={args.n}, {args.moduli} moduli, {args.mode} mode",
        "value": v, "unit": "TFLOPS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (rand-0.5)*exp(phi*randn), phi=%g" % args.phi,
        "config": {"workload": f"DGEMM m=n=k={args.n} per GPU (column block of B/C), {args.moduli} moduli, "
                               f"{args.mode}", "sample": sample},
        "cpu_baseline": {"value": v, "unit": "TFLOPS", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU helpers
def gen_device(rows, cols, phi, seed, dtype, device, chunk=2048):
    """paper generator on the device: column-major (rows x cols) tensor, drawn
    column block by column block (no full-size temporaries at n = 65536)"""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((cols, rows), dtype=dtype, device=device)
    for j0 in range(0, cols, chunk):
        j1 = min(cols, j0 + chunk)
        x = torch.rand((j1 - j0, rows), generator=g, device=device, dtype=torch.float64)
        x = (1.0 - x) - 0.5  # rand in (0, 1]
        if phi:
            x.mul_(torch.exp(phi * torch.randn((j1 - j0, rows), generator=g, device=device, dtype=torch.float64)))
        out[j0:j1].copy_(x)
    return out.t()


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


def load_traffic():
    """DRAM bytes per K2 launch from the committed ncu --set full summary (or None)"""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
    except OSError:
        return {}


def native_gemm_tflops(n, dtype, steps=5):
    import torch

    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(2):
        torch.mm(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        torch.mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return 2.0 * n ** 3 / (ms * 1e-3) / 1e12


def int8_library_tops(n):
    """cuBLASLt int8 GEMM (torch._int_mm) on the same GPU: the library baseline for K2"""
    import torch

    a = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8)
    b = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8).t().contiguous().t()
    for _ in range(2):
        torch._int_mm(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    return 2.0 * n ** 3 / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e12


# ------------------------------------------------------------------ main arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2508_03984_b200 import Context, EmuConfig, Precision, ScaleMode
    from paper_2508_03984_b200.distributed import gemm_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if os.environ.get("OZK_BENCH_ONE_DEVICE") else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    from paper_2508_03984_b200.distributed import column_shard

    n_total = args.n
    m = k = args.n
    if args.scaling == "strong":
        j0, n = column_shard(n_total, world, rank)  # this rank's share of the n columns
        n_done = n_total
    else:
        n, n_done = args.n, args.n * world
    mode = ScaleMode.Fast if args.mode == "fast" else ScaleMode.Accurate
    cfg = EmuConfig(n_moduli=args.moduli, mode=mode, precision=Precision.Fp64)
    stream = torch.cuda.current_stream()
    ctx = Context(local)
    ctx.set_stream(stream.cuda_stream)

    A = gen_device(m, k, args.phi, 1, torch.float64, dev)
    B = gen_device(k, n, args.phi, 2 + rank, torch.float64, dev)  # this rank's column block
    C = torch.empty((n, m), dtype=torch.float64, device=dev).t()
    torch.cuda.empty_cache()
    # footprint cap: the caller's operands + the handle's workspace
    ws_cap = int(args.footprint_gb * 1e9) - torch.cuda.memory_allocated(dev) - (1 << 30)
    ctx.set_workspace_limit(max(ws_cap, 1 << 30))

    def step():
        if world > 1:
            # column shard: A broadcast from rank 0 + (accurate) row-bound all-reduce
            gemm_sharded(ctx, A, B, cfg, C, row_block=args.row_block or None)
        else:
            ctx.gemm(A, B, cfg, C)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    ctx.profile(True)
    ctx.profile_read(reset=True)
    launches0 = ctx.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches = ctx.kernel_launches - launches0
    prof = ctx.profile_read(reset=True)
    ctx.profile(False)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    flop = 2.0 * m * n * k  # this rank's share
    value = 2.0 * m * n_done * k / (ms * 1e-3) / 1e12
    free_b, total_b = torch.cuda.mem_get_info(dev)
    memory = {"abc_gb": torch.cuda.memory_allocated(dev) / 1e9, "workspace_gb": ctx.workspace_bytes / 1e9,
              "device_used_gb": (total_b - free_b) / 1e9, "device_total_gb": total_b / 1e9,
              "plan": ctx.last_plan}

    # ---- roofline of the dominant kernel (K2, tensor-bound) and of K1 / K3 (HBM) ----
    peaks = load_peaks()
    # per step: the streamed multi-GPU path launches K2 once per row block of A,
    # the panelled path once per panel
    k2_ms = prof["products"][0] / args.steps
    k2_ops = args.moduli * 2.0 * m * n * k  # algorithmic int8 ops per step
    achieved = k2_ops / (k2_ms * 1e-3) / 1e12
    bf16 = peaks.get("bf16_tflops")
    peak = 2.0 * bf16 if bf16 else 2.0 * 1590.0
    traffic = load_traffic().get(f"products_n{args.n}_N{args.moduli}_{args.mode}") if world == 1 else None
    hbm = peaks.get("hbm_gbs") or 7700.0
    # K1 / K3 in the step: K1's two streams overlap, so its wall time is the
    # step's total minus K2 and K3 (which run after the join on one stream)
    tot_ms = prof["total"][0] / args.steps
    k3_ms = prof["reconstruct"][0] / args.steps
    k1_ms = max(tot_ms - k2_ms - k3_ms, 1e-9)
    es = 8
    k1_bytes = (m * k + k * n) * (es + args.moduli)  # compulsory: read A, B; write N planes each
    k3_bytes = m * n * (args.moduli + 8)             # read N residues, write C per element
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "residue_gemm_kernel (K2, tcgen05.mma kind::i8)",
                "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops (dense INT8 = 2 x dense BF16 on sm_100)"
                                if bf16 else "2 x fallback 1.59 PFLOP/s bf16 (B200_PROFILING.md)"),
                "traffic_source": "profiles/roofline_traffic.json (ncu --set full, dram__bytes_read+write per launch)",
                "k2_launches_per_step": prof["products"][1] / args.steps, "k2_ms": k2_ms,
                # the memory-bound stages against MEASURED_PEAKS.json hbm_gbs, in the step
                "k1_ms": k1_ms, "k1_gbps": k1_bytes / (k1_ms * 1e-3) / 1e9,
                "k1_frac_hbm": k1_bytes / (k1_ms * 1e-3) / 1e9 / hbm,
                "k3_ms": k3_ms, "k3_gbps": k3_bytes / (k3_ms * 1e-3) / 1e9,
                "k3_frac_hbm": k3_bytes / (k3_ms * 1e-3) / 1e9 / hbm,
                "hbm_peak_gbps": hbm,
                "stage_ms": {kname: v[0] / args.steps for kname, v in prof.items()}}
    if peaks.get("bf16_tflops_sustained"):
        # K2 runs inside a long step: the sustained-clock denominator, for reference
        roofline["peak_sustained"] = 2.0 * peaks["bf16_tflops_sustained"]
        roofline["frac_sustained"] = achieved / roofline["peak_sustained"]

    out = {
        "metric": f"emulated DGEMM TFLOPS (2mnk/s) at n={args.n}, {args.moduli} moduli, {args.mode} mode",
        "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (rand-0.5)*exp(phi*randn), phi={args.phi}, generated on device",
        "config": {"workload": (f"DGEMM m=n=k={args.n} per GPU (column block of B/C), {args.moduli} moduli, {args.mode}"
                                if args.scaling == "weak" else
                                f"DGEMM m=n=k={args.n} split by columns over {world} GPU(s), {args.moduli} moduli, "
                                f"{args.mode}"),
                   "l2": "inputs (2 x 8 n^2 bytes) larger than L2; no flush", "parallelism": f"colshard{world}",
                   "a_broadcast": (f"row blocks of {args.row_block}" if world > 1 and args.row_block
                                   and args.mode == "fast" else ("whole" if world > 1 else "none")),
                   "footprint_cap_gb": args.footprint_gb},
        "gpu_launches": int(launches), "roofline": roofline, "clocks": clk.summary(), "memory": memory,
    }

    # ---- end to end through the host-pointer C ABI (ozk_gemm_host) ----------------
    big = args.n > 32768 and not args.e2e_force  # 3 x 8 n^2 bytes of pinned host memory
    if not args.no_e2e and world == 1 and not big:
        import numpy as np

        Ah = torch.empty((k, m), dtype=torch.float64, pin_memory=True)
        Bh = torch.empty((n, k), dtype=torch.float64, pin_memory=True)
        Ch = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A.t())
        Bh.copy_(B.t())
        an, bn, cn = (np.asfortranarray(x.numpy().T) for x in (Ah, Bh, Ch))  # zero-copy column-major views
        for _ in range(1):
            ctx.gemm_host(an, bn, cfg, c=cn)
        e_steps = max(2, min(args.steps, 4))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            ctx.gemm_host(an, bn, cfg, c=cn)
        e_s = (time.perf_counter() - t0) / e_steps
        out["e2e"] = {"value": flop / e_s / 1e12, "unit": "TFLOPS", "h2d_bytes_per_step": 2 * 8 * m * k,
                      "d2h_bytes_per_step": 8 * m * n, "ms_per_step": e_s * 1e3,
                      "path": "ozk_gemm_host (pinned host A, B, C)"}
        del Ah, Bh, Ch, an, bn, cn
        # the same call from pageable host memory (what a crtgemm Matrix<T>, a
        # std::vector, hands over): the handle's pinned staging ring
        ap = np.asfortranarray(A.cpu().numpy())
        bp = np.asfortranarray(B.cpu().numpy())
        cp = np.zeros((m, n), order="F")
        ctx.gemm_host(ap, bp, cfg, c=cp)
        t0 = time.perf_counter()
        for _ in range(2):
            ctx.gemm_host(ap, bp, cfg, c=cp)
        e_p = (time.perf_counter() - t0) / 2
        out["e2e_pageable"] = {"value": flop / e_p / 1e12, "unit": "TFLOPS", "ms_per_step": e_p * 1e3,
                               "path": "ozk_gemm_host (pageable numpy A, B, C: pinned staging ring, host_stage.cpp)"}
        del ap, bp, cp
        dropin = dropin_e2e(args.n, args.moduli, args.mode)
        if dropin:
            out["e2e_dropin"] = dropin
    elif not args.no_e2e and world > 1 and not big:
        # N > 1: host buffers on every rank (A on the source rank only): H2D of A
        # (rank 0) and of each rank's B block, the column-sharded GEMM with A's
        # row-streamed broadcast, D2H of each C block; wall clock, max over ranks
        Ah = torch.empty((k, m), dtype=torch.float64, pin_memory=True)
        Bh = torch.empty((n, k), dtype=torch.float64, pin_memory=True)
        Ch = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A.t())
        Bh.copy_(B.t())

        def e2e_step():
            if rank == 0:
                A.t().copy_(Ah, non_blocking=True)
            B.t().copy_(Bh, non_blocking=True)
            step()
            Ch.copy_(C.t(), non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        dist.barrier()
        e_steps = max(2, min(args.steps, 4))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        e_s = (time.perf_counter() - t0) / e_steps
        t = torch.tensor([e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_s = float(t.item())
        out["e2e"] = {"value": 2.0 * m * n_done * k / e_s / 1e12, "unit": "TFLOPS",
                      "h2d_bytes_per_step": 8 * (m * k + k * n * world), "d2h_bytes_per_step": 8 * m * n * world,
                      "ms_per_step": e_s * 1e3,
                      "path": "pinned host A (rank 0), B and C blocks (every rank) -> H2D -> gemm_sharded -> D2H"}
    elif not args.no_e2e:
        out["e2e_note"] = f"host-buffer leg skipped at n={args.n} (needs {3 * 8 * args.n ** 2 / 1e9:.0f} GB pinned; --e2e)"

    # ---- extras: native FP64/FP32, moduli sweep, accuracy, int8 library -----------
    if not args.no_extra and world == 1 and args.n <= 16384:
        extra = {}
        extra["native_fp64_tflops"] = native_gemm_tflops(n, torch.float64, 3)
        extra["native_fp32_tflops"] = native_gemm_tflops(n, torch.float32, 3)
        extra["int8_cublaslt_tops"] = int8_library_tops(n)
        exact = ExactPool()

        def timed(Ax, Bx, c2, Cx, reps=2, **kw):
            ctx.gemm(Ax, Bx, c2, Cx, **kw)
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(reps):
                ctx.gemm(Ax, Bx, c2, Cx, **kw)
            s1.record(stream)
            torch.cuda.synchronize()
            mm, nn = Cx.shape
            kk = Ax.shape[0] if kw.get("trans_a") else Ax.shape[1]
            return 2.0 * mm * nn * kk / (s0.elapsed_time(s1) / reps * 1e-3) / 1e12

        # accuracy at the bench size against the reference's exact GMP oracle
        # (oracle.cpp exact_gemm / compare) on 64 x 64 sampled entries of C, full k
        rows, cols = sample_idx(m, 64, 7), sample_idx(n, 64, 8)
        exact.submit("main", A, B, rows, cols)
        sweep, acc = {}, {}
        for N in (12, 14, 15, 16, 18, 20):
            for md in (ScaleMode.Fast, ScaleMode.Accurate):
                key = f"{md.name.lower()}{N}"
                sweep[key] = timed(A, B, EmuConfig(n_moduli=N, mode=md), C)
                acc[key] = C[rows][:, cols].cpu().numpy()
        Cn = torch.mm(A, B)
        acc["native_fp64"] = Cn[rows][:, cols].cpu().numpy()
        del Cn
        extra["dgemm_sweep_tflops"] = sweep
        # BLAS transposes (square problem: the stored operands are read as op(X) = X^T)
        extra["transposes_tflops"] = {"TN"[not ta] + "TN"[not tb]: timed(A, B, cfg, C, trans_a=ta, trans_b=tb)
                                      for ta, tb in ((False, False), (True, False), (False, True), (True, True))}
        # SGEMM emulation (BASELINE configs[2]): FP32 inputs, FP32 C, N = 6..10, vs native FP32
        A32, B32 = A.float(), B.float()
        C32 = torch.empty((n, m), dtype=torch.float32, device=dev).t()
        exact.submit("sgemm", A32, B32, rows, cols)
        ssweep, sacc = {}, {}
        for N in (6, 7, 8, 9, 10):
            for md in (ScaleMode.Fast, ScaleMode.Accurate):
                key = f"{md.name.lower()}{N}"
                ssweep[key] = timed(A32, B32, EmuConfig(n_moduli=N, mode=md, precision=Precision.Fp32), C32)
                sacc[key] = C32[rows][:, cols].double().cpu().numpy()
        sacc["native_fp32"] = torch.mm(A32, B32)[rows][:, cols].double().cpu().numpy()
        extra["sgemm_sweep_tflops"] = ssweep
        del A32, B32, C32
        # input dynamic range (BASELINE configs[4]): phi sweep, 1024^2 outputs with full k,
        # exact errors on 64 x 64 sampled entries
        phi_acc = {}
        r1, c1 = sample_idx(1024, 64, 9), sample_idx(1024, 64, 10)
        for phi in (0.5, 1.0, 1.5, 2.0, 3.0, 4.0):
            Ap = gen_device(1024, k, phi, 11, torch.float64, dev)
            Bp = gen_device(k, 1024, phi, 12, torch.float64, dev)
            exact.submit(f"phi{phi}", Ap, Bp, r1, c1)
            Cp = torch.empty((1024, 1024), dtype=torch.float64, device=dev).t()
            d = {}
            for N in (14, 16, 18):
                for md in (ScaleMode.Fast, ScaleMode.Accurate):
                    ctx.gemm(Ap, Bp, EmuConfig(n_moduli=N, mode=md), Cp)
                    d[f"{md.name.lower()}{N}"] = Cp[r1][:, c1].cpu().numpy()
            d["native_fp64"] = torch.mm(Ap, Bp)[r1][:, c1].cpu().numpy()
            phi_acc[str(phi)] = d
            del Ap, Bp, Cp
        # rectangular m = n = 8192, k = 65536 (configs[4]) and n = 32768 (configs[3] per-GPU problem)
        del C
        torch.cuda.empty_cache()
        Ar = gen_device(8192, 65536, args.phi, 21, torch.float64, dev)
        Br = gen_device(65536, 8192, args.phi, 22, torch.float64, dev)
        Cr = torch.empty((8192, 8192), dtype=torch.float64, device=dev).t()
        r2, c2 = sample_idx(8192, 64, 11), sample_idx(8192, 64, 12)
        exact.submit("rect", Ar, Br, r2, c2)
        rect, racc = {}, {}
        for md in (ScaleMode.Fast, ScaleMode.Accurate):
            key = f"{md.name.lower()}{args.moduli}"
            rect[key] = timed(Ar, Br, EmuConfig(n_moduli=args.moduli, mode=md), Cr)
            racc[key] = Cr[r2][:, c2].cpu().numpy()
        racc["native_fp64"] = torch.mm(Ar, Br)[r2][:, c2].cpu().numpy()
        extra["rect_8192x8192x65536_tflops"] = rect
        del Ar, Br, Cr
        torch.cuda.empty_cache()
        if not os.environ.get("OZK_BENCH_NO_32K"):
            n2 = 32768
            A2 = gen_device(n2, n2, args.phi, 31, torch.float64, dev)
            B2 = gen_device(n2, n2, args.phi, 32, torch.float64, dev)
            C2 = torch.empty((n2, n2), dtype=torch.float64, device=dev).t()
            extra["dgemm_32768_tflops"] = {f"{md.name.lower()}{args.moduli}": timed(
                A2, B2, EmuConfig(n_moduli=args.moduli, mode=md), C2, reps=1)
                for md in (ScaleMode.Fast, ScaleMode.Accurate)}
            extra["native_fp64_32768_tflops"] = native_gemm_tflops(n2, torch.float64, 1)
            del A2, B2, C2
            torch.cuda.empty_cache()
        # errors (componentwise relative, the reference's compare()) per configuration
        errs = {"main": exact.errors("main", acc), "sgemm": exact.errors("sgemm", sacc),
                "rect": exact.errors("rect", racc)}
        extra["accuracy_exact"] = {
            "how": "max / median |c - r| / |r| over 64 x 64 sampled entries of C (full k) against the exact "
                   "product (reference oracle.cpp exact_gemm, GMP), phi=%g" % args.phi,
            "dgemm_16384": errs["main"], "sgemm_16384": errs["sgemm"], "rect_8192x8192x65536": errs["rect"]}
        extra["phi_sweep_exact_max_rel"] = {ph: {key: v[0] for key, v in exact.errors(f"phi{ph}", d).items()}
                                            for ph, d in phi_acc.items()}
        # the speed-up at matching accuracy: the fastest emulation whose max and
        # median errors are both no larger than native FP64's
        nat = errs["main"]["native_fp64"]
        ok = [(sweep[key], key) for key, e in errs["main"].items()
              if key in sweep and e[0] <= nat[0] and e[1] <= nat[1]]
        if ok:
            tf, key = max(ok)
            extra["at_native_fp64_accuracy"] = {
                "config": key, "tflops": tf, "max_rel": errs["main"][key][0], "median_rel": errs["main"][key][1],
                "native_max_rel": nat[0], "native_median_rel": nat[1],
                "native_fp64_tflops": extra["native_fp64_tflops"],
                "speedup_vs_native_fp64": tf / extra["native_fp64_tflops"]}
            out["tflops_at_native_fp64_accuracy"] = tf
        exact.close()
        out["extra"] = extra

    if world == 1 and not os.environ.get("OZK_BENCH_NO_CPU"):  # the CPU leg: rank 0 at N = 1 only
        cb = cpu_reference_sample(args.cpu_sample, k, args.moduli, 0 if args.mode == "fast" else 1, args.phi)
        out["cpu_baseline"] = {
            "value": cb["tflops"], "unit": "TFLOPS", "cores": cb["threads"], "kind": "reference",
            "sample": f"C block {args.cpu_sample}x{args.cpu_sample} of the {n}^3 problem (full k={k}), "
                      f"oracle/_ref gemm_emulated, {cb['runs']} runs, {cb['seconds_per_sample']:.2f} s each"}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def sample_idx(size, count, seed):
    """sorted sample of `count` indices of [0, size) including the first and the last"""
    import numpy as np

    rng = np.random.default_rng(seed)
    inner = rng.choice(np.arange(1, size - 1), count - 2, replace=False)
    return np.array(sorted(set(inner.tolist()) | {0, size - 1}))


class ExactPool:
    """the reference's exact GMP product of sampled rows x columns, computed on
    host threads while the GPU keeps timing (oracle/_ref; checker only)"""

    def __init__(self):
        from concurrent.futures import ThreadPoolExecutor

        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from _oracle import RefLib

        self.ref = RefLib() if RefLib.available() else None
        self.pool = ThreadPoolExecutor(4)
        self.jobs = {}

    def submit(self, name, A, B, rows, cols):
        import numpy as np
        import torch

        if self.ref is None:
            return
        a = np.asfortranarray(A[torch.from_numpy(rows).to(A.device)].cpu().numpy())
        b = np.asfortranarray(B[:, torch.from_numpy(cols).to(B.device)].cpu().numpy())
        prec = 1 if a.dtype == np.float32 else 0
        self.jobs[name] = self.pool.submit(self.ref.exact_rounded, a, b, prec)

    def errors(self, name, results):
        """{key: (max_rel, median_rel)} of each candidate block in `results`"""
        import numpy as np

        if name not in self.jobs:
            return {}
        from _oracle import RefLib

        ex = self.jobs[name].result()
        out = {}
        for key, c in results.items():
            e = RefLib.rel_errors(c, ex)
            out[key] = (float(e.max()), float(np.median(e)))
        return out

    def close(self):
        self.pool.shutdown()


def dropin_e2e(n, moduli, mode):
    """the reference-facing C++ API end to end: tools/dropin_bench (built against
    include/crtgemm and the product library) times crtgemm::gemm_emulated on
    Matrix<double> (std::vector storage) at n^3"""
    exe = os.path.join(ROOT, "paper_2508_03984_b200", "lib", "dropin_bench")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe, str(n), str(moduli), "0" if mode == "fast" else "1", "2"], capture_output=True,
                           text=True, timeout=600)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001  (reported, not fatal)
        return {"error": str(e)[:200]}


if __name__ == "__main__":
    main()

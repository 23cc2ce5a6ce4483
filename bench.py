#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for this repo.

Headline workload (BASELINE.json configs[3], the config the metric's
"1/2/4/8 B200" and the >=70%-of-FP64-peak target are quoted on): square fp64
GEMM C = A.B at N = 16384, A and B uniform [-1,1) from splitmix64 seeds 0/1,
resident in rank 0's HBM.  One step = one master/worker round (the
reference's master_run / worker_run, protocol.hpp:50-147; bracket first send
-> last receive, protocol.hpp:63,105):
  * 1 GPU: the round is one multiply (no communicator, no exchange);
  * N GPUs: row blocks of A by split_rows over the N ranks, B broadcast and A
    scattered over NCCL, each worker's C rows stored by its GEMM epilogue
    straight into rank 0's C over NVLink (CUDA IPC; NCCL C-slices if IPC is
    unavailable).  Total work is fixed as N grows ("strong" scaling).
Sub-objects of the same line: `fp32` (configs[4]: N=32768 normal(0,1), FFMA2
path, same round at N ranks), `sweep` (configs[1]: the paper's N=10..2000 on
one GPU), `exact_n4099` (configs[2]: integer inputs, sha256 against the
reference-generated golden), `e2e` (pinned host buffers) + `e2e_pageable`
(plain numpy arrays, what a std::vector-backed mmws::Matrix hands the
drop-in), `emulated_fp64` (opt-in int8-tensor-core emulation, 1 GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W]        # our arm
  python bench.py --impl reference [--steps K] [--warmup W]  # reference arm

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches
the N ranks itself (one process per GPU, RANK/LOCAL_RANK/WORLD_SIZE/
MASTER_ADDR=127.0.0.1) and relays rank 0's line; under torchrun it checks
WORLD_SIZE == --gpus.  --dry-run runs the launcher, the row-block message
plan over gloo and the line assembly on the CPU (no GPU, no multiply) -- a
test of the plumbing, not a measurement.

The reference arm times the reference's own CPU code (oracle/_ref: the
unmodified mmws headers compiled by oracle/Makefile; mmws::matmul_threads with
every host thread) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC_FALLBACK = "GFLOP/s (2N³/time) for N×N GEMM at 1/2/4/8 B200 vs FP64/FP32 peak"
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4
DATA = "synthetic: splitmix64 uniform[-1,1), seed 0 (A) / 1 (B), generated on the device"
SWEEP_NS = (10, 50, 100, 250, 500, 1000, 1500, 2000)


def metric_name() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return METRIC_FALLBACK


def workload_config(n: int, n_gpus: int, mode: str) -> dict:
    """The same dict for both arms (the arm label is the line's `impl`)."""
    if n_gpus == 1:
        what = (f"configs[3]: square fp64 GEMM N={n} on 1 GPU -- the master/worker round of a "
                "1-GPU world is one multiply (no exchange); A, B resident in HBM")
    else:
        what = (f"configs[3]: square fp64 GEMM N={n}, row-block master/worker over {n_gpus} GPUs: "
                "B broadcast + A row blocks scattered via NCCL, worker C rows stored by the GEMM "
                "epilogue into rank 0's C over NVLink (A, B resident on rank 0)")
    return {"workload": what, "n": n, "mode": mode, "parallelism": f"rowblock{n_gpus}",
            "l2": "no flush: inputs are 3 x 8N^2 = %.1f GB >> 126 MB L2" % (3 * 8 * n * n / 1e9)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_reference_sample(n: int, repeats: int = 1, serial: bool = False):
    """The reference's matmul_threads (all host threads) on a row sample of the
    N x N workload: C[0:r, :] = A[0:r, :] . B with r = #host threads (one row
    per worker, static_partition).  Bitwise the same rows the full product
    would give.  Returns dict(value GFLOP/s, seconds, cores, kind, sample), plus
    the serial matmul_seq on one row ("serial") when asked."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402  (test infrastructure: CPU baseline only)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    rows = cores
    b = O.fill(O.DIST_UNIFORM, 1, n, n, threads=cores)
    a = O.fill(O.DIST_UNIFORM, 0, rows, n, threads=cores)
    if O.ref_available():
        kind = "reference"
        best, _ = O.ref_time_matmul(a, b, cores, repeats=repeats)
    else:  # the C restatement, same loop order and threading
        kind = "port"
        t0 = time.perf_counter()
        O.matmul_threads(a, b, cores)
        best = time.perf_counter() - t0
    flops = 2.0 * rows * n * n
    out = {"value": flops / best / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": kind,
           "seconds": best,
           "sample": f"{rows} rows x {n} cols of C = A.B (N={n}, uniform seeds 0/1) via "
                     f"{'mmws::matmul_threads' if kind == 'reference' else 'oracle_matmul_threads'}"
                     f"({cores} workers), time_model bracket; full product extrapolated"}
    if serial:  # the serial path on one core: the first row of the same sample
        a1 = a[:1]
        if kind == "reference":
            t1, _ = O.ref_time_matmul(a1, b, 0, repeats=1)
        else:
            t0 = time.perf_counter()
            O.matmul_seq(a1, b)
            t1 = time.perf_counter() - t0
        out["serial"] = {
            "value": 2.0 * n * n / t1 / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": kind,
            "seconds": t1,
            "sample": f"1 row x {n} cols of C = A.B via "
                      f"{'mmws::matmul_seq' if kind == 'reference' else 'oracle_matmul_seq'}"}
    return out


def cpu_sweep(ns=(10, 50, 100, 250, 500, 1000)):
    """The reference's matmul_seq (1 core) and matmul_threads (all cores) over
    the paper's small sizes, full products (CPU-baseline leg only)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402
    if not O.ref_available():
        return None
    cores = len(os.sched_getaffinity(0))
    out = []
    for n in ns:
        a = O.fill(O.DIST_UNIFORM, 0, n, n)
        b = O.fill(O.DIST_UNIFORM, 1, n, n)
        reps = 3 if n <= 500 else 1
        ts, _ = O.ref_time_matmul(a, b, 0, repeats=reps)
        tt, _ = O.ref_time_matmul(a, b, cores, repeats=reps)
        out.append({"n": n, "seq_us": ts * 1e6, "threads_us": tt * 1e6, "threads_cores": cores,
                    "seq_gflops": 2 * n ** 3 / ts / 1e9, "threads_gflops": 2 * n ** 3 / tt / 1e9})
    return out


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times = []
    sample = None
    for step in range(args.warmup + args.steps):
        sample = cpu_reference_sample(args.n, serial=step == args.warmup + args.steps - 1)
        if step >= args.warmup:
            times.append(sample["seconds"])
    rows = sample["cores"]
    flops = 2.0 * rows * args.n * args.n
    value = flops * len(times) / sum(times) / 1e9
    line = {
        "impl": "reference", "metric": metric_name(), "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA.replace(
            "generated on the device", "generated on the host"),
        "config": workload_config(args.n, args.gpus, args.mode),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": sample["cores"],
                         "kind": sample["kind"], "sample": sample["sample"],
                         "serial": sample["serial"]},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], 0.0, set()
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) < 8:
                    continue
                try:
                    sm.append(float(p[0]))
                    mx = max(mx, float(p[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, p[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def measured_hbm_gbs() -> float:
    """HBM copy bandwidth of this pool (MEASURED_PEAKS.json, driver-written),
    else the profiling recipe's fallback (6.65 TB/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def profiled_traffic(n: int, rows: int, plan: str, dtype: str = "f64"):
    """dram bytes per launch of the dominant kernel from the committed ncu
    captures (profiles/*_ncu_summary*.json) for this N, this rank's row count
    and kernel configuration (ctx.last_plan)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_summary*.json")), reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
            for k in d.get("kernels", []):
                if (k.get("n") == n and k.get("role") == "dominant" and k.get("plan") == plan
                        and k.get("rows", n) == rows and k.get("dtype", "f64") == dtype):
                    return k.get("dram_bytes"), os.path.relpath(p, ROOT)
        except Exception:
            continue
    return None, None


def golden(key: str):
    with open(os.path.join(ROOT, "tests", "golden", "ref_big.json")) as f:
        return json.load(f)[key]


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ----------------------------------------------------------------------------- launcher
def launch_ranks(args) -> int:
    """One process per GPU (the driver may call plain `python bench.py --gpus N`):
    children get RANK/LOCAL_RANK/WORLD_SIZE/MASTER_ADDR/MASTER_PORT; rank 0's
    stdout is relayed; any failing rank fails the run, and -- like the
    reference's ProcessGroup (launch.hpp:73,113-127) -- the first rank to fail
    takes the others down instead of leaving them blocked on their peers."""
    port = str(free_port())
    out = tempfile.TemporaryFile()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=out if r == 0 else sys.stderr.fileno()))
    failed = None
    while True:
        states = [p.poll() for p in procs]  # every rank, every time (no short-circuit)
        if all(st is not None for st in states):
            break
        bad = [r for r, st in enumerate(states) if st not in (None, 0)]
        if bad and failed is None:
            failed = bad
            for p in procs:
                if p.poll() is None:
                    p.terminate()
            deadline = time.time() + 15
            while any(p.poll() is None for p in procs) and time.time() < deadline:
                time.sleep(0.1)
            for p in procs:
                if p.poll() is None:
                    p.kill()
        time.sleep(0.05)
    codes = [p.wait() for p in procs]
    out.seek(0)
    sys.stdout.write(out.read().decode())
    sys.stdout.flush()
    bad = [(r, c) for r, c in enumerate(codes) if c != 0]
    if bad:
        sys.stderr.write(f"bench.py: rank(s) failed: {bad}" +
                         (f" (first: {failed})" if failed else "") + "\n")
        return 1
    return 0


def world_from_env(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    return rank, world, local


# ----------------------------------------------------------------------------- dry run (CPU)
def run_dry(args) -> None:
    """The launcher, the max-over-ranks timing and the line, on the CPU: the
    row-block message plan (the product library's mmws_gpu_rowblock_plan)
    replayed over gloo with zero payloads and no multiply."""
    import torch
    import torch.distributed as dist

    import paper_1012_2273_b200 as P
    rank, world, _ = world_from_env(args)
    if os.environ.get("MMWS_BENCH_DRY_FAIL_RANK") == str(rank):  # launcher test: this rank dies
        sys.exit(3)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = args.n
    plan = P.rowblock_plan(n, n, n, world)
    off, rows = P.split_rows(n, world)[rank]

    def step():
        b = torch.zeros((n, n), dtype=torch.float64)
        for e in plan:
            if e["dir"] == "broadcast":
                dist.broadcast(b, 0)
            elif rank == 0:
                buf = torch.zeros(e["count"], dtype=torch.float64)
                (dist.send if e["dir"] == "sent" else dist.recv)(buf, e["peer"])
            elif e["peer"] == rank:
                buf = torch.zeros(e["count"], dtype=torch.float64)
                (dist.recv if e["dir"] == "sent" else dist.send)(buf, 0)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dist.barrier()
    ms = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([ms], dtype=torch.float64)
    per_rank = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(per_rank, t)
    ms_max = max(float(x[0]) for x in per_rank)
    if rank == 0:
        line = {
            "metric": metric_name(), "value": 2.0 * n ** 3 * args.steps / (ms_max / 1e3) / 1e9,
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "none: dry run (zero payloads)",
            "config": workload_config(n, world, args.mode), "dry_run": True,
            "per_rank_ms": [float(x[0]) for x in per_rank],
            "messages_rank0": len(plan), "rows_rank0": rows,
            "note": "launcher + gloo replay of the row-block message plan, no multiply: "
                    "a plumbing test, not a measurement",
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1012_2273_b200 as P

    rank, world, local = world_from_env(args)
    # MMWS_BENCH_ONE_GPU_WORLD=1 (tests only): every rank on GPU 0, gloo for
    # the plumbing, with MMWS_GPU_NCCL_LIB naming tests/fake_nccl -- runs the
    # N>1 code path of this file on one GPU; its times are not measurements
    one_gpu = os.environ.get("MMWS_BENCH_ONE_GPU_WORLD") == "1" and world > 1
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = P.Context(local)
    if world > 1:
        P.bootstrap_comm(ctx)
    mode = {"auto": P.MODE_AUTO, "dmma": P.MODE_DMMA, "exact": P.MODE_EXACT,
            "ozaki": P.MODE_OZAKI}[args.mode]
    n = args.n
    root = rank == 0
    flops = 2.0 * n ** 3

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def gather_all(values):
        """[per-rank list of `values`] on every rank."""
        t = torch.tensor(values, dtype=torch.float64, device="cpu" if one_gpu else "cuda")
        if world == 1:
            return [values]
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [o.tolist() for o in out]

    ext = torch.cuda.ExternalStream(ctx.stream)

    def timed_rounds(fn, steps):
        """Device time of `steps` rounds on this rank's stream (ms) and the
        per-round kernel times, bracketed by barrier + synchronize."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(ext)
        kern = []
        for _ in range(steps):
            fn()
            kern.append(ctx.last_kernel_ms)
        e1.record(ext)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1), kern

    # ------------------------------------------------------------ headline: configs[3]
    A = B = C = None
    if root:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
    torch.cuda.synchronize()
    dmma_peak = max(ctx.peak_probe(P.PROBE_DMMA, 20000) for _ in range(3))  # live roofline denominator

    def round64():
        ctx.rowblock(n, n, n, A, B, C, mode=mode)

    barrier()
    for _ in range(args.warmup):
        round64()
    barrier()
    sampler = ClockSampler(local) if root else None
    if sampler:
        sampler.start()
    l0 = ctx.launches
    ms, kern_ms = timed_rounds(round64, args.steps)
    launches = ctx.launches - l0
    clocks = sampler.stop() if sampler else None
    plan = ctx.last_plan
    active, gather = ctx.last_round
    b_panels = ctx.last_b_panels
    per_rank = gather_all([ms, float(launches), sum(kern_ms) / len(kern_ms)])
    ms_max = max(r[0] for r in per_rank)
    launches_total = int(sum(r[1] for r in per_rank))
    value = flops * args.steps / (ms_max / 1e3) / 1e9
    rows0 = P.split_rows(n, active)[0][1]
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    achieved = 2.0 * rows0 * n * n / (kern_avg_ms / 1e3) / 1e12
    traffic, traffic_src = profiled_traffic(n, rows0, plan)

    # ------------------------------------------------------------ link calibration (f3)
    link = None
    if world > 1:
        bcast = ctx.link_probe(1 << 28, 5)
        p2p = ctx.p2p_probe(1 << 28, 5)
        rates = gather_all([bcast, p2p])
        per_gpu_rate = 2.0 * rows0 * n * n / (kern_avg_ms / 1e3)
        t_pred = P.rowblock_cost(n, n, n, world, 8, min(bcast, p2p), per_gpu_rate)[0]
        link = {"broadcast_GBps": bcast / 1e9, "p2p_GBps": p2p / 1e9,
                "p2p_GBps_per_rank": [r[1] / 1e9 for r in rates],
                "source": "mmws_gpu_link_probe (5 x 256 MiB NCCL broadcasts from rank 0) and "
                          "mmws_gpu_p2p_probe (5 x 256 MiB rank 0 -> each worker)",
                "predicted_ms_per_step": t_pred * 1e3, "measured_ms_per_step": ms_max / args.steps,
                "model": "mmws_gpu_rowblock_cost at the measured link (min of the two) and this "
                         "run's per-GPU kernel rate"}

    # ------------------------------------------------------------ e2e through the host entry
    # master_run with host matrices (the call a user makes): H2D of A and B,
    # the round, D2H of C inside the bracket; rank 0's host wall clock.
    e2e_steps = max(2, min(args.steps, 3))
    a_pin = b_pin = c_pin = a_np = b_np = None
    if root:
        a_np = A.cpu().numpy()            # plain (pageable) numpy, as a std::vector hands it
        b_np = B.cpu().numpy()
        a_pin = torch.from_numpy(a_np).pin_memory().numpy()
        b_pin = torch.from_numpy(b_np).pin_memory().numpy()
        c_pin = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()

    def host_round(a, b, c):
        if root:
            ctx.master_run_host(a, b, c, mode=mode)
        else:
            ctx.master_run_host(None, None, None, mode=mode, m=n, n=n, k=n)

    def e2e_wall(a, b, c, steps):
        # workers wait for rank 0's host-side preparation here (torch's own
        # collective timeout), not inside the round's 30 s deadline
        barrier()
        host_round(a, b, c)  # warm-up (staging buffers, IPC mappings)
        barrier()
        walls = []
        for _ in range(steps):
            t0 = time.perf_counter()
            host_round(a, b, c)
            walls.append(time.perf_counter() - t0)
        barrier()
        return max(r[0] for r in gather_all([sum(walls) / len(walls)]))

    e2e_s = e2e_wall(a_pin, b_pin, c_pin, e2e_steps)
    del c_pin
    c_np = np.empty((n, n)) if root else None
    e2e_pg_s = e2e_wall(a_np, b_np, c_np, 2)
    bytes_in, bytes_out = 2 * 8 * n * n, 8 * n * n
    e2e = {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": bytes_in,
           "d2h_bytes_per_step": bytes_out, "seconds_per_step": e2e_s,
           "entry": "mmws_gpu_master_run_host (C ABI), pinned host A/B/C, rank 0 host wall clock "
                    "(perf_counter) per call, max over ranks"}
    e2e_pageable = {"value": flops / e2e_pg_s / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": bytes_in, "d2h_bytes_per_step": bytes_out,
                    "seconds_per_step": e2e_pg_s,
                    "entry": "mmws_gpu_master_run_host with plain (pageable) numpy arrays -- what "
                             "a std::vector-backed mmws::Matrix hands the drop-in; host wall clock"}
    if root:
        del a_pin, b_pin, c_np
        del A, B, C
    torch.cuda.empty_cache()
    barrier()

    # ------------------------------------------------------------ emulated fp64 (opt-in mode, 1 GPU)
    emulated = None
    if root and world == 1 and not args.no_emulated and not args.quick:
        emulated = measure_emulated(ctx, P, torch, n, args, local, a_np, b_np, flops)
    barrier()

    # ------------------------------------------------------------ fp32: configs[4]
    fp32 = None
    if not args.no_fp32:
        fp32 = measure_fp32(ctx, P, torch, dist, args, rank, world, local, barrier, gather_all,
                            timed_rounds)
    barrier()

    # ------------------------------------------------------------ paper sweep + exactness (rank 0)
    sweep = exact = None
    if root and not args.quick:
        sweep = measure_sweep(ctx, P, torch, np)
        exact = measure_exact(ctx, P, torch)
    barrier()

    # ------------------------------------------------------------ CPU baseline (rank 0, every N)
    cpu = None
    if root and not args.no_cpu_baseline:
        s = cpu_reference_sample(n, serial=True)
        cpu = {k: s[k] for k in ("value", "unit", "cores", "kind", "sample", "serial")}
        if not args.quick:
            cpu["sweep"] = cpu_sweep()
        cpu["fp32_note"] = "the reference has no fp32 path (its Matrix is fp64 only)"
    barrier()

    if root:
        line = {
            "metric": metric_name(), "value": value, "unit": "GFLOP/s", "n_gpus": world,
            **({"plumbing_test": "MMWS_BENCH_ONE_GPU_WORLD: every rank on one GPU with the "
                                 "loopback NCCL stand-in -- a code-path test, not a "
                                 "measurement"} if one_gpu else {}),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "config": workload_config(n, world, args.mode),
            "per_rank_ms_per_step": [r[0] / args.steps for r in per_rank],
            "per_rank_kernel_ms": [r[2] for r in per_rank],
            "round": {"active_ranks": active, "gather": gather, "b_panels": b_panels,
                      "rows_rank0": rows0, "plan_rank0": plan},
            "roofline": {
                "bound": "tensor", "achieved": achieved, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": achieved / dmma_peak, "traffic": traffic,
                "kernel": plan + " (DMMA.8x8x4)",
                "peak_source": "measured live in this run: DMMA.8x8x4 throughput probe "
                               "(FP64 tensor pipe; MEASURED_PEAKS.json has no fp64 figure)",
                "peak_nominal": NOMINAL_FP64_TFLOPS, "frac_of_nominal": achieved / NOMINAL_FP64_TFLOPS,
                "flops_per_launch": 2.0 * rows0 * n * n, "kernel_ms_avg": kern_avg_ms,
                "kernel_scope": "rank 0's multiply (all its sub-block launches) per round",
                "traffic_source": traffic_src,
                "traffic_note": (None if traffic is None else
                                 "ncu dram bytes per round of rank 0's multiply vs %.2f GB "
                                 "algorithmic: A/B panels are re-streamed per wave of tiles "
                                 "(they exceed the 126 MB L2); %.1f%% of HBM bandwidth over "
                                 "the kernel, the FP64 tensor pipe is the bound"
                                 % (8.0 * (2 * rows0 * n + n * n) / 1e9,
                                    100.0 * traffic / (kern_avg_ms / 1e3) / 1e9
                                    / measured_hbm_gbs())),
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            "gpu_launches": launches_total,
            "link": link,
            "fp32": fp32,
            "sweep": sweep,
            "exact_n4099": exact,
            "emulated_fp64": emulated,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def measure_emulated(ctx, P, torch, n, args, local, a_np, b_np, flops):
    """The same multiply emulated on the int8 tensor cores (MODE_OZAKI,
    opt-in; the headline stays on the FP64 tensor path): device-resident,
    CUDA events, plus its normwise difference from the DMMA product."""
    A = torch.from_numpy(a_np).cuda()
    B = torch.from_numpy(b_np).cuda()
    C = ctx.dgemm(A, B, mode=P.MODE_AUTO)
    C_oz = torch.empty_like(C)
    ctx.dgemm(A, B, C_oz, mode=P.MODE_OZAKI)
    torch.cuda.synchronize()
    oz_steps = max(3, min(args.steps, 5))
    sampler = ClockSampler(local)
    sampler.start()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(oz_steps):
        ctx.dgemm(A, B, C_oz, mode=P.MODE_OZAKI)
    f1.record()
    torch.cuda.synchronize()
    oz_clocks = sampler.stop()
    oz_ms = f0.elapsed_time(f1) / oz_steps
    diff = float(torch.linalg.norm(C_oz - C) / torch.linalg.norm(C))
    moduli, bits = P.ozaki_plan(n)
    del A, B, C, C_oz
    torch.cuda.empty_cache()
    a_pin = torch.from_numpy(a_np).pin_memory().numpy()
    b_pin = torch.from_numpy(b_np).pin_memory().numpy()
    c_pin = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
    ctx.master_run_host(a_pin, b_pin, c_pin, mode=P.MODE_OZAKI)
    walls = []
    for _ in range(2):
        t0 = time.perf_counter()
        ctx.master_run_host(a_pin, b_pin, c_pin, mode=P.MODE_OZAKI)
        walls.append(time.perf_counter() - t0)
    oz_s = sum(walls) / len(walls)
    return {
        "mode": f"ozaki (fp64 emulated exactly on int8 tcgen05 tensor cores, CRT over {moduli} "
                f"moduli, {bits}-bit scaling)",
        "value": flops / (oz_ms / 1e3) / 1e9, "unit": "GFLOP/s", "ms_per_step": oz_ms,
        "steps": oz_steps, "int8_gemms": moduli,
        "int8_tops_equivalent": moduli * flops / (oz_ms / 1e3) / 1e12,
        "int8_tensor_peak_nominal_tops": 4500.0,
        "normwise_diff_vs_dmma": diff, "clocks": oz_clocks,
        "note": "opt-in MMWS_GPU_MODE_OZAKI; error ~1e-14 vs the fp64 oracle (tests), "
                "integer inputs bit-exact",
        "e2e": {"value": flops / oz_s / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": 2 * 8 * n * n, "d2h_bytes_per_step": 8 * n * n,
                "seconds_per_step": oz_s,
                "entry": "mmws_gpu_master_run_host (C ABI, pinned host A/B/C), MODE_OZAKI, "
                         "host wall clock"},
    }


def measure_fp32(ctx, P, torch, dist, args, rank, world, local, barrier, gather_all, timed_rounds):
    """configs[4]: fp32 N=32768, normal(0,1) seeds 0/1, FFMA2 path, the same
    row-block round over all ranks; roofline against the live FFMA2 probe;
    normwise error of sampled rows against an fp64 product of the widened
    inputs (torch fp64 on the GPU as the checker, not measured)."""
    n = args.n32
    root = rank == 0
    A = B = C = None
    if root:
        A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
        B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
        C = torch.empty_like(A)
    torch.cuda.synchronize()
    ffma2_peak = max(ctx.peak_probe(P.PROBE_FFMA2, 100000) for _ in range(3))
    # the outer-product operand pattern in registers (one fresh register
    # operand per FFMA2): one register-only loop of it, not a ceiling -- the
    # rate depends on where ptxas puts the operands
    pattern_peak = max(ctx.peak_probe(P.PROBE_FFMA2_OUTER, 20000) for _ in range(3))

    def round32():
        ctx.rowblock(n, n, n, A, B, C, mode=P.MODE_FFMA, f32=True)

    barrier()
    round32()  # warm-up
    sampler = ClockSampler(local) if root else None
    if sampler:
        sampler.start()
    steps = args.steps32
    ms, kern = timed_rounds(round32, steps)
    clocks = sampler.stop() if sampler else None
    plan = ctx.last_plan
    active, gather = ctx.last_round
    per_rank = gather_all([ms, sum(kern) / len(kern)])
    ms_max = max(r[0] for r in per_rank)
    rows0 = P.split_rows(n, active)[0][1]
    kern_ms = sum(kern) / len(kern)
    achieved = 2.0 * rows0 * n * n / (kern_ms / 1e3) / 1e12
    traffic, traffic_src = profiled_traffic(n, rows0, plan, "f32")

    # e2e through the host entry, as for the headline: master_run with pinned
    # host fp32 matrices (H2D of A and B, the round, D2H of C inside the
    # bracket), rank 0's host wall clock, max over ranks
    e2e = None
    if not args.quick:
        hA = hB = hC = None
        if root:
            hA = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
            hB = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
            hC = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
            hA.copy_(A)
            hB.copy_(B)
            hA, hB, hC = hA.numpy(), hB.numpy(), hC.numpy()

        def host_round32():
            if root:
                ctx.master_run_host(hA, hB, hC, mode=P.MODE_FFMA)
            else:
                ctx.master_run_host(None, None, None, mode=P.MODE_FFMA, m=n, n=n, k=n, f32=True)

        barrier()  # rank 0 pinned 3 x 4 GiB meanwhile: outside the round's deadline
        host_round32()  # warm-up
        barrier()
        walls = []
        for _ in range(2):
            t0 = time.perf_counter()
            host_round32()
            walls.append(time.perf_counter() - t0)
        barrier()
        e2e_s = max(r[0] for r in gather_all([sum(walls) / len(walls)]))
        same = None
        if root:  # the host entry's C is the device round's C, bitwise
            same = bool(torch.equal(torch.from_numpy(hC).view(torch.int32),
                                    C.cpu().view(torch.int32)))
        e2e = {"value": 2.0 * n ** 3 / e2e_s / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": 2 * 4 * n * n, "d2h_bytes_per_step": 4 * n * n,
               "seconds_per_step": e2e_s, "bitwise_equal_device_round": same,
               "entry": "mmws_gpu_master_run_host_f32 (C ABI), pinned host A/B/C, MODE_FFMA, "
                        "rank 0 host wall clock (perf_counter) per call, max over ranks"}
        del hA, hB, hC
    out = None
    if root:
        rows = sorted({0, 1, n // 3, n // 2, (2 * n) // 3, n - 2, n - 1, 12345 % n})
        idx = torch.tensor(rows, device=A.device)
        ref = A.index_select(0, idx).double() @ B.double()
        got = C.index_select(0, idx).double()
        err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
        flops = 2.0 * n ** 3
        out = {
            "workload": f"configs[4]: square fp32 GEMM N={n}, normal(0,1) seeds 0/1 (device "
                        f"Box-Muller), FFMA2 path, row-block round over {world} GPU(s)",
            "value": flops * steps / (ms_max / 1e3) / 1e9, "unit": "GFLOP/s", "steps": steps,
            "warmup": 1, "ms_per_step": ms_max / steps, "dtype": "f32",
            "per_rank_ms_per_step": [r[0] / steps for r in per_rank],
            "round": {"active_ranks": active, "gather": gather, "rows_rank0": rows0,
                      "b_panels": ctx.last_b_panels, "plan_rank0": plan},
            "roofline": {"bound": "fp32 pipe (FFMA2)", "achieved": achieved, "peak": ffma2_peak,
                         "unit": "TFLOP/s", "frac": achieved / ffma2_peak, "traffic": traffic,
                         "traffic_source": traffic_src, "kernel_ms_avg": kern_ms,
                         "flops_per_launch": 2.0 * rows0 * n * n,
                         "peak_source": "measured live in this run: FFMA2 (fma.rn.f32x2) "
                                        "throughput probe",
                         "peak_nominal": NOMINAL_FP32_TFLOPS,
                         "pattern_probe": pattern_peak,
                         "pattern_note": "register-only FFMA2 outer-product loop at the kernel's "
                                         "shape (8 warps/SM, 64 pairs per lane, one fresh "
                                         "broadcast operand per instruction): "
                                         "mmws_gpu_peak_probe(FFMA2_OUTER); not a ceiling -- "
                                         "such loops measure 62-71 TFLOP/s depending on the "
                                         "register assignment (profiles/r02_ffma2_shape_probe.txt)"
                                         ", and the kernel with A staged k-major beats this one",
                         "transpose_pass": "A is transposed once per launch (HBM-bound, 0.17% of "
                                           "the multiply at N=32768) inside the timed region"},
            "accuracy": {"normwise_rel_error": err, "bound": 1e-5, "ok": err <= 1e-5,
                         "rows": rows,
                         "reference": "fp64 product of the widened fp32 rows (torch fp64 on the "
                                      "GPU, checker only); tests pin the same rows against the "
                                      "CPU oracle"},
            "clocks": clocks,
            "e2e": e2e,
        }
    del A, B, C
    torch.cuda.empty_cache()
    return out


def measure_sweep(ctx, P, torch, np):
    """configs[1]: the paper's sweep N=10..2000, fp64 AUTO (small-N latency
    path / small-tile DMMA), one GPU.  Per N: device time per multiply with
    the launch queue kept full, CUDA-graph replay device time, the host wall
    time of one eager launch + synchronize and of one graph launch +
    synchronize, and the host-buffer entry (pageable numpy in/out, the call a
    user makes); GFLOP/s and achieved HBM GB/s on the algorithmic 3 x 8N^2
    bytes."""
    s = torch.cuda.current_stream()
    hbm = measured_hbm_gbs()

    def dev_time(fn, reps, inner):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(int(inner * 40e-6 * 2e9))  # keeps host submission off the clock
            e0.record(s)
            for _ in range(inner):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3 / inner)
        return best

    def wall(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts), statistics.median(ts)

    out = []
    for n in SWEEP_NS:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
        reps = 20 if n <= 500 else 8
        inner = 20 if n <= 1000 else 3
        t = dev_time(lambda: ctx.dgemm(A, B, C), reps, inner)
        # EXACT (bitwise matmul_seq): what the C++ drop-in's matmul_seq /
        # matmul_threads / master_run run by default
        plan = ctx.last_plan
        tx = dev_time(lambda: ctx.dgemm(A, B, C, mode=P.MODE_EXACT), reps, inner)
        plan_x = ctx.last_plan
        g = ctx.graph_dgemm(A, B, C)
        tg = dev_time(lambda: g.launch(), reps, inner)
        tw, tw_med = wall(lambda: ctx.dgemm(A, B, C), reps)
        tgw, tgw_med = wall(lambda: g.launch(), reps)
        g.close()
        a, b = A.cpu().numpy(), B.cpu().numpy()
        c = np.empty_like(a)
        for _ in range(5):
            ctx.matmul_host(a, b, out=c)
        th = []
        for _ in range(reps if n > 500 else 60):
            t0 = time.perf_counter()
            ctx.matmul_host(a, b, out=c)
            th.append(time.perf_counter() - t0)
        flops = 2.0 * n ** 3
        byt = 3 * 8.0 * n * n
        out.append({"n": n, "plan": plan,
                    "device_us": t * 1e6, "graph_device_us": tg * 1e6,
                    "exact_plan": plan_x, "exact_device_us": tx * 1e6,
                    "gflops_exact_device": 2.0 * n ** 3 / tx / 1e9,
                    "launch_wall_us": tw * 1e6, "graph_wall_us": tgw * 1e6,
                    "graph_wall_median_us": tgw_med * 1e6,
                    "host_entry_wall_us": min(th) * 1e6,
                    "host_entry_wall_median_us": statistics.median(th) * 1e6,
                    "gflops_device": flops / t / 1e9, "gflops_graph_wall": flops / tgw / 1e9,
                    "gflops_host_entry": flops / min(th) / 1e9,
                    "hbm_GBps_device": byt / t / 1e9, "hbm_frac": byt / t / 1e9 / hbm})
        del A, B, C
    # the resident latency server (N <= 96): host-buffer calls without a
    # launch or a copy engine (mmws_gpu_server_dgemm); it holds SMs, so it
    # runs last and is stopped again
    torch.cuda.synchronize()
    ctx.server_start()
    try:
        for rec in out:
            n = rec["n"]
            if n > 96:
                continue
            a = np.random.default_rng(n).uniform(-1, 1, (n, n))
            b = np.random.default_rng(n + 1).uniform(-1, 1, (n, n))
            c = np.empty_like(a)
            for _ in range(50):
                ctx.server_matmul(a, b, out=c)
            ts = []
            for _ in range(500):
                t0 = time.perf_counter()
                ctx.server_matmul(a, b, out=c)
                ts.append(time.perf_counter() - t0)
            rec["server_wall_us"] = min(ts) * 1e6
            rec["server_wall_median_us"] = statistics.median(ts) * 1e6
    finally:
        ctx.server_stop()
    return out


def measure_exact(ctx, P, torch):
    """configs[2]: N=4099 (non-tile-aligned), integer inputs in [-8,8] seeds
    0/1: AUTO (DMMA, packed operands) and EXACT, device time per call and the
    sha256 of C against the golden produced by the reference's own
    matmul_threads (tests/golden/ref_big.json)."""
    n = 4099
    A = ctx.fill(P.DIST_INT8, 0, n, n)
    B = ctx.fill(P.DIST_INT8, 1, n, n)
    C = torch.empty_like(A)
    want = golden("n4099_int8_sha256")
    out = {"n": n, "inputs": "integers in [-8,8] (splitmix64 seeds 0/1) stored as fp64",
           "golden": "sha256 of the reference matmul_threads product (tests/golden/ref_big.json)"}
    for name, mode in (("auto", P.MODE_AUTO), ("exact", P.MODE_EXACT)):
        ctx.dgemm(A, B, C, mode=mode)
        torch.cuda.synchronize()
        sha = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            ctx.dgemm(A, B, C, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        out[name] = {"ms": t * 1e3, "gflops": 2.0 * n ** 3 / t / 1e9, "plan": ctx.last_plan,
                     "sha256": sha, "bitwise_equal_golden": sha == want}
    del A, B, C
    torch.cuda.empty_cache()
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--n32", type=int, default=32768, help="fp32 sub-object size (configs[4])")
    ap.add_argument("--steps32", type=int, default=3)
    ap.add_argument("--mode", choices=["auto", "dmma", "exact", "ozaki"], default="auto")
    ap.add_argument("--no-emulated", action="store_true",
                    help="skip the MODE_OZAKI measurement added to the JSON line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="headline, e2e, fp32 and the CPU sample only (no sweep / exactness / emulation)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: launcher + gloo replay of the message plan, no GPU")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1 or args.gpus < 1:
        sys.exit("steps must be >= 1, warmup >= 0, gpus >= 1")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.dry_run:
        run_dry(args)
        return
    try:
        run_ours(args)
    except Exception as exc:  # a failed run still leaves a line saying why
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": metric_name(), "value": None, "unit": "GFLOP/s",
                              "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                              "error": f"{type(exc).__name__}: {exc}"}), flush=True)
        raise


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for this repo.

Workload (BASELINE.json configs[3], the config the metric's "1/2/4/8 B200" and
the >=70%-of-FP64-peak target are quoted on): square fp64 GEMM C = A.B at
N = 16384, A and B uniform [-1,1) from splitmix64 seeds 0/1, row-block
(master/worker) partition of A over the n_gpus ranks, B broadcast and A
scattered over NCCL, each worker's C rows stored by its GEMM epilogue straight
into rank 0's C over NVLink (CUDA IPC) -- the reference's master_run / worker_run
(protocol.hpp:50-147) on B200s.  One step = one master/worker round with A, B
resident in rank 0's HBM (first send -> last receive, protocol.hpp:63,105).
Total work is fixed as n_gpus grows ("strong" scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W]            # our arm
  python bench.py --impl reference [--steps K] [--warmup W]      # reference arm

The reference arm times the reference's own CPU code (oracle/_ref: the
unmodified mmws headers compiled by oracle/Makefile; mmws::matmul_threads with
every host thread) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC_FALLBACK = "GFLOP/s (2N³/time) for N×N GEMM at 1/2/4/8 B200 vs FP64/FP32 peak"
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz
DATA = "synthetic: splitmix64 uniform[-1,1), seed 0 (A) / 1 (B), generated on the device"


def metric_name() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return METRIC_FALLBACK


def workload_config(n: int, n_gpus: int, mode: str) -> dict:
    return {
        "workload": f"configs[3]: square fp64 GEMM N={n}, row-block master/worker over {n_gpus} GPU(s), "
                    "B broadcast + A scatter via NCCL, C rows stored by the GEMM epilogue into rank 0 "
                    "over NVLink (A,B resident on rank 0)",
        "n": n, "mode": mode, "parallelism": f"rowblock{n_gpus}",
        "l2": "no flush: inputs are 3 x 8N^2 = %.1f GB >> 126 MB L2" % (3 * 8 * n * n / 1e9),
    }


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
                     f"({cores} workers), time_model bracket"}
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
        "config": workload_config(args.n, args.gpus, "reference-cpu"),
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


# ----------------------------------------------------------------------------- our arm
def measured_hbm_gbs() -> float:
    """HBM copy bandwidth of this pool (MEASURED_PEAKS.json, driver-written),
    else the profiling recipe's fallback (6.65 TB/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def profiled_traffic(n: int, plan: str):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/*_ncu_summary*.json), if one matches this N and kernel
    configuration (ctx.last_plan)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_summary*.json")), reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
            for k in d.get("kernels", []):
                if k.get("n") == n and k.get("role") == "dominant" and k.get("plan") == plan:
                    return k.get("dram_bytes"), os.path.relpath(p, ROOT)
        except Exception:
            continue
    return None, None


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1012_2273_b200 as P

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = P.Context(local)
    if world > 1:
        P.bootstrap_comm(ctx)
    mode = {"auto": P.MODE_AUTO, "dmma": P.MODE_DMMA, "exact": P.MODE_EXACT,
            "ozaki": P.MODE_OZAKI}[args.mode]
    n = args.n
    root = rank == 0

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    A = B = C = None
    if root:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
    torch.cuda.synchronize()

    # live FP64 tensor-pipe peak (roofline denominator), same box, same run
    dmma_peak = max(ctx.peak_probe(P.PROBE_DMMA, 20000) for _ in range(3))

    for _ in range(args.warmup):
        ctx.rowblock(n, n, n, A, B, C, mode=mode)
    barrier()
    # cost-model calibration: NCCL broadcast bandwidth out of rank 0 (collective)
    link_bw = ctx.link_probe(1 << 28, 5) if world > 1 else None
    barrier()

    sampler = ClockSampler(local) if root else None
    if sampler:
        sampler.start()
    ext = torch.cuda.ExternalStream(ctx.stream)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    l0 = ctx.launches
    e0.record(ext)
    kern_ms = []
    for _ in range(args.steps):
        ctx.rowblock(n, n, n, A, B, C, mode=mode)
        kern_ms.append(ctx.last_kernel_ms)
    plan = ctx.last_plan
    e1.record(ext)
    torch.cuda.synchronize()
    launches = ctx.launches - l0
    barrier()
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms, float(launches)], dtype=torch.float64, device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms, launches_total = float(tmax[0]), int(t[1])
    else:
        launches_total = launches
    ms_per_step = ms / args.steps
    flops = 2.0 * n ** 3
    value = flops * args.steps / (ms / 1e3) / 1e9

    # dominant kernel roofline (rank 0's DMMA launch; events on its stream)
    active = P.rowblock_ranks(n, n, n, world)  # = world at this size
    rows0 = P.split_rows(n, active)[0][1]
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    achieved = 2.0 * rows0 * n * n / (kern_avg_ms / 1e3) / 1e12
    traffic, traffic_src = profiled_traffic(n, plan) if world == 1 else (None, None)

    # The same multiply emulated on the int8 tensor cores (MODE_OZAKI, opt-in;
    # the headline above stays on the FP64 tensor path): device-resident, CUDA
    # events, plus its normwise difference from the DMMA product of this run.
    emulated = None
    if root and world == 1 and not args.no_emulated:
        C_oz = torch.empty_like(C)
        ctx.dgemm(A, B, C_oz, mode=P.MODE_OZAKI)
        torch.cuda.synchronize()
        oz_steps = max(3, min(args.steps, 5))
        oz_sampler = ClockSampler(local)
        oz_sampler.start()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(oz_steps):
            ctx.dgemm(A, B, C_oz, mode=P.MODE_OZAKI)
        f1.record()
        torch.cuda.synchronize()
        oz_clocks = oz_sampler.stop()
        oz_ms = f0.elapsed_time(f1) / oz_steps
        diff = float(torch.linalg.norm(C_oz - C) / torch.linalg.norm(C))
        moduli, _bits = P.ozaki_plan(n)
        emulated = {
            "mode": f"ozaki (fp64 emulated exactly on int8 tcgen05 tensor cores, CRT over {moduli} moduli, {_bits}-bit scaling)",
            "value": flops / (oz_ms / 1e3) / 1e9, "unit": "GFLOP/s", "ms_per_step": oz_ms,
            "steps": oz_steps, "int8_gemms": moduli,
            "int8_tops_equivalent": moduli * flops / (oz_ms / 1e3) / 1e12,
            "int8_tensor_peak_nominal_tops": 4500.0,
            "normwise_diff_vs_dmma": diff,
            "clocks": oz_clocks,
            "note": "opt-in MMWS_GPU_MODE_OZAKI; error ~1e-14 vs the fp64 oracle (tests), "
                    "integer inputs bit-exact",
        }
        del C_oz

    # e2e: the public host-buffer entry (master_run with host matrices): H2D of
    # A and B, the round, D2H of C inside the bracket, pinned host buffers.
    e2e_steps = max(2, min(args.steps, 4))
    if root:
        a_h = A.cpu().pin_memory().numpy()
        b_h = B.cpu().pin_memory().numpy()
        c_t = torch.empty((n, n), dtype=torch.float64).pin_memory()
        c_h = c_t.numpy()
        del A, B, C
        torch.cuda.empty_cache()
    barrier()
    e2e_t = []
    for i in range(1 + e2e_steps):
        t0 = time.perf_counter()
        if root:
            _, el = ctx.master_run_host(a_h, b_h, c_h, mode=mode)
        else:
            _, el = ctx.master_run_host(None, None, None, mode=mode, m=n, n=n, k=n)
        wall = time.perf_counter() - t0
        if i > 0:
            e2e_t.append(max(el, 0.0) if root else wall)
    e2e_s = sum(e2e_t) / len(e2e_t)
    if emulated is not None:  # the emulated mode through the same host entry
        oz_e2e = [ctx.master_run_host(a_h, b_h, c_h, mode=P.MODE_OZAKI)[1] for _ in range(3)][1:]
        oz_s = sum(oz_e2e) / len(oz_e2e)
        emulated["e2e"] = {"value": flops / oz_s / 1e9, "unit": "GFLOP/s",
                           "h2d_bytes_per_step": 2 * 8 * n * n, "d2h_bytes_per_step": 8 * n * n,
                           "seconds_per_step": oz_s,
                           "entry": "mmws_gpu_master_run_host (C ABI, pinned host A/B/C), MODE_OZAKI"}

    cpu = None
    if root and world == 1 and not args.no_cpu_baseline:
        s = cpu_reference_sample(n, serial=True)
        cpu = {k: s[k] for k in ("value", "unit", "cores", "kind", "sample", "serial")}

    if root and world > 1:  # cost model of this schedule at the measured 1-GPU kernel rate
        t_model, _, _ = P.rowblock_cost(n, n, n, world, 8, link_bw,
                                        2.0 * rows0 * n * n / (kern_avg_ms / 1e3))
        model = {"predicted_ms_per_step": t_model * 1e3, "link_GBps": link_bw / 1e9,
                 "link_source": "mmws_gpu_link_probe: 5 x 256 MiB NCCL broadcasts from rank 0"}
    else:
        model = None
    if root:
        line = {
            "metric": metric_name(), "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "config": workload_config(n, world, args.mode),
            "roofline": {
                "bound": "tensor", "achieved": achieved, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": achieved / dmma_peak, "traffic": traffic,
                "kernel": plan + " (DMMA.8x8x4)",
                "peak_source": "measured live in this run: DMMA.8x8x4 throughput probe "
                               "(FP64 tensor pipe; MEASURED_PEAKS.json has no fp64 figure)",
                "peak_nominal": NOMINAL_FP64_TFLOPS, "frac_of_nominal": achieved / NOMINAL_FP64_TFLOPS,
                "flops_per_launch": 2.0 * rows0 * n * n, "kernel_ms_avg": kern_avg_ms,
                "traffic_source": traffic_src,
                "traffic_note": (None if traffic is None else
                                 "ncu dram bytes per launch vs %.2f GB algorithmic: each wave of "
                                 "148 tiles streams its ~24 A/B panels (16 MB each) from HBM "
                                 "again because they exceed the 126 MB L2; %.1f%% of HBM "
                                 "bandwidth over the launch, the FP64 tensor pipe is the bound"
                                 % (8.0 * (2 * rows0 * n + n * n) / 1e9,
                                    100.0 * traffic / (kern_avg_ms / 1e3) / 1e9
                                    / measured_hbm_gbs())),
            },
            "cpu_baseline": cpu,
            "e2e": {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 2 * 8 * n * n, "d2h_bytes_per_step": 8 * n * n,
                    "seconds_per_step": e2e_s,
                    "entry": "mmws_gpu_master_run_host (C ABI, pinned host A/B/C)"},
            "gpu_launches": launches_total,
            "cost_model": model,
            "emulated_fp64": emulated,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--mode", choices=["auto", "dmma", "exact", "ozaki"], default="auto")
    ap.add_argument("--no-emulated", action="store_true",
                    help="skip the MODE_OZAKI measurement added to the JSON line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        sys.exit("steps must be >= 1 and warmup >= 0")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

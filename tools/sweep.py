"""configs[1] sweep: square fp64 GEMM at N in {10..2000}, uniform [-1,1) seeds
0/1, one GPU.  Per N: device time of one multiply (CUDA events, min over
reps) for eager launches and for CUDA-graph replay, the host-buffer call
(H2D + multiply + D2H through the C ABI), the resident latency server for
N <= 96 (host buffers, min and median of 200 calls), and the reference CPU time
(oracle/_ref matmul_seq on 1 thread and matmul_threads on all threads, full
product, time_model bracket) where it finishes quickly.  Writes one JSON line
per N to stdout."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402  (CPU reference timing only)
import paper_1012_2273_b200 as P  # noqa: E402


def dev_time(fn, reps, inner=1):
    """Device time per call: CUDA events around `inner` back-to-back calls
    queued behind a sleep kernel, so the host's submission time (Python,
    ctypes, argument checks) never shows up as idle GPU time between them."""
    s = torch.cuda.current_stream()
    best = 1e9
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(inner * 40e-6 * 2e9))  # longer than queuing `inner` calls
        e0.record(s)
        for _ in range(inner):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / inner)
    return best


def wall_time(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    ctx = P.Context(0)
    cores = len(os.sched_getaffinity(0))
    ns = [int(x) for x in sys.argv[1:]] or [10, 50, 96, 100, 250, 500, 1000, 1500, 2000]
    for n in ns:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
        reps = 50 if n <= 500 else 20
        rec = {"n": n, "flops": 2 * n ** 3}
        for name, mode in (("auto", P.MODE_AUTO), ("exact", P.MODE_EXACT)):
            inner = 20 if n <= 1000 else 3
            t = dev_time(lambda: ctx.dgemm(A, B, C, mode=mode), reps, inner)
            g = ctx.graph_dgemm(A, B, C, mode=mode)
            tg = dev_time(lambda: g.launch(), reps, inner)
            tw = wall_time(lambda: ctx.dgemm(A, B, C, mode=mode), reps)
            twg = wall_time(lambda: g.launch(), reps)
            g.close()
            # device_s / graph_device_s: per call with the launch queue kept full;
            # wall_s / graph_wall_s: one call + synchronize, as a caller sees it
            rec[name] = {"device_s": t, "graph_device_s": tg, "wall_s": tw, "graph_wall_s": twg,
                         "gflops": 2 * n ** 3 / t / 1e9,
                         "gflops_graph_wall": 2 * n ** 3 / twg / 1e9,
                         "hbm_gbs": 3 * 8 * n * n / t / 1e9}
        a, b = A.cpu().numpy(), B.cpu().numpy()
        th = min(ctx.matmul_host(a, b)[1] for _ in range(5))
        rec["host_entry_s"] = th
        if n <= 96:
            # resident latency server: host buffers in, host buffers out, no launch
            ctx.server_start()
            for mode_name, mode in (("server_auto_s", P.MODE_AUTO), ("server_exact_s", P.MODE_EXACT)):
                for _ in range(20):
                    ctx.server_matmul(a, b, mode=mode)
                ts = sorted(ctx.server_matmul(a, b, mode=mode)[1] for _ in range(200))
                rec[mode_name] = ts[0]
                rec[mode_name.replace("_s", "_median_s")] = ts[len(ts) // 2]
            ctx.server_stop()
        if O.ref_available() and n <= 2000:
            reps_cpu = 3 if n <= 1000 else 1
            if n <= 1500:
                rec["ref_seq_s"], _ = O.ref_time_matmul(a, b, 0, repeats=reps_cpu)
            rec["ref_threads_s"], _ = O.ref_time_matmul(a, b, cores, repeats=reps_cpu)
            rec["ref_threads_cores"] = cores
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

"""DMMA tile plans at small / mid sizes: per-call time of back-to-back
device-pointer multiplies (CUDA events around `reps` calls queued behind a
sleep kernel, min of 5 rounds)
for each MMWS_GPU_DMMA_PLAN override ("<cfg>" one-shot, "<cfg>s<CTAs/SM>"
stream-K; cfg 0 = 128x128, 1 = 64x64, 2 = 128x64, 3 = 64x64 with 8 math
warps, 4 = 32x32, 5 = 32x64) against the default plan, and checks every plan's bits
against the default's.
Usage: python tools/dmma_plan_probe.py [N ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

PLANS = os.environ.get("PLANS", "1,4,5,0s1,1s2,1s3,3s1,4s4,5s2,5s4").split(",")


def per_call_ms(fn, reps):
    """GPU time per call of `reps` back-to-back calls: a sleep kernel holds the
    stream while the host queues them, so host-side call overhead (Python,
    ctypes) does not show up as idle time between the timed kernels."""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(reps * 40e-6 * 2e9))  # > host time to queue the calls
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def main():
    ctx = P.Context(0)
    sizes = [int(x) for x in sys.argv[1:]] or [300, 400, 500, 640, 750, 1000, 1250, 1500,
                                                1750, 2000, 2500, 3000]
    for n in sizes:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        ref = torch.empty_like(A)
        reps = max(5, min(200, int(2e10 / (2 * n ** 3))))
        ctx.tune("MMWS_GPU_DMMA_PLAN", None)
        rec = {"n": n, "reps": reps}
        ms = per_call_ms(lambda: ctx.dgemm(A, B, ref, mode=P.MODE_AUTO), reps)
        rec["auto"] = {"us": ms * 1e3, "tflops": 2 * n ** 3 / ms / 1e9}
        for plan in PLANS:
            ctx.tune("MMWS_GPU_DMMA_PLAN", plan)
            C = torch.empty_like(A)
            try:
                ctx.dgemm(A, B, C, mode=P.MODE_DMMA)
            except Exception as exc:  # plan not usable at this size
                rec[plan] = {"skip": str(exc)[:60]}
                continue
            torch.cuda.synchronize()
            same = bool(torch.equal(C.view(torch.int64), ref.view(torch.int64)))
            ms = per_call_ms(lambda: ctx.dgemm(A, B, C, mode=P.MODE_DMMA), reps)
            rec[plan] = {"us": ms * 1e3, "tflops": 2 * n ** 3 / ms / 1e9, "bitwise": same}
        ctx.tune("MMWS_GPU_DMMA_PLAN", None)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

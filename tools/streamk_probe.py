"""Stream-K vs one-shot DMMA launches at mid sizes (CUDA events, min of reps).
Usage: python tools/streamk_probe.py [N ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402


def best_ms(fn, reps=20):
    """Min GPU time of one call, queued behind a sleep kernel so the host's
    submission time is not counted."""
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100000)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


ctx = P.Context(0)
for n in [int(x) for x in sys.argv[1:]] or [1600, 2000, 2048, 2304, 2500, 3000, 4099, 8192]:
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    rec = {"n": n}
    for name, env, mode in (("auto", {}, P.MODE_AUTO),
                            ("no_streamk", {"MMWS_GPU_NO_STREAMK": "1"}, P.MODE_AUTO),
                            ("exact", {}, P.MODE_EXACT),
                            ("exact_no_streamk", {"MMWS_GPU_NO_STREAMK": "1"}, P.MODE_EXACT)):
        ctx.tune("MMWS_GPU_NO_STREAMK", env.get("MMWS_GPU_NO_STREAMK"))
        ms = best_ms(lambda: ctx.dgemm(A, B, C, mode=mode))
        rec[name] = {"ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}
    ctx.tune("MMWS_GPU_NO_STREAMK", None)
    print(json.dumps(rec), flush=True)

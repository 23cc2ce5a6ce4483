"""MODE_OZAKI (fp64 emulated on the int8 tensor cores): accuracy against the
fp64 oracle on sampled rows / integer inputs, and rate vs the DMMA path.
Usage: python tools/ozaki_probe.py [N ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402  (accuracy reference only)
import paper_1012_2273_b200 as P  # noqa: E402


def best_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


ctx = P.Context(0)
for n in [int(x) for x in sys.argv[1:]] or [512, 2048, 4096, 8192, 16384]:
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    rec = {"n": n}
    ctx.dgemm(A, B, C, mode=P.MODE_OZAKI)
    rows = sorted({0, n // 3, n - 1})
    a, b = A.cpu().numpy(), B.cpu().numpy()
    want = O.matmul_rows(rows, a, b)
    got = C.cpu().numpy()[rows]
    rec["normwise_err"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    for name, mode in (("ozaki", P.MODE_OZAKI), ("dmma", P.MODE_AUTO)):
        ms = best_ms(lambda: ctx.dgemm(A, B, C, mode=mode))
        rec[name] = {"ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}
    Ai = ctx.fill(P.DIST_INT8, 0, n, n)
    Bi = ctx.fill(P.DIST_INT8, 1, n, n)
    ci = ctx.dgemm(Ai, Bi, mode=P.MODE_OZAKI).cpu().numpy()[rows]
    wi = O.matmul_rows(rows, Ai.cpu().numpy(), Bi.cpu().numpy())
    rec["int8_bit_exact"] = bool((ci == wi).all())
    if os.environ.get("OZAKI_PROBE_F32"):
        Af, Bf = A.float(), B.float()
        Cf = torch.empty_like(Af)
        for name, mode in (("f32_ozaki", P.MODE_OZAKI), ("f32_ffma", P.MODE_AUTO)):
            ms = best_ms(lambda: ctx.sgemm(Af, Bf, Cf, mode=mode))
            rec[name] = {"ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}
        ctx.sgemm(Af, Bf, Cf, mode=P.MODE_OZAKI)
        wf = O.matmul_rows(rows, Af.cpu().numpy(), Bf.cpu().numpy())
        rec["f32_ozaki_err"] = float(np.linalg.norm(Cf.cpu().numpy()[rows] - wf) / np.linalg.norm(wf))
    print(json.dumps(rec), flush=True)

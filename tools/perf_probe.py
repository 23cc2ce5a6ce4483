"""Quick device-side timing of every kernel family (development aid)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1012_2273_b200 as P


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return min(ts), sorted(ts)[len(ts) // 2]


def main():
    ctx = P.Context(0)
    out = {"num_sms": ctx.num_sms, "max_clock_khz": ctx.max_clock_khz}
    for name, w in [("dmma", P.PROBE_DMMA), ("dfma", P.PROBE_DFMA), ("dmul_dadd", P.PROBE_DMUL_DADD),
                    ("ffma", P.PROBE_FFMA), ("ffma2", P.PROBE_FFMA2)]:
        out["probe_" + name] = [ctx.peak_probe(w, 20000) for _ in range(3)]
    print(json.dumps(out), flush=True)
    sizes = [int(x) for x in (sys.argv[1:] or ["16384"])]
    for n in sizes:
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
        for mname, mode in [("dmma", P.MODE_DMMA), ("dmma_small", P.MODE_DMMA_SMALL), ("exact", P.MODE_EXACT)]:
            if mode == P.MODE_EXACT and n > 8192:
                continue
            reps = 3 if n >= 8192 else 10
            tmin, tmed = timeit(lambda: ctx.dgemm(A, B, C, mode=mode), reps=reps)
            print(json.dumps({"n": n, "mode": mname, "t_min": tmin, "t_med": tmed,
                              "tflops": 2 * n**3 / tmin / 1e12}), flush=True)
        del A, B, C
    for n in [8192, 16384, 32768]:
        A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
        B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
        C = torch.empty_like(A)
        tmin, tmed = timeit(lambda: ctx.sgemm(A, B, C), reps=3)
        print(json.dumps({"n": n, "mode": "ffma", "t_min": tmin, "t_med": tmed,
                          "tflops": 2 * n**3 / tmin / 1e12}), flush=True)


if __name__ == "__main__":
    main()

"""Where the small-N host-buffer multiply's wall time goes: the Python API
(ctx.matmul_host), the bare ctypes call of mmws_gpu_matmul_host with
precomputed pointers, and the library's own device-event bracket, pageable
and pinned buffers.  python tools/host_entry_probe.py [N ...]"""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402


def med(fn, reps=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6, min(ts) * 1e6


ctx = P.Context(0)
lib = P._abi.load()
for n in [int(x) for x in sys.argv[1:]] or [10, 50, 100, 250]:
    a = np.random.rand(n, n)
    b = np.random.rand(n, n)
    c = np.empty((n, n))
    for label, (aa, bb, cc) in (("pageable", (a, b, c)),
                                ("pinned", tuple(torch.from_numpy(x).pin_memory().numpy()
                                                 for x in (a, b, c)))):
        api = med(lambda: ctx.matmul_host(aa, bb, out=cc))
        el = C.c_double()
        args = (ctx.handle, n, n, n, aa.ctypes.data, bb.ctypes.data, cc.ctypes.data, 0, C.byref(el))
        raw = med(lambda: lib.mmws_gpu_matmul_host(*args))
        lib.mmws_gpu_matmul_host(*args)
        print(f"N={n} {label}: api {api[0]:.1f} us (min {api[1]:.1f}), bare ctypes {raw[0]:.1f} "
              f"(min {raw[1]:.1f}), library bracket {el.value * 1e6:.1f}", flush=True)

"""SM clock / power while MODE_OZAKI runs back to back at N=16384 (power cap check)."""
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

samples = []
stop = False


def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout
        samples.append(out.strip())
        time.sleep(0.1)


ctx = P.Context(0)
n = 16384
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
C = torch.empty_like(A)
for mode_name, mode in (("dmma", P.MODE_AUTO), ("ozaki", P.MODE_OZAKI)):
    ctx.dgemm(A, B, C, mode=mode)
    torch.cuda.synchronize()
    samples.clear()
    stop = False
    th = threading.Thread(target=sampler)
    th.start()
    t0 = time.time()
    reps = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        ctx.dgemm(A, B, C, mode=mode)
        torch.cuda.synchronize()
        reps += 1
    e1.record()
    torch.cuda.synchronize()
    stop = True
    th.join()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"mode": mode_name, "ms_per_call": ms, "tflops": 2 * n ** 3 / ms / 1e9,
                      "samples": samples[-12:]}), flush=True)

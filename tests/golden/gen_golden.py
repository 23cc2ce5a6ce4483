"""Generate tests/golden/*.json|npz from the REFERENCE ITSELF (oracle/_ref).

Run here (the build container, where /root/reference exists):
    make -C oracle && python tests/golden/gen_golden.py [--big]

Everything written is produced by the reference's own code compiled from
/root/reference/proj/include (mmws::random_matrix, mmws::matmul_seq,
mmws::matmul_threads, mmws::split_rows, mmws::static_partition,
mmws::op_count) via oracle/ref_shim.cpp.  Inputs for the configs use the
frozen generators of SURVEY.md s8(d) built on the reference's splitmix64
stream (oracle/mmws_oracle.c oracle_fill); their agreement with
mmws::random_matrix is itself one of the goldens.

--big adds the full-size pins (several minutes on 8 cores):
  * N=1000 uniform[-1,1) seeds 0/1: sha256 of matmul_threads(A, B) (== seq);
  * N=4099 integer [-8,8] seeds 0/1: sha256 of matmul_threads(A, B);
  * N=16384 uniform seeds 0/1: sha256 of 8 sampled rows of C, computed by
    matmul_threads on the A row slice (bitwise the same rows of matmul_seq).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

ACCEPT_NS = list(range(1, 17)) + [31, 32, 33, 64]          # acceptance.cpp:91-93
BIG_ROWS_16384 = [0, 1, 2047, 2048, 4095, 8191, 12288, 16383]


def hexbits(x: np.ndarray):
    return [format(int(v), "016x") for v in O.bits(x).ravel()]


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def small(out_path: str) -> None:
    g = {"source": "oracle/_ref (reference headers compiled unchanged)"}
    # random_matrix first draws (matrix.hpp:101-107)
    g["random_matrix"] = {str(s): hexbits(O.ref_random_matrix(2, 4, s))
                          for s in (0, 1, 42, 0xDEADBEEF)}
    # hand-computed products (test_matrix.cpp:105-120)
    g["matmul_2x2"] = hexbits(O.ref_matmul_seq(np.array([[1., 2], [3, 4]]),
                                               np.array([[5., 6], [7, 8]])))
    g["matmul_1x1"] = hexbits(O.ref_matmul_seq(np.array([[3.25]]), np.array([[-2.0]])))
    # acceptance-style products: seeds 1000+N / 2000+N (acceptance.cpp:95-96),
    # and the rectangular cases of test_matrix.cpp:148-156 / test_workshare.cpp:160-163
    prods = {}
    for n in ACCEPT_NS:
        a = O.ref_random_matrix(n, n, 1000 + n)
        b = O.ref_random_matrix(n, n, 2000 + n)
        prods[f"sq{n}"] = hexbits(O.ref_matmul_seq(a, b))
    for (m, k, n, sa, sb) in [(2, 5, 4, 303, 304), (4, 7, 3, 27, 28), (5, 7, 4, 31, 32)]:
        a = O.ref_random_matrix(m, k, sa)
        b = O.ref_random_matrix(k, n, sb)
        prods[f"rect{m}x{k}x{n}"] = hexbits(O.ref_matmul_seq(a, b))
    g["products_unit"] = prods
    # split_rows fixtures and a grid (test_protocol.cpp:22-54), static_partition,
    # op_count (test_matrix.cpp:159-165)
    g["split_rows"] = {f"{n},{w}": O.ref_split_rows(n, w)
                       for n in (2, 4, 6, 33, 4099, 16384) for w in (1, 2, 3, 4, 5, 8, 16)}
    g["static_partition"] = {f"{n},{w}": O.ref_static_partition(n, w)
                             for n in (0, 3, 8, 50, 1000) for w in (1, 2, 4, 9)}
    g["op_count"] = {str(n): O.ref_op_count(n) for n in (1, 100, 1000, 4099, 16384, 32768)}
    # bench.hpp harness pieces: derive_seed (:83-86) and mflops (:70-73)
    g["derive_seed"] = {f"{s},{n},{w}": O.ref_derive_seed(s, n, w)
                        for s in (0, 42, 2**63 + 5) for n in (1, 100, 1000, 16384) for w in (0, 1)}
    g["mflops"] = {f"{n},{t}": O.ref_mflops(n, t)
                   for n in (100, 500, 1000, 2000) for t in (0.03, 2.09, 22.52, 240.97)}
    with open(out_path, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)


def big(out_path: str) -> None:
    g = {"source": "oracle/_ref matmul_threads (reference headers compiled unchanged)",
         "workers": os.cpu_count()}
    w = os.cpu_count() or 8
    t0 = time.time()
    a = O.fill(O.DIST_UNIFORM, 0, 1000, 1000)
    b = O.fill(O.DIST_UNIFORM, 1, 1000, 1000)
    g["n1000_uniform_sha256"] = sha(O.ref_matmul_threads(a, b, w))
    print("n1000", time.time() - t0, flush=True)
    a = O.fill(O.DIST_INT8, 0, 4099, 4099)
    b = O.fill(O.DIST_INT8, 1, 4099, 4099)
    c = O.ref_matmul_threads(a, b, w)
    g["n4099_int8_sha256"] = sha(c)
    g["n4099_int8_absmax"] = float(np.abs(c).max())
    g["n4099_int8_row0_first8"] = hexbits(c[0, :8])
    print("n4099", time.time() - t0, flush=True)
    del a, b, c
    n = 16384
    b = O.fill(O.DIST_UNIFORM, 1, n, n)
    rows = BIG_ROWS_16384
    a_rows = np.stack([O.fill(O.DIST_UNIFORM, 0, 1, n, first=r * n)[0] for r in rows])
    c_rows = O.ref_matmul_threads(a_rows, b, len(rows))
    g["n16384_rows"] = rows
    g["n16384_rows_sha256"] = [sha(c_rows[i]) for i in range(len(rows))]
    g["n16384_rows_first4"] = [hexbits(c_rows[i, :4]) for i in range(len(rows))]
    print("n16384", time.time() - t0, flush=True)
    with open(out_path, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    if not O.ref_available():
        sys.exit("oracle/_ref/libmmws_ref.so missing: run `make -C oracle` where /root/reference exists")
    small(os.path.join(HERE, "ref_small.json"))
    if args.big:
        big(os.path.join(HERE, "ref_big.json"))

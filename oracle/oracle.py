"""ctypes access to the CPU oracle (oracle/_build) and the reference shim (oracle/_ref).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
The C restatement lives in oracle/mmws_oracle.c (each function cites the
reference file:line it follows); libmmws_ref.so is the reference's own headers
compiled by oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmmws_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmmws_ref.so")

DIST_UNIT, DIST_UNIFORM, DIST_INT8, DIST_NORMAL = 0, 1, 2, 3

_i64, _u64, _i32, _u32 = C.c_int64, C.c_uint64, C.c_int32, C.c_uint32
_pd, _pf, _pi64, _pu64 = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                          C.POINTER(C.c_int64), C.POINTER(C.c_uint64))


def build() -> None:
    """Compile the oracle (and, where /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_splitmix64_draw.restype = _u64
        L.oracle_splitmix64_draw.argtypes = [_u64, _u64]
        L.oracle_fill.argtypes = [C.c_int, _u64, _u64, _u64, _pd, _pf, C.c_int]
        L.oracle_matmul_seq.argtypes = [_i64, _i64, _i64, _pd, _i64, _pd, _i64, _pd, _i64]
        L.oracle_worker_block.argtypes = [_i64, _i64, _i64, _pd, _pd, _pd]
        L.oracle_matmul_rows.argtypes = [_i64, _pi64, _i64, _i64, _i64, _pd, _i64, _pd, _i64,
                                         _pd, C.c_int]
        L.oracle_matmul_rows_f32w.argtypes = [_i64, _pi64, _i64, _i64, _i64, _pf, _i64, _pf,
                                              _i64, _pd, C.c_int]
        L.oracle_static_partition.argtypes = [_u64, _u32, _pu64, _pu64]
        L.oracle_split_rows.argtypes = [_i64, _i32, _pi64, _pi64]
        L.oracle_op_count.argtypes = [_i64, _pu64]
        L.oracle_matmul_threads.argtypes = [_i64, _i64, _i64, _pd, _pd, _pd, _u32]
        L.oracle_first_difference.restype = _i64
        L.oracle_first_difference.argtypes = [_pd, _pd, _i64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference's own matmul code (oracle/_ref/libmmws_ref.so)."""
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_random_matrix.argtypes = [_i64, _i64, _u64, _pd]
        L.ref_identity.argtypes = [_i64, _pd]
        L.ref_matmul_seq.argtypes = [_i64, _i64, _i64, _i64, _pd, _pd, _pd]
        L.ref_matmul_threads.argtypes = [_i64, _i64, _i64, _i64, _pd, _pd, _pd, C.c_uint]
        L.ref_time_matmul.argtypes = [_i64, _i64, _i64, _pd, _pd, C.c_uint, C.c_int, _pd, _pd]
        L.ref_static_partition.argtypes = [_u64, C.c_uint, _pu64, _pu64]
        L.ref_op_count.argtypes = [_i64, _pu64]
        L.ref_split_rows.argtypes = [_i64, C.c_int, _pi64, _pi64]
        L.ref_derive_seed.argtypes = [_u64, _i64, C.c_int, _pu64]
        L.ref_mflops.argtypes = [_i64, C.c_double, C.POINTER(C.c_double)]
        _ref = L
    return _ref


# ----------------------------------------------------------------------------- oracle wrappers
def fill(dist: int, seed: int, rows: int, cols: int, dtype=np.float64, first: int = 0,
         threads: int = 0) -> np.ndarray:
    out = np.empty((rows, cols), dtype=dtype)
    if dtype == np.float64:
        rc = lib().oracle_fill(dist, seed, first, rows * cols, _ptr(out, _pd), None, threads)
    else:
        rc = lib().oracle_fill(dist, seed, first, rows * cols, None, _ptr(out, _pf), threads)
    if rc:
        raise ValueError(f"oracle_fill rc={rc}")
    return out


def matmul_seq(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    c = np.empty((m, n), dtype=np.float64)
    rc = lib().oracle_matmul_seq(m, n, k, _ptr(a, _pd), k, _ptr(b, _pd), n, _ptr(c, _pd), n)
    if rc:
        raise ValueError(f"oracle_matmul_seq rc={rc}")
    return c


def matmul_threads(a: np.ndarray, b: np.ndarray, workers: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m, k = a.shape
    _, n = b.shape
    c = np.empty((m, n), dtype=np.float64)
    rc = lib().oracle_matmul_threads(m, n, k, _ptr(a, _pd), _ptr(b, _pd), _ptr(c, _pd),
                                     workers or os.cpu_count() or 1)
    if rc:
        raise ValueError(f"oracle_matmul_threads rc={rc}")
    return c


def worker_block(a_slice: np.ndarray, b: np.ndarray) -> np.ndarray:
    a_slice = np.ascontiguousarray(a_slice, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    rows, k = a_slice.shape
    _, n = b.shape
    c = np.empty((rows, n), dtype=np.float64)
    rc = lib().oracle_worker_block(rows, n, k, _ptr(a_slice, _pd), _ptr(b, _pd), _ptr(c, _pd))
    if rc:
        raise ValueError(f"oracle_worker_block rc={rc}")
    return c


def matmul_rows(rows, a: np.ndarray, b: np.ndarray, threads: int = 0) -> np.ndarray:
    """Bitwise matmul_seq restricted to the listed rows (fp64), or the fp64
    product of widened fp32 inputs when a/b are float32."""
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    m, k = a.shape
    _, n = b.shape
    out = np.empty((len(rows), n), dtype=np.float64)
    if a.dtype == np.float32:
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b, dtype=np.float32)
        rc = lib().oracle_matmul_rows_f32w(len(rows), _ptr(rows, _pi64), m, n, k, _ptr(a, _pf),
                                           a.strides[0] // 4, _ptr(b, _pf), b.strides[0] // 4,
                                           _ptr(out, _pd), threads)
    else:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        rc = lib().oracle_matmul_rows(len(rows), _ptr(rows, _pi64), m, n, k, _ptr(a, _pd),
                                      a.strides[0] // 8, _ptr(b, _pd), b.strides[0] // 8,
                                      _ptr(out, _pd), threads)
    if rc:
        raise ValueError(f"oracle_matmul_rows rc={rc}")
    return out


def split_rows(n_rows: int, n_workers: int):
    off = np.zeros(max(n_workers, 1), dtype=np.int64)
    rows = np.zeros(max(n_workers, 1), dtype=np.int64)
    rc = lib().oracle_split_rows(n_rows, n_workers, _ptr(off, _pi64), _ptr(rows, _pi64))
    if rc:
        raise ValueError("split_rows domain error")
    return list(zip(off.tolist(), rows.tolist()))


def static_partition(iterations: int, workers: int):
    st = np.zeros(max(workers, 1), dtype=np.uint64)
    ln = np.zeros(max(workers, 1), dtype=np.uint64)
    rc = lib().oracle_static_partition(iterations, workers, _ptr(st, _pu64), _ptr(ln, _pu64))
    if rc:
        raise ValueError("static_partition domain error")
    return list(zip(st.tolist(), ln.tolist()))


def op_count(n: int) -> int:
    out = C.c_uint64()
    if lib().oracle_op_count(n, C.byref(out)):
        raise ValueError("op_count domain error")
    return out.value


def first_difference(x: np.ndarray, y: np.ndarray):
    if x.shape != y.shape:
        return 0
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = lib().oracle_first_difference(_ptr(x, _pd), _ptr(y, _pd), x.size)
    return None if r < 0 else int(r)


# ----------------------------------------------------------------------------- reference shim
def ref_random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    rc = ref().ref_random_matrix(rows, cols, seed, _ptr(out, _pd))
    if rc:
        raise ValueError(f"ref_random_matrix rc={rc}")
    return out


def ref_matmul_seq(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
    rc = ref().ref_matmul_seq(a.shape[0], a.shape[1], b.shape[0], b.shape[1], _ptr(a, _pd),
                              _ptr(b, _pd), _ptr(c, _pd))
    if rc:
        raise ValueError(f"ref_matmul_seq rc={rc}")
    return c


def ref_matmul_threads(a: np.ndarray, b: np.ndarray, workers: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
    rc = ref().ref_matmul_threads(a.shape[0], a.shape[1], b.shape[0], b.shape[1], _ptr(a, _pd),
                                  _ptr(b, _pd), _ptr(c, _pd), workers)
    if rc:
        raise ValueError(f"ref_matmul_threads rc={rc}")
    return c


def ref_time_matmul(a: np.ndarray, b: np.ndarray, workers: int, repeats: int = 1,
                    want_c: bool = False):
    """Reference matmul_seq (workers=0) / matmul_threads timed with the
    reference's time_model bracket (bench.hpp:99-111): (best_s, C or None)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64) if want_c else None
    best = C.c_double()
    rc = ref().ref_time_matmul(a.shape[0], a.shape[1], b.shape[1], _ptr(a, _pd), _ptr(b, _pd),
                               workers, repeats, C.byref(best),
                               _ptr(c, _pd) if c is not None else None)
    if rc:
        raise ValueError(f"ref_time_matmul rc={rc}")
    return best.value, c


def ref_split_rows(n_rows: int, n_workers: int):
    off = np.zeros(max(n_workers, 1), dtype=np.int64)
    rows = np.zeros(max(n_workers, 1), dtype=np.int64)
    rc = ref().ref_split_rows(n_rows, n_workers, _ptr(off, _pi64), _ptr(rows, _pi64))
    if rc:
        raise ValueError(f"ref_split_rows rc={rc}")
    return list(zip(off.tolist(), rows.tolist()))


def ref_static_partition(iterations: int, workers: int):
    st = np.zeros(max(workers, 1), dtype=np.uint64)
    ln = np.zeros(max(workers, 1), dtype=np.uint64)
    rc = ref().ref_static_partition(iterations, workers, _ptr(st, _pu64), _ptr(ln, _pu64))
    if rc:
        raise ValueError(f"ref_static_partition rc={rc}")
    return list(zip(st.tolist(), ln.tolist()))


def ref_op_count(n: int) -> int:
    out = C.c_uint64()
    rc = ref().ref_op_count(n, C.byref(out))
    if rc:
        raise ValueError(f"ref_op_count rc={rc}")
    return out.value


def ref_derive_seed(seed: int, n: int, which: int) -> int:
    out = C.c_uint64()
    rc = ref().ref_derive_seed(seed, n, which, C.byref(out))
    if rc:
        raise ValueError(f"ref_derive_seed rc={rc}")
    return out.value


def ref_mflops(n: int, elapsed: float) -> float:
    out = C.c_double()
    rc = ref().ref_mflops(n, elapsed, C.byref(out))
    if rc:
        raise ValueError(f"ref_mflops rc={rc}")
    return out.value


def bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)

"""ctypes binding of libmmws_gpu.so (the C ABI declared in include/mmws_gpu.h).

This is the binding a Python caller of the reference would add (see
INTEGRATION.md); the product itself is the in-tree shared library.  Loading
fails loudly if the library has not been built -- there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libmmws_gpu.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "mmws_gpu.h")

(OK, ERR_DIMENSION, ERR_DOMAIN, ERR_CUDA, ERR_NCCL, ERR_RANK, ERR_PROTOCOL, ERR_STATE, ERR_ALLOC,
 ERR_TIMEOUT) = range(10)
GATHER_NONE, GATHER_FUSED, GATHER_NCCL = range(3)
MODE_AUTO, MODE_EXACT, MODE_DMMA, MODE_DMMA_SMALL, MODE_FFMA, MODE_OZAKI = range(6)
DIST_UNIT, DIST_UNIFORM, DIST_INT8, DIST_NORMAL = range(4)
PROBE_DMMA, PROBE_DFMA, PROBE_DMUL_DADD, PROBE_FFMA, PROBE_FFMA2, PROBE_FFMA2_OUTER = range(6)

_v, _i, _i32, _i64, _u32, _u64 = C.c_void_p, C.c_int, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
_p = C.POINTER
_d, _f = C.c_double, C.c_float

# name -> (restype, argtypes); mirrors include/mmws_gpu.h one to one
SIGNATURES = {
    "mmws_gpu_abi_version": (_i, []),
    "mmws_gpu_last_error": (C.c_char_p, []),
    "mmws_gpu_init": (_i, [_i, _p(_v)]),
    "mmws_gpu_destroy": (_i, [_v]),
    "mmws_gpu_device_info": (_i, [_v, _p(_i), _p(_i), _p(_i), _p(_i)]),
    "mmws_gpu_launch_count": (_u64, [_v]),
    "mmws_gpu_stream": (_v, [_v]),
    "mmws_gpu_tune": (_i, [_v, C.c_char_p, C.c_char_p]),
    "mmws_gpu_split_rows": (_i, [_i64, _i, _p(_i64), _p(_i64)]),
    "mmws_gpu_static_partition": (_i, [_u64, _u32, _p(_u64), _p(_u64)]),
    "mmws_gpu_op_count": (_i, [_i64, _p(_u64)]),
    "mmws_gpu_dgemm": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _i, _v]),
    "mmws_gpu_sgemm": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _i, _v]),
    "mmws_gpu_dgemm_acc": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _v, _i64, _i,
                                _v]),
    "mmws_gpu_sgemm_acc": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _v, _i64, _i,
                                _v]),
    "mmws_gpu_matmul_host": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_matmul_host_f32": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_fill": (_i, [_v, _i, _u64, _v, _i64, _i64, _i64, _i, _u64, _v]),
    "mmws_gpu_graph_dgemm": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _i, _p(_v)]),
    "mmws_gpu_graph_launch": (_i, [_v, _v]),
    "mmws_gpu_graph_destroy": (_i, [_v]),
    "mmws_gpu_server_start": (_i, [_v]),
    "mmws_gpu_server_dgemm": (_i, [_v, _i64, _i64, _i64, _v, _i64, _v, _i64, _v, _i64, _i, _p(_d)]),
    "mmws_gpu_server_stop": (_i, [_v]),
    "mmws_gpu_synchronize": (_i, [_v]),
    "mmws_gpu_ipc_export": (_i, [_v, _v, _p(C.c_uint8)]),
    "mmws_gpu_ipc_open": (_i, [_v, _p(C.c_uint8), _p(_v)]),
    "mmws_gpu_ozaki_plan": (_i, [_i64, _p(_i), _p(_i)]),
    "mmws_gpu_peak_probe": (_i, [_v, _i, _i, _p(_d)]),
    "mmws_gpu_gemm_probe": (_i, [_v, _i64, _i, _i, _p(_d)]),
    "mmws_gpu_link_probe": (_i, [_v, _i64, _i, _p(_d)]),
    "mmws_gpu_p2p_probe": (_i, [_v, _i64, _i, _p(_d)]),
    "mmws_gpu_last_round": (_i, [_v, _p(_i), _p(_i), _p(_i)]),
    "mmws_gpu_set_timeout": (_i, [_v, _d]),
    "mmws_gpu_nccl_unique_id": (_i, [_p(C.c_uint8)]),
    "mmws_gpu_comm_init": (_i, [_v, _i, _i, _p(C.c_uint8)]),
    "mmws_gpu_comm_destroy": (_i, [_v]),
    "mmws_gpu_rowblock_dgemm": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_rowblock_sgemm": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_master_run_host": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_master_run_host_f32": (_i, [_v, _i64, _i64, _i64, _v, _v, _v, _i, _p(_d)]),
    "mmws_gpu_last_kernel_ms": (_i, [_v, _p(_d)]),
    "mmws_gpu_last_plan": (_i, [_v, _p(C.c_char_p)]),
    "mmws_gpu_rowblock_cost": (_i, [_i64, _i64, _i64, _i, _i, _d, _d, _p(_d), _p(_d), _p(_d)]),
    "mmws_gpu_rowblock_ranks": (_i, [_i64, _i64, _i64, _i, _i, _p(_i)]),
    "mmws_gpu_rowblock_plan": (_i, [_i64, _i64, _i64, _i, _p(_i32), _p(_i32), _p(_i32), _p(_i64),
                                    _p(_i64), _p(_i32), _p(_i32)]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libmmws_gpu.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make -C paper_1012_2273_b200`). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().mmws_gpu_last_error()
    return msg.decode() if msg else ""

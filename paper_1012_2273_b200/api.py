"""Python host mirror of the reference's hot-path API over the C ABI.

The reference is C++ (namespace mmws); its drop-in for C++ callers is
include/mmws_gpu.hpp.  This module is the same surface for Python callers,
tests and bench.py: reference names (split_rows, static_partition, op_count,
matmul / master_run analogues), reference error classes, and device tensors
handed to the CUDA kernels through ctypes.  Every compute call goes to
libmmws_gpu.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _abi
from ._abi import (DIST_INT8, DIST_NORMAL, DIST_UNIFORM, DIST_UNIT, MODE_AUTO, MODE_DMMA,  # noqa: F401
                   MODE_DMMA_SMALL, MODE_EXACT, MODE_FFMA, MODE_OZAKI, PROBE_DFMA, PROBE_DMMA,
                   PROBE_DMUL_DADD, PROBE_FFMA, PROBE_FFMA2,
                   PROBE_FFMA2_OUTER)


# --------------------------------------------------------------------------- errors
# Names and bases follow the reference's error.hpp:9-53.
class DimensionError(ValueError):
    """Invalid matrix shapes (error.hpp:9-12)."""


class DomainError(ValueError):
    """Arguments outside an operation's domain (error.hpp:14-17)."""


class RankError(IndexError):
    """Unaddressable rank (error.hpp:19-22)."""


class ProtocolError(RuntimeError):
    """Row-block exchange failed (error.hpp:29-32)."""


class TimeoutError(RuntimeError):  # noqa: A001 -- the reference's name (error.hpp:36-39)
    """A distributed step made no progress within the deadline (error.hpp:36-39)."""


class GpuError(RuntimeError):
    """CUDA / NCCL / allocation failure (no reference counterpart)."""


_ERRORS = {
    _abi.ERR_DIMENSION: DimensionError,
    _abi.ERR_DOMAIN: DomainError,
    _abi.ERR_RANK: RankError,
    _abi.ERR_PROTOCOL: ProtocolError,
    _abi.ERR_TIMEOUT: TimeoutError,
}


def _check(rc: int) -> None:
    if rc != _abi.OK:
        raise _ERRORS.get(rc, GpuError)(f"[mmws_gpu rc={rc}] {_abi.last_error()}")


def _lib():
    return _abi.load()


# --------------------------------------------------------------------------- host-only helpers
def split_rows(n_rows: int, n_workers: int) -> List[Tuple[int, int]]:
    """split_rows (protocol.hpp:33-46) -> [(offset, rows)] per worker."""
    n = max(int(n_workers), 1)
    off = (C.c_int64 * n)()
    rows = (C.c_int64 * n)()
    _check(_lib().mmws_gpu_split_rows(n_rows, n_workers, off, rows))
    return [(off[i], rows[i]) for i in range(n)]


def static_partition(iterations: int, workers: int) -> List[Tuple[int, int]]:
    """static_partition (workshare.hpp:33-46) -> [(start, len)] per worker."""
    n = max(int(workers), 1)
    st = (C.c_uint64 * n)()
    ln = (C.c_uint64 * n)()
    _check(_lib().mmws_gpu_static_partition(iterations, workers, st, ln))
    return [(st[i], ln[i]) for i in range(n)]


def op_count(n: int) -> int:
    """op_count (matrix.hpp:130-134): N^2 (2N - 1)."""
    out = C.c_uint64()
    _check(_lib().mmws_gpu_op_count(n, C.byref(out)))
    return out.value


def rowblock_plan(m: int, n: int, k: int, nranks: int):
    """Rank 0's message plan for the row-block exchange, in issue order: list of
    dicts(peer, tag, kind, count, row0, dir) with dir in {sent, received, broadcast}."""
    cnt = C.c_int32(0)
    _check(_lib().mmws_gpu_rowblock_plan(m, n, k, nranks, None, None, None, None, None, None,
                                         C.byref(cnt)))
    e = cnt.value
    peer, tag, kind, dirs = ((C.c_int32 * max(e, 1))() for _ in range(4))
    count, row0 = ((C.c_int64 * max(e, 1))() for _ in range(2))
    _check(_lib().mmws_gpu_rowblock_plan(m, n, k, nranks, peer, tag, kind, count, row0, dirs,
                                         C.byref(cnt)))
    names = {0: "sent", 1: "received", 2: "broadcast"}
    return [dict(peer=peer[i], tag=tag[i], kind=kind[i], count=count[i], row0=row0[i],
                 dir=names[dirs[i]]) for i in range(e)]


def rowblock_cost(m: int, n: int, k: int, nranks: int, elem_bytes: int = 8,
                  link_bytes_per_s: float = 770e9, gemm_flops_per_s: float = 36.4e12):
    """Predicted row-block round (seconds, rank 0 egress bytes, ingress bytes);
    defaults: measured B200 peer-copy bandwidth per direction
    (B200_PROFILING.md) and the measured 1-GPU fp64 DMMA rate."""
    t, eg, ing = C.c_double(), C.c_double(), C.c_double()
    _check(_lib().mmws_gpu_rowblock_cost(m, n, k, nranks, elem_bytes, link_bytes_per_s,
                                         gemm_flops_per_s, C.byref(t), C.byref(eg), C.byref(ing)))
    return t.value, eg.value, ing.value


def rowblock_ranks(m: int, n: int, k: int, nranks: int, elem_bytes: int = 8) -> int:
    """How many ranks a row-block round over nranks GPUs uses: nranks when
    the distributed round is predicted to beat rank 0 alone, else 1
    (mmws_gpu_rowblock_ranks)."""
    out = C.c_int()
    _check(_lib().mmws_gpu_rowblock_ranks(m, n, k, nranks, elem_bytes, C.byref(out)))
    return out.value


def ozaki_plan(k: int):
    """MODE_OZAKI plan for inner dimension k: (int8 GEMMs, integer bits)."""
    s, t = C.c_int(), C.c_int()
    _check(_lib().mmws_gpu_ozaki_plan(k, C.byref(s), C.byref(t)))
    return s.value, t.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib().mmws_gpu_nccl_unique_id(buf))
    return bytes(buf)


# --------------------------------------------------------------------------- context
def _ptr(t) -> int:
    return t.data_ptr()


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the default stream torch reports as 0


_RAW_STREAM = None


def _stream(stream) -> int:
    """Launch stream for a call: torch's current stream by default, so the
    kernels order with surrounding torch work and torch events time them.
    Read as a raw handle when torch offers it (no Stream object per call:
    ~3 us of the ~12 us a small dgemm call costs from Python)."""
    global _RAW_STREAM
    if stream is None:
        import torch
        if _RAW_STREAM is None:
            _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
        if _RAW_STREAM:
            stream = _RAW_STREAM(torch.cuda.current_device())
        else:
            stream = torch.cuda.current_stream().cuda_stream
    stream = int(stream)
    return stream if stream else _CUDA_STREAM_LEGACY


def _ld(t) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise DimensionError("expected a 2-D row-major tensor with unit column stride")
    return t.stride(0)


def _device_operands(A, B, C_, dtype, who: str, device: Optional[int] = None):
    """Shapes (m, n, k) of C_ = A . B on the device; every tensor must be a
    2-D CUDA tensor of `dtype` on the context's device, and C_ (if given) at
    least m x n."""
    for name, t in (("A", A), ("B", B), ("C", C_)):
        if t is None:
            continue
        if t.dtype != dtype:
            raise DomainError(f"{who}: {name} must be {dtype}, got {t.dtype}")
        if not t.is_cuda:
            raise DomainError(f"{who}: {name} must be a CUDA tensor")
        if device is not None and t.device.index != device:
            raise DomainError(f"{who}: {name} is on {t.device}, the context on cuda:{device}")
        if t.dim() != 2:
            raise DimensionError(f"{who}: {name} must be 2-D, got {t.dim()}-D")
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise DimensionError(f"matmul: inner dimensions differ, {k} vs {k2}")
    if C_ is not None and (C_.shape[0] < m or C_.shape[1] < n):
        raise DimensionError(f"{who}: C is {tuple(C_.shape)}, needs at least ({m}, {n})")
    return m, n, k


def _host_out(out, m: int, n: int, dt, who: str):
    """The caller's output array for an (m, n) host result, checked; or a new one."""
    if out is None:
        return np.empty((m, n), dtype=dt)
    if not isinstance(out, np.ndarray):
        raise DomainError(f"{who}: out must be a numpy array")
    if out.shape != (m, n):
        raise DimensionError(f"{who}: out is {out.shape}, expected {(m, n)}")
    if out.dtype != dt:
        raise DomainError(f"{who}: out must be {np.dtype(dt)}, got {out.dtype}")
    if not out.flags["C_CONTIGUOUS"] or not out.flags["WRITEABLE"]:
        raise DimensionError(f"{who}: out must be C-contiguous and writeable")
    return out


class Graph:
    """A captured fp64 multiply (small-N path: one graph launch per call)."""

    def __init__(self, ctx: "Context", handle: int, keep):
        self._ctx, self._h, self._keep = ctx, handle, keep

    def launch(self, stream=None) -> None:
        _check(_lib().mmws_gpu_graph_launch(self._h, _stream(stream)))

    def close(self) -> None:
        if self._h:
            _lib().mmws_gpu_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One CUDA device (sm_100a) + its stream, workspaces and NCCL communicator."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib().mmws_gpu_init(device, C.byref(h)))
        self._h = h.value
        self.device = device
        sms, ma, mi, clk = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_lib().mmws_gpu_device_info(self._h, C.byref(sms), C.byref(ma), C.byref(mi),
                                           C.byref(clk)))
        self.num_sms, self.cc, self.max_clock_khz = sms.value, (ma.value, mi.value), clk.value

    # -- lifecycle
    def close(self) -> None:
        if self._h:
            _lib().mmws_gpu_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> int:
        return self._h

    @property
    def launches(self) -> int:
        return int(_lib().mmws_gpu_launch_count(self._h))

    def tune(self, knob: str, value=None) -> None:
        """Set one MMWS_GPU_* knob on this context (None: default)."""
        _check(_lib().mmws_gpu_tune(self._h, knob.encode(),
                                    None if value is None else str(value).encode()))

    @property
    def stream(self) -> int:
        return int(_lib().mmws_gpu_stream(self._h) or 0)

    # -- device-pointer multiply (torch CUDA tensors)
    def dgemm(self, A, B, C_=None, mode: int = MODE_AUTO, stream=None, accumulate=None):
        """C_ = A . B; with `accumulate`, C_ = accumulate + A . B continuing its
        chains (mmws_gpu_dgemm_acc; `accumulate` may be C_ itself; K splits are
        bitwise the one call when every call takes the same kernel family --
        see include/mmws_gpu.h)."""
        import torch
        m, n, k = _device_operands(A, B, C_, torch.float64, "dgemm", self.device)
        if C_ is None:
            C_ = torch.empty((m, n), dtype=torch.float64, device=A.device)
        if accumulate is not None:
            _device_operands(A, B, accumulate, torch.float64, "dgemm", self.device)
            _check(_lib().mmws_gpu_dgemm_acc(self._h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                             _ptr(accumulate), _ld(accumulate), _ptr(C_), _ld(C_),
                                             mode, _stream(stream)))
            return C_
        _check(_lib().mmws_gpu_dgemm(self._h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                     _ptr(C_), _ld(C_), mode, _stream(stream)))
        return C_

    def sgemm(self, A, B, C_=None, mode: int = MODE_AUTO, stream=None, accumulate=None):
        """fp32 C_ = A . B; with `accumulate`, C_ = accumulate + A . B
        (mmws_gpu_sgemm_acc)."""
        import torch
        m, n, k = _device_operands(A, B, C_, torch.float32, "sgemm", self.device)
        if C_ is None:
            C_ = torch.empty((m, n), dtype=torch.float32, device=A.device)
        if accumulate is not None:
            _device_operands(A, B, accumulate, torch.float32, "sgemm", self.device)
            _check(_lib().mmws_gpu_sgemm_acc(self._h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                             _ptr(accumulate), _ld(accumulate), _ptr(C_), _ld(C_),
                                             mode, _stream(stream)))
            return C_
        _check(_lib().mmws_gpu_sgemm(self._h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                     _ptr(C_), _ld(C_), mode, _stream(stream)))
        return C_

    # -- host-buffer multiply (the matmul_seq / matmul_threads replacement)
    def matmul_host(self, a: np.ndarray, b: np.ndarray, mode: int = MODE_AUTO,
                    out: Optional[np.ndarray] = None) -> Tuple[np.ndarray, float]:
        if a.ndim != 2 or b.ndim != 2:
            raise DimensionError("matmul expects 2-D matrices")
        if a.shape[1] != b.shape[0]:
            raise DimensionError(f"matmul: inner dimensions differ, {a.shape[1]} vs {b.shape[0]}")
        f32 = a.dtype == np.float32
        dt = np.float32 if f32 else np.float64
        a = np.ascontiguousarray(a, dtype=dt)
        b = np.ascontiguousarray(b, dtype=dt)
        m, k = a.shape
        n = b.shape[1]
        c = _host_out(out, m, n, dt, "matmul")
        el = C.c_double()
        fn = _lib().mmws_gpu_matmul_host_f32 if f32 else _lib().mmws_gpu_matmul_host
        _check(fn(self._h, m, n, k, a.ctypes.data, b.ctypes.data, c.ctypes.data, mode,
                  C.byref(el)))
        return c, el.value

    # -- generators
    def fill(self, dist: int, seed: int, rows: int, cols: int, dtype=None, first: int = 0,
             out=None, stream=None):
        import torch
        dtype = dtype or torch.float64
        if dtype not in (torch.float64, torch.float32):
            raise DomainError(f"fill: dtype must be float64 or float32, got {dtype}")
        if out is not None:
            if out.dtype not in (torch.float64, torch.float32):
                raise DomainError(f"fill: out must be float64 or float32, got {out.dtype}")
            if not out.is_cuda or out.device.index != self.device:
                raise DomainError(f"fill: out is on {out.device}, the context on cuda:{self.device}")
            if out.dim() != 2 or out.shape[0] < rows or out.shape[1] < cols:
                raise DimensionError(f"fill: out is {tuple(out.shape)}, needs at least ({rows}, {cols})")
        t = out if out is not None else torch.empty((rows, cols), dtype=dtype,
                                                    device=f"cuda:{self.device}")
        _check(_lib().mmws_gpu_fill(self._h, dist, seed, _ptr(t), rows, cols, _ld(t),
                                    int(t.dtype == torch.float32), first, _stream(stream)))
        return t

    # -- graphs
    def graph_dgemm(self, A, B, C_, mode: int = MODE_AUTO) -> Graph:
        import torch
        if C_ is None:
            raise DomainError("graph_dgemm: C must be given (the graph writes into it on every replay)")
        m, n, k = _device_operands(A, B, C_, torch.float64, "graph_dgemm", self.device)
        g = C.c_void_p()
        _check(_lib().mmws_gpu_graph_dgemm(self._h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                           _ptr(C_), _ld(C_), mode, C.byref(g)))
        return Graph(self, g.value, (A, B, C_))

    # -- measurement
    def peak_probe(self, which: int, iters: int = 4096) -> float:
        out = C.c_double()
        _check(_lib().mmws_gpu_peak_probe(self._h, which, iters, C.byref(out)))
        return out.value

    def gemm_probe(self, n: int = 4096, mode: int = MODE_AUTO, iters: int = 3) -> float:
        """Device-resident n x n multiply rate in FLOP/s (cost-model calibration)."""
        out = C.c_double()
        _check(_lib().mmws_gpu_gemm_probe(self._h, n, mode, iters, C.byref(out)))
        return out.value

    def link_probe(self, nbytes: int = 1 << 28, iters: int = 5) -> float:
        """Collective: broadcast bandwidth from rank 0 in bytes/s (needs comm_init)."""
        out = C.c_double()
        _check(_lib().mmws_gpu_link_probe(self._h, nbytes, iters, C.byref(out)))
        return out.value

    def p2p_probe(self, nbytes: int = 1 << 28, iters: int = 5) -> float:
        """Collective: rank 0 -> each worker point-to-point copy rate in bytes/s
        (slowest peer on rank 0; 0 in a 1-rank world)."""
        out = C.c_double()
        _check(_lib().mmws_gpu_p2p_probe(self._h, nbytes, iters, C.byref(out)))
        return out.value

    def set_timeout(self, seconds: float) -> None:
        """Deadline of one distributed step (default 30 s, MMWS_GPU_TIMEOUT_S)."""
        _check(_lib().mmws_gpu_set_timeout(self._h, float(seconds)))

    @property
    def last_round(self):
        """(ranks that multiplied, gather) of the latest row-block call;
        gather in {"none", "fused-ipc", "nccl"}."""
        act, g = C.c_int(), C.c_int()
        _check(_lib().mmws_gpu_last_round(self._h, C.byref(act), C.byref(g), None))
        return act.value, {0: "none", 1: "fused-ipc", 2: "nccl"}[g.value]

    @property
    def last_b_panels(self) -> int:
        """k-panels B was broadcast in during the latest row-block call."""
        p = C.c_int()
        _check(_lib().mmws_gpu_last_round(self._h, None, None, C.byref(p)))
        return p.value

    # -- row-block distribution
    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(_lib().mmws_gpu_comm_init(self._h, nranks, rank, buf))

    def comm_destroy(self) -> None:
        _check(_lib().mmws_gpu_comm_destroy(self._h))

    def rowblock(self, m: int, n: int, k: int, A=None, B=None, C_=None, mode: int = MODE_AUTO,
                 f32: bool = False) -> float:
        """Collective master/worker multiply; rank 0 passes dense A (m x k), B
        (k x n), C (m x n) device tensors, the other ranks nothing."""
        if A is not None or B is not None or C_ is not None:
            import torch
            if A is None or B is None or C_ is None:
                raise DomainError("rowblock: rank 0 passes A, B and C")
            dt = torch.float32 if f32 else torch.float64
            _device_operands(A, B, C_, dt, "rowblock", self.device)
            if tuple(A.shape) != (m, k) or tuple(B.shape) != (k, n) or tuple(C_.shape) != (m, n):
                raise DimensionError(f"rowblock: shapes {tuple(A.shape)} x {tuple(B.shape)} -> "
                                     f"{tuple(C_.shape)} do not match m={m} n={n} k={k}")
            if not (A.is_contiguous() and B.is_contiguous() and C_.is_contiguous()):
                raise DimensionError("rowblock: A, B and C must be dense (contiguous)")
        # The round runs on the context's own stream (mmws_gpu.h): order it
        # after the work already queued on torch's current stream (e.g. the
        # kernels that produced A and B), as every other call here is.
        import torch
        torch.cuda.ExternalStream(self.stream, device=f"cuda:{self.device}").wait_stream(
            torch.cuda.current_stream(self.device))
        el = C.c_double(0.0)
        fn = _lib().mmws_gpu_rowblock_sgemm if f32 else _lib().mmws_gpu_rowblock_dgemm
        _check(fn(self._h, m, n, k, _ptr(A) if A is not None else None,
                  _ptr(B) if B is not None else None, _ptr(C_) if C_ is not None else None,
                  mode, C.byref(el)))
        return el.value


def _master_run_host(self, a=None, b=None, out=None, mode: int = MODE_AUTO, m=None, n=None,
                     k=None, f32: bool = False):
    """master_run (protocol.hpp:50-108) with host matrices on rank 0 (numpy
    arrays, pinned for full PCIe bandwidth); other ranks pass nothing but the
    shape.  Returns (C or None, elapsed_s)."""
    if a is not None:
        if b is None:
            raise DomainError("master_run: rank 0 passes both A and B")
        if a.ndim != 2 or b.ndim != 2:
            raise DimensionError("master_run expects 2-D matrices")
        if a.shape[1] != b.shape[0]:
            raise DimensionError(f"master_run: inner dimensions disagree, {a.shape[1]} vs {b.shape[0]}")
        m, k = a.shape
        n = b.shape[1]
        f32 = a.dtype == np.float32
        if a.dtype not in (np.float32, np.float64) or b.dtype != a.dtype:
            raise DomainError("master_run: A and B must both be float64 or both float32")
        out = _host_out(out, m, n, a.dtype, "master_run")
        for x in (a, b):
            if not x.flags["C_CONTIGUOUS"]:
                raise DimensionError("master_run: host matrices must be C-contiguous")
    elif m is None or n is None or k is None:
        raise DomainError("master_run: a worker rank passes the shape (m, n, k)")
    el = C.c_double()
    fn = _lib().mmws_gpu_master_run_host_f32 if f32 else _lib().mmws_gpu_master_run_host
    ptr = (lambda x: x.ctypes.data if x is not None else None)
    _check(fn(self._h, m, n, k, ptr(a), ptr(b), ptr(out), mode, C.byref(el)))
    return out, el.value


def _server_start(self) -> None:
    """Start the resident latency server (tiny multiplies, m, n, k <= 96)."""
    _check(_lib().mmws_gpu_server_start(self._h))


def _server_matmul(self, a: np.ndarray, b: np.ndarray, mode: int = MODE_AUTO,
                   out: Optional[np.ndarray] = None) -> Tuple[np.ndarray, float]:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape[1] != b.shape[0]:
        raise DimensionError(f"matmul: inner dimensions differ, {a.shape[1]} vs {b.shape[0]}")
    m, k = a.shape
    n = b.shape[1]
    c = _host_out(out, m, n, np.float64, "server_matmul")
    el = C.c_double()
    _check(_lib().mmws_gpu_server_dgemm(self._h, m, n, k, a.ctypes.data, k, b.ctypes.data, n,
                                        c.ctypes.data, n, mode, C.byref(el)))
    return c, el.value


def _server_stop(self) -> None:
    _check(_lib().mmws_gpu_server_stop(self._h))


Context.server_start = _server_start
Context.server_matmul = _server_matmul
Context.server_stop = _server_stop


def _last_kernel_ms(self) -> float:
    out = C.c_double()
    _check(_lib().mmws_gpu_last_kernel_ms(self._h, C.byref(out)))
    return out.value


def _last_plan(self) -> str:
    out = C.c_char_p()
    _check(_lib().mmws_gpu_last_plan(self._h, C.byref(out)))
    return (out.value or b"").decode()


Context.master_run_host = _master_run_host
Context.last_kernel_ms = property(_last_kernel_ms)
Context.last_plan = property(_last_plan)


def bootstrap_comm(ctx: Context) -> None:
    """NCCL communicator for the current torch.distributed world: rank 0 makes
    the unique id, torch.distributed ships it (plumbing only)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.comm_init(world, rank, obj[0])

"""paper_1012_2273_b200 -- B200-native dense N x N matmul (the hot path of
arxiv/paper_1012_2273's "mmws" reference) behind the reference's API.

Product: libmmws_gpu.so (csrc/, sm_100a CUDA + NCCL) with the C ABI in
include/mmws_gpu.h and the C++ drop-in adapter include/mmws_gpu.hpp.  This
Python package is the ctypes binding used by tests and bench.py.
"""
from .api import (Context, DimensionError, DomainError, GpuError, Graph, ProtocolError,  # noqa: F401
                  RankError, TimeoutError, bootstrap_comm, nccl_unique_id, op_count, ozaki_plan, rowblock_cost,
                  rowblock_ranks,
                  rowblock_plan,
                  split_rows, static_partition)
from ._abi import (GATHER_FUSED, GATHER_NCCL, GATHER_NONE, DIST_INT8, DIST_NORMAL, DIST_UNIFORM, DIST_UNIT, MODE_AUTO, MODE_DMMA,  # noqa: F401
                   MODE_DMMA_SMALL, MODE_EXACT, MODE_FFMA, MODE_OZAKI, PROBE_DFMA, PROBE_DMMA,
                   PROBE_DMUL_DADD, PROBE_FFMA, PROBE_FFMA2,
                   PROBE_FFMA2_OUTER)

"""Multi-process (gloo, CPU) test of the row-block master/worker host logic.

The GPU engine (csrc/rowblock.cu) executes, on every rank, split_rows(m, P)
and rank 0's message plan (mmws_gpu_rowblock_plan): A-slices out, one B
broadcast, C-slices back into C's row blocks.  Only one GPU is available to
this build, so the N > 1 path is exercised here with real processes: the same
plan from the product library, the exchange over torch.distributed gloo, and
the oracle's worker_block (protocol.hpp:132-141) standing in for the GPU
kernel.  Mirrors the reference's msg-vs-seq matrix (acceptance.cpp:112-133,
test_protocol.cpp:76-89): bitwise equal to matmul_seq, idle workers included.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _b_span(e, k, n):
    """Elements of B a broadcast entry covers: all of it (row0 -1) or the
    k-panel of rows [row0, row0 + count / n)."""
    lo = 0 if e["row0"] < 0 else e["row0"] * n
    assert e["count"] % n == 0 and lo + e["count"] <= k * n
    return slice(lo, lo + e["count"])


def _rank_main(rank, world, port, cases, failures):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_1012_2273_b200 as P

    dist.init_process_group("gloo", rank=rank, world_size=world,
                            init_method=f"tcp://127.0.0.1:{port}")
    try:
        for (m, k, n, sa, sb) in cases:
            # rank 0's plan is the single schedule; a worker follows the
            # entries addressed to it, in order (as the NCCL engine does)
            plan = P.rowblock_plan(m, n, k, world)
            off, rows = P.split_rows(m, world)[rank]
            if rank == 0:
                a = O.fill(O.DIST_UNIT, sa, m, k)
                b = O.fill(O.DIST_UNIT, sb, k, n)
                c = np.full((m, n), np.nan)
                if rows:
                    c[off:off + rows] = O.worker_block(a[off:off + rows], b)
                for e in plan:
                    if e["dir"] == "broadcast":                # B, or one k-panel of it
                        dist.broadcast(torch.from_numpy(b).reshape(-1)[_b_span(e, k, n)], 0)
                    elif e["dir"] == "sent":               # tag 1: A sub-slice
                        r0, nr = e["row0"], e["count"] // k
                        dist.send(torch.from_numpy(np.ascontiguousarray(a[r0:r0 + nr])), e["peer"])
                    else:                                  # tag 2: C sub-slice
                        r0, nr = e["row0"], e["count"] // n
                        buf = torch.empty((nr, n), dtype=torch.float64)
                        dist.recv(buf, e["peer"])
                        c[r0:r0 + nr] = buf.numpy()
                want = O.matmul_seq(a, b)
                if O.first_difference(c, want) is not None:
                    failures.append(f"m={m} k={k} n={n} world={world}")
                covered = sum(e["count"] // n for e in plan if e["dir"] == "received") + rows
                if world > 1 and covered != m:
                    failures.append(f"coverage m={m} world={world}")
            else:
                a_loc = np.zeros((rows, k))
                b = torch.empty((k, n), dtype=torch.float64)
                for e in plan:
                    if e["dir"] == "broadcast":
                        dist.broadcast(b.reshape(-1)[_b_span(e, k, n)], 0)
                    elif e["peer"] != rank:
                        continue
                    elif e["dir"] == "sent":
                        r0, nr = e["row0"] - off, e["count"] // k
                        buf = torch.empty((nr, k), dtype=torch.float64)
                        dist.recv(buf, 0)
                        a_loc[r0:r0 + nr] = buf.numpy()
                    else:                                  # multiply the sub-block, reply
                        r0, nr = e["row0"] - off, e["count"] // n
                        c_sub = O.worker_block(a_loc[r0:r0 + nr], b.numpy())
                        dist.send(torch.from_numpy(c_sub), 0)
    finally:
        dist.destroy_process_group()


def _run(world, cases):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    failures = mgr.list()
    port = _free_port()
    mp.spawn(_rank_main, args=(world, port, cases, failures), nprocs=world, join=True)
    return list(failures)


ACCEPT = [(n, n, n, 3000 + n, 4000 + n) for n in (1, 2, 3, 4, 8, 16, 33)]
RECT = [(5, 7, 4, 31, 32), (2, 2, 2, 61, 62), (513, 67, 129, 7, 8)]
SUBBLOCKS = [(2048 * 5 + 3, 7, 5, 9, 10)]   # >= 1024 rows per rank: two sub-blocks each
# B big enough to go out in k-panels (>= 64 Mi elements): 2 panels of 1024 rows
PANELS = [(3, 2048, 32768, 11, 12)]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_rowblock_gloo_bitwise_equals_seq(world):
    assert _run(world, ACCEPT + RECT + SUBBLOCKS) == []


def test_rowblock_gloo_b_in_k_panels():
    # the panel plan (first A sub-blocks, B as k-panels, the other A
    # sub-blocks, C-slices) replayed by 2 processes; workers multiply only
    # after every panel landed here (the GPU continues accumulators panel by
    # panel -- bitwise the same, tests/test_gpu_parity.py accumulate tests)
    m, k, n = PANELS[0][:3]
    plan = __import__("paper_1012_2273_b200").rowblock_plan(m, n, k, 2)
    assert [e["dir"] for e in plan].count("broadcast") == 2
    assert _run(2, PANELS) == []


# ----------------------------------------------------------------------------- fused gather
def _rank_main_fused(rank, world, port, cases, failures, refuse_rank):
    """The default (fused) C gather of csrc/rowblock.cu, replayed by real
    processes: rank 0 "exports" its C (a shared-memory file standing in for
    the CUDA IPC handle) and broadcasts the handle; every rank maps it and
    votes (allreduce-min) -- a rank that cannot map it (refuse_rank) sends the
    whole world to the NCCL-style C-slice messages; B is broadcast, the A
    sub-slices sent; each worker stores its rows straight into the mapped C
    (the GEMM epilogue's peer stores); an allreduce of a token after every
    rank's last multiply is the completion barrier, after which rank 0's C
    must be bitwise matmul_seq."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from multiprocessing import shared_memory

    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_1012_2273_b200 as P

    dist.init_process_group("gloo", rank=rank, world_size=world,
                            init_method=f"tcp://127.0.0.1:{port}")
    try:
        for ci, (m, k, n, sa, sb) in enumerate(cases):
            plan = P.rowblock_plan(m, n, k, world)
            off, rows = P.split_rows(m, world)[rank]
            shm = None
            # ---- handle broadcast (80 bytes in the engine)
            name = [f"mmws_fused_{port}_{ci}" if rank == 0 else None]
            if rank == 0:
                shm = shared_memory.SharedMemory(name=name[0], create=True, size=8 * m * n)
            dist.broadcast_object_list(name, src=0)
            ok_here = 1
            if rank != 0:
                try:
                    if rank == refuse_rank:
                        raise OSError("cannot map")
                    shm = shared_memory.SharedMemory(name=name[0])
                except OSError:
                    ok_here = 0
            # ---- vote: allreduce-min
            vote = torch.tensor([ok_here], dtype=torch.int32)
            dist.all_reduce(vote, op=dist.ReduceOp.MIN)
            fused = bool(vote.item())
            c = np.ndarray((m, n), dtype=np.float64, buffer=shm.buf) if shm is not None else None
            if rank == 0:
                c[:] = np.nan
                a = O.fill(O.DIST_UNIT, sa, m, k)
                b = O.fill(O.DIST_UNIT, sb, k, n)
            else:
                a = np.zeros((rows, k))
                b = np.zeros((k, n))
            bt = torch.from_numpy(b)
            c_loc = np.zeros((rows, n))
            for e in plan:
                if e["dir"] == "broadcast":
                    dist.broadcast(bt.reshape(-1)[_b_span(e, k, n)], 0)
                elif e["dir"] == "sent":                       # A sub-slices
                    r0, nr = e["row0"], e["count"] // k
                    if rank == 0:
                        dist.send(torch.from_numpy(np.ascontiguousarray(a[r0:r0 + nr])), e["peer"])
                    elif e["peer"] == rank:
                        buf = torch.empty((nr, k), dtype=torch.float64)
                        dist.recv(buf, 0)
                        a[r0 - off:r0 - off + nr] = buf.numpy()
            b = bt.numpy()
            # ---- every rank multiplies its rows; fused: stores into rank 0's C
            if rows:
                block = O.worker_block(a[off:off + rows] if rank == 0 else a, b)
                if rank == 0 or fused:
                    c[off:off + rows] = block
                else:
                    c_loc[:] = block
            if fused:                                          # completion barrier
                token = torch.zeros(1, dtype=torch.int32)
                dist.all_reduce(token)
            else:                                              # C-slice messages
                for e in plan:
                    if e["dir"] != "received":
                        continue
                    r0, nr = e["row0"], e["count"] // n
                    if rank == 0:
                        buf = torch.empty((nr, n), dtype=torch.float64)
                        dist.recv(buf, e["peer"])
                        c[r0:r0 + nr] = buf.numpy()
                    elif e["peer"] == rank:
                        dist.send(torch.from_numpy(np.ascontiguousarray(
                            c_loc[r0 - off:r0 - off + nr])), 0)
            if rank == 0:
                want = O.matmul_seq(a, b)
                if O.first_difference(c, want) is not None:
                    failures.append(f"fused={fused} m={m} k={k} n={n} world={world}")
                if fused != (refuse_rank is None or refuse_rank >= world):
                    failures.append(f"vote gave fused={fused} with refuse_rank={refuse_rank}")
            dist.barrier()
            if shm is not None:
                shm.close()
                if rank == 0:
                    shm.unlink()
    finally:
        dist.destroy_process_group()


def _run_fused(world, cases, refuse_rank):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    failures = mgr.list()
    port = _free_port()
    mp.spawn(_rank_main_fused, args=(world, port, cases, failures, refuse_rank), nprocs=world,
             join=True)
    return list(failures)


@pytest.mark.parametrize("world,refuse_rank", [(2, None), (3, None), (5, None), (3, 2)])
def test_rowblock_gloo_fused_gather_bitwise_equals_seq(world, refuse_rank):
    assert _run_fused(world, ACCEPT[:5] + RECT + SUBBLOCKS, refuse_rank) == []


def test_rowblock_gloo_fused_gather_with_b_panels():
    assert _run_fused(2, PANELS, None) == []

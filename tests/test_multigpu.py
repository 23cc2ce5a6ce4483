"""Row-block master/worker across real GPUs (one process per GPU, NCCL).

The reference's msg-vs-seq matrix (acceptance.cpp:112-133,
test_protocol.cpp:76-89,139-157) and its dead-worker test
(test_protocol.cpp:171-178) on B200s: P-GPU products are bitwise the 1-GPU
product (every rank runs the same kernel configuration with an
M-independent k-order), exact-mode rows match the reference-generated
goldens, idle ranks and ragged blocks work, both C gathers (fused peer
stores over NVLink, NCCL C-slices) give the same bits, and a worker that
leaves the world surfaces on rank 0 as a ProtocolError naming it.

Tests that need P GPUs skip on boxes with fewer; the 1-GPU failure-detection
tests run everywhere a GPU is.
"""
import hashlib
import os
import socket
import time

import numpy as np
import pytest

import paper_1012_2273_b200 as P

pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _need(p):
    if _gpus() < p:
        pytest.skip(f"needs {p} GPUs, this box has {_gpus()}")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ----------------------------------------------------------------------------- rank driver
def _rank_main(rank, world, port, job, results):
    """One rank: NCCL world over torch.distributed (plumbing), then `job`."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = P.Context(rank)
    try:
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_timeout(60)
        ctx.comm_init(world, rank, uid[0])
        out = JOBS[job](ctx, rank, world, dist)
        results.put((rank, "ok", out))
    except Exception as exc:  # reported to the parent
        results.put((rank, "error", f"{type(exc).__name__}: {exc}"))
    finally:
        try:
            ctx.close()
        except Exception:
            pass
        dist.destroy_process_group()


def _run(world, job, timeout=600):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, job, results))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    deadline = time.time() + timeout
    while len(out) < world and time.time() < deadline:
        try:
            r, status, val = results.get(timeout=5)
            out[r] = (status, val)
        except Exception:
            if all(not p.is_alive() for p in procs) and results.empty():
                break
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    return out


def _ok(out, world):
    assert len(out) == world, out
    bad = {r: v for r, v in out.items() if v[0] != "ok"}
    assert not bad, bad
    return {r: v[1] for r, v in out.items()}


# ----------------------------------------------------------------------------- jobs
def _bits_sha(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def _job_fp64(ctx, rank, world, dist):
    """configs[3] N=16384 fp64 AUTO and a ragged N=4099 integer case; rank 0
    compares with its own 1-GPU product."""
    import torch
    res = {}
    for (n, dist_kind, modes) in ((16384, P.DIST_UNIFORM, (P.MODE_AUTO,)),
                                  (4099, P.DIST_INT8, (P.MODE_AUTO, P.MODE_EXACT)),
                                  (2053, P.DIST_UNIFORM, (P.MODE_AUTO, P.MODE_EXACT))):
        for mode in modes:
            ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
            if rank == 0:
                A = ctx.fill(dist_kind, 0, n, n)
                B = ctx.fill(dist_kind, 1, n, n)
                C = torch.empty_like(A)
                ctx.rowblock(n, n, n, A, B, C, mode=mode)
                active, gather = ctx.last_round
                want = ctx.dgemm(A, B, mode=mode)
                torch.cuda.synchronize()
                res[(n, mode)] = {"bitwise_1gpu": bool(torch.equal(C.view(torch.int64),
                                                                     want.view(torch.int64))),
                                  "active": active, "gather": gather, "sha": _bits_sha(C)}
                del A, B, C, want
            else:
                ctx.rowblock(n, n, n, mode=mode)
    return res


def _job_fp32(ctx, rank, world, dist):
    """configs[4] N=32768 fp32 FFMA: bitwise the 1-GPU product; sampled rows
    normwise against an fp64 product of the widened inputs."""
    import torch
    n = 32768
    if rank != 0:
        ctx.rowblock(n, n, n, mode=P.MODE_FFMA, f32=True)
        return None
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
    C = torch.empty_like(A)
    ctx.rowblock(n, n, n, A, B, C, mode=P.MODE_FFMA, f32=True)
    active, gather = ctx.last_round
    want = ctx.sgemm(A, B, mode=P.MODE_FFMA)
    rows = torch.tensor([0, 1, n // 2, n - 1], device=A.device)
    ref = A.index_select(0, rows).double() @ B.double()
    err = float(torch.linalg.norm(C.index_select(0, rows).double() - ref) / torch.linalg.norm(ref))
    torch.cuda.synchronize()
    return {"bitwise_1gpu": bool(torch.equal(C.view(torch.int32), want.view(torch.int32))),
            "err": err, "active": active, "gather": gather}


def _job_exact_rows(ctx, rank, world, dist):
    """configs[3] in exact mode: sampled rows against the sha256 of the
    reference's own matmul_seq rows (tests/golden/ref_big.json)."""
    import json
    import torch
    n = 16384
    if rank != 0:
        ctx.rowblock(n, n, n, mode=P.MODE_EXACT)
        return None
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    ctx.rowblock(n, n, n, A, B, C, mode=P.MODE_EXACT)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "ref_big.json")) as f:
        g = json.load(f)
    got = [hashlib.sha256(C[r].cpu().numpy().tobytes()).hexdigest() for r in g["n16384_rows"]]
    return {"match": got == g["n16384_rows_sha256"], "gather": ctx.last_round[1]}


def _job_idle_and_gathers(ctx, rank, world, dist):
    """m < P (idle ranks still take part, protocol.hpp:122-123), tiny and
    rectangular shapes, forced distribution, both gathers."""
    import torch
    res = {}
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    for gather_knob in (None, "1"):
        ctx.tune("MMWS_GPU_NCCL_GATHER", gather_knob)
        for (m, k, n) in ((1, 1, 1), (2, 3, 2), (world - 1, 5, 7), (33, 33, 33), (1031, 517, 263)):
            for mode in (P.MODE_AUTO, P.MODE_EXACT):
                if rank == 0:
                    A = ctx.fill(P.DIST_UNIFORM, 3000 + m, m, k)
                    B = ctx.fill(P.DIST_UNIFORM, 4000 + m, k, n)
                    C = torch.full((m, n), float("nan"), dtype=torch.float64, device=A.device)
                    ctx.rowblock(m, n, k, A, B, C, mode=mode)
                    want = ctx.dgemm(A, B, mode=mode)
                    torch.cuda.synchronize()
                    res[(gather_knob, m, k, n, mode)] = (
                        bool(torch.equal(C.view(torch.int64), want.view(torch.int64))),
                        ctx.last_round)
                else:
                    ctx.rowblock(m, n, k, mode=mode)
    return res


def _job_dead_worker(ctx, rank, world, dist):
    """Rank 1 joins the world, then leaves without serving the round
    (test_protocol.cpp:171-178's "join-only" worker)."""
    import torch
    if rank == 1:
        return "left"
    ctx.set_timeout(10)
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    n = 512
    A = ctx.fill(P.DIST_UNIFORM, 81, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 82, n, n)
    C = torch.empty_like(A)
    t0 = time.time()
    try:
        ctx.rowblock(n, n, n, A, B, C)
    except (P.ProtocolError, P.TimeoutError) as exc:
        took = time.time() - t0
        # afterwards: every row-block call fails until the communicator is rebuilt
        try:
            ctx.rowblock(n, n, n, A, B, C)
            state = "no error"
        except P.GpuError as e2:
            state = str(e2)
        ctx.comm_destroy()
        ctx.rowblock(n, n, n, A, B, C)  # no communicator: one multiply
        return {"type": type(exc).__name__, "msg": str(exc), "took": took, "after": state}
    return {"type": None}


JOBS = {"fp64": _job_fp64, "fp32": _job_fp32, "exact_rows": _job_exact_rows,
        "idle": _job_idle_and_gathers, "dead": _job_dead_worker}


# ----------------------------------------------------------------------------- tests
@pytest.mark.parametrize("world", [2, 4, 8])
def test_rowblock_fp64_bitwise_equals_one_gpu(world):
    _need(world)
    res = _ok(_run(world, "fp64"), world)[0]
    for key, v in res.items():
        assert v["bitwise_1gpu"], (key, v)
        assert v["active"] == world and v["gather"] == "fused-ipc", (key, v)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "ref_big.json")) as f:
        import json
        want = json.load(f)["n4099_int8_sha256"]
    assert res[(4099, P.MODE_AUTO)]["sha"] == want
    assert res[(4099, P.MODE_EXACT)]["sha"] == want


@pytest.mark.parametrize("world", [2, 8])
def test_rowblock_fp32_bitwise_equals_one_gpu(world):
    _need(world)
    res = _ok(_run(world, "fp32"), world)[0]
    assert res["bitwise_1gpu"] and res["err"] <= 1e-5 and res["active"] == world, res


def test_rowblock_exact_rows_match_reference_goldens():
    world = _gpus()
    _need(2)
    res = _ok(_run(world, "exact_rows"), world)[0]
    assert res["match"], res


@pytest.mark.parametrize("world", [2, 3])
def test_rowblock_idle_ranks_and_both_gathers(world):
    _need(world)
    res = _ok(_run(world, "idle"), world)[0]
    for key, (same, (active, gather)) in res.items():
        assert same, key
        assert active == world, key
        assert gather == ("nccl" if key[0] == "1" else "fused-ipc"), (key, gather)


def test_dead_worker_is_a_protocol_error_naming_the_rank():
    _need(2)
    out = _ok(_run(2, "dead", timeout=300), 2)
    r0 = out[0]
    assert r0["type"] == "ProtocolError", r0
    assert "rank 1" in r0["msg"], r0
    assert r0["took"] < 40, r0
    assert "destroy" in r0["after"], r0


# --------------------------------------------------------------- one GPU: the deadline itself
def test_comm_init_times_out_when_the_world_never_assembles():
    """A 2-rank world whose rank 1 never calls comm_init: rank 0 gives up at
    the deadline with TimeoutError (comm.hpp:144's "deadlock-suspected"),
    its context stays usable, and a new communicator can be built."""
    import torch
    c = P.Context(0)
    try:
        c.set_timeout(3)
        t0 = time.time()
        with pytest.raises(P.TimeoutError) as ei:
            c.comm_init(2, 0, P.nccl_unique_id())
        took = time.time() - t0
        assert 2.5 < took < 30, took
        assert "deadlock-suspected" in str(ei.value)
        n = 300
        A = c.fill(P.DIST_UNIFORM, 0, n, n)
        B = c.fill(P.DIST_UNIFORM, 1, n, n)
        C = torch.empty_like(A)
        c.comm_init(1, 0, P.nccl_unique_id())          # the context recovers
        c.rowblock(n, n, n, A, B, C, mode=P.MODE_EXACT)
        assert torch.equal(C, c.dgemm(A, B, mode=P.MODE_EXACT))
        c.comm_destroy()
    finally:
        c.close()


def test_one_rank_world_reports_gather_and_forced_nccl_gather():
    import torch
    c = P.Context(0)
    try:
        c.comm_init(1, 0, P.nccl_unique_id())
        n = 2304
        A = c.fill(P.DIST_UNIFORM, 0, n, n)
        B = c.fill(P.DIST_UNIFORM, 1, n, n)
        want = c.dgemm(A, B)
        for knob, gather in ((None, "fused-ipc"), ("1", "nccl"), (None, "fused-ipc")):
            c.tune("MMWS_GPU_NCCL_GATHER", knob)
            C = torch.empty_like(A)  # a new allocation: a new handle, a new vote
            c.rowblock(n, n, n, A, B, C)
            assert c.last_round == (1, gather)
            assert torch.equal(C.view(torch.int64), want.view(torch.int64))
        a, b = A.cpu().numpy(), B.cpu().numpy()
        c.tune("MMWS_GPU_NCCL_GATHER", None)
        got, el = c.master_run_host(a, b)
        assert el > 0 and np.array_equal(got.view(np.int64), want.cpu().numpy().view(np.int64))
        assert c.p2p_probe(1 << 20, 2) == 0.0          # no peers in a 1-rank world
        assert c.link_probe(1 << 20, 2) > 0
        c.comm_destroy()
        assert c.last_round[0] == 1
    finally:
        c.close()


def test_tune_rejects_unknown_knobs(ctx):
    with pytest.raises(P.DomainError):
        ctx.tune("MMWS_GPU_NOT_A_KNOB", "1")
    ctx.tune("MMWS_GPU_TIMEOUT_S", "30")
    with pytest.raises(P.DomainError):
        ctx.set_timeout(0)


def test_one_rank_host_round_streams_b_in_panels():
    """master_run from host memory in a 1-rank world with a B big enough for
    k-panels: rank 0 copies its rows and B's panels in over PCIe piece by
    piece and multiplies panel by panel as they land (accumulator
    continuation), its own C rows go back before the round's barrier --
    bitwise the one-call product, pinned and pageable."""
    import torch
    c = P.Context(0)
    try:
        c.comm_init(1, 0, P.nccl_unique_id())
        m, k, n = 1100, 8192, 8192          # B = 64 Mi elements: 2 panels of 4096 rows
        A = c.fill(P.DIST_UNIFORM, 5, m, k)
        B = c.fill(P.DIST_UNIFORM, 6, k, n)
        a, b = A.cpu().numpy(), B.cpu().numpy()
        for mode in (P.MODE_AUTO, P.MODE_EXACT):
            want = c.dgemm(A, B, mode=mode).cpu().numpy()
            got, el = c.master_run_host(a, b, mode=mode)                       # pageable
            assert el > 0 and c.last_b_panels == 2 and c.last_round == (1, "fused-ipc")
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), mode
            ap = torch.from_numpy(a).pin_memory().numpy()
            bp = torch.from_numpy(b).pin_memory().numpy()
            cp = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
            got, _ = c.master_run_host(ap, bp, cp, mode=mode)                  # pinned
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), mode
        # fp32 through the same host round (panel edges at multiples of 1024)
        Af, Bf = A.float(), B.float()
        want = c.sgemm(Af, Bf).cpu().numpy()
        got, _ = c.master_run_host(Af.cpu().numpy(), Bf.cpu().numpy())
        assert np.array_equal(got.view(np.int32), want.view(np.int32))
        # MODE_OZAKI cannot continue accumulators: its host round keeps B in one piece
        want = c.dgemm(A, B, mode=P.MODE_OZAKI).cpu().numpy()
        got, _ = c.master_run_host(a, b, mode=P.MODE_OZAKI)
        assert c.last_b_panels == 1
        assert np.array_equal(got.view(np.int64), want.view(np.int64))
        # device-resident rounds in a 1-rank world keep B in one piece
        C = torch.empty((m, n), dtype=torch.float64, device="cuda")
        c.rowblock(m, n, k, A, B, C)
        assert c.last_b_panels == 1
        c.comm_destroy()
    finally:
        c.close()

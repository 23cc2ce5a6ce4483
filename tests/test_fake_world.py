"""The row-block master/worker engine with every rank's side executing on the
GPU -- several processes on ONE B200.

NCCL refuses two ranks on one device, so these tests load a loopback
stand-in for its entry points (tests/fake_nccl/fake_nccl.cpp, test
infrastructure only: device-to-device copies between the processes' buffers
through CUDA IPC, host rendezvous in shared memory) via MMWS_GPU_NCCL_LIB.
Everything else is the product path: the workers receive their A rows and
B (in k-panels where the round uses them), multiply panel by panel with
accumulator continuation, store their C rows straight into rank 0's C
through the CUDA IPC mapping (fused gather) or send them back (NCCL-style
gather), mark their progress on rank 0's board, and rank 0 names a worker
that left (test_protocol.cpp:171-178).  Results must be bitwise rank 0's own
one-GPU product.  No kernel waits on another process's kernel (the B200
profiling guide's Xid-109 warning): cross-process ordering is host
rendezvous plus stream waits on IPC events.
"""
import os
import secrets
import subprocess
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fake_lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("fake_nccl") / "libfake_nccl.so"
    subprocess.run(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cpp"), "-o", str(out),
                    "-L/usr/local/cuda/lib64/stubs", "-lcuda"], check=True)
    return str(out)


def _uid(name: str) -> bytes:
    raw = name.encode()
    return raw + b"\0" * (128 - len(raw))


def _rank_main(rank, world, lib, name, job, results):
    os.environ["MMWS_GPU_NCCL_LIB"] = lib
    import sys
    sys.path.insert(0, ROOT)
    import paper_1012_2273_b200 as P
    ctx = P.Context(0)
    try:
        ctx.set_timeout(60)
        ctx.comm_init(world, rank, _uid(name))
        out = JOBS[job](P, ctx, rank, world)
        results.put((rank, "ok", out))
    except Exception as exc:
        results.put((rank, "error", f"{type(exc).__name__}: {exc}"))
    finally:
        try:
            ctx.close()
        except Exception:
            pass


def _run(world, lib, job, timeout=600):
    import torch.multiprocessing as mp
    mpc = mp.get_context("spawn")
    results = mpc.Queue()
    name = "/mmws_fake_nccl_" + secrets.token_hex(8)
    procs = [mpc.Process(target=_rank_main, args=(r, world, lib, name, job, results))
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


def _same(a, b):
    import torch
    return bool(torch.equal(a.view(torch.int64 if a.dtype == torch.float64 else torch.int32),
                            b.view(torch.int64 if b.dtype == torch.float64 else torch.int32)))


# ----------------------------------------------------------------------------- jobs
CASES = [  # (m, k, n, dtype, mode name): one-piece B with two sub-blocks, B in k-panels
    (2304, 2304, 2304, "f64", "auto"), (2304, 2304, 2304, "f64", "exact"),
    (2100, 8192, 8192, "f64", "auto"), (2100, 8192, 8192, "f32", "ffma"),
]


def _job_rounds(P, ctx, rank, world):
    import torch
    modes = {"auto": P.MODE_AUTO, "exact": P.MODE_EXACT, "ffma": P.MODE_FFMA}
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    res = []
    for gather in (None, "1"):
        ctx.tune("MMWS_GPU_NCCL_GATHER", gather)
        for (m, k, n, dt, mode_name) in CASES:
            mode, f32 = modes[mode_name], dt == "f32"
            tdt = torch.float32 if f32 else torch.float64
            dist = P.DIST_NORMAL if f32 else P.DIST_UNIFORM
            if rank == 0:
                A = ctx.fill(dist, 11, m, k, dtype=tdt)
                B = ctx.fill(dist, 12, k, n, dtype=tdt)
                C = torch.full((m, n), float("nan"), dtype=tdt, device="cuda")
                ctx.rowblock(m, n, k, A, B, C, mode=mode, f32=f32)
                info = (ctx.last_round, ctx.last_b_panels)
                want = (ctx.sgemm if f32 else ctx.dgemm)(A, B, mode=mode)
                torch.cuda.synchronize()
                res.append((gather, m, k, n, dt, mode_name, info, _same(C, want)))
                del A, B, C, want
            else:
                ctx.rowblock(m, n, k, mode=mode, f32=f32)
    # master_run from pageable host memory (the e2e entry), B in k-panels
    ctx.tune("MMWS_GPU_NCCL_GATHER", None)
    m, k, n = 2100, 8192, 8192
    if rank == 0:
        A = ctx.fill(P.DIST_UNIFORM, 21, m, k)
        B = ctx.fill(P.DIST_UNIFORM, 22, k, n)
        want = ctx.dgemm(A, B).cpu().numpy()
        got, el = ctx.master_run_host(A.cpu().numpy(), B.cpu().numpy())
        res.append(("host", m, k, n, "f64", "auto", (ctx.last_round, ctx.last_b_panels),
                    bool(np.array_equal(got.view(np.int64), want.view(np.int64))) and el > 0))
    else:
        ctx.master_run_host(None, None, None, m=m, n=n, k=k)
    return res


def _job_dead(P, ctx, rank, world):
    """rank 1 joins, then leaves without serving a round"""
    import torch
    if rank == 1:
        return "left"
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
        try:
            ctx.rowblock(n, n, n, A, B, C)
            after = "no error"
        except P.GpuError as e2:
            after = str(e2)
        ctx.comm_destroy()
        ctx.rowblock(n, n, n, A, B, C)   # no communicator: one multiply
        ok = _same(C, ctx.dgemm(A, B))
        return {"type": type(exc).__name__, "msg": str(exc), "took": took, "after": after,
                "recovered": ok}
    return {"type": None}


def _job_ragged(P, ctx, rank, world):
    """configs[2] over `world` ranks: N=4099 integer inputs, ragged split_rows
    blocks (513 x 3 + 512 x 5 at 8 ranks), AUTO and EXACT -- sha256 of C
    against the reference-generated golden; then idle ranks (m < P)."""
    import hashlib
    import json
    import torch
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    out = {}
    n = 4099
    for name, mode in (("auto", P.MODE_AUTO), ("exact", P.MODE_EXACT)):
        if rank == 0:
            A = ctx.fill(P.DIST_INT8, 0, n, n)
            B = ctx.fill(P.DIST_INT8, 1, n, n)
            C = torch.empty_like(A)
            ctx.rowblock(n, n, n, A, B, C, mode=mode)
            out[name] = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()
            del A, B, C
        else:
            ctx.rowblock(n, n, n, mode=mode)
    if rank == 0:
        with open(os.path.join(ROOT, "tests", "golden", "ref_big.json")) as f:
            out["golden"] = json.load(f)["n4099_int8_sha256"]
        out["split"] = P.split_rows(n, world)
    m = world - 2                      # idle ranks: fewer rows than ranks
    if rank == 0:
        A = ctx.fill(P.DIST_UNIFORM, 3, m, 33)
        B = ctx.fill(P.DIST_UNIFORM, 4, 33, 17)
        C = torch.full((m, 17), float("nan"), dtype=torch.float64, device="cuda")
        ctx.rowblock(m, 17, 33, A, B, C, mode=P.MODE_EXACT)
        out["idle"] = _same(C, ctx.dgemm(A, B, mode=P.MODE_EXACT))
    else:
        ctx.rowblock(m, 17, 33, mode=P.MODE_EXACT)
    return out


def _job_config3(P, ctx, rank, world):
    """configs[3] at its real size over `world` ranks (S = 2 sub-blocks, B in
    8 k-panels): bitwise the one-GPU product, AUTO fp64 and fp32 FFMA."""
    import torch
    n = 16384
    out = {}
    for f32 in (False, True):
        mode = P.MODE_FFMA if f32 else P.MODE_AUTO
        if rank == 0:
            dt = torch.float32 if f32 else torch.float64
            dist = P.DIST_NORMAL if f32 else P.DIST_UNIFORM
            A = ctx.fill(dist, 0, n, n, dtype=dt)
            B = ctx.fill(dist, 1, n, n, dtype=dt)
            C = torch.empty_like(A)
            ctx.rowblock(n, n, n, A, B, C, mode=mode, f32=f32)
            panels = ctx.last_b_panels
            want = (ctx.sgemm if f32 else ctx.dgemm)(A, B, mode=mode)
            out["f32" if f32 else "f64"] = (_same(C, want), panels, ctx.last_round)
            del A, B, C, want
            torch.cuda.empty_cache()
        else:
            ctx.rowblock(n, n, n, mode=mode, f32=f32)
    return out


def _job_slow(P, ctx, rank, world):
    """test_protocol.cpp:160-168: a worker that stalls before serving is waited
    for (no false deadline), and the round's result is still exact."""
    import torch
    ctx.set_timeout(5)
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    n = 300
    if rank == 1:
        time.sleep(3)                   # stalls before the round, within the deadline
    if rank != 0:
        ctx.rowblock(n, n, n, mode=P.MODE_EXACT)
        return None
    A = ctx.fill(P.DIST_UNIFORM, 71, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 72, n, n)
    C = torch.empty_like(A)
    t0 = time.time()
    el = ctx.rowblock(n, n, n, A, B, C, mode=P.MODE_EXACT)
    return {"same": _same(C, ctx.dgemm(A, B, mode=P.MODE_EXACT)), "waited": time.time() - t0,
            "elapsed": el}


def _job_random(P, ctx, rank, world):
    """Seeded random rounds (every rank draws the same sequence): shapes from
    1 row to B in k-panels, ragged and idle-rank splits, AUTO / EXACT / DMMA
    fp64 and FFMA fp32, both gathers, device and host entries -- rank 0
    compares each round with its own one-GPU product, bitwise."""
    import torch
    # MMWS_FAKE_SOAK=<rounds>:<seed> lengthens it (soak runs, tools/README.md)
    rounds, seed = 24, 4242
    if os.environ.get("MMWS_FAKE_SOAK"):
        rounds, seed = (int(v) for v in os.environ["MMWS_FAKE_SOAK"].split(":"))
    rng = np.random.default_rng(seed)
    modes = [("auto", P.MODE_AUTO, False), ("exact", P.MODE_EXACT, False),
             ("dmma", P.MODE_DMMA, False), ("ffma", P.MODE_FFMA, True)]
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    res = []
    for case in range(rounds):
        r = rng.random()
        if r < 0.3:
            m, k, n = (int(v) for v in rng.integers(1, 40, size=3))
        elif r < 0.85:
            m, k, n = (int(v) for v in rng.integers(40, 1500, size=3))
        else:  # B in k-panels: k * n >= 64 Mi elements
            m, k, n = int(rng.integers(600, 2500)), 8192, int(rng.integers(8192, 9000))
        name, mode, f32 = modes[int(rng.integers(0, len(modes)))]
        gather = None if rng.random() < 0.6 else "1"
        host = not f32 and rng.random() < 0.25
        ctx.tune("MMWS_GPU_NCCL_GATHER", gather)
        tdt = torch.float32 if f32 else torch.float64
        dist = P.DIST_NORMAL if f32 else [P.DIST_UNIFORM, P.DIST_INT8][case % 2]
        if rank == 0:
            A = ctx.fill(dist, 100 + case, m, k, dtype=tdt)
            B = ctx.fill(dist, 200 + case, k, n, dtype=tdt)
            want = (ctx.sgemm if f32 else ctx.dgemm)(A, B, mode=mode)
            if host:
                got, _ = ctx.master_run_host(A.cpu().numpy(), B.cpu().numpy(), mode=mode)
                got = torch.from_numpy(got)
            else:
                C = torch.full((m, n), float("nan"), dtype=tdt, device="cuda")
                ctx.rowblock(m, n, k, A, B, C, mode=mode, f32=f32)
                got = C.cpu()
            torch.cuda.synchronize()
            w = want.cpu()
            iv = torch.int32 if f32 else torch.int64
            rows_bad = (got.view(iv) != w.view(iv)).any(dim=1).nonzero().flatten().tolist()
            same = not rows_bad
            res.append((case, m, k, n, name, gather, host, ctx.last_round, ctx.last_b_panels,
                        rows_bad[:3] + ([len(rows_bad)] if rows_bad else []), same))
            del A, B, want
        elif host:
            ctx.master_run_host(None, None, None, mode=mode, m=m, n=n, k=k)
        else:
            ctx.rowblock(m, n, k, mode=mode, f32=f32)
    return res


def _job_fresh_c(P, ctx, rank, world):
    """Every round gets a freshly allocated C on rank 0 (new IPC handle): the
    workers map each one for the fused gather and close the least recently
    used beyond a few, so old C allocations do not stay mapped; results stay
    bitwise, including a C seen again after its mapping was evicted."""
    import torch
    ctx.tune("MMWS_GPU_ROWBLOCK_RANKS", "all")
    m, n, k = 600, 520, 300
    out = []
    keep = None
    for i in range(9):
        if rank == 0:
            A = ctx.fill(P.DIST_UNIFORM, 900 + i, m, k)
            B = ctx.fill(P.DIST_UNIFORM, 950 + i, k, n)
            if i == 8:
                C = keep                                  # an early C again
            else:
                C = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
            ctx.rowblock(m, n, k, A, B, C)
            out.append((i, ctx.last_round, _same(C, ctx.dgemm(A, B)), C.data_ptr()))
            if i == 1:
                keep = C
            else:
                del C
            torch.cuda.synchronize()
            torch.cuda.empty_cache()                      # the next C is a new allocation
        else:
            ctx.rowblock(m, n, k)
    return out


JOBS = {"rounds": _job_rounds, "dead": _job_dead, "ragged": _job_ragged, "config3": _job_config3,
        "slow": _job_slow, "random": _job_random, "fresh_c": _job_fresh_c}


@pytest.mark.timeout(600)
def test_fresh_c_every_round_keeps_few_mappings(fake_lib):
    res = _ok(_run(3, fake_lib, "fresh_c"), 3)[0]
    assert len(res) == 9
    for i, (active, how), same, _ in res:
        assert same and active == 3 and how == "fused-ipc", (i, active, how)
    # the allocator hands the same address to later C's (new allocations,
    # new IPC handles): the workers' stale mappings of it must not get in
    # the way (cudaErrorAlreadyMapped -> close the idle round mappings)
    ptrs = [p for *_, p in res]
    assert len(set(ptrs)) < len(ptrs), ptrs


@pytest.mark.timeout(900)
def test_random_rounds_bitwise_over_3_ranks(fake_lib):
    world = int(os.environ.get("MMWS_FAKE_SOAK_WORLD", "3"))  # soak runs: other worlds
    res = _ok(_run(world, fake_lib, "random"), world)[0]
    assert len(res) == (int(os.environ["MMWS_FAKE_SOAK"].split(":")[0])
                        if os.environ.get("MMWS_FAKE_SOAK") else 24)
    bad = [r for r in res if not r[-1]]
    if bad:
        pytest.fail(f"rounds differing from the one-GPU product: {bad}")


@pytest.mark.timeout(300)
def test_slow_worker_is_waited_for(fake_lib):
    res = _ok(_run(3, fake_lib, "slow", timeout=240), 3)[0]
    assert res["same"] and res["waited"] > 2.0 and res["elapsed"] > 0, res


@pytest.mark.timeout(900)
def test_config3_at_size_over_8_ranks_bitwise(fake_lib):
    res = _ok(_run(8, fake_lib, "config3"), 8)[0]
    for key in ("f64", "f32"):
        same, panels, (active, gather) = res[key]
        assert same and panels == 8 and active == 8 and gather == "fused-ipc", (key, res[key])


@pytest.mark.timeout(900)
def test_ragged_n4099_over_8_ranks_matches_reference_golden(fake_lib):
    res = _ok(_run(8, fake_lib, "ragged"), 8)[0]
    assert [r for _, r in res["split"]] == [513] * 3 + [512] * 5
    assert res["auto"] == res["golden"] and res["exact"] == res["golden"], res
    assert res["idle"]


# ----------------------------------------------------------------------------- tests
@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 3])
def test_worker_side_executes_bitwise_on_one_gpu(fake_lib, world):
    res = _ok(_run(world, fake_lib, "rounds"), world)[0]
    assert len(res) == 2 * len(CASES) + 1
    for gather, m, k, n, dt, mode, ((active, how), panels), same in res:
        assert same, (gather, m, k, n, dt, mode)
        assert active == world
        if gather != "host":
            assert how == ("nccl" if gather == "1" else "fused-ipc"), (gather, how)
        assert panels == (2 if k * n >= 64 * 2 ** 20 else 1), (m, k, n, panels)


@pytest.mark.timeout(300)
def test_dead_worker_named_on_one_gpu(fake_lib):
    out = _ok(_run(2, fake_lib, "dead", timeout=240), 2)
    r0 = out[0]
    assert r0["type"] == "ProtocolError", r0
    assert "rank 1" in r0["msg"], r0
    assert r0["took"] < 60, r0
    assert "destroy" in r0["after"] and r0["recovered"], r0


@pytest.mark.timeout(900)
def test_bench_multi_rank_line_on_one_gpu(fake_lib):
    """bench.py's N>1 path (self-launched ranks, the row-block rounds with B in
    k-panels, link probes, host-round e2e, fp32 rounds, per-rank gathering)
    on one GPU with the stand-in: one complete JSON line (times meaningless)."""
    import json
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(MMWS_GPU_NCCL_LIB=fake_lib, MMWS_BENCH_ONE_GPU_WORLD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--n", "8192",
                        "--n32", "8192", "--steps", "2", "--warmup", "1", "--steps32", "1",
                        "--quick"], capture_output=True, text=True, cwd=ROOT, env=env,
                       timeout=800)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "plumbing_test" in d and d["value"] > 0
    assert d["round"]["active_ranks"] == 2 and d["round"]["gather"] == "fused-ipc"
    assert d["round"]["b_panels"] == 2 and len(d["per_rank_ms_per_step"]) == 2
    assert d["link"]["broadcast_GBps"] > 0 and d["link"]["p2p_GBps"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e_pageable"]["value"] > 0
    assert d["fp32"]["accuracy"]["ok"] and d["fp32"]["round"]["b_panels"] == 2
    assert d["cpu_baseline"]["cores"] >= 1 and d["gpu_launches"] > 0


@pytest.mark.timeout(600)
def test_cpp_dropin_master_worker_over_3_processes(fake_lib):
    """The C++ drop-in end to end over 3 processes on one GPU: the reference's
    own launcher starts the workers (launch_with_master / connect_from_env),
    mmws::gpu::comm_init_from ships the NCCL id over its Communicator, and
    master_run / worker_run run the rounds; the harness gates every record
    against mmws::matmul_seq (tools/cpp_world_rehearsal.sh)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "mmws_gpu_bench_ref")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/mmws_gpu_bench_ref not built (needs the reference headers)")
    env = dict(os.environ, MMWS_GPU_NCCL_LIB=fake_lib, MMWS_BENCH_ONE_GPU_WORLD="1",
               MMWS_GPU_ROWBLOCK_RANKS="all")
    r = subprocess.run([exe, "--gpus", "3", "--dims", "1,10,500,2000,4099",
                        "--models", "gpu-rowblock", "--repeats", "2"],
                       capture_output=True, text=True, env=env, timeout=500)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    rows = [ln.split() for ln in r.stdout.splitlines() if ln.startswith("gpu-rowblock")]
    assert [int(x[1]) for x in rows] == [1, 10, 500, 2000, 4099], r.stdout
    for x in rows:
        assert int(x[2]) == 3 and float(x[5]) <= 1e-12, x


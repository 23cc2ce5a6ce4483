"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/mmws_gpu.h declares, its host-only logic matches the reference
(split_rows, static_partition, op_count, the row-block message plan), the C++
adapter compiles against the reference's own Matrix type, and there is no CPU
fallback (no compute calls here)."""
import os
import re
import subprocess

import pytest

import paper_1012_2273_b200 as P
from paper_1012_2273_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def header_functions():
    with open(os.path.join(ROOT, "include", "mmws_gpu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|uint64_t|void\*)\s+(mmws_gpu_\w+)\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    declared = header_functions()
    assert len(declared) >= 25
    nm = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r" T (mmws_gpu_\w+)", nm))
    assert set(declared) <= exported, set(declared) - exported
    assert set(declared) == set(_abi.SIGNATURES), set(declared) ^ set(_abi.SIGNATURES)
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.mmws_gpu_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_no_cpu_fallback_without_gpu():
    # No GPU in this container: creating a context must fail loudly.
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.GpuError):
        P.Context(0)


def test_split_rows_matches_reference(oracle, golden_small):
    for key, want in golden_small["split_rows"].items():
        n, w = (int(x) for x in key.split(","))
        assert [list(x) for x in P.split_rows(n, w)] == want
    assert P.split_rows(4, 3) == [(0, 2), (2, 1), (3, 1)]
    assert P.split_rows(2, 3) == [(0, 1), (1, 1), (2, 0)]
    for n in range(0, 201, 13):
        for w in range(1, 17):
            assert P.split_rows(n, w) == oracle.split_rows(n, w)
    with pytest.raises(P.DomainError):
        P.split_rows(4, 0)
    with pytest.raises(P.DomainError):
        P.split_rows(-1, 2)


def test_static_partition_and_op_count_match_reference(golden_small):
    for key, want in golden_small["static_partition"].items():
        n, w = (int(x) for x in key.split(","))
        assert [list(x) for x in P.static_partition(n, w)] == want
    with pytest.raises(P.DomainError):
        P.static_partition(3, 0)
    for n, want in golden_small["op_count"].items():
        assert P.op_count(int(n)) == want
    with pytest.raises(P.DomainError):
        P.op_count(0)
    with pytest.raises(P.DomainError):
        P.op_count(-5)


def test_rowblock_plan_shape():
    # The reference's protocol shape test (test_protocol.cpp:99-137) on a 4x4
    # problem over 2 workers; here rank 0 also computes, so 3 ranks = rank 0 +
    # 2 remote workers, metadata is derived locally (no scalar messages), and B
    # is one broadcast (first: nothing can finish without all of B) instead of
    # per-worker copies.
    plan = P.rowblock_plan(4, 4, 4, 3)
    assert [(e["dir"], e["tag"], e["peer"], e["count"], e["row0"]) for e in plan] == [
        ("broadcast", 1, -1, 16, -1), ("sent", 1, 1, 4, 2), ("sent", 1, 2, 4, 3),
        ("received", 2, 1, 4, 2), ("received", 2, 2, 4, 3)]
    # idle ranks (P > N) exchange nothing but still join the broadcast
    plan = P.rowblock_plan(2, 2, 2, 5)
    assert [e["peer"] for e in plan if e["dir"] == "sent"] == [1]
    assert P.rowblock_plan(7, 7, 7, 1) == []
    # N=16384 over 8 GPUs: two sub-blocks per rank; A and C slices tile rows
    # 2048..16383 exactly once each; B goes out once, as 8 k-panels (row
    # panels of B, edges at multiples of 1024) after the first A sub-blocks
    m, n, k, world = 16384, 16384, 16384, 8
    plan = P.rowblock_plan(m, n, k, world)
    rows0 = P.split_rows(m, world)[0][1]
    dirs = [e["dir"] for e in plan]
    first_b = dirs.index("broadcast")
    assert dirs[:first_b] == ["sent"] * (world - 1)              # A sub-block 0 of every worker
    panels = [(e["row0"], e["row0"] + e["count"] // n) for e in plan if e["dir"] == "broadcast"]
    assert len(panels) == 8 and panels[0][0] == 0 and panels[-1][1] == k
    assert all(a[1] == b[0] for a, b in zip(panels, panels[1:]))
    assert all(lo % 1024 == 0 for lo, _ in panels)
    assert dirs[first_b:first_b + 8] == ["broadcast"] * 8
    for d, width in (("sent", k), ("received", n)):
        spans = sorted((e["row0"], e["row0"] + e["count"] // width) for e in plan if e["dir"] == d)
        assert len(spans) == 2 * (world - 1)
        assert spans[0][0] == rows0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    # every sub-block is a whole number of 128-row bands (wave quantisation)
    assert all(e["count"] // k % 128 == 0 for e in plan if e["dir"] == "sent")
    with pytest.raises(P.DimensionError):
        P.rowblock_plan(0, 4, 4, 2)


def _compile_adapter(tmp_path):
    exe = tmp_path / "test_adapter"
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror",
                    f"-I{ROOT}/include", f"{ROOT}/tests/cpp/test_adapter.cpp", "-o", str(exe),
                    f"-L{ROOT}/paper_1012_2273_b200", "-lmmws_gpu",
                    f"-Wl,-rpath,{ROOT}/paper_1012_2273_b200"], check=True)
    return exe


def test_cpp_adapter_host_checks(tmp_path):
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    exe = _compile_adapter(tmp_path)
    if gpu:
        pytest.skip("host-only variant asserts that no GPU is present")
    r = subprocess.run([str(exe), "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_INC, "mmws", "matrix.hpp")),
                    reason="reference headers not present (GPU box)")
def test_cpp_adapter_is_dropin_for_reference_matrix():
    json_dir = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "print-json-dir"],
                              capture_output=True, text=True).stdout.strip()
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                    f"-I{REF_INC}", f"-I{json_dir}", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/ref_dropin_check.cpp"], check=True)


@pytest.mark.gpu
def test_cpp_adapter_gpu_checks(tmp_path):
    exe = _compile_adapter(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_rowblock_cost_model():
    # The reference's cost-model checks (test_cost_model.cpp / acceptance.cpp:172-202)
    # transposed to this schedule: traffic formulas, monotone in N and P.
    n, bw, fl = 16384, 770e9, 36.4e12
    t1, e1, i1 = P.rowblock_cost(n, n, n, 1, 8, bw, fl)
    assert t1 == pytest.approx(2 * n ** 3 / fl) and e1 == 0 and i1 == 0
    for p in (2, 4, 8):
        t, eg, ing = P.rowblock_cost(n, n, n, p, 8, bw, fl)
        rows0 = P.split_rows(n, p)[0][1]
        assert eg == 8 * (n * n + (n - rows0) * n)       # B once + the workers' A rows
        assert ing == 8 * (n - rows0) * n                # the workers' C rows
        assert t < t1 and t1 / (p * t) > 0.85            # >= 85% efficiency target
    prev = 0.0
    for nn in (1000, 2000, 4096, 8192):
        t, _, _ = P.rowblock_cost(nn, nn, nn, 8, 8, bw, fl)
        assert t > prev
        prev = t
    # fp32 halves the bytes
    _, eg64, _ = P.rowblock_cost(4096, 4096, 4096, 4, 8, bw, fl)
    _, eg32, _ = P.rowblock_cost(4096, 4096, 4096, 4, 4, bw, fl)
    assert eg32 * 2 == eg64
    with pytest.raises(P.DomainError):
        P.rowblock_cost(10, 10, 10, 2, 3, bw, fl)


def test_rowblock_distributes_only_where_it_pays(monkeypatch):
    # north_star (3): the row-block exchange is used only where N is large
    # enough to amortise the transfers -- rank 0 alone below that.
    monkeypatch.delenv("MMWS_GPU_ROWBLOCK_RANKS", raising=False)
    for n in (10, 100, 500, 1000):
        assert P.rowblock_ranks(n, n, n, 8) == 1, n
    for n in (2000, 4096, 16384):
        assert P.rowblock_ranks(n, n, n, 8) == 8, n
        assert P.rowblock_ranks(n, n, n, 2, 4) == 2, n
    assert P.rowblock_ranks(32768, 32768, 32768, 8, 4) == 8
    assert P.rowblock_ranks(16384, 16384, 16384, 1) == 1
    # monotone: once distributed, every larger square problem is too
    seen = False
    for n in range(200, 4000, 50):
        d = P.rowblock_ranks(n, n, n, 4) == 4
        assert d or not seen, n
        seen = seen or d
    assert seen
    # it is the cost model's own comparison (plus the fixed round latency)
    t1, _, _ = P.rowblock_cost(3000, 3000, 3000, 1, 8, 770e9, 36.3e12)
    t8, _, _ = P.rowblock_cost(3000, 3000, 3000, 8, 8, 770e9, 36.3e12)
    assert (t8 + 60e-6 < t1) == (P.rowblock_ranks(3000, 3000, 3000, 8) == 8)
    monkeypatch.setenv("MMWS_GPU_ROWBLOCK_RANKS", "all")
    assert P.rowblock_ranks(10, 10, 10, 8) == 8
    monkeypatch.setenv("MMWS_GPU_ROWBLOCK_RANKS", "1")
    assert P.rowblock_ranks(16384, 16384, 16384, 8) == 1
    with pytest.raises(P.DimensionError):
        P.rowblock_ranks(0, 4, 4, 2)
    with pytest.raises(P.DomainError):
        P.rowblock_ranks(4, 4, 4, 2, 3)


REF_CP = os.path.join(ROOT, "oracle", "_ref", "ref_control_plane")


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_INC, "mmws", "launch.hpp")),
                    reason="reference headers not present (GPU box)")
def test_nccl_id_over_the_reference_control_plane():
    # the reference's own launcher (launch_with_master /
    # connect_from_env) and TCP Communicator ship the NCCL id to every rank
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    r = subprocess.run([REF_CP, "master", "4"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "4 ranks share one NCCL id" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_master_run_over_a_world_bootstrapped_by_the_reference_launcher():
    if not os.path.exists(REF_CP):
        pytest.skip("ref_control_plane not built (needs the reference headers at build time)")
    r = subprocess.run([REF_CP, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok: master_run" in r.stdout, r.stdout + r.stderr


def test_python_output_buffer_checks_without_a_gpu():
    # the wrappers validate outputs before the C ABI
    # writes m*n elements into them (host heap / device out-of-bounds writes)
    import numpy as np
    import torch

    from paper_1012_2273_b200 import api
    assert api._host_out(None, 3, 4, np.float64, "t").shape == (3, 4)
    ok = np.empty((3, 4))
    assert api._host_out(ok, 3, 4, np.float64, "t") is ok
    with pytest.raises(P.DimensionError):
        api._host_out(np.empty((3, 3)), 3, 4, np.float64, "t")
    with pytest.raises(P.DomainError):
        api._host_out(np.empty((3, 4), dtype=np.float32), 3, 4, np.float64, "t")
    with pytest.raises(P.DimensionError):
        api._host_out(np.empty((4, 3)).T, 3, 4, np.float64, "t")
    ro = np.empty((3, 4))
    ro.setflags(write=False)
    with pytest.raises(P.DimensionError):
        api._host_out(ro, 3, 4, np.float64, "t")
    a = torch.zeros((3, 2), dtype=torch.float64)
    b = torch.zeros((2, 4), dtype=torch.float64)
    with pytest.raises(P.DomainError):            # host tensors are not device operands
        api._device_operands(a, b, None, torch.float64, "t")
    with pytest.raises(P.DomainError):
        api._device_operands(a.float(), b, None, torch.float64, "t")


def test_device_operand_checks_name_the_context_device():
    # operands on another GPU than the context's would be read through UVA by
    # the kernels (an illegal address without peer access): refused up front
    import torch

    from paper_1012_2273_b200 import api

    class FakeCuda:
        def __init__(self, shape, index):
            self.shape, self.dtype, self.is_cuda = shape, torch.float64, True
            self.device = torch.device("cuda", index)

        def dim(self):
            return 2

    a, b = FakeCuda((3, 2), 1), FakeCuda((2, 4), 1)
    assert api._device_operands(a, b, None, torch.float64, "t", 1) == (3, 4, 2)
    with pytest.raises(P.DomainError, match="cuda:1.*cuda:0"):
        api._device_operands(a, b, None, torch.float64, "t", 0)


def test_master_run_host_argument_checks_without_a_gpu():
    import numpy as np

    from paper_1012_2273_b200 import api

    class Ctx:  # the checks run before the C ABI is reached
        _h = None

    with pytest.raises(P.DomainError):
        api._master_run_host(Ctx(), np.zeros((2, 2)))
    with pytest.raises(P.DimensionError):
        api._master_run_host(Ctx(), np.zeros(4), np.zeros((2, 2)))
    with pytest.raises(P.DomainError):
        api._master_run_host(Ctx(), m=4, n=None, k=4)

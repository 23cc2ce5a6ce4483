"""The benchmark harness with GPU models (include/mmws_gpu_bench.hpp,
tools/mmws_gpu_bench.cpp): host-side pieces pinned against the reference's own
bench.hpp values (golden), and an end-to-end sweep on the GPU with the
correctness gate."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
LIB = ["-L" + os.path.join(ROOT, "paper_1012_2273_b200"), "-lmmws_gpu",
       "-Wl,-rpath," + os.path.join(ROOT, "paper_1012_2273_b200")]


def _build(src, out, extra=()):
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror",
                    "-I" + os.path.join(ROOT, "include"), *extra, src, "-o", str(out), *LIB],
                   check=True)
    return str(out)


def test_harness_host_pieces_match_reference(tmp_path, golden_small):
    exe = _build(os.path.join(ROOT, "tests", "cpp", "test_harness.cpp"), tmp_path / "th")
    got = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    assert {k: int(v) for k, v in got["derive_seed"].items()} == golden_small["derive_seed"]
    for key, want in golden_small["mflops"].items():
        n, t = key.split(",")
        assert got["mflops"][f"{n},{float(t):.6g}"] == want
    assert got["random0"] == 0.88331080821364261
    assert got["csv"] == ("model,n,workers,elapsed_s,mflops,speedup|"
                          "gpu,1000,1,0.000123457,16191.2,|gpu-exact,1000,1,0.5,3998,2.5|")
    assert got["mflops_zero_throws"] is True


def _series(svg_path):
    import re
    text = open(svg_path).read()
    out = {}
    for name, pts, rest in re.findall(r'data-series="([^"]+)" data-points="([^"]*)"( [^>]*)?', text):
        out[name] = [tuple(float(v) for v in p.split(":")) for p in pts.split(";")]
        out[name + "#dashed"] = "stroke-dasharray" in text.split(f'data-series="{name}"')[0].rsplit("<polyline", 1)[1]
    return text, out


def test_plots_series_and_cost_overlay(tmp_path):
    import paper_1012_2273_b200 as P
    exe = _build(os.path.join(ROOT, "tests", "cpp", "test_harness.cpp"), tmp_path / "th")
    d = tmp_path / "plots"
    got = json.loads(subprocess.run([exe, str(d)], capture_output=True, text=True,
                                    check=True).stdout)
    assert got["empty_throws"] is True and got["io_error"] is True
    assert sorted(os.listdir(d)) == ["mflops.svg", "runtime.svg", "speedup.svg"]
    text, s = _series(d / "runtime.svg")
    assert text.startswith("<svg") and "Running time vs matrix dimension" in text
    assert s["gpu"] == [(100.0, 0.0001), (500.0, 0.002)]           # sorted by N
    assert s["gpu-exact"] == [(100.0, 0.0002)]
    assert s["gpu-rowblock"] == [(2048.0, 0.003), (4096.0, 0.01)]
    want = [(float(n), P.rowblock_cost(n, n, n, 4, 8, 500e9, 3e13)[0]) for n in (2048, 4096)]
    assert [x for x, _ in s["cost-model"]] == [x for x, _ in want]
    for (_, a), (_, b) in zip(s["cost-model"], want):
        assert abs(a - b) <= 1e-5 * b                                  # %.6g in the attribute
    assert s["cost-model#dashed"] and not s["gpu#dashed"]
    assert "cost-model overlay: link=5e+11 B/s (B200 peer-copy reference)" in text
    _, m = _series(d / "mflops.svg")
    assert m["gpu-rowblock"] == [(2048.0, 5.7e6), (4096.0, 1.3e7)] and "cost-model" not in m
    _, sp = _series(d / "speedup.svg")
    assert sp == {"gpu": [(100.0, 4.0), (500.0, 30.0)], "gpu#dashed": False}


def test_cli_builds_standalone_and_against_reference(tmp_path):
    _build(os.path.join(ROOT, "tools", "mmws_gpu_bench.cpp"), tmp_path / "b1")
    if os.path.exists(os.path.join(REF_INC, "mmws", "matrix.hpp")):
        _build(os.path.join(ROOT, "tools", "mmws_gpu_bench.cpp"), tmp_path / "b2",
               extra=("-I" + REF_INC,))
        json_dir = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"),
                                   "print-json-dir"], capture_output=True, text=True).stdout.strip()
        exe = _build(os.path.join(ROOT, "tools", "mmws_gpu_bench.cpp"), tmp_path / "b3",
                     extra=("-I" + REF_INC, "-I" + json_dir, "-pthread"))
        # --gpus P needs a GPU per rank; without one the context fails loudly
        r = subprocess.run([exe, "--dims", "64", "--models", "gpu-rowblock", "--gpus", "1"],
                           capture_output=True, text=True, timeout=120)
        assert r.returncode != 0 or "gpu-rowblock" in r.stdout


@pytest.mark.gpu
def test_cli_sweep_with_gate(tmp_path):
    exe = _build(os.path.join(ROOT, "tools", "mmws_gpu_bench.cpp"), tmp_path / "b")
    csv = tmp_path / "out.csv"
    r = subprocess.run([exe, "--dims", "10,100,257,1000", "--models", "gpu,gpu-exact,gpu-rowblock",
                        "--repeats", "2", "--csv", str(csv), "--plots", str(tmp_path / "svg"),
                        "--calibrate"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = csv.read_text().splitlines()
    assert lines[0] == "model,n,workers,elapsed_s,mflops,speedup"
    assert len(lines) == 1 + 12
    models = [ln.split(",")[0] for ln in lines[1:]]
    assert models == ["gpu"] * 4 + ["gpu-exact"] * 4 + ["gpu-rowblock"] * 4
    assert "calibration: link 7.7e+11 B/s (B200 peer-copy reference), gemm" in r.stdout
    _, s = _series(tmp_path / "svg" / "runtime.svg")
    assert [x for x, _ in s["cost-model"]] == [10.0, 100.0, 257.0, 1000.0]
    assert [x for x, _ in s["gpu-rowblock"]] == [10.0, 100.0, 257.0, 1000.0]
    for ln in lines[1:]:
        f = ln.split(",")
        assert float(f[3]) > 0 and float(f[4]) > 0 and f[5] == ""
    # an impossible tolerance trips the normwise gate: exit code 2 (bench_main.cpp:175-177)
    r = subprocess.run([exe, "--dims", "300", "--models", "gpu", "--tolerance", "0"],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "correctness gate" in r.stderr


@pytest.mark.gpu
def test_cli_with_latency_server(tmp_path):
    # --server: N <= 96 calls go through the resident kernel; the gate still holds
    exe = _build(os.path.join(ROOT, "tools", "mmws_gpu_bench.cpp"), tmp_path / "b")
    csv = tmp_path / "out.csv"
    r = subprocess.run([exe, "--dims", "10,50,96,100", "--models", "gpu,gpu-exact", "--server",
                        "--repeats", "3", "--csv", str(csv)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(csv.read_text().splitlines()) == 1 + 8


@pytest.mark.gpu
def test_cli_gpus_mode_through_the_reference_launcher(tmp_path):
    # --gpus P: the reference's launcher spawns ranks 1..P-1 and ships the NCCL
    # id; on this one-GPU box P = 1 (a 1-rank NCCL world, same code path)
    exe = os.path.join(ROOT, "oracle", "_ref", "mmws_gpu_bench_ref")
    if not os.path.exists(exe):
        pytest.skip("mmws_gpu_bench_ref not built (needs the reference headers at build time)")
    csv = tmp_path / "out.csv"
    r = subprocess.run([exe, "--dims", "100,1000", "--models", "gpu-rowblock", "--gpus", "1",
                        "--repeats", "2", "--csv", str(csv), "--calibrate"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = csv.read_text().splitlines()
    assert [ln.split(",")[:3] for ln in lines[1:]] == [["gpu-rowblock", "100", "1"],
                                                       ["gpu-rowblock", "1000", "1"]]
    assert "calibration: link" in r.stdout   # 1 rank: no link to measure (nominal)


@pytest.mark.gpu
def test_cli_cpu_models_through_the_reference_suite(tmp_path):
    # --cpu-models: the reference's own run_suite times seq / threads first (its
    # own gate included); their seq times give every GPU record its speedup
    exe = os.path.join(ROOT, "oracle", "_ref", "mmws_gpu_bench_ref")
    if not os.path.exists(exe):
        pytest.skip("mmws_gpu_bench_ref not built (needs the reference headers at build time)")
    csv = tmp_path / "out.csv"
    r = subprocess.run([exe, "--dims", "10,200", "--models", "gpu,gpu-exact",
                        "--cpu-models", "seq,threads", "--csv", str(csv),
                        "--plots", str(tmp_path / "svg")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [ln.split(",") for ln in csv.read_text().splitlines()[1:]]
    assert [(f[0], f[1]) for f in rows] == [("seq", "10"), ("seq", "200"), ("threads", "10"),
                                            ("threads", "200"), ("gpu", "10"), ("gpu", "200"),
                                            ("gpu-exact", "10"), ("gpu-exact", "200")]
    seq = {f[1]: float(f[3]) for f in rows if f[0] == "seq"}
    for f in rows:
        assert f[5] != "", f                              # every record paired with seq
        assert abs(float(f[5]) - seq[f[1]] / float(f[3])) <= 1e-4 * float(f[5])
    _, s = _series(tmp_path / "svg" / "speedup.svg")
    assert {"seq", "threads", "gpu", "gpu-exact"} <= set(k for k in s if "#" not in k)

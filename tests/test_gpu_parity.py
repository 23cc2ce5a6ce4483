"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): bit-exact for integer-valued inputs and for
the exact-order mode; fp64 DMMA normwise <= 1e-12, fp32 FFMA normwise <= 1e-5
against the fp64 oracle of the widened inputs.  Golden fixtures in
tests/golden/ were produced by the reference itself (gen_golden.py).
"""
import hashlib

import numpy as np
import pytest

import paper_1012_2273_b200 as P

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12   # north_star: fp64 normwise relative error
FP32_TOL = 1e-5    # north_star: fp32 normwise relative error vs fp64 oracle
FP64_MODES = [P.MODE_EXACT, P.MODE_DMMA, P.MODE_DMMA_SMALL, P.MODE_AUTO]


def torch():
    import torch as T
    return T


def dev(x):
    T = torch()
    return T.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch().cuda.synchronize()
    return t.cpu().numpy()


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def from_hex(h, shape):
    return np.array([int(v, 16) for v in h], dtype=np.uint64).view(np.float64).reshape(shape)


def normwise(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


# ----------------------------------------------------------------------------- known answers
@pytest.mark.parametrize("mode", FP64_MODES)
def test_hand_computed_2x2_and_1x1(ctx, golden_small, mode):
    # test_matrix.cpp:105-120 (and over msg, test_protocol.cpp:56-67)
    c = host(ctx.dgemm(dev(np.array([[1., 2], [3, 4]])), dev(np.array([[5., 6], [7, 8]])),
                       mode=mode))
    assert c.tolist() == [[19.0, 22.0], [43.0, 50.0]]
    assert (bits(c).ravel() == bits(from_hex(golden_small["matmul_2x2"], (2, 2))).ravel()).all()
    c = host(ctx.dgemm(dev(np.array([[3.25]])), dev(np.array([[-2.0]])), mode=mode))
    assert c[0, 0] == 3.25 * -2.0


@pytest.mark.parametrize("mode", FP64_MODES)
def test_identity_is_bitwise_neutral(ctx, oracle, mode):
    # test_matrix.cpp:122-141
    for n in (1, 2, 5, 13, 130):
        a = oracle.ref_random_matrix(n, n, 1000 + n) if oracle.ref_available() else \
            oracle.fill(0, 1000 + n, n, n)
        eye = np.eye(n)
        assert (bits(host(ctx.dgemm(dev(a), dev(eye), mode=mode))) == bits(a)).all()
        assert (bits(host(ctx.dgemm(dev(eye), dev(a), mode=mode))) == bits(a)).all()


def test_acceptance_products_match_reference_golden(ctx, oracle, golden_small):
    # acceptance.cpp:90-109 dims, seeds 1000+N / 2000+N; golden = mmws::matmul_seq
    for n in [int(k[2:]) for k in golden_small["products_unit"] if k.startswith("sq")]:
        a = oracle.fill(oracle.DIST_UNIT, 1000 + n, n, n)
        b = oracle.fill(oracle.DIST_UNIT, 2000 + n, n, n)
        want = from_hex(golden_small["products_unit"][f"sq{n}"], (n, n))
        got = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_EXACT))
        assert (bits(got) == bits(want)).all(), f"exact N={n}"
        for mode in (P.MODE_DMMA, P.MODE_DMMA_SMALL):
            got = host(ctx.dgemm(dev(a), dev(b), mode=mode))
            assert normwise(got, want) <= FP64_TOL, f"mode={mode} N={n}"


def test_rectangular_products(ctx, oracle, golden_small):
    # test_matrix.cpp:148-156, test_workshare.cpp:160-163, test_protocol.cpp:91-97
    for key, (m, k, n, sa, sb) in {"rect2x5x4": (2, 5, 4, 303, 304),
                                   "rect4x7x3": (4, 7, 3, 27, 28),
                                   "rect5x7x4": (5, 7, 4, 31, 32)}.items():
        a = oracle.fill(oracle.DIST_UNIT, sa, m, k)
        b = oracle.fill(oracle.DIST_UNIT, sb, k, n)
        want = from_hex(golden_small["products_unit"][key], (m, n))
        for mode in FP64_MODES:
            got = host(ctx.dgemm(dev(a), dev(b), mode=mode))
            assert got.shape == (m, n)
            if mode == P.MODE_EXACT:
                assert (bits(got) == bits(want)).all()
            else:
                assert normwise(got, want) <= FP64_TOL


# ----------------------------------------------------------------------------- exact mode, any input
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 3, 5), (64, 64, 64), (127, 129, 131),
                                   (200, 33, 257), (300, 1000, 17), (513, 257, 260)])
def test_exact_mode_bitwise_equals_matmul_seq(ctx, oracle, shape):
    m, k, n = shape
    a = oracle.fill(oracle.DIST_UNIFORM, 11, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 12, k, n)
    want = oracle.matmul_seq(a, b)
    got = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_EXACT))
    assert oracle.first_difference(got, want) is None


@pytest.mark.parametrize("shape", [(4, 1_000_000, 4), (3, 500_001, 130), (1_000_003, 16, 97),
                                   (7, 97, 300_001)])
def test_extreme_aspect_ratios_bit_exact(ctx, oracle, shape):
    # very long K (one tile, a million-step chain), very tall A, very wide B:
    # integer inputs, so every mode must reproduce the oracle's sampled rows
    # bitwise (fp32 too while the partial sums stay below 2^24)
    m, k, n = shape
    a = oracle.fill(oracle.DIST_INT8, 1, m, k)
    b = oracle.fill(oracle.DIST_INT8, 2, k, n)
    rows = sorted({0, m // 2, m - 1})
    want = oracle.matmul_rows(rows, a, b)
    A, B = dev(a), dev(b)
    for mode in (P.MODE_AUTO, P.MODE_DMMA, P.MODE_EXACT):
        got = host(ctx.dgemm(A, B, mode=mode))[rows]
        assert (bits(got) == bits(want)).all(), (shape, mode)
    af, bf = a.astype(np.float32), b.astype(np.float32)
    gf = host(ctx.sgemm(dev(af), dev(bf)))[rows].astype(np.float64)
    assert normwise(gf, oracle.matmul_rows(rows, af, bf)) <= FP32_TOL, shape


def test_exact_mode_signed_zeros_and_specials(ctx, oracle):
    # -0 handling: acc starts at +0, so all-zero rows give +0 (matrix.hpp:120)
    a = np.array([[-0.0, 0.0], [1e308, 1e308], [1.0, -1.0]])
    b = np.array([[0.0, -0.0], [-0.0, 3.0]])
    want = oracle.matmul_seq(a, b)
    for mode in FP64_MODES:
        got = host(ctx.dgemm(dev(a), dev(b), mode=mode))
        if mode == P.MODE_EXACT:
            assert oracle.first_difference(got, want) is None
        assert (np.signbit(got[0]) == np.signbit(want[0])).all()


# ----------------------------------------------------------------------------- integer inputs: bit-exact everywhere
@pytest.mark.parametrize("mode", FP64_MODES)
@pytest.mark.parametrize("n", [1, 2, 3, 17, 100, 129, 255, 1001])
def test_integer_inputs_bit_exact_all_modes(ctx, oracle, mode, n):
    a = oracle.fill(oracle.DIST_INT8, 0, n, n)
    b = oracle.fill(oracle.DIST_INT8, 1, n, n)
    want = oracle.matmul_threads(a, b)
    got = host(ctx.dgemm(dev(a), dev(b), mode=mode))
    assert oracle.first_difference(got, want) is None


def test_config_c3_n4099_integer_bit_exact(ctx, oracle, golden_big):
    # BASELINE configs[2]: odd, non-tile-aligned N, DMMA path packs for TMA.
    n = 4099
    A = ctx.fill(P.DIST_INT8, 0, n, n)
    B = ctx.fill(P.DIST_INT8, 1, n, n)
    for mode in (P.MODE_AUTO, P.MODE_DMMA, P.MODE_EXACT):
        c = host(ctx.dgemm(A, B, mode=mode))
        assert sha(c) == golden_big["n4099_int8_sha256"], f"mode {mode}"


@pytest.mark.parametrize("shape", [(2000, 2000, 2000), (1536, 999, 1664), (1280, 5000, 1920),
                                   (1536, 16, 1664), (2100, 1001, 2303), (2304, 2304, 2304),
                                   (1000, 1000, 1000), (1100, 701, 1100)])
def test_stream_k_is_bitwise_the_one_shot_kernel(ctx, oracle, monkeypatch, shape):
    # 148..1183 tiles of 128x128 with a partial last wave take the stream-K
    # launch (accumulators of a cut tile continued by the next CTA); it must
    # reproduce the one-shot kernels' bits exactly.  The last two shapes have
    # fewer 128x128 tiles than SMs: the exact mode's 64x64 stream-K.
    m, k, n = shape
    A = ctx.fill(P.DIST_UNIFORM, 31, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 32, k, n)
    for mode in (P.MODE_AUTO, P.MODE_DMMA):
        got = host(ctx.dgemm(A, B, mode=mode))
        ctx.tune("MMWS_GPU_NO_STREAMK", "1")
        want = host(ctx.dgemm(A, B, mode=mode))
        ctx.tune("MMWS_GPU_NO_STREAMK", None)
        assert (bits(got) == bits(want)).all(), (shape, mode)
    again = host(ctx.dgemm(A, B))                 # flags were left clean for the next launch
    assert (bits(again) == bits(got)).all()
    rows = [0, m // 2, m - 1]
    want_rows = oracle.matmul_rows(rows, host(A), host(B))
    assert normwise(got[rows], want_rows) <= FP64_TOL
    # exact order: stream-K form of the exact kernel, bitwise matmul_seq
    ex = host(ctx.dgemm(A, B, mode=P.MODE_EXACT))
    assert (bits(ex[rows]) == bits(want_rows)).all()
    ctx.tune("MMWS_GPU_NO_STREAMK", "1")
    ex1 = host(ctx.dgemm(A, B, mode=P.MODE_EXACT))
    ctx.tune("MMWS_GPU_NO_STREAMK", None)
    assert (bits(ex) == bits(ex1)).all()


@pytest.mark.parametrize("shape", [(1000, 1000, 1000), (777, 513, 1001), (33, 4099, 65),
                                   (4099, 300, 257), (1600, 1600, 1600)])
def test_every_dmma_tile_plan_gives_the_same_bits(ctx, oracle, monkeypatch, shape):
    # AUTO picks among 128x128 / 64x64 / 128x64 / 32x32 / 32x64 tiles, one-shot
    # or stream-K, by tile count; each element is the same DMMA chain in
    # ascending k from +0.0 in all of them, so every plan must give the same
    # bits (odd pitches go through the packing path first).
    m, k, n = shape
    A = ctx.fill(P.DIST_UNIFORM, 41, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 42, k, n)
    want = host(ctx.dgemm(A, B, mode=P.MODE_DMMA))
    rows = [0, m // 2, m - 1]
    assert normwise(want[rows], oracle.matmul_rows(rows, host(A), host(B))) <= FP64_TOL
    sms = torch().cuda.get_device_properties(0).multi_processor_count
    tried = 0
    # (tile rows, tile columns, resident CTAs per SM) of each configuration
    cfgs = [(128, 128, 1), (64, 64, 3), (128, 64, 1), (64, 64, 1), (32, 32, 6), (32, 64, 4),
            (32, 32, 2), (16, 16, 4)]
    for cfg, (bm, bn, per_sm) in enumerate(cfgs):
        tiles = -(-m // bm) * -(-n // bn)
        plans = [str(cfg)] + [f"{cfg}s{r}" for r in (1, 2, 3, 4)
                              if r <= per_sm and tiles >= r * sms and r * bm * bn <= 128 * 128]
        for plan in plans:
            ctx.tune("MMWS_GPU_DMMA_PLAN", plan)
            # strided C inside a canary frame: the plan writes exactly C
            buf = torch().full((m + 2, n + 3), -7.5, dtype=torch().float64, device="cuda")
            ctx.dgemm(A, B, buf[1:m + 1, 1:n + 1], mode=P.MODE_DMMA)
            b = host(buf)
            assert (bits(b[1:m + 1, 1:n + 1]) == bits(want)).all(), (shape, plan)
            assert (b[0] == -7.5).all() and (b[m + 1] == -7.5).all(), (shape, plan)
            assert (b[:, 0] == -7.5).all() and (b[:, n + 1:] == -7.5).all(), (shape, plan)
            tried += 1
    ctx.tune("MMWS_GPU_DMMA_PLAN", None)
    for mode in (P.MODE_AUTO, P.MODE_DMMA_SMALL):
        assert (bits(host(ctx.dgemm(A, B, mode=mode))) == bits(want)).all(), (shape, mode)
    assert tried >= 6
    ctx.tune("MMWS_GPU_DMMA_PLAN", "0s2")  # more CTAs than can be resident
    try:
        with pytest.raises(P.DomainError):
            ctx.dgemm(A, B, mode=P.MODE_DMMA)
    finally:
        ctx.tune("MMWS_GPU_DMMA_PLAN", None)


@pytest.mark.parametrize("seed", range(4))
def test_random_shapes_and_strides(ctx, oracle, seed):
    # Seeded fuzz over shapes (1..420), leading dimensions (dense or padded
    # views, odd pitches that force packing / the cp.async fallbacks) and all
    # modes: EXACT bitwise matmul_seq, tensor modes <= 1e-12 normwise and
    # bit-exact on integer inputs, fp32 <= 1e-5.
    T = torch()
    rng = np.random.default_rng(1000 + seed)
    for case in range(12):
        m, k, n = (int(v) for v in rng.integers(1, 421, size=3))
        pa, pb = (int(v) for v in rng.integers(0, 5, size=2))
        dist = oracle.DIST_INT8 if case % 3 == 0 else oracle.DIST_UNIFORM
        a = oracle.fill(dist, 7 * seed + case, m, k)
        b = oracle.fill(dist, 7 * seed + case + 100, k, n)
        A = T.zeros((m, k + pa), dtype=T.float64, device="cuda")[:, :k]
        B = T.zeros((k, n + pb), dtype=T.float64, device="cuda")[:, :n]
        A.copy_(T.from_numpy(a))
        B.copy_(T.from_numpy(b))
        want = oracle.matmul_seq(a, b)
        for mode in FP64_MODES:
            got = host(ctx.dgemm(A, B, mode=mode))
            if mode == P.MODE_EXACT or dist == oracle.DIST_INT8:
                assert oracle.first_difference(got, want) is None, (m, k, n, pa, pb, mode)
            else:
                assert normwise(got, want) <= FP64_TOL, (m, k, n, pa, pb, mode)
        af, bf = a.astype(np.float32), b.astype(np.float32)
        Af = T.zeros((m, k + pa), dtype=T.float32, device="cuda")[:, :k]
        Bf = T.zeros((k, n + pb), dtype=T.float32, device="cuda")[:, :n]
        Af.copy_(T.from_numpy(af))
        Bf.copy_(T.from_numpy(bf))
        gotf = host(ctx.sgemm(Af, Bf)).astype(np.float64)
        wantf = oracle.matmul_rows(list(range(m)), af, bf)
        if dist == oracle.DIST_INT8:   # |sums| < 2^24: exact in fp32 too
            assert (gotf == wantf).all(), (m, k, n, pa, pb)
        else:
            assert normwise(gotf, wantf) <= FP32_TOL, (m, k, n, pa, pb)


# ----------------------------------------------------------------------------- fp64 on the int8 tensor cores
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 3, 5), (128, 128, 128), (129, 1000, 131),
                                   (300, 17, 257), (1000, 37, 999), (513, 260, 1030),
                                   (2048, 2048, 2048), (64, 131072, 64), (1, 131072, 1)])
def test_ozaki_mode_accuracy_and_integer_exactness(ctx, oracle, shape):
    m, k, n = shape
    a = oracle.fill(oracle.DIST_UNIFORM, 51, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 52, k, n)
    rows = sorted({0, m // 2, m - 1})
    got = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_OZAKI))
    want = oracle.matmul_rows(rows, a, b)
    assert normwise(got[rows], want) <= 1e-13        # bound 1e-12; expected ~1e-15..1e-14
    ai = oracle.fill(oracle.DIST_INT8, 53, m, k)
    bi = oracle.fill(oracle.DIST_INT8, 54, k, n)
    gi = host(ctx.dgemm(dev(ai), dev(bi), mode=P.MODE_OZAKI))
    assert oracle.first_difference(gi[rows], oracle.matmul_rows(rows, ai, bi)) is None


def test_ozaki_mode_fp32(ctx, oracle):
    # fp32 operands through the same integer scheme (30-bit scaling): error at
    # the fp32 output rounding (~3e-8), far inside the 1e-5 bound
    T = torch()
    for (m, k, n) in [(1, 1, 1), (129, 1000, 131), (1000, 37, 999), (2048, 2048, 2048)]:
        A = ctx.fill(P.DIST_NORMAL, 81, m, k, dtype=T.float32)
        B = ctx.fill(P.DIST_NORMAL, 82, k, n, dtype=T.float32)
        got = host(ctx.sgemm(A, B, mode=P.MODE_OZAKI)).astype(np.float64)
        rows = sorted({0, m // 2, m - 1})
        want = oracle.matmul_rows(rows, host(A), host(B))
        assert normwise(got[rows], want) <= 1e-7, (m, k, n)
    ai = oracle.fill(oracle.DIST_INT8, 83, 300, 500).astype(np.float32)
    bi = oracle.fill(oracle.DIST_INT8, 84, 500, 200).astype(np.float32)
    gi = host(ctx.sgemm(dev(ai), dev(bi), mode=P.MODE_OZAKI))
    assert (gi.astype(np.float64) == oracle.matmul_rows(list(range(300)), ai, bi)).all()


def test_ozaki_mode_host_entry(ctx, oracle):
    a = oracle.fill(oracle.DIST_UNIFORM, 95, 1500, 1300)
    b = oracle.fill(oracle.DIST_UNIFORM, 96, 1300, 1700)
    want = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_OZAKI))
    c, el = ctx.matmul_host(a, b, mode=P.MODE_OZAKI)
    assert el > 0 and (bits(c) == bits(want)).all()
    cf, _ = ctx.matmul_host(a.astype(np.float32), b.astype(np.float32), mode=P.MODE_OZAKI)
    assert (cf == host(ctx.sgemm(dev(a.astype(np.float32)), dev(b.astype(np.float32)),
                                 mode=P.MODE_OZAKI))).all()
    # big enough for the panel pipeline (B prepared once, A in 512-row panels,
    # a ragged last one): still the one-shot bits, fp64 and fp32
    for (m, k, n) in [(2500, 4100, 1000), (1100, 3000, 3100)]:
        a = oracle.fill(oracle.DIST_UNIFORM, 97, m, k)
        b = oracle.fill(oracle.DIST_UNIFORM, 98, k, n) * 1e-3
        want = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_OZAKI))
        c, el = ctx.matmul_host(a, b, mode=P.MODE_OZAKI)
        assert el > 0 and (bits(c) == bits(want)).all(), (m, k, n)
        af, bf = a.astype(np.float32), b.astype(np.float32)
        cf, _ = ctx.matmul_host(af, bf, mode=P.MODE_OZAKI)
        assert (cf == host(ctx.sgemm(dev(af), dev(bf), mode=P.MODE_OZAKI))).all(), (m, k, n)


def test_ozaki_mode_tall_and_wide(ctx, oracle):
    # more rows than a grid dimension holds (row loops) and a 1-column B
    for (m, k, n) in [(70000, 24, 8), (5, 40, 70001), (70000, 3, 1)]:
        A = ctx.fill(P.DIST_INT8, 11, m, k)
        B = ctx.fill(P.DIST_INT8, 12, k, n)
        got = host(ctx.dgemm(A, B, mode=P.MODE_OZAKI))
        rows = [0, m // 2, m - 1]
        want = oracle.matmul_rows(rows, host(A), host(B))
        assert oracle.first_difference(got[rows], want) is None, (m, k, n)


def test_ozaki_mode_in_a_cuda_graph(ctx):
    # captured across its two streams; replays give the eager bits
    T = torch()
    A = ctx.fill(P.DIST_UNIFORM, 91, 512, 700)
    B = ctx.fill(P.DIST_UNIFORM, 92, 700, 300)
    want = host(ctx.dgemm(A, B, mode=P.MODE_OZAKI))
    C2 = T.full((512, 300), float("nan"), dtype=T.float64, device="cuda")
    g = ctx.graph_dgemm(A, B, C2, mode=P.MODE_OZAKI)
    g.launch()
    g.launch()
    assert (bits(host(C2)) == bits(want)).all()
    g.close()


def test_ozaki_mode_long_k_and_limits(ctx, oracle):
    # k beyond the headline (plan: 14 moduli, t = 46 at k = 65536) and the
    # int32-accumulation limit
    m, k, n = 64, 65536 + 40, 96
    A = ctx.fill(P.DIST_UNIFORM, 71, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 72, k, n)
    got = host(ctx.dgemm(A, B, mode=P.MODE_OZAKI))
    rows = [0, 31, 63]
    assert normwise(got[rows], oracle.matmul_rows(rows, host(A), host(B))) <= 1e-13
    assert P.ozaki_plan(65536) == (14, 46) and P.ozaki_plan(65576) == (15, 49)
    with pytest.raises(P.DimensionError):
        ctx.dgemm(ctx.fill(P.DIST_UNIFORM, 1, 2, 131073), ctx.fill(P.DIST_UNIFORM, 2, 131073, 2),
                  mode=P.MODE_OZAKI)


def test_ozaki_mode_row_slices_strides_scales_and_specials(ctx, oracle):
    T = torch()
    m, k, n = 700, 513, 600
    a = oracle.fill(oracle.DIST_UNIFORM, 61, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 62, k, n)
    a[3] *= 1e-200                                   # per-row / per-column power-of-two scaling
    a[5] *= 1e250
    b[:, 7] *= 3e-300
    full = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_OZAKI))
    for r0, r1 in ((0, 128), (128, 333), (333, 700)):    # row slices: same bits
        part = host(ctx.dgemm(dev(a[r0:r1]), dev(b), mode=P.MODE_OZAKI))
        assert (bits(part) == bits(full[r0:r1])).all()
    rows = [3, 5, 100]
    want = oracle.matmul_rows(rows, a, b)
    for i, r in enumerate(rows):                     # row-wise relative accuracy (overflow-safe)
        scale = np.max(np.abs(want[i]))
        assert np.linalg.norm((full[r] - want[i]) / scale) <= 1e-13 * np.linalg.norm(want[i] / scale)
    big = T.zeros((m, k + 3), dtype=T.float64, device="cuda")[:, 1:k + 1]   # misaligned view
    big.copy_(T.from_numpy(a))
    assert (bits(host(ctx.dgemm(big, dev(b), mode=P.MODE_OZAKI))) == bits(full)).all()
    a2 = a.copy()
    a2[10, 20] = np.inf
    b2 = b.copy()
    b2[30, 40] = np.nan
    g = host(ctx.dgemm(dev(a2), dev(b2), mode=P.MODE_OZAKI))
    assert np.isnan(g[10]).all() and np.isnan(g[:, 40]).all()
    assert (bits(np.delete(np.delete(g, 10, 0), 40, 1)) ==
            bits(np.delete(np.delete(full, 10, 0), 40, 1))).all()


# ----------------------------------------------------------------------------- real inputs: tolerance
def test_config_c1_n1000(ctx, oracle, golden_big):
    n = 1000
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    exact = host(ctx.dgemm(A, B, mode=P.MODE_EXACT))
    assert sha(exact) == golden_big["n1000_uniform_sha256"]
    for mode in (P.MODE_AUTO, P.MODE_DMMA, P.MODE_DMMA_SMALL):
        assert normwise(host(ctx.dgemm(A, B, mode=mode)), exact) <= FP64_TOL


@pytest.mark.parametrize("n", [10, 50, 100, 250, 500, 1500, 2000])
def test_config_c2_sweep(ctx, oracle, n):
    a = oracle.fill(oracle.DIST_UNIFORM, 0, n, n)
    b = oracle.fill(oracle.DIST_UNIFORM, 1, n, n)
    rows = sorted({0, n // 3, n // 2, n - 1})
    want = oracle.matmul_rows(rows, a, b)
    A, B = dev(a), dev(b)
    got = host(ctx.dgemm(A, B, mode=P.MODE_EXACT))
    assert (bits(got[rows]) == bits(want)).all()
    for mode in (P.MODE_AUTO, P.MODE_DMMA, P.MODE_DMMA_SMALL):
        assert normwise(host(ctx.dgemm(A, B, mode=mode))[rows], want) <= FP64_TOL
    # graph replay (small-N latency path) gives the same bits as an eager call
    C1 = ctx.dgemm(A, B, mode=P.MODE_AUTO)
    C2 = torch().full_like(C1, float("nan"))
    g = ctx.graph_dgemm(A, B, C2, mode=P.MODE_AUTO)
    g.launch()
    g.launch()
    assert (bits(host(C1)) == bits(host(C2))).all()
    g.close()


def test_config_c4_n16384_sampled_rows(ctx, oracle, golden_big):
    n = 16384
    rows = golden_big["n16384_rows"]
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    a_rows = host(A[rows])
    b = host(B)
    # oracle rows on the box, pinned against the reference's own rows (sha256)
    want = oracle.matmul_rows(list(range(len(rows))), a_rows, b)
    assert [sha(want[i]) for i in range(len(rows))] == golden_big["n16384_rows_sha256"]
    C = ctx.dgemm(A, B, mode=P.MODE_AUTO)
    got = host(C[rows])
    assert normwise(got, want) <= FP64_TOL
    for i in range(len(rows)):
        assert normwise(got[i], want[i]) <= FP64_TOL
    exact = host(ctx.dgemm(A, B, mode=P.MODE_EXACT)[rows])
    assert (bits(exact) == bits(want)).all()


def test_config_c5_n32768_fp32_sampled_rows(ctx, oracle):
    n = 32768
    T = torch()
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=T.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=T.float32)
    rows = [0, 1, 4095, 4096, 16383, 16384, 24575, 32767]
    C = ctx.sgemm(A, B)
    got = host(C[rows]).astype(np.float64)
    a_rows = host(A[rows])
    b = host(B)
    want = oracle.matmul_rows(list(range(len(rows))), a_rows, b)
    err = normwise(got, want)
    assert err <= FP32_TOL, err


def test_fp32_small_shapes(ctx, oracle):
    # aligned shapes take the TMA kernel, the others the cp.async kernel
    for (m, k, n) in [(1, 1, 1), (3, 5, 7), (128, 128, 128), (129, 1000, 131), (1000, 37, 999),
                      (200, 1000, 1004), (257, 36, 260), (1, 4, 4)]:
        a = oracle.fill(oracle.DIST_NORMAL, 3, m, k, dtype=np.float32)
        b = oracle.fill(oracle.DIST_NORMAL, 4, k, n, dtype=np.float32)
        want = oracle.matmul_rows(list(range(m)), a, b)
        got = host(ctx.sgemm(dev(a), dev(b))).astype(np.float64)
        assert normwise(got, want) <= FP32_TOL


# ----------------------------------------------------------------------------- row-block semantics on one GPU
@pytest.mark.parametrize("P_", [2, 3, 4, 8])
def test_rowblock_slices_bitwise_equal_full_product(ctx, P_):
    # split_rows blocks multiplied separately == 1-GPU product, bitwise: the
    # property that makes P-GPU results identical to 1-GPU results.
    n = 1031
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    for mode in (P.MODE_AUTO, P.MODE_DMMA, P.MODE_EXACT):
        full = host(ctx.dgemm(A, B, mode=mode))
        for off, rows in P.split_rows(n, P_):
            if rows == 0:
                continue
            part = host(ctx.dgemm(A[off:off + rows].contiguous(), B, mode=mode))
            assert (bits(part) == bits(full[off:off + rows])).all()


def test_rowblock_single_rank_entry(ctx, oracle):
    n = 300
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch().empty_like(A)
    el = ctx.rowblock(n, n, n, A, B, C, mode=P.MODE_EXACT)
    assert el > 0
    want = oracle.matmul_seq(host(A), host(B))
    assert oracle.first_difference(host(C), want) is None


def test_rowblock_orders_after_the_callers_stream(ctx):
    # the round runs on the context stream; the Python entry orders it after
    # torch's current stream, where fill queued A and B behind a long sleep
    # (found by the randomized one-GPU-world rounds: without the ordering a
    # round could read its inputs before they were written)
    T = torch()
    n = 512
    for _ in range(2):
        T.cuda._sleep(100_000_000)                      # ~50 ms on the current stream
        A = ctx.fill(P.DIST_UNIFORM, 91, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 92, n, n)
        C = T.full((n, n), float("nan"), dtype=T.float64, device="cuda")
        ctx.rowblock(n, n, n, A, B, C)
        want = ctx.dgemm(A, B)
        assert (bits(host(C)) == bits(host(want))).all()


@pytest.mark.parametrize("mode", ["dmma", "sgemm", "ozaki"])
def test_calls_on_two_streams_do_not_share_a_workspace(ctx, mode):
    # Operands TMA cannot read are packed into a workspace, and MODE_OZAKI
    # keeps its residues in one: a call on stream s2 must not overwrite the
    # workspace a still-running call on stream s1 reads.  s1: a long
    # multiply of packed operands; s2: a short sleep, then the same-shaped
    # multiply of other operands, packed while the first one runs.
    T = torch()
    n = 4099 if mode != "ozaki" else 3001
    dt = T.float32 if mode == "sgemm" else T.float64
    call = ctx.sgemm if mode == "sgemm" else ctx.dgemm
    kw = {} if mode == "sgemm" else {"mode": P.MODE_OZAKI if mode == "ozaki" else P.MODE_AUTO}
    big = [ctx.fill(P.DIST_UNIFORM, 300 + i, n, n + 1, dtype=dt) for i in range(4)]
    ops = [x[:, 1:] for x in big]                     # misaligned views: packed
    A1, B1, A2, B2 = ops[0], ops[1][:, :n], ops[2], ops[3][:, :n]
    want1 = host(call(A1, B1, **kw))
    want2 = host(call(A2, B2, **kw))
    s1, s2 = T.cuda.Stream(), T.cuda.Stream()
    T.cuda.synchronize()
    for _ in range(3):
        with T.cuda.stream(s1):
            C1 = call(A1, B1, **kw)
        with T.cuda.stream(s2):
            T.cuda._sleep(2_000_000)                  # ~1 ms: lands mid-multiply on s1
            C2 = call(A2, B2, **kw)
        T.cuda.synchronize()
        assert (bits(host(C1)) == bits(want1)).all(), mode
        assert (bits(host(C2)) == bits(want2)).all(), mode


def test_many_streams_keep_a_bounded_set_of_workspaces(ctx):
    # per-stream workspaces (packing, stream-K) are capped: cycling through
    # more streams than the cap frees the least recently used ones (after a
    # device synchronisation) -- results unchanged
    T = torch()
    n = 2051                                          # odd: packed operands
    big = ctx.fill(P.DIST_UNIFORM, 41, n, n + 1)
    A, B = big[:, 1:], big[:, :n]
    want = bits(host(ctx.dgemm(A, B, mode=P.MODE_DMMA)))   # stream-K + packing
    streams = [T.cuda.Stream() for _ in range(40)]
    for rep in range(2):
        outs = []
        for s in streams:
            with T.cuda.stream(s):
                outs.append(ctx.dgemm(A, B, mode=P.MODE_DMMA))
        T.cuda.synchronize()
        for o in outs:
            assert (bits(host(o)) == want).all()


def test_one_context_from_four_threads(ctx):
    # The ABI is reentrant per context (a mutex; ctypes drops the GIL): four
    # threads, each on its own torch stream, mix device multiplies (AUTO,
    # EXACT, packed views, fp32, OZAKI) and host-buffer multiplies (pageable
    # and pinned) on one context; every result equals its single-threaded
    # reference, bitwise.
    import threading
    T = torch()
    rng = np.random.default_rng(77)
    jobs = []
    for i in range(24):
        n = int(rng.integers(40, 700))
        kind = ["auto", "exact", "packed", "f32", "ozaki", "host", "host_pinned"][i % 7]
        dt = T.float32 if kind == "f32" else T.float64
        big = ctx.fill(P.DIST_UNIFORM, 500 + i, n, n + 1, dtype=dt)
        A = big[:, 1:] if kind == "packed" else big[:, :n].contiguous()
        B = ctx.fill(P.DIST_UNIFORM, 600 + i, n, n, dtype=dt)
        jobs.append((kind, A, B))

    def run(kind, A, B):
        if kind == "f32":
            return host(ctx.sgemm(A, B))
        if kind in ("host", "host_pinned"):
            a, b = host(A), host(B)
            if kind == "host_pinned":
                a = T.from_numpy(a).pin_memory().numpy()
                b = T.from_numpy(b).pin_memory().numpy()
            return ctx.matmul_host(a, b, mode=P.MODE_EXACT)[0].copy()
        mode = {"auto": P.MODE_AUTO, "exact": P.MODE_EXACT, "packed": P.MODE_AUTO,
                "ozaki": P.MODE_OZAKI}[kind]
        return host(ctx.dgemm(A, B, mode=mode))

    want = [run(*j) for j in jobs]
    T.cuda.synchronize()
    errors = []

    def worker(t):
        s = T.cuda.Stream()
        with T.cuda.stream(s):
            for rep in range(3):
                for i in range(t, len(jobs), 4):
                    got = run(*jobs[i])
                    if not (bits(got) == bits(want[i])).all():
                        errors.append((t, rep, i, jobs[i][0]))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=240)
    assert not any(th.is_alive() for th in threads)
    assert not errors, errors


def test_graph_outliving_its_context_is_an_error_not_a_crash():
    # mmws_gpu_destroy releases the device resources of the context's live
    # graphs and detaches them: launching one afterwards is an error, and
    # destroying it just frees the handle
    T = torch()
    c = P.Context(0)
    A = c.fill(P.DIST_UNIFORM, 1, 100, 100)
    C_ = T.empty_like(A)
    g = c.graph_dgemm(A, A, C_)
    g.launch()
    T.cuda.synchronize()
    c.close()
    with pytest.raises(P.GpuError):
        g.launch()
    g.close()
    g.close()                                          # idempotent


def test_rowblock_nccl_path_single_rank(oracle):
    # The NCCL engine (dlopen of the process's libnccl, communicator, broadcast,
    # grouped exchanges, two sub-blocks, stream joins) in a 1-rank world -- the
    # only multi-rank code this one-GPU box can execute.  Bitwise equal to the
    # plain multiply.
    T = torch()
    c2 = P.Context(0)
    try:
        c2.comm_init(1, 0, P.nccl_unique_id())
        n = 2304  # >= 1024 rows per rank: two sub-blocks
        A = c2.fill(P.DIST_UNIFORM, 0, n, n)
        B = c2.fill(P.DIST_UNIFORM, 1, n, n)
        C = T.empty_like(A)
        rows = [0, 1, 1151, 1152, n - 1]   # both sub-blocks
        ref_rows = oracle.matmul_rows(rows, host(A), host(B))
        for mode in (P.MODE_AUTO, P.MODE_EXACT):
            el = c2.rowblock(n, n, n, A, B, C, mode=mode)
            assert el > 0
            want = host(c2.dgemm(A, B, mode=mode))
            assert (bits(host(C)) == bits(want)).all()
            got_rows = host(C)[rows]
            if mode == P.MODE_EXACT:       # the engine's rows against the CPU oracle
                assert (bits(got_rows) == bits(ref_rows)).all()
            else:
                assert normwise(got_rows, ref_rows) <= FP64_TOL
            c, el = c2.master_run_host(host(A), host(B), mode=mode)
            assert el > 0 and (bits(c) == bits(want)).all()
        # fp32 through the same engine
        Af, Bf = A.float(), B.float()
        Cf = T.empty_like(Af)
        c2.rowblock(n, n, n, Af, Bf, Cf, f32=True)
        assert (host(Cf) == host(c2.sgemm(Af, Bf))).all()
        # cost-model calibration probes (bench_main.cpp:64-93 analogue)
        assert c2.link_probe(1 << 24, 3) > 1e9
        c2.comm_destroy()
        with pytest.raises(P.GpuError):
            c2.link_probe(1 << 20, 1)                                 # needs a communicator
    finally:
        c2.close()


def test_gemm_probe_rate(ctx):
    r = ctx.gemm_probe(2048, P.MODE_AUTO, 3)
    assert 5e12 < r < 40e12                       # FP64 tensor pipe: <= 37.2 TFLOP/s
    assert ctx.gemm_probe(512, P.MODE_EXACT, 2) < r
    with pytest.raises(P.DomainError):
        ctx.gemm_probe(0)


def _ipc_child(conn):
    import ctypes
    import paper_1012_2273_b200 as P2
    handle, m, n, k = conn.recv()
    ctx = P2.Context(0)
    lib = P2._abi.load()
    ptr = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 72).from_buffer_copy(handle)
    assert lib.mmws_gpu_ipc_open(ctx.handle, buf, ctypes.byref(ptr)) == 0, P2._abi.last_error()
    A = ctx.fill(P2.DIST_UNIFORM, 5, m, k)
    B = ctx.fill(P2.DIST_UNIFORM, 6, k, n)
    import torch as T
    T.cuda.synchronize()
    # this process's GEMM stores straight into the other process's buffer
    assert lib.mmws_gpu_dgemm(ctx.handle, m, n, k, A.data_ptr(), k, B.data_ptr(), n, ptr.value,
                              n, P2.MODE_AUTO, None) == 0, P2._abi.last_error()
    assert lib.mmws_gpu_synchronize(ctx.handle) == 0
    conn.send("done")
    ctx.close()


def test_ipc_peer_stores_from_another_process(ctx):
    # The fused C gather of the row-block path: a worker's GEMM epilogue writes
    # its rows into rank 0's C through a CUDA IPC mapping.  Two processes on one
    # GPU exercise the same export/open/store path (no kernel waits on another).
    import ctypes
    import multiprocessing as mp
    T = torch()
    m, n, k = 700, 900, 500
    Cbig = T.zeros((m + 8, n), dtype=T.float64, device="cuda")
    out = (ctypes.c_uint8 * 72)()
    lib = P._abi.load()
    assert lib.mmws_gpu_ipc_export(ctx.handle, Cbig[4:].data_ptr(), out) == 0, P._abi.last_error()
    mpc = mp.get_context("spawn")
    a, b = mpc.Pipe()
    proc = mpc.Process(target=_ipc_child, args=(b,))
    proc.start()
    a.send((bytes(out), m, n, k))
    assert a.poll(240) and a.recv() == "done"
    proc.join(60)
    assert proc.exitcode == 0
    A = ctx.fill(P.DIST_UNIFORM, 5, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 6, k, n)
    want = host(ctx.dgemm(A, B))
    got = host(Cbig)
    assert (bits(got[4:4 + m]) == bits(want)).all()
    assert (got[:4] == 0).all() and (got[4 + m:] == 0).all()


# ----------------------------------------------------------------------------- boundary behaviour
def test_host_entry_matches_device_entry(ctx, oracle):
    a = oracle.fill(oracle.DIST_UNIFORM, 5, 257, 300)
    b = oracle.fill(oracle.DIST_UNIFORM, 6, 300, 129)
    for mode in FP64_MODES:
        c, el = ctx.matmul_host(a, b, mode=mode)
        assert el > 0
        assert (bits(c) == bits(host(ctx.dgemm(dev(a), dev(b), mode=mode)))).all()
    c, _ = ctx.matmul_host(a, b, mode=P.MODE_EXACT)
    assert oracle.first_difference(c, oracle.matmul_seq(a, b)) is None
    af, bf = a.astype(np.float32), b.astype(np.float32)
    cf, _ = ctx.matmul_host(af, bf)
    assert normwise(cf.astype(np.float64), oracle.matmul_rows(list(range(257)), af, bf)) <= FP32_TOL


def test_host_entry_pinned_panels_match_pageable_and_device(ctx, oracle):
    # host buffers take the row-panel pipeline from m*n*k = 1e8 on (8 panels
    # pinned; 4 / 2 / 8 pageable by size): same bits either way, and the
    # device entry's
    T = torch()
    for (m, k, n) in [(700, 600, 900), (1001, 999, 1003), (333, 2000, 700)]:
        a = oracle.fill(oracle.DIST_UNIFORM, 7, m, k)
        b = oracle.fill(oracle.DIST_UNIFORM, 8, k, n)
        want = host(ctx.dgemm(dev(a), dev(b)))
        ap = T.from_numpy(a).pin_memory().numpy()
        bp = T.from_numpy(b).pin_memory().numpy()
        cp = T.empty((m, n), dtype=T.float64).pin_memory().numpy()
        got, _ = ctx.matmul_host(ap, bp, out=cp)
        assert (bits(got) == bits(want)).all(), (m, k, n, "pinned")
        got, _ = ctx.matmul_host(a, b)
        assert (bits(got) == bits(want)).all(), (m, k, n, "pageable")
        ex, _ = ctx.matmul_host(ap, bp, mode=P.MODE_EXACT, out=cp)
        rows = [0, m // 2, m - 1]
        assert (bits(ex[rows]) == bits(oracle.matmul_rows(rows, a, b))).all()


def test_host_entry_any_panel_count_gives_the_same_bits(ctx, oracle):
    # MMWS_GPU_HOST_PANELS forces the row-panel count of a host-buffer
    # multiply: every count (one panel .. more panels than 128-row bands)
    # gives the device entry's bits, pageable and pinned, AUTO and EXACT
    T = torch()
    m, k, n = 777, 515, 1029
    a = oracle.fill(oracle.DIST_UNIFORM, 31, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 32, k, n)
    ap = T.from_numpy(a).pin_memory().numpy()
    bp = T.from_numpy(b).pin_memory().numpy()
    try:
        for mode in (P.MODE_AUTO, P.MODE_EXACT):
            want = bits(host(ctx.dgemm(dev(a), dev(b), mode=mode)))
            for panels in ("1", "2", "3", "4", "8", "64"):
                ctx.tune("MMWS_GPU_HOST_PANELS", panels)
                for x, y in ((a, b), (ap, bp)):
                    got, _ = ctx.matmul_host(x, y, mode=mode)
                    assert (bits(got) == want).all(), (mode, panels, x.flags.c_contiguous)
    finally:
        ctx.tune("MMWS_GPU_HOST_PANELS", "0")


@pytest.mark.timeout(180, method="thread")
@pytest.mark.parametrize("ctas", [None, "1", "3"])
def test_latency_server_bitwise_equals_device_entry(oracle, monkeypatch, ctas):
    # While the resident server kernel runs, a device-wide synchronize
    # (torch.cuda.synchronize) would wait for it forever: the expected results
    # are computed before server_start, and only stream-ordered copies are used.
    if ctas is not None:
        monkeypatch.setenv("MMWS_GPU_SERVER_CTAS", ctas)
    shapes = [(1, 1, 1), (2, 3, 4), (10, 10, 10), (17, 96, 5), (50, 50, 50), (96, 96, 96),
              (96, 1, 96), (64, 96, 80), (95, 93, 91), (3, 96, 96)]
    c = P.Context(0)
    try:
        cases = []
        for seed, (m, k, n) in enumerate(shapes):
            a = oracle.fill(oracle.DIST_UNIFORM, 100 + seed, m, k)
            b = oracle.fill(oracle.DIST_UNIFORM, 200 + seed, k, n)
            want = {mode: host(c.dgemm(dev(a), dev(b), mode=mode))
                    for mode in (P.MODE_AUTO, P.MODE_EXACT)}
            cases.append((a, b, want))
        with pytest.raises(P.GpuError):
            c.server_matmul(np.ones((2, 2)), np.ones((2, 2)))       # not started
        c.server_start()
        c.server_start()                                             # idempotent
        for a, b, want in cases:
            for mode in (P.MODE_AUTO, P.MODE_EXACT):
                got, el = c.server_matmul(a, b, mode=mode)
                assert el > 0
                assert (bits(got) == bits(want[mode])).all(), (a.shape, b.shape, mode)
            got, _ = c.server_matmul(a, b, mode=P.MODE_EXACT)
            assert oracle.first_difference(got, oracle.matmul_seq(a, b)) is None
        for a, b, want in cases:                                     # routed by matmul_host
            for mode in (P.MODE_AUTO, P.MODE_EXACT):
                assert (bits(c.matmul_host(a, b, mode=mode)[0]) == bits(want[mode])).all()
        a = oracle.fill(oracle.DIST_UNIFORM, 1, 50, 50)
        first, _ = c.server_matmul(a, a)
        for _ in range(200):                                         # repeated requests
            again, _ = c.server_matmul(a, a)
        assert (bits(again) == bits(first)).all()
        # the server does not block stream-ordered work of the same context
        x = dev(a)
        y = c.dgemm(x, x, mode=P.MODE_EXACT).cpu().numpy()
        assert oracle.first_difference(y, oracle.matmul_seq(a, a)) is None
        # nor host-buffer calls it does not take, even when they must grow the
        # context's device buffers (cudaFree would wait for the server)
        for nn in (100, 300, 700):
            big = oracle.fill(oracle.DIST_INT8, nn, nn, nn)
            got, _ = c.matmul_host(big, big, mode=P.MODE_EXACT)
            assert oracle.first_difference(got, oracle.matmul_threads(big, big)) is None
        with pytest.raises(P.DimensionError):
            c.server_matmul(np.ones((97, 2)), np.ones((2, 2)))
        with pytest.raises(P.DimensionError):
            c.server_matmul(np.ones((2, 3)), np.ones((2, 2)))
        with pytest.raises(P.DomainError):
            c.server_matmul(a, a, mode=P.MODE_DMMA)
        c.server_stop()
        c.server_start()                                             # restart after stop
        got, _ = c.server_matmul(a, a, mode=P.MODE_EXACT)
        assert oracle.first_difference(got, oracle.matmul_seq(a, a)) is None
    finally:
        c.close()                                                    # stops the server too


@pytest.mark.parametrize("shape", [(1301, 1299, 1303), (2048, 1024, 4096), (2100, 1000, 2500)])
def test_host_pipeline_bitwise_equals_device(ctx, oracle, shape):
    # big enough to take the overlapped (row-panel x column-block) host path
    T = torch()
    m, k, n = shape
    a = oracle.fill(oracle.DIST_UNIFORM, 21, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 22, k, n)
    ap = T.from_numpy(a).pin_memory().numpy()
    bp = T.from_numpy(b).pin_memory().numpy()
    for mode in (P.MODE_AUTO, P.MODE_EXACT):
        want = host(ctx.dgemm(dev(a), dev(b), mode=mode))
        for (x, y) in ((a, b), (ap, bp)):
            c, el = ctx.matmul_host(x, y, mode=mode)
            assert el > 0 and (bits(c) == bits(want)).all()
        c, el = ctx.master_run_host(ap, bp, mode=mode)
        assert (bits(c) == bits(want)).all()
    rows = [0, m // 2, m - 1]
    assert oracle.first_difference(c[rows], oracle.matmul_rows(rows, a, b)) is None
    af, bf = a.astype(np.float32), b.astype(np.float32)
    cf, _ = ctx.matmul_host(af, bf)
    assert (cf == host(ctx.sgemm(dev(af), dev(bf)))).all()


def test_streamed_host_path_random_shapes(ctx):
    # host_multiply_streamed (one persistent DMMA kernel fed by PCIe bands,
    # arrival flags, per-row-band copy-out): seeded random shapes with ragged
    # last bands (m, n not multiples of 256 / 512, k small to large), pageable
    # and pinned, AUTO and DMMA -- bitwise the device-pointer call
    T = torch()
    rng = np.random.default_rng(5150)
    seen = 0
    for case in range(10):
        m = int(rng.integers(2200, 4200))
        n = int(rng.integers(1100, 2100)) * 2
        k = int(rng.integers(8, 2100)) * 2
        A = ctx.fill(P.DIST_UNIFORM, 700 + case, m, k)
        B = ctx.fill(P.DIST_UNIFORM, 800 + case, k, n)
        mode = P.MODE_AUTO if case % 2 else P.MODE_DMMA
        want = bits(host(ctx.dgemm(A, B, mode=mode)))
        a, b = host(A), host(B)
        if case % 3 == 0:
            a = T.from_numpy(a).pin_memory().numpy()
            b = T.from_numpy(b).pin_memory().numpy()
        got, el = ctx.matmul_host(a, b, mode=mode)
        seen += "streamed" in ctx.last_plan
        assert el > 0 and (bits(got) == want).all(), (m, k, n, mode)
    assert seen >= 8, seen


def test_pageable_host_buffers_bigger_than_the_staging_ring(ctx, oracle):
    # pageable numpy buffers go through the pinned chunk ring (4 x 32 MB):
    # 128 MB operands wrap it several times; fp64 streamed path, fp32 panel
    # path, exact panel path -- all bitwise the device-pointer results
    n = 4096
    A = ctx.fill(P.DIST_UNIFORM, 41, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 42, n, n)
    a, b = host(A), host(B)
    for mode in (P.MODE_AUTO, P.MODE_EXACT):
        c, el = ctx.matmul_host(a, b, mode=mode)
        assert el > 0 and (bits(c) == bits(host(ctx.dgemm(A, B, mode=mode)))).all(), mode
    af, bf = a.astype(np.float32), b.astype(np.float32)
    cf, _ = ctx.matmul_host(af, bf)
    assert (cf == host(ctx.sgemm(dev(af), dev(bf)))).all()
    # ragged rows / a view with a row pitch (np.ascontiguousarray copies it)
    a2 = np.ascontiguousarray(a[:4000, :3001])
    b2 = np.ascontiguousarray(b[:3001, :4093])
    c2, _ = ctx.matmul_host(a2, b2, mode=P.MODE_EXACT)
    rows = [0, 1999, 3999]
    assert oracle.first_difference(c2[rows], oracle.matmul_rows(rows, a2, b2)) is None


def test_strided_views_and_unaligned_leading_dims(ctx, oracle):
    T = torch()
    big_a = ctx.fill(P.DIST_UNIFORM, 7, 300, 301)
    big_b = ctx.fill(P.DIST_UNIFORM, 8, 211, 259)
    A = big_a[3:203, 1:212]   # odd offset -> misaligned base, lda = 301
    B = big_b[:, 2:201]       # ldb = 259
    a, b = host(A.contiguous()), host(B.contiguous())
    want = oracle.matmul_seq(a, b)
    Cbig = T.zeros((200, 205), dtype=T.float64, device="cuda")
    Cv = Cbig[:, 3:202]
    for mode in FP64_MODES:
        ctx.dgemm(A, B, Cv, mode=mode)
        got = host(Cv.contiguous())
        if mode == P.MODE_EXACT:
            assert oracle.first_difference(got, want) is None
        else:
            assert normwise(got, want) <= FP64_TOL
        cb = host(Cbig)
        assert (cb[:, :3] == 0).all() and (cb[:, 202:] == 0).all()


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 3, 7), (129, 200, 131), (300, 17, 257),
                                   (1000, 64, 1001), (2400, 300, 2500)])
def test_no_writes_outside_c(ctx, shape):
    # canary frame around a strided C view: every mode must write exactly C
    T = torch()
    m, k, n = shape
    A = ctx.fill(P.DIST_UNIFORM, 1, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 2, k, n)
    for mode in FP64_MODES:
        buf = T.full((m + 2, n + 3), -7.5, dtype=T.float64, device="cuda")
        C = buf[1:m + 1, 1:n + 1]
        ctx.dgemm(A, B, C, mode=mode)
        b = host(buf)
        assert (b[0] == -7.5).all() and (b[m + 1] == -7.5).all(), mode
        assert (b[:, 0] == -7.5).all() and (b[:, n + 1:] == -7.5).all(), mode
        assert not np.isnan(b[1:m + 1, 1:n + 1]).any()
    Af, Bf = A.float(), B.float()
    for sl in (slice(None), slice(0, k)):
        buf = T.full((m + 2, n + 5), -7.5, dtype=T.float32, device="cuda")
        C = buf[1:m + 1, 4:n + 4]
        ctx.sgemm(Af[:, sl], Bf[sl], C)
        b = host(buf)
        assert (b[0] == -7.5).all() and (b[m + 1] == -7.5).all()
        assert (b[:, :4] == -7.5).all() and (b[:, n + 4:] == -7.5).all()


def test_errors_map_to_reference_types(ctx):
    T = torch()
    a = T.zeros((2, 3), dtype=T.float64, device="cuda")
    b = T.zeros((2, 2), dtype=T.float64, device="cuda")
    with pytest.raises(P.DimensionError):
        ctx.dgemm(a, b)                       # inner mismatch (matrix.hpp:113-116)
    with pytest.raises(P.DomainError):
        ctx.dgemm(a, a.t().contiguous(), mode=99)
    with pytest.raises(P.DimensionError):
        ctx.matmul_host(np.zeros((2, 3)), np.zeros((2, 2)))


def test_device_generators_match_oracle(ctx, oracle):
    for dist in (oracle.DIST_UNIT, oracle.DIST_UNIFORM, oracle.DIST_INT8):
        for (r, c, first) in [(1, 1, 0), (17, 23, 0), (64, 100, 12345)]:
            want = oracle.fill(dist, 42, r, c, first=first)
            got = host(ctx.fill(dist, 42, r, c, first=first))
            assert (bits(got) == bits(want)).all()
    T = torch()
    got = host(ctx.fill(P.DIST_NORMAL, 3, 50, 70, dtype=T.float32))
    want = oracle.fill(oracle.DIST_NORMAL, 3, 50, 70, dtype=np.float32)
    assert np.allclose(got, want, rtol=1e-6, atol=1e-6)


def test_launch_accounting(ctx):
    before = ctx.launches
    T = torch()
    a = T.ones((64, 64), dtype=T.float64, device="cuda")
    ctx.dgemm(a, a, mode=P.MODE_DMMA)
    ctx.dgemm(a, a, mode=P.MODE_EXACT)
    assert ctx.launches - before == 2


def test_peak_probes_run(ctx):
    for which in (P.PROBE_DMMA, P.PROBE_DFMA, P.PROBE_DMUL_DADD, P.PROBE_FFMA, P.PROBE_FFMA2,
                  P.PROBE_FFMA2_OUTER):
        tf = ctx.peak_probe(which, 256)
        assert 0.5 < tf < 200, (which, tf)
    # the GEMM operand pattern cannot beat the plain FFMA2 peak
    outer = max(ctx.peak_probe(P.PROBE_FFMA2_OUTER, 20000) for _ in range(2))
    plain = max(ctx.peak_probe(P.PROBE_FFMA2, 100000) for _ in range(2))
    assert 40 < outer <= plain * 1.02, (outer, plain)
    with pytest.raises(P.DomainError):
        ctx.peak_probe(6, 10)


def test_auto_tile_plan_by_size(ctx):
    # AUTO's plan (mmws_gpu_last_plan): the DFMA latency kernel while n, k <= 96,
    # 16x16 DMMA tiles below one 32x32 tile per SM, 32x32 tiles below three
    # 128x128 tiles per SM, 64x64 tiles up to 64 per SM, 128x128 above;
    # MODE_DMMA keeps 128x128 tiles (stream-K from one tile per SM).
    T = torch()
    sms = T.cuda.get_device_properties(0).multi_processor_count
    for (m, n, k), want in [((64, 64, 64), "dgemm_small_kernel<DFMA"),
                            ((96, 96, 96), "dgemm_small_kernel<DFMA"),
                            ((64, 97, 64), "dgemm_dmma_kernel<16x16"),
                            ((250, 250, 250), "dgemm_dmma_kernel<16x16"),
                            ((400, 400, 400), "dgemm_dmma_kernel<32x32"),
                            ((1000, 1000, 1000), "dgemm_dmma_kernel<32x32"),
                            ((128 * 3 * sms, 128, 64), "dgemm_dmma_kernel<64x64"),
                            ((128 * 64 * sms, 128, 16), "dgemm_dmma_kernel<128x128")]:
        A = T.zeros((m, k), dtype=T.float64, device="cuda")
        B = T.zeros((k, n), dtype=T.float64, device="cuda")
        ctx.dgemm(A, B, mode=P.MODE_AUTO)
        assert ctx.last_plan.startswith(want), ((m, n, k), ctx.last_plan)
    A = T.zeros((2048, 2048), dtype=T.float64, device="cuda")
    ctx.dgemm(A, A, mode=P.MODE_DMMA)
    assert ctx.last_plan == "dgemm_dmma_kernel<128x128, 8 math warps, stream-K>"
    ctx.dgemm(A, A, mode=P.MODE_DMMA_SMALL)
    assert ctx.last_plan.startswith("dgemm_dmma_kernel<32x32")
    ctx.dgemm(A, A, mode=P.MODE_EXACT)
    assert ctx.last_plan == "dgemm_exact_tma_kernel<128x128, stream-K>"
    A = T.zeros((1000, 1000), dtype=T.float64, device="cuda")
    ctx.dgemm(A, A, mode=P.MODE_EXACT)             # 256 tiles of 64x64: uneven one-shot
    assert ctx.last_plan == "dgemm_exact_tma_kernel<64x64, stream-K>"
    A = T.zeros((1300, 1300), dtype=T.float64, device="cuda")
    ctx.dgemm(A, A, mode=P.MODE_EXACT)             # 441 tiles: 2.98 per SM, one-shot
    assert ctx.last_plan == "dgemm_exact_tma_kernel<64x64>"
    A = T.zeros((500, 500), dtype=T.float64, device="cuda")
    ctx.dgemm(A, A, mode=P.MODE_EXACT)             # 64 tiles of 64x64: 32x32 tiles
    assert ctx.last_plan == "dgemm_exact_tma_kernel<32x32>"
    A = T.zeros((160, 160), dtype=T.float64, device="cuda")
    ctx.dgemm(A, A, mode=P.MODE_EXACT)
    assert ctx.last_plan.startswith("dgemm_small_kernel<exact")
    T.cuda.synchronize()


@pytest.mark.parametrize("shape", [(193, 200, 202), (500, 500, 500), (128, 1000, 998),
                                   (257, 32, 300), (33, 700, 1000), (640, 18, 250)])
def test_exact_32x32_tma_tiles_are_matmul_seq(ctx, oracle, shape):
    # the 32x32 exact TMA plan (few-tile problems): ragged M / N edges, K not
    # a multiple of the 16-wide k-stage; bitwise the reference chain, and
    # bitwise the other exact kernels (latency kernel / cp.async layout)
    m, k, n = shape
    a = oracle.fill(oracle.DIST_UNIFORM, 61, m, k)
    b = oracle.fill(oracle.DIST_UNIFORM, 62, k, n)
    got = host(ctx.dgemm(dev(a), dev(b), mode=P.MODE_EXACT))
    assert ctx.last_plan == "dgemm_exact_tma_kernel<32x32>", (shape, ctx.last_plan)
    if m * n * k <= 40_000_000:
        assert oracle.first_difference(got, oracle.matmul_seq(a, b)) is None, shape
    else:
        rows = [0, 1, m // 2, m - 1]
        assert (bits(got[rows]) == bits(oracle.matmul_rows(rows, a, b))).all(), shape
    # an odd row pitch sends the same problem to the plain-load kernels
    T = torch()
    big_a = T.zeros((m, k + 1), dtype=T.float64, device="cuda")
    big_a[:, :k] = dev(a)
    other = host(ctx.dgemm(big_a[:, :k], dev(b), mode=P.MODE_EXACT))
    assert (bits(other) == bits(got)).all(), shape


# ----------------------------------------------------------------------------- round-2 fixes
def test_fp32_unaligned_layouts_are_packed_and_bitwise_the_aligned_call(ctx, oracle):
    # lda / ldb not multiples of 4 floats and misaligned bases: the operands
    # are packed for the TMA kernel, so the bits equal the dense call's
    T = torch()
    big_a = ctx.fill(P.DIST_NORMAL, 5, 301, 1031, dtype=T.float32)
    big_b = ctx.fill(P.DIST_NORMAL, 6, 1030, 517, dtype=T.float32)
    A = big_a[1:300, 3:1030]      # lda 1031, base off by 3 floats
    B = big_b[1:1028, 1:516]      # ldb 517
    dense = host(ctx.sgemm(A.contiguous(), B.contiguous()))
    got = host(ctx.sgemm(A, B))
    assert (got.view(np.int32) == dense.view(np.int32)).all()
    rows = [0, 150, 298]
    ref = oracle.matmul_rows(rows, host(A.contiguous()).astype(np.float64),
                             host(B.contiguous()).astype(np.float64))
    assert normwise(got[rows].astype(np.float64), ref) <= FP32_TOL
    assert ctx.last_plan.startswith("sgemm_tma_kernel")


def test_fp32_k_major_staging_is_bitwise_the_row_major_kernel(ctx, oracle):
    # wide fp32 problems transpose A first and stage it k-major (sgemm_tma.cu):
    # same FFMA chain per element, so the same bits as the kernel that stages A
    # as it lies -- ragged shapes, unaligned / strided A, accumulate
    T = torch()
    rng = np.random.default_rng(77)
    shapes = [(128, 16, 2048), (129, 1025, 2049), (333, 3001, 2307), (1, 7, 5), (700, 2048, 2560)]
    try:
        for m, k, n in shapes:
            big_a = ctx.fill(P.DIST_NORMAL, 11 + m, m + 2, k + 5, dtype=T.float32)
            B = ctx.fill(P.DIST_NORMAL, 12 + m, k, n, dtype=T.float32)
            for A in (big_a[1:m + 1, 3:k + 3], big_a[:m, :k].contiguous()):
                ctx.tune("MMWS_GPU_SGEMM_AT", "0")
                want = ctx.sgemm(A, B)
                assert "k-major" not in ctx.last_plan
                ctx.tune("MMWS_GPU_SGEMM_AT", "1")
                got = ctx.sgemm(A, B)
                assert "k-major" in ctx.last_plan
                assert bool((got.view(T.int32) == want.view(T.int32)).all()), (m, k, n)
                if k > 1024:  # accumulate continuation at the 1024-k chunk
                    C = ctx.sgemm(A[:, :1024], B[:1024])
                    ctx.sgemm(A[:, 1024:], B[1024:], C, accumulate=C)
                    assert bool((C.view(T.int32) == want.view(T.int32)).all()), (m, k, n)
        # more than 65535 * 32 rows: the transposition runs on a 1-D grid
        m, k, n = 2_200_000, 4, 2048
        A = ctx.fill(P.DIST_NORMAL, 3, m, k, dtype=T.float32)
        B = ctx.fill(P.DIST_NORMAL, 4, k, n, dtype=T.float32)
        ctx.tune("MMWS_GPU_SGEMM_AT", "0")
        want = ctx.sgemm(A, B)
        ctx.tune("MMWS_GPU_SGEMM_AT", "1")
        got = ctx.sgemm(A, B)
        assert bool(T.equal(got.view(T.int32), want.view(T.int32)))
        del want, got, A, B
        T.cuda.empty_cache()
        # the size rule: from n = 2048 (and at least one 128-row tile)
        ctx.tune("MMWS_GPU_SGEMM_AT", None)
        A = ctx.fill(P.DIST_NORMAL, 1, 256, 64, dtype=T.float32)
        for n, want_at in ((2047, False), (2048, True)):
            ctx.sgemm(A, ctx.fill(P.DIST_NORMAL, 2, 64, n, dtype=T.float32))
            assert ("k-major" in ctx.last_plan) == want_at, (n, ctx.last_plan)
        rows = [0, 127, 255]
        Bn = ctx.fill(P.DIST_NORMAL, 2, 64, 2048, dtype=T.float32)
        got = host(ctx.sgemm(A, Bn))
        ref = oracle.matmul_rows(rows, host(A).astype(np.float64), host(Bn).astype(np.float64))
        assert normwise(got[rows].astype(np.float64), ref) <= FP32_TOL
    finally:
        ctx.tune("MMWS_GPU_SGEMM_AT", None)


def test_graph_keeps_its_own_workspace(ctx, oracle):
    # a graph whose multiply packs its operands must not
    # share the context's workspace -- an eager call that regrows it, or runs
    # meanwhile, must leave the graph's replays correct.
    T = torch()
    big = ctx.fill(P.DIST_UNIFORM, 51, 401, 403)
    A = big[:, 1:400]              # odd leading dimension: packed
    B = ctx.fill(P.DIST_UNIFORM, 52, 399, 397)
    C = T.empty((401, 397), dtype=T.float64, device="cuda")
    want = host(ctx.dgemm(A.contiguous(), B))
    g = ctx.graph_dgemm(A, B, C)
    try:
        g.launch()
        T.cuda.synchronize()
        assert (bits(host(C)) == bits(want)).all()
        # eager calls that need a much bigger packing workspace (regrow)
        big2 = ctx.fill(P.DIST_UNIFORM, 53, 3001, 3003)
        ctx.dgemm(big2[:, 1:3002], big2[:3001, 2:3003])
        T.cuda.synchronize()
        C.zero_()
        g.launch()
        T.cuda.synchronize()
        assert (bits(host(C)) == bits(want)).all()
    finally:
        g.close()


def test_host_pipeline_narrow_tail_block_keeps_the_whole_problem_bits(ctx):
    # m = n = 1060, k = 96 from pinned buffers splits panel 0
    # into column blocks; a narrow last block must not drop onto the latency
    # kernel (it is folded into the previous block)
    T = torch()
    m = n = 1060
    k = 96
    A = ctx.fill(P.DIST_UNIFORM, 61, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 62, k, n)
    want = host(ctx.dgemm(A, B))
    a = T.from_numpy(host(A)).pin_memory().numpy()
    b = T.from_numpy(host(B)).pin_memory().numpy()
    c = T.empty((m, n), dtype=T.float64).pin_memory().numpy()
    got, _ = ctx.matmul_host(a, b, out=c)
    assert (bits(got) == bits(want)).all()


def test_host_and_device_output_checks(ctx):
    # wrong output buffers are rejected before any write
    T = torch()
    a = np.ones((4, 3))
    b = np.ones((3, 5))
    with pytest.raises(P.DimensionError):
        ctx.matmul_host(a, b, out=np.empty((4, 4)))
    with pytest.raises(P.DomainError):
        ctx.matmul_host(a, b, out=np.empty((4, 5), dtype=np.float32))
    with pytest.raises(P.DimensionError):
        ctx.matmul_host(a, b, out=np.empty((5, 4)).T)
    A = ctx.fill(P.DIST_UNIFORM, 1, 4, 3)
    B = ctx.fill(P.DIST_UNIFORM, 2, 3, 5)
    with pytest.raises(P.DimensionError):
        ctx.dgemm(A, B, T.empty((3, 5), dtype=T.float64, device="cuda"))
    with pytest.raises(P.DomainError):
        ctx.dgemm(A, B, T.empty((4, 5), dtype=T.float32, device="cuda"))
    with pytest.raises(P.DomainError):
        ctx.dgemm(A, B, T.empty((4, 5), dtype=T.float64))          # host tensor
    with pytest.raises(P.DomainError):
        ctx.graph_dgemm(A, B.float(), T.empty((4, 5), dtype=T.float64, device="cuda"))
    with pytest.raises(P.DimensionError):
        ctx.rowblock(4, 5, 3, A, B, T.empty((4, 6), dtype=T.float64, device="cuda"))


def test_tuning_knobs_apply_on_a_live_context(ctx):
    n = 2000
    A = ctx.fill(P.DIST_UNIFORM, 71, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 72, n, n)
    ctx.dgemm(A, B, mode=P.MODE_DMMA)
    assert "stream-K" in ctx.last_plan
    ctx.tune("MMWS_GPU_NO_STREAMK", "1")
    ctx.dgemm(A, B, mode=P.MODE_DMMA)
    assert "stream-K" not in ctx.last_plan
    ctx.tune("MMWS_GPU_NO_STREAMK", None)
    ctx.dgemm(A, B, mode=P.MODE_DMMA)
    assert "stream-K" in ctx.last_plan


@pytest.mark.parametrize("mode,shape,cuts", [
    (P.MODE_AUTO, (1000, 777, 2048), (512, 1024)),
    (P.MODE_DMMA, (1000, 777, 2048), (16, 1040)),
    (P.MODE_DMMA_SMALL, (257, 300, 800), (400,)),
    (P.MODE_EXACT, (257, 300, 800), (16, 32, 784)),
    (P.MODE_EXACT, (1500, 1100, 1600), (800,)),
    (P.MODE_AUTO, (4099, 1000, 4099), (2048,)),
])
def test_accumulate_in_k_panels_is_bitwise_one_call(ctx, oracle, mode, shape, cuts):
    # mmws_gpu_dgemm_acc: C = Cin + A.B continues Cin's chains, so a K split
    # at multiples of 16 chained through the accumulator reproduces the
    # one-call bits (what the row-block workers do while B is arriving)
    T = torch()
    m, n, k = shape
    A = ctx.fill(P.DIST_UNIFORM, 81, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 82, k, n)
    want = host(ctx.dgemm(A, B, mode=mode))
    edges = (0,) + tuple(cuts) + (k,)
    C = T.empty((m, n), dtype=T.float64, device="cuda")
    ctx.dgemm(A[:, :edges[1]], B[:edges[1]], C, mode=mode)
    for k0, k1 in zip(edges[1:-1], edges[2:]):
        ctx.dgemm(A[:, k0:k1], B[k0:k1], C, mode=mode, accumulate=C)   # in place
    assert (bits(host(C)) == bits(want)).all(), (mode, shape, cuts)
    # out of place: Cin untouched, C = Cin + A.B
    Cin = T.empty_like(C)
    ctx.dgemm(A[:, :edges[-2]], B[:edges[-2]], Cin, mode=mode)
    keep = host(Cin)
    C2 = T.full_like(C, float("nan"))
    ctx.dgemm(A[:, edges[-2]:], B[edges[-2]:], C2, mode=mode, accumulate=Cin)
    assert (bits(host(C2)) == bits(want)).all()
    assert (bits(host(Cin)) == bits(keep)).all()
    if mode == P.MODE_EXACT:
        rows = [0, m // 2, m - 1]
        assert (bits(want[rows]) == bits(oracle.matmul_rows(rows, host(A), host(B)))).all()


def test_accumulate_fp32_chunks_and_limits(ctx):
    T = torch()
    m, n, k = 700, 900, 3072
    A = ctx.fill(P.DIST_NORMAL, 91, m, k, dtype=T.float32)
    B = ctx.fill(P.DIST_NORMAL, 92, k, n, dtype=T.float32)
    want = host(ctx.sgemm(A, B))
    C = ctx.sgemm(A[:, :1024], B[:1024])
    ctx.sgemm(A[:, 1024:], B[1024:], C, accumulate=C)       # split at the 1024-k chunk
    assert (host(C).view(np.int32) == want.view(np.int32)).all()
    Ad = A.double()
    Bd = B.double()
    with pytest.raises(P.DomainError):
        ctx.dgemm(Ad, Bd, mode=P.MODE_OZAKI, accumulate=T.zeros((m, n), dtype=T.float64,
                                                                 device="cuda"))
    with pytest.raises(P.DimensionError):
        ctx.dgemm(Ad, Bd, accumulate=T.zeros((m - 1, n), dtype=T.float64, device="cuda"))

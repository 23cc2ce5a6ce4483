"""CPU tests: the oracle is pinned against the reference (golden vectors that the
reference itself produced, and -- where oracle/_ref is built -- the reference
code directly), plus the reference's own properties (test_matrix.cpp,
test_workshare.cpp, test_protocol.cpp, acceptance.cpp)."""
import numpy as np
import pytest


def from_hex(h, shape):
    return np.array([int(v, 16) for v in h], dtype=np.uint64).view(np.float64).reshape(shape)


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


needs_ref = pytest.mark.skipif(
    not __import__("os").path.exists(
        __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "oracle", "_ref",
                                   "libmmws_ref.so")),
    reason="oracle/_ref not built")


def test_random_stream_matches_reference_golden(oracle, golden_small):
    for seed, hx in golden_small["random_matrix"].items():
        got = oracle.fill(oracle.DIST_UNIT, int(seed), 2, 4)
        assert (bits(got).ravel() == bits(from_hex(hx, (2, 4))).ravel()).all()
    # pinned first draws recorded by the survey
    assert oracle.fill(oracle.DIST_UNIT, 0, 1, 1)[0, 0] == 0.88331080821364261
    assert oracle.fill(oracle.DIST_UNIT, 1, 1, 1)[0, 0] == 0.5665615751722809


def test_counter_based_stream_offsets(oracle):
    full = oracle.fill(oracle.DIST_UNIFORM, 9, 7, 11)
    part = oracle.fill(oracle.DIST_UNIFORM, 9, 2, 11, first=3 * 11)
    assert (bits(full[3:5]) == bits(part)).all()


def test_derived_distributions(oracle):
    u = oracle.fill(oracle.DIST_UNIT, 5, 64, 64)
    assert (oracle.fill(oracle.DIST_UNIFORM, 5, 64, 64) == 2.0 * u - 1.0).all()
    i = oracle.fill(oracle.DIST_INT8, 5, 300, 300)
    assert i.min() == -8 and i.max() == 8 and (i == np.round(i)).all()
    assert len(np.unique(i)) == 17
    z = oracle.fill(oracle.DIST_NORMAL, 5, 400, 400, dtype=np.float32)
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1) < 0.01


def test_known_products(oracle, golden_small):
    c = oracle.matmul_seq(np.array([[1., 2], [3, 4]]), np.array([[5., 6], [7, 8]]))
    assert c.tolist() == [[19, 22], [43, 50]]
    assert (bits(c).ravel() == bits(from_hex(golden_small["matmul_2x2"], (2, 2))).ravel()).all()
    c = oracle.matmul_seq(np.array([[3.25]]), np.array([[-2.0]]))
    assert c[0, 0] == 3.25 * -2.0


def test_oracle_products_match_reference_golden(oracle, golden_small):
    for key, hx in golden_small["products_unit"].items():
        if key.startswith("sq"):
            n = int(key[2:])
            a = oracle.fill(oracle.DIST_UNIT, 1000 + n, n, n)
            b = oracle.fill(oracle.DIST_UNIT, 2000 + n, n, n)
            shape = (n, n)
        else:
            m, k, n = (int(x) for x in key[4:].split("x"))
            seeds = {"rect2x5x4": (303, 304), "rect4x7x3": (27, 28), "rect5x7x4": (31, 32)}[key]
            a = oracle.fill(oracle.DIST_UNIT, seeds[0], m, k)
            b = oracle.fill(oracle.DIST_UNIT, seeds[1], k, n)
            shape = (m, n)
        want = from_hex(hx, shape)
        for got in (oracle.matmul_seq(a, b), oracle.matmul_threads(a, b, 3),
                    oracle.matmul_rows(list(range(shape[0])), a, b),
                    oracle.worker_block(a, b)):
            assert oracle.first_difference(got, want) is None, key


def test_row_sampled_oracle_is_bitwise(oracle):
    a = oracle.fill(oracle.DIST_UNIFORM, 0, 120, 333)
    b = oracle.fill(oracle.DIST_UNIFORM, 1, 333, 97)
    full = oracle.matmul_seq(a, b)
    rows = [0, 5, 64, 119]
    assert oracle.first_difference(oracle.matmul_rows(rows, a, b, threads=4), full[rows]) is None
    # fp32 widened variant == fp64 oracle of the widened inputs
    af, bf = a.astype(np.float32), b.astype(np.float32)
    want = oracle.matmul_seq(af.astype(np.float64), bf.astype(np.float64))
    assert oracle.first_difference(oracle.matmul_rows(rows, af, bf), want[rows]) is None


def test_identity_and_signed_zero(oracle):
    for n in (1, 2, 5, 13):
        a = oracle.fill(oracle.DIST_UNIT, 1000 + n, n, n)
        eye = np.eye(n)
        assert oracle.first_difference(oracle.matmul_seq(a, eye), a) is None
        assert oracle.first_difference(oracle.matmul_seq(eye, a), a) is None
    z1, z2 = np.array([[0.0]]), np.array([[-0.0]])
    assert oracle.first_difference(z1, z2) == 0   # memcmp semantics (matrix.hpp:136-145)
    c = oracle.matmul_seq(np.array([[-0.0]]), np.array([[1.0]]))
    assert not np.signbit(c[0, 0])                 # acc starts at +0.0


def test_partitions_and_op_count(oracle, golden_small):
    for key, want in golden_small["split_rows"].items():
        n, w = (int(x) for x in key.split(","))
        assert [list(x) for x in oracle.split_rows(n, w)] == want
    for key, want in golden_small["static_partition"].items():
        n, w = (int(x) for x in key.split(","))
        assert [list(x) for x in oracle.static_partition(n, w)] == want
    for n, want in golden_small["op_count"].items():
        assert oracle.op_count(int(n)) == want
    assert oracle.split_rows(4, 3) == [(0, 2), (2, 1), (3, 1)]     # test_protocol.cpp:23-24
    assert oracle.split_rows(6, 3) == [(0, 2), (2, 2), (4, 2)]
    assert oracle.split_rows(2, 3) == [(0, 1), (1, 1), (2, 0)]
    with pytest.raises(ValueError):
        oracle.split_rows(4, 0)
    with pytest.raises(ValueError):
        oracle.op_count(0)
    assert oracle.op_count(1000) == 1_999_000_000


@needs_ref
def test_oracle_equals_reference_code_directly(oracle):
    rng_dims = [(1, 1, 1), (3, 7, 2), (33, 17, 65), (64, 64, 64), (100, 3, 50)]
    for (m, k, n) in rng_dims:
        a = oracle.ref_random_matrix(m, k, m * 7 + k)
        b = oracle.ref_random_matrix(k, n, n * 11 + k)
        want = oracle.ref_matmul_seq(a, b)
        assert oracle.first_difference(oracle.matmul_seq(a, b), want) is None
        assert oracle.first_difference(oracle.ref_matmul_threads(a, b, 4), want) is None
    for n in range(0, 60, 7):
        for w in range(1, 10):
            assert oracle.static_partition(n, w) == oracle.ref_static_partition(n, w)
            assert oracle.split_rows(n, w) == oracle.ref_split_rows(n, w)


def test_split_rows_grid_properties(oracle):
    # test_protocol.cpp:32-54 / acceptance.cpp:136-169
    for n in range(1, 201, 7):
        for w in range(1, 17):
            parts = oracle.split_rows(n, w)
            nxt = 0
            for i, (off, rows) in enumerate(parts):
                assert off == nxt and rows == n // w + (1 if i < n % w else 0)
                nxt += rows
            assert nxt == n

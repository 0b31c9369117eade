"""Pin the CPU oracle (oracle/patchlift_oracle.c) before trusting it.

* against the reference tests' known-answer vectors (cited file:line);
* against tests/golden/golden.npz, generated from the reference itself;
* bit for bit against the reference library (oracle/_ref) on randomised cases
  with the reference tests' own seeds where it is built.
"""
import math

import numpy as np
import pytest

from oracle import OracleError


# ---- known answers from the reference's own tests ---------------------------
def test_worked_kernel_example(orc):
    # banded_kernel_test.cpp:75-94 
    band, _ = orc.banded_kernel([1, 2, 3, 4], 1, 1)
    at = lambda i, j: band[i, j - i + 1]
    assert [at(0, 0), at(1, 1), at(2, 2), at(3, 3)] == [6.0, 14.0, 29.0, 41.0]
    assert [at(0, 1), at(1, 2), at(2, 3)] == [9.0, 20.0, 34.0]
    dist = orc.distance_band([1, 2, 3, 4], 1, 1)
    assert [dist[0, 2], dist[1, 2], dist[2, 2], dist[1, 1]] == [2.0, 3.0, 2.0, 0.0]
    assert math.isnan(band[0, 0]) and math.isnan(band[3, 2])  # sentinels


def test_naive_distance_examples(orc):
    # banded_kernel_test.cpp:200-207
    assert orc.patch_distance([1, 2, 3, 4], 0, 1, 1) == 2.0
    assert orc.patch_distance([1, 2, 3, 4], 0, 3, 1) == 17.0
    assert orc.patch_distance([1, 2, 3, 4], 2, 2, 1) == 0.0
    assert orc.patch_distance([1, 2, 3, 4], 0, 0, 4) == 0.0


def test_worked_filter_example(orc):
    # nlm_test.cpp:52-66 
    e1 = math.exp(-1.0)
    for naive in (False, True):
        out = orc.nlm_1d([0, 0, 10], 1, 0, 10.0, naive=naive)
        assert abs(out[1] - 10 * e1 / (2 + e1)) < 1e-9
        assert abs(out[1] - 1.5536253) < 1e-6 * (1 + 1.5536253)  # doctest Approx scale
        assert abs(out[0]) < 1e-12
        assert abs(out[2] - 10 / (e1 + 1)) < 1e-9


def test_weight(orc):
    # nlm_test.cpp:45-50
    assert orc.weight(0.0, 10.0) == 1.0
    assert abs(orc.weight(1.0, 1.0) - math.exp(-1)) < 1e-14
    assert abs(orc.weight(50.0, 5.0) - math.exp(-2)) < 1e-14
    assert orc.weight(1e9, 1.0) == 0.0


def test_mirror_examples(orc):
    # core_types_test.cpp:53-61 and the mirror rule for every pad (:63-80)
    assert list(orc.extend_symmetric([1, 2, 3, 4], 1)) == [1, 1, 2, 3, 4, 4]
    assert list(orc.extend_symmetric([1, 2, 3], 2)) == [2, 1, 1, 2, 3, 3, 2]
    f = [5, -1, 0.25, 9, 13]
    for pad in range(len(f) + 1):
        e = orc.extend_symmetric(f, pad)
        for t in range(pad):
            assert e[pad - 1 - t] == f[t] and e[pad + len(f) + t] == f[len(f) - 1 - t]
    with pytest.raises(OracleError, match="insufficient signal for symmetric extension"):
        orc.extend_symmetric(f, 6)


def test_validation_messages(orc):
    # core_types_test.cpp:37-51 (exact strings)
    cases = [((-1, 0, 1.0, 8), "search radius must be nonnegative"),
             ((0, -1, 1.0, 8), "patch radius must be nonnegative"),
             ((0, 9, 1.0, 8), "patch radius exceeds signal length"),
             ((1, 1, 0.0, 8), "smoothing parameter h must be positive"),
             ((1, 1, -2.0, 8), "smoothing parameter h must be positive")]
    for args, msg in cases:
        with pytest.raises(OracleError, match=msg):
            orc.validate_params(*args)
    orc.validate_params(0, 0, 1.0, 1)
    orc.validate_geometry(100, 8, 8)


def test_integer_kernel_exact_vs_direct(orc):
    # banded_kernel_test.cpp:96-118: integer data -> recursion == direct sum exactly
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(1, 41))
        K = int(rng.integers(0, n + 1))
        S = int(rng.integers(0, 12))
        f = rng.integers(0, 256, n).astype(np.float64)
        a = orc.distance_band(f, S, K)
        b = orc.distance_band_direct(f, S, K)
        assert np.array_equal(a, b, equal_nan=True)


def test_op_count_closed_form(orc):
    # banded_kernel_test.cpp:247-279
    rng = np.random.default_rng(15)
    for _ in range(40):
        n = int(rng.integers(1, 101))
        K = min(n, int(rng.integers(0, 6)))
        S = int(rng.integers(0, 14))
        _, (adds, muls) = orc.banded_kernel(rng.uniform(0, 255, n), S, K)
        ea = sum(2 * K + 2 * (n - d - 1) for d in range(min(S, n - 1) + 1))
        em = sum(2 * K + 1 + 2 * (n - d - 1) for d in range(min(S, n - 1) + 1))
        assert (adds, muls) == (ea, em)


# ---- golden fixtures (generated from the reference, tests/golden/make_golden.py)
def test_golden_lines(orc, golden):
    for t, (n, S, K, h, integer) in enumerate(golden["line_cases"]):
        n, S, K = int(n), int(S), int(K)
        f = golden[f"l{t}_f"]
        assert np.array_equal(orc.distance_band(f, S, K), golden[f"l{t}_dist"], equal_nan=True)
        assert np.array_equal(orc.nlm_1d(f, S, K, h), golden[f"l{t}_nlm"])


def test_golden_images(orc, golden):
    for t, (r, c, S, K, h) in enumerate(golden["image_cases"]):
        img = golden[f"i{t}_img"]
        for op in ("row", "col", "rc", "cr", "snlm"):
            assert np.array_equal(orc.filter(op, img, int(S), int(K), h), golden[f"i{t}_{op}"]), op


def test_golden_c1(orc, golden):
    from paper_1407_2343_b200 import workloads
    S, K, h = workloads.params("c1")
    f = workloads.make_config("c1").astype(np.float64)
    assert np.allclose(golden["c1_input_sum"], [f.sum(), (f * f).sum()], rtol=0, atol=0)
    assert np.array_equal(orc.nlm_1d(f, S, K, h).astype(np.float32), golden["c1_nlm"])
    assert np.array_equal(orc.distance_band(f[:4096], S, K), golden["c1_dist_head"], equal_nan=True)


def test_golden_metrics(orc, golden):
    for t, _ in enumerate(golden["metric_cases"]):
        got = orc.metrics(golden[f"m{t}_a"], golden[f"m{t}_b"])
        assert np.array_equal(np.array(got), golden[f"m{t}_metrics"]), t


def test_metrics_edge_cases(orc):
    a = np.random.default_rng(3).uniform(0, 255, (12, 15))
    mse, psnr, ssim = orc.metrics(a, a)
    assert mse == 0.0 and psnr == float("inf") and ssim == 1.0
    from oracle import OracleError
    with pytest.raises(OracleError, match="11x11 structural window"):
        orc.metrics(a[:10], a[:10])


# ---- bit for bit against the reference library -----------------------------
def test_oracle_equals_reference_1d(orc, ref):
    rng = np.random.default_rng(101)
    for _ in range(300):
        n = int(rng.integers(1, 200))
        K = int(rng.integers(0, min(n, 9) + 1))
        S = int(rng.integers(0, 20))
        h = float(np.exp(rng.uniform(np.log(0.5), np.log(5000.0))))
        f = rng.uniform(0, 255, n)
        assert np.array_equal(orc.distance_band(f, S, K), ref.distance_band(f, S, K), equal_nan=True)
        band_o, _ = orc.banded_kernel(f, S, K)
        band_r, _ = ref.banded_kernel(f, S, K)
        assert np.array_equal(band_o, band_r, equal_nan=True)
        assert np.array_equal(orc.nlm_1d(f, S, K, h), ref.nlm_1d(f, S, K, h))
        assert np.array_equal(orc.nlm_1d(f, S, K, h, naive=True), ref.nlm_1d(f, S, K, h, naive=True))


def test_oracle_equals_reference_images(orc, ref):
    rng = np.random.default_rng(105)
    for _ in range(12):
        r, c = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        S = int(rng.integers(0, 12))
        K = int(rng.integers(0, min(r, c, 5) + 1))
        h = float(np.exp(rng.uniform(np.log(0.5), np.log(5000.0))))
        img = rng.uniform(0, 255, (r, c))
        for op in ("row", "col", "rc", "cr", "snlm"):
            assert np.array_equal(orc.filter(op, img, S, K, h, threads=3),
                                  ref.filter(op, img, S, K, h, threads=2)), op


def test_oracle_ops_equal_reference(orc, ref):
    f = np.random.default_rng(29).uniform(0, 255, 100)
    a, b = [0] * 4, [0] * 4
    orc.nlm_1d(f, 6, 2, 40.0, ops=a)
    ref.nlm_1d(f, 6, 2, 40.0, ops=b)
    assert a == b


def test_oracle_metrics_equal_reference(orc, ref):
    rng = np.random.default_rng(105)
    for _ in range(6):
        r, c = int(rng.integers(11, 60)), int(rng.integers(11, 60))
        a = rng.uniform(0, 255, (r, c))
        b = np.clip(a + rng.normal(0, 15, (r, c)), 0, 255)
        assert orc.metrics(a, b) == ref.metrics(a, b)

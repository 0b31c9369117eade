"""Parity of the CUDA path (through the C ABI) against the oracle.

Tolerance tiers:
  T0  distances on integer inputs: bit-exact (int32 and fp32 exports)
  T1  distances on float inputs:   |dd| <= 1e-5 (1 + E_i + E_j) + 4 sqrt(C+S) 2^-24 (2K+1) M^2
                                   (E = patch energy, M = max |f|, C = segment length)
  T2  filter outputs:              max abs error <= 1e-3 on the [0, 255] scale
  T3  structural invariants:       exact (transpose equivariance, constant
                                   fixpoints, S=0 identity, batch/launch invariance)
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1407_2343_b200 as pl  # noqa: E402
from paper_1407_2343_b200 import workloads  # noqa: E402

T2 = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    pl.lib()  # fail loudly if the native library is missing
    yield


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rand_line(rng, n, integer):
    if integer:
        return rng.integers(0, 256, n).astype(np.float32)
    return rng.uniform(0, 255, n).astype(np.float32)


# ---- T0 / T1: distances -------------------------------------------------------
def test_integer_distances_bit_exact(orc):
    rng = np.random.default_rng(11)
    for _ in range(150):
        n = int(rng.integers(1, 300))
        K = int(rng.integers(0, min(n, 8) + 1))
        S = int(rng.integers(0, 34))
        f = rand_line(rng, n, True)
        want = orc.distance_band(f, S, K)
        got32 = host(pl.distance_band(dev(f), S, K, dtype=torch.int32))[0]
        gotf = host(pl.distance_band(dev(f), S, K))[0]
        mask = np.isnan(want)
        assert np.array_equal(np.where(mask, -1, want).astype(np.int64), got32.astype(np.int64)), (n, S, K)
        assert np.array_equal(want, gotf.astype(np.float64), equal_nan=True), (n, S, K)


def test_c4_distances_bit_exact(orc):
    # config 4 shape: 2048-sample integer rows of the quantised synthetic image
    S, K, _ = workloads.params("c4")
    img = workloads.make_config("c4", batch=1)[0]
    rows = img[::64]  # 32 rows across the image
    got = host(pl.distance_band(dev(rows), S, K, dtype=torch.int32))
    for r in range(rows.shape[0]):
        want = orc.distance_band(rows[r].astype(np.float64), S, K)
        want = np.where(np.isnan(want), -1, want).astype(np.int64)
        assert np.array_equal(want, got[r].astype(np.int64)), r


def test_float_distances_t1(orc):
    rng = np.random.default_rng(12)
    for _ in range(60):
        n = int(rng.integers(8, 600))
        K = int(rng.integers(0, 9))
        S = int(rng.integers(1, 26))
        f = rand_line(rng, n, False).astype(np.float64)
        want = orc.distance_band(f, S, K)
        got = host(pl.distance_band(dev(f), S, K))[0].astype(np.float64)
        kern, _ = orc.banded_kernel(f, S, K)
        energy = kern[:, S]
        i = np.arange(n)[:, None]
        j = i + np.arange(-S, S + 1)[None, :]
        ok = ~np.isnan(want)
        # relative to patch energy, plus the running sum's rounding scale: each
        # update rounds at 2^-24 of a sum bounded by (2K+1) M^2, random-walked
        # over at most C+S steps since the segment's anchor
        steps = pl.segment_length(n, S) + S
        walk = 4 * math.sqrt(steps) * 2.0 ** -24 * (2 * K + 1) * float(np.abs(f).max()) ** 2
        tol = 1e-5 * (1 + energy[i.repeat(2 * S + 1, 1)] + energy[np.clip(j, 0, n - 1)]) + walk
        assert np.array_equal(np.isnan(got), ~ok)
        assert np.all(np.abs(got - want)[ok] <= tol[ok]), (n, S, K)


def test_banded_kernel_f64_bit_equal(orc):
    rng = np.random.default_rng(13)
    for _ in range(60):
        n = int(rng.integers(1, 120))
        K = int(rng.integers(0, min(n, 8) + 1))
        S = int(rng.integers(0, 20))
        f = rng.uniform(0, 255, n)
        want, _ = orc.banded_kernel(f, S, K)
        got = host(pl.banded_kernel_f64(dev(f, torch.float64), S, K))[0]
        assert np.array_equal(want, got, equal_nan=True), (n, S, K)


# ---- T2: filter outputs ----------------------------------------------------------
def test_lines_vs_oracle(orc):
    rng = np.random.default_rng(21)
    worst = 0.0
    for t in range(200):
        n = int(rng.integers(1, 400))
        S = int(rng.integers(0, 40))
        K = int(rng.integers(0, min(n, 9) + 1))
        h = float(np.exp(rng.uniform(np.log(15.0), np.log(1000.0))))
        f = rand_line(rng, n, t % 3 == 0)
        want = orc.nlm_1d(f.astype(np.float64), S, K, h)
        got = host(pl.nlm_1d_patchlift(dev(f), (S, K, h))).astype(np.float64)
        worst = max(worst, float(np.abs(got - want).max()))
        assert np.abs(got - want).max() <= T2, (n, S, K, h)
    print("worst T2 error over random lines:", worst)


def test_naive_route_vs_oracle(orc):
    rng = np.random.default_rng(22)
    for _ in range(40):
        n = int(rng.integers(1, 200))
        S = int(rng.integers(0, 20))
        K = int(rng.integers(0, min(n, 6) + 1))
        h = float(np.exp(rng.uniform(np.log(15.0), np.log(1000.0))))
        f = rand_line(rng, n, False)
        want = orc.nlm_1d(f.astype(np.float64), S, K, h, naive=True)
        got = host(pl.nlm_1d_naive(dev(f), (S, K, h))).astype(np.float64)
        assert np.abs(got - want).max() <= T2


def test_c1_full_vs_golden(golden):
    S, K, h = workloads.params("c1")
    f = workloads.make_config("c1")
    got = host(pl.nlm_1d_patchlift(dev(f), (S, K, h)))
    err = np.abs(got.astype(np.float64) - golden["c1_nlm"].astype(np.float64)).max()
    assert err <= T2, err


def test_images_vs_oracle(orc):
    rng = np.random.default_rng(26)
    shapes = [(1, 1), (1, 7), (7, 1), (2, 3), (14, 9), (24, 17), (33, 40), (64, 64), (130, 257),
              (300, 129)]
    for r, c in shapes:
        for S, K in [(0, 0), (1, 0), (4, 2), (10, 3), (15, 5), (25, 7), (40, 1)]:
            if K > min(r, c):
                continue
            h = float(np.exp(rng.uniform(np.log(15.0), np.log(1000.0))))
            img = rng.uniform(0, 255, (r, c)).astype(np.float32)
            x = dev(img)
            for op, fn in (("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass),
                           ("rc", pl.snlm_2d_row_col), ("cr", pl.snlm_2d_col_row),
                           ("snlm", pl.snlm_2d)):
                want = orc.filter(op, img.astype(np.float64), S, K, h, threads=4)
                got = host(fn(x, (S, K, h))).astype(np.float64)
                assert np.abs(got - want).max() <= T2, (r, c, S, K, op)


def test_small_h_strict_t2_default_policy(orc):
    """Small h on 8-bit data, default precision policy (PL_PRECISION_AUTO):
    every reference-API filter holds the strict T2 = 1e-3 against the oracle
    at any h.  Below pl_fast_h_threshold() (48 per 255 of data range) the
    library measures the input's range and runs the call in double on the
    device (route "f64<...>"); the host-buffer pipeline follows the same rule."""
    rng = np.random.default_rng(41)
    assert pl.fast_h_threshold() == 48.0
    for t in range(12):
        r, c = int(rng.integers(20, 200)), int(rng.integers(20, 200))
        S, K = int(rng.integers(2, 26)), int(rng.integers(0, 3))
        h = float(rng.uniform(5.0, 47.0))
        img = rng.uniform(0, 255, (r, c)).astype(np.float32)
        x = dev(img)
        for op, fn in (("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass),
                       ("rc", pl.snlm_2d_row_col), ("cr", pl.snlm_2d_col_row),
                       ("snlm", pl.snlm_2d)):
            want = orc.filter(op, img.astype(np.float64), S, K, h, threads=4)
            err = np.abs(host(fn(x, (S, K, h))).astype(np.float64) - want).max()
            assert pl.last_route().startswith("f64"), (op, pl.last_route())
            assert err <= T2, (op, r, c, S, K, h, err)
        if t < 4:
            want = orc.filter("rc", img.astype(np.float64), S, K, h, threads=4)
            got = pl.snlm_2d_row_col_host(img[None], (S, K, h))
            assert np.abs(np.asarray(got)[0].astype(np.float64) - want).max() <= T2, (r, c, S, K, h)
    # 1D lines through the same policy; with a line stride ld > n via the C ABI
    n, S, K, h = 700, 10, 3, 9.0
    sig = rng.uniform(0, 255, (5, n)).astype(np.float32)
    got = host(pl.nlm_1d_patchlift(dev(sig), (S, K, h)))
    assert pl.last_route().startswith("f64")
    padded = np.full((5, n + 3), 1e9, np.float32)  # the padding must not widen the measured range
    padded[:, :n] = sig
    xp = dev(padded)
    yp = torch.full_like(xp, -7.0)
    pl._check(pl.lib().pl_nlm_lines(xp.data_ptr(), yp.data_ptr(), 5, n, n + 3,
                                    pl._params((S, K, h)), pl._stream(xp)))
    yp = host(yp)
    assert np.all(yp[:, n:] == -7.0)
    for l in range(5):
        want = orc.nlm_1d(sig[l].astype(np.float64), S, K, h)
        assert np.abs(got[l].astype(np.float64) - want).max() <= T2
        assert np.array_equal(yp[l, :n], got[l])


def test_precision_policy_routes(orc):
    """The policy is scale-aware and never touches the configs' settings:
    h >= 48 goes straight to the fp32 kernels (no range measurement), a small
    h on small-range data stays on them (h / range decides), PL_PRECISION_FAST
    pins them, and a CUDA graph (fp32 only) refuses an h it cannot bound."""
    rng = np.random.default_rng(43)
    img = rng.uniform(0, 255, (96, 130)).astype(np.float32)
    x = dev(img)
    pl.snlm_2d_row_col(x, (10, 3, 74.8))
    assert not pl.last_route().startswith("f64"), pl.last_route()
    pl.snlm_2d_row_col(x, (10, 3, 12.0))
    assert pl.last_route().startswith("f64"), pl.last_route()
    # the same image on a [0, 1] scale with h scaled alike is the same problem:
    # unit-range data with h = 0.3 (= 76.5 per 255) is a fast-route call
    unit = (img / 255.0).astype(np.float32)
    got = host(pl.snlm_2d_row_col(dev(unit), (10, 3, 0.3)))
    assert not pl.last_route().startswith("f64"), pl.last_route()
    want = orc.filter("rc", unit.astype(np.float64), 10, 3, 0.3, threads=4)
    assert np.abs(got.astype(np.float64) - want).max() <= T2 / 255.0
    # the partition-level entry points are fp32 only: they refuse such an h
    # unless the caller pins the fp32 kernels
    with pytest.raises(RuntimeError, match="runs the fp32 kernels only"):
        pl.nlm_row_pass_blocked(x, (10, 3, 12.0), 65)
    with pl.precision_policy("fast"):
        pl.nlm_row_pass_blocked(x, (10, 3, 12.0), 65)
        fast = host(pl.snlm_2d_row_col(x, (10, 3, 12.0)))
        assert not pl.last_route().startswith("f64"), pl.last_route()
        g = pl.RCGraph(x, (10, 3, 12.0))  # allowed when pinned fast
        del g
    with pytest.raises(RuntimeError, match="graph capture covers the fp32 kernels only"):
        pl.RCGraph(x, (10, 3, 12.0))
    # fp32 characterisation (what the policy protects from): the fast route's
    # error at small h stays within T2 (25/h)^2 single pass / (36/h)^2 composite
    want = orc.filter("rc", img.astype(np.float64), 10, 3, 12.0, threads=4)
    assert np.abs(fast.astype(np.float64) - want).max() <= T2 * (36.0 / 12.0) ** 2


def test_small_h_fast_policy_bounds(orc):
    """PL_PRECISION_FAST at small h (the fp32 kernels' own behaviour).  The fp32
    moving sums carry an absolute rounding error ~ ulp(max d') that grows like
    1/h^2, and a two-pass composite amplifies the first pass's output rounding
    by the second pass's condition number (~ 2 |df| |f - out| / h^2): single
    passes stay within T2 (25/h)^2, composites within T2 (36/h)^2 (worst over
    ~25,000 random cases, tools/fuzz_parity.py: 0.84 and 0.65 of these)."""
    rng = np.random.default_rng(41)
    with pl.precision_policy("fast"):
        for t in range(12):
            r, c = int(rng.integers(20, 200)), int(rng.integers(20, 200))
            S, K = int(rng.integers(2, 26)), int(rng.integers(0, 3))
            h = float(rng.uniform(5.0, 25.0))
            img = rng.uniform(0, 255, (r, c)).astype(np.float32)
            x = dev(img)
            for op, fn in (("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass),
                           ("rc", pl.snlm_2d_row_col), ("cr", pl.snlm_2d_col_row)):
                want = orc.filter(op, img.astype(np.float64), S, K, h, threads=4)
                err = np.abs(host(fn(x, (S, K, h))).astype(np.float64) - want).max()
                tol = T2 * max(1.0, ((25.0 if op in ("row", "col") else 36.0) / h) ** 2)
                assert err <= tol, (op, r, c, S, K, h, err)


def test_golden_images_t2(golden):
    for t, (r, c, S, K, h) in enumerate(golden["image_cases"]):
        x = dev(golden[f"i{t}_img"])
        for op, fn in (("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass),
                       ("rc", pl.snlm_2d_row_col), ("cr", pl.snlm_2d_col_row), ("snlm", pl.snlm_2d)):
            got = host(fn(x, (int(S), int(K), h))).astype(np.float64)
            assert np.abs(got - golden[f"i{t}_{op}"]).max() <= T2, (t, op)


def test_c2_rc_vs_oracle(orc):
    S, K, h = workloads.params("c2")
    img = workloads.make_config("c2")[0]
    want = orc.snlm_rc(img.astype(np.float64), S, K, h, threads=8)
    got = host(pl.snlm_2d_row_col(dev(img), (S, K, h))).astype(np.float64)
    assert np.abs(got - want).max() <= T2


@pytest.mark.slow
def test_c3_rc_vs_oracle(orc):
    S, K, h = workloads.params("c3")
    img = workloads.make_config("c3")[0]
    got = host(pl.snlm_2d_row_col(dev(img), (S, K, h))).astype(np.float64)
    rows = slice(0, 4096, 97)  # a sampled stripe keeps the CPU check to seconds
    want_rows = orc.row_pass(img.astype(np.float64), S, K, h, threads=8)
    want = orc.col_pass(want_rows, S, K, h, threads=8)
    assert np.abs(got[rows] - want[rows]).max() <= T2


def test_c4_batch_rc_vs_oracle(orc):
    S, K, h = workloads.params("c4")
    imgs = workloads.make_config("c4", batch=2)
    got = host(pl.snlm_2d_row_col(dev(imgs), (S, K, h))).astype(np.float64)
    for b in range(2):
        want = orc.snlm_rc(imgs[b].astype(np.float64), S, K, h, threads=8)
        assert np.abs(got[b] - want).max() <= T2


# ---- T3: structural invariants ----------------------------------------------------
def test_transpose_equivariance_bitwise():
    rng = np.random.default_rng(3001)
    for r, c, S, K, h in [(24, 17, 5, 2, 50.0), (12, 15, 5, 1, 55.0), (200, 333, 15, 5, 140.0),
                          (64, 300, 10, 3, 74.8)]:
        img = rng.uniform(0, 255, (r, c)).astype(np.float32)
        x, xt = dev(img), dev(img.T)
        p = (S, K, h)
        assert np.array_equal(host(pl.snlm_2d(xt, p)), host(pl.snlm_2d(x, p)).T)
        assert np.array_equal(host(pl.snlm_2d_row_col(xt, p)), host(pl.snlm_2d_col_row(x, p)).T)
        assert np.array_equal(host(pl.snlm_2d_col_row(xt, p)), host(pl.snlm_2d_row_col(x, p)).T)
        assert np.array_equal(host(pl.nlm_col_pass(x, p)), host(pl.nlm_row_pass(xt, p)).T)


@pytest.mark.parametrize("shape,p", [((40, 52), (5, 1, 52.0)), ((2, 300, 256), (10, 3, 60.0)),
                                     ((1, 130, 128), (15, 5, 90.0)), ((1, 90, 64), (25, 7, 99.0)),
                                     ((37, 1), (5, 1, 52.0)), ((1, 29), (4, 1, 52.0)),
                                     ((33, 70), (40, 2, 52.0)), ((3, 20, 24), (6, 9, 52.0))])
def test_snlm_is_mean_of_orders_bitwise(shape, p):
    """snlm_2d fuses the average into RC's final column-pass store (every
    walker and the direct route): bitwise (RC + CR) / 2."""
    img = np.random.default_rng(27).uniform(0, 255, shape).astype(np.float32)
    x = dev(img)
    rc = host(pl.snlm_2d_row_col(x, p))
    cr = host(pl.snlm_2d_col_row(x, p))
    assert np.array_equal(host(pl.snlm_2d(x, p)), (rc + cr) / np.float32(2))


def test_constant_fixpoints_exact():
    for c in (0.0, 0.5, 100.0, 255.0):
        f = np.full(40, c, np.float32)
        assert np.array_equal(host(pl.nlm_1d_patchlift(dev(f), (5, 2, 30.0))), f)
        img = np.full((12, 17), c, np.float32)
        for fn in (pl.snlm_2d, pl.snlm_2d_row_col, pl.nlm_row_pass, pl.nlm_col_pass, pl.nlm_2d_naive):
            assert np.array_equal(host(fn(dev(img), (6, 2, 30.0))), img)
        big = np.full((3, 300, 260), c, np.float32)
        assert np.array_equal(host(pl.snlm_2d_row_col(dev(big), (15, 5, 30.0))), big)


def test_s0_identity_exact():
    rng = np.random.default_rng(22)
    f = rng.uniform(0, 255, 33).astype(np.float32)
    assert np.array_equal(host(pl.nlm_1d_patchlift(dev(f), (0, 3, 25.0))), f)
    img = rng.uniform(0, 255, (9, 13)).astype(np.float32)
    for fn in (pl.snlm_2d, pl.snlm_2d_row_col, pl.snlm_2d_col_row):
        assert np.array_equal(host(fn(dev(img), (0, 3, 25.0))), img)


def test_h_infinity_window_mean():
    # nlm_test.cpp:114-141 re-tiered: fp32 window mean, tolerance 1e-4
    f = np.random.default_rng(23).uniform(0, 255, 64).astype(np.float32)
    S = 7
    got = host(pl.nlm_1d_patchlift(dev(f), (S, 2, 1e9)))
    for i in range(64):
        lo, hi = max(0, i - S), min(63, i + S)
        assert abs(got[i] - f[lo:hi + 1].astype(np.float64).mean()) <= 1e-4


def test_convex_bounds():
    # acceptance_main.cpp:258-283 on the device: output inside [min, max] of input
    rng = np.random.default_rng(105)
    for t in range(40):
        img = rng.uniform(0, 255, (64, 64)).astype(np.float32)
        p = (1 + int(rng.integers(0, 8)), int(rng.integers(0, 5)),
             float(np.exp(rng.uniform(np.log(0.5), np.log(5000.0)))))
        for fn in (pl.snlm_2d, pl.nlm_2d_naive):
            out = host(fn(dev(img), p))
            assert out.min() >= img.min() and out.max() <= img.max(), (t, p)


def test_batch_and_launch_invariance_bitwise():
    rng = np.random.default_rng(28)
    imgs = rng.uniform(0, 255, (5, 150, 190)).astype(np.float32)
    p = (10, 3, 74.8)
    whole = host(pl.snlm_2d_row_col(dev(imgs), p))
    for b in range(5):
        assert np.array_equal(host(pl.snlm_2d_row_col(dev(imgs[b]), p)), whole[b])
    again = host(pl.snlm_2d_row_col(dev(imgs), p))
    assert np.array_equal(whole, again)  # deterministic


def test_lines_batch_invariance_bitwise():
    rng = np.random.default_rng(30)
    x = rng.uniform(0, 255, (37, 1000)).astype(np.float32)
    p = (15, 5, 140.0)
    allr = host(pl.nlm_1d_patchlift(dev(x), p))
    for r in (0, 5, 36):
        assert np.array_equal(host(pl.nlm_1d_patchlift(dev(x[r]), p)), allr[r])


def test_blocked_row_pass_layout():
    rng = np.random.default_rng(31)
    img = rng.uniform(0, 255, (96, 256)).astype(np.float32)
    p = (10, 3, 74.8)
    plain = host(pl.nlm_row_pass(dev(img), p))
    for cb in (32, 64, 128, 256):
        blk = host(pl.nlm_row_pass_blocked(dev(img), p, cb))
        want = plain.reshape(96, 256 // cb, cb).transpose(1, 0, 2).reshape(-1)
        assert np.array_equal(blk.reshape(-1), want), cb


def test_host_e2e_matches_device():
    rng = np.random.default_rng(32)
    imgs = rng.uniform(0, 255, (3, 128, 200)).astype(np.float32)
    p = (10, 3, 74.8)
    dev_out = host(pl.snlm_2d_row_col(dev(imgs), p))
    host_out = pl.snlm_2d_row_col_host(imgs, p)
    assert np.array_equal(dev_out, host_out)


@pytest.mark.parametrize("shape,p", [
    ((1, 1100, 8200), (10, 3, 74.8)),   # 3 column segments, 1 per block
    ((2, 5000, 1800), (15, 5, 140.0)),  # 11 segments, two images through the same buffers
    ((1, 9000, 1000), (25, 7, 136.9)),  # 8+ segments (multiple of 8), interior/edge bodies
])
def test_host_e2e_streamed_large_images(shape, p):
    """Images of 32 MiB and more go through pl_snlm_2d_row_col_host's
    intra-image pipeline (row chunks up, row pass per chunk, column pass per
    block of whole segments as soon as its rows are there, output rows down):
    bitwise the device result."""
    rng = np.random.default_rng(shape[1])
    imgs = rng.uniform(0, 255, shape).astype(np.float32)
    dev_out = host(pl.snlm_2d_row_col(dev(imgs), p))
    host_out = pl.snlm_2d_row_col_host(imgs, p)
    assert np.array_equal(dev_out, np.asarray(host_out))


def test_validation_errors_raise():
    x = dev(np.ones((5, 9), np.float32))
    with pytest.raises(pl.ValidationError, match="patch radius exceeds signal length"):
        pl.snlm_2d(x, (2, 6, 5.0))
    with pytest.raises(pl.ValidationError, match="smoothing parameter h must be positive"):
        pl.snlm_2d(x, (2, 1, -1.0))
    with pytest.raises(pl.ValidationError, match="search radius must be nonnegative"):
        pl.nlm_1d_patchlift(dev(np.ones(5, np.float32)), (-1, 1, 5.0))


def test_nlm_2d_naive_vs_reference(ref):
    rng = np.random.default_rng(33)
    img = rng.uniform(0, 255, (23, 17)).astype(np.float32)
    for p in [(4, 1, 35.0), (3, 2, 60.0)]:
        want = ref.filter("nlm2d", img.astype(np.float64), *p)
        got = host(pl.nlm_2d_naive(dev(img), p)).astype(np.float64)
        assert np.abs(got - want).max() <= T2


def test_rc_vs_reference_library(ref):
    """The CUDA path against the reference's own snlm_2d_row_col (oracle/_ref)."""
    S, K, h = workloads.params("c2")
    img = workloads.make_config("c2")[0][:256, :320]
    want = ref.filter("rc", img.astype(np.float64), S, K, h, threads=0)
    got = host(pl.snlm_2d_row_col(dev(img), (S, K, h))).astype(np.float64)
    assert np.abs(got - want).max() <= T2


def test_cpp_dropin_library():
    """libpatchlift_b200 through the reference's C++ API (tests/cpp/dropin_check.cpp)."""
    import os
    import subprocess
    exe = os.path.join(pl.LIBDIR, "dropin_check")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_hot_kernel_line_modes_bitwise():
    """The hot kernel's lines per lane and warps per CTA (performance choices,
    pinned through pl_debug_set_route): every combination, with every staging
    / flush mode (row pass, column pass, transposed-intermediate RC, S-NLM
    with the fused average), gives the same bits."""
    rng = np.random.default_rng(8)
    cases = [(2, 200, 256, 10, 3), (1, 130, 192, 15, 5), (1, 120, 96, 25, 7)]
    xs = [dev(rng.uniform(0, 255, (b, r, c))) for (b, r, c, S, K) in cases]
    runs = []
    for lines, wpc in ((0, 0), (1, 0), (2, 0), (0, 8), (0, 2), (1, 8)):
        outs = {}
        with pl.debug_route(0, lines, wpc):
            for x, (b, r, c, S, K) in zip(xs, cases):
                p = (S, K, 40.0 + 5 * S)
                for nm, f in (("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass),
                              ("rc", pl.snlm_2d_row_col), ("snlm", pl.snlm_2d)):
                    outs[f"{S}_{nm}"] = host(f(x, p))
                    assert pl.last_route().startswith("hot<"), pl.last_route()
        runs.append(outs)
    for other in runs[1:]:
        for key in runs[0]:
            assert np.array_equal(runs[0][key], other[key]), key


def test_portable_and_production_walkers_bitwise_equal():
    """The hot kernel (walk3), the production walker (smem-staged, packed
    f32x2, walk2) and the portable one (plgpu_walk.cuh) run the same per-line
    arithmetic: outputs are bitwise equal."""
    rng = np.random.default_rng(5)
    cases = [(2, 300, 517, 10, 3), (1, 260, 700, 15, 5), (1, 333, 290, 25, 7),
             (3, 64, 128, 4, 2), (1, 40, 1000, 32, 7), (2, 1100, 96, 10, 3), (1, 70, 1500, 15, 5),
             (1, 900, 100, 25, 7), (1, 7, 3000, 10, 3), (1, 40, 9000, 25, 7), (1, 1700, 64, 25, 7),
             (1, 64, 2000, 15, 5), (1, 1600, 96, 15, 5), (1, 33, 16384, 25, 7), (1, 96, 300, 12, 0),
             (2, 50, 1030, 8, 1)]
    xs = [dev(rng.uniform(0, 255, (b, r, c))) for (b, r, c, S, K) in cases]
    runs = []
    for walker in (0, 1, 2):  # default (walk3/walk2), portable only, walk2 (no hot kernel)
        outs = {}
        with pl.debug_route(walker):
            for x, (b, r, c, S, K) in zip(xs, cases):
                p = (S, K, 50.0 + 10 * S)
                outs[f"{r}x{c}_rc"] = host(pl.snlm_2d_row_col(x, p))
                outs[f"{r}x{c}_cr"] = host(pl.snlm_2d_col_row(x, p))
        runs.append(outs)
    for key in runs[0]:
        assert np.array_equal(runs[0][key], runs[1][key]), key
        assert np.array_equal(runs[0][key], runs[2][key]), key


def test_slab_transpose_emulated_bitwise():
    """c5's row-slab -> all-to-all -> column-slab path, with G ranks emulated on
    one GPU (the exchange is a host-side regrouping of the send blocks): the
    stitched column slabs equal the single-device RC bit for bit."""
    from paper_1407_2343_b200.distributed import SlabPlan
    G, H, W = 4, 256, 512
    S, K, h = 10, 3, 74.8
    img = workloads.make_image(H, W, 20, 25.0, seed=4)
    want = host(pl.snlm_2d_row_col(dev(img), (S, K, h)))
    sends = []
    for g in range(G):
        plan = SlabPlan(H, W, G, g)
        r0, r1 = plan.rows
        sends.append(host(pl.nlm_row_pass_blocked(dev(img[r0:r1]), (S, K, h), W // G))
                     .reshape(G, H // G, W // G))
    for g in range(G):
        colslab = np.concatenate([sends[src][g] for src in range(G)], axis=0)  # recv layout
        got = host(pl.nlm_col_pass(dev(colslab), (S, K, h)))
        assert np.array_equal(got, want[:, g * (W // G):(g + 1) * (W // G)]), g


@pytest.mark.parametrize("S,K", [(10, 3), (15, 5), (25, 7), (4, 1), (12, 2), (6, 9)])
def test_col_pass_window_bitwise(S, K):
    """Windowed column pass (halo form): for first, middle, last and full
    segment ranges, the window's output rows equal the whole-image column pass
    bit for bit, with the window embedded in NaN guard rows (a read outside
    pl_col_window's range would poison the output) and the output in a -7
    guard (a stray write would show)."""
    rng = np.random.default_rng(S * 10 + K)
    b, H, W = 2, 2048, 96
    x = rng.uniform(0, 255, (b, H, W)).astype(np.float32)
    p = (S, K, 55.0)
    want = host(pl.nlm_col_pass(dev(x), p))
    nseg = pl.col_segments(H, p)
    assert nseg >= 4
    for a, e in [(0, 1), (1, 3), (nseg - 1, nseg), (0, nseg), (2, nseg - 1)]:
        in_lo, in_hi, out_lo, out_hi = pl.col_window(H, a, e, p)
        assert in_lo <= out_lo < out_hi <= in_hi
        G = 64
        rows = in_hi - in_lo
        win = dev(x[:, in_lo:in_hi])
        outbuf = torch.full((b * (out_hi - out_lo) * W + 2 * 4096,), -7.0, device="cuda")
        out = outbuf[4096:4096 + b * (out_hi - out_lo) * W].view(b, out_hi - out_lo, W)
        got = host(pl.nlm_col_pass_window(win, in_lo, H, a, e, p, out=out))
        assert np.array_equal(got, want[:, out_lo:out_hi]), (a, e)
        assert (host(outbuf[:4096]) == -7).all() and (host(outbuf[-4096:]) == -7).all()
        # one image with NaN rows right outside its window (batch 1)
        one = torch.full((rows + 2 * G, W), float("nan"), device="cuda")
        one[G:G + rows] = dev(x[0, in_lo:in_hi])
        got1 = host(pl.nlm_col_pass_window(one[G:G + rows], in_lo, H, a, e, p))
        assert np.array_equal(got1, want[0, out_lo:out_hi]), (a, e)
    with pytest.raises(IndexError):  # window too small
        in_lo, in_hi, _, _ = pl.col_window(H, 1, 2, p)
        pl.nlm_col_pass_window(dev(x[0, in_lo + 1:in_hi]), in_lo + 1, H, 1, 2, p)


@pytest.mark.parametrize("G,S,K", [(4, 10, 3), (8, 25, 7), (3, 15, 5)])
def test_halo_exchange_emulated_bitwise(G, S, K):
    """c5's halo-exchange path with G ranks emulated on one GPU (row pass of
    each rank's rows into its window buffer, the plan's transfers as device
    copies between the ranks' buffers, windowed column pass): the stitched
    row slabs equal the single-device RC bit for bit."""
    from paper_1407_2343_b200.distributed import HaloPlan
    H, W = 8192, 128
    h = 60.0
    img = workloads.make_image(H, W, 40, 25.0, seed=6)
    want = host(pl.snlm_2d_row_col(dev(img), (S, K, h)))
    plans = [HaloPlan(H, W, G, r, (S, K, h)) for r in range(G)]
    ys = []
    for r, plan in enumerate(plans):
        (olo, ohi), (wlo, whi) = plan.rows, plan.window_rows
        y = torch.full((whi - wlo, W), float("nan"), device="cuda")
        pl.nlm_row_pass(dev(img[olo:ohi]), (S, K, h), out=y[olo - wlo:ohi - wlo])
        ys.append(y)
    for s, d, lo, hi in plans[0].transfers():
        ys[d][lo - plans[d].window_rows[0]:hi - plans[d].window_rows[0]] = \
            ys[s][lo - plans[s].window_rows[0]:hi - plans[s].window_rows[0]]
    got = np.concatenate([host(pl.nlm_col_pass_window(ys[r], plans[r].window_rows[0], H,
                                                      *plans[r].segments, (S, K, h)))
                          for r in range(G)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("rows,cols,S,K", [(300, 517, 10, 3), (200, 300, 25, 7), (160, 256, 15, 5),
                                           (130, 200, 5, 2), (64, 90, 0, 2), (40, 300, 10, 9)])
def test_row_pass_fanout_bitwise(rows, cols, S, K):
    """pl_nlm_row_pass_fanout: dst is bit-identical to the plain row pass and
    every fanned-out row to the corresponding dst row (hot kernel's row flush,
    portable walker, direct route + copies); nothing outside the targets is
    written."""
    img = np.random.default_rng(rows + S).uniform(0, 255, (rows, cols)).astype(np.float32)
    p = (S, K, 60.0)
    x = dev(img)
    want = host(pl.nlm_row_pass(x, p))
    ranges = [(0, min(rows, 37)), (max(0, rows - 50), rows)]
    bufs = [torch.full((hi - lo + 3, cols), float("nan"), device="cuda") for lo, hi in ranges]
    out = pl.nlm_row_pass_fanout(x, p, extras=[(b, lo, hi) for b, (lo, hi) in zip(bufs, ranges)])
    assert np.array_equal(host(out), want)
    for b, (lo, hi) in zip(bufs, ranges):
        got = host(b)
        assert np.array_equal(got[:hi - lo], want[lo:hi])
        assert np.isnan(got[hi - lo:]).all()
    assert np.array_equal(host(pl.nlm_row_pass_fanout(x, p)), want)  # no targets
    with pytest.raises(RuntimeError):  # PL_ERR_ARG: more than PL_MAX_FANOUT targets
        pl.nlm_row_pass_fanout(x, p, extras=[(bufs[0], 0, 1)] * 3)
    with pytest.raises(RuntimeError):  # PL_ERR_ARG: rows outside the image
        pl.nlm_row_pass_fanout(x, p, extras=[(bufs[0], 5, rows + 1)])


@pytest.mark.parametrize("G,S,K", [(4, 10, 3), (8, 25, 7), (3, 15, 5), (2, 25, 7)])
def test_fused_halo_emulated_bitwise(G, S, K):
    """The fused halo path with G ranks emulated on one GPU: each rank's row
    pass (pl_nlm_row_pass_fanout) stores its halo rows straight into the other
    ranks' window buffers (NaN-filled: any row not delivered shows), then the
    windowed column passes; the stitched rows equal the single-device RC bit
    for bit.  No rank waits on another inside a kernel: phase 1 runs for every
    rank, then phase 2."""
    from paper_1407_2343_b200.distributed import HaloPlan, halo_cols_fused, halo_rows_fused
    H, W = 8192, 96
    p = (S, K, 60.0)
    img = workloads.make_image(H, W, 40, 25.0, seed=9)
    want = host(pl.snlm_2d_row_col(dev(img), p))
    plans = [HaloPlan(H, W, G, r, p) for r in range(G)]
    cap = plans[0].window_capacity
    wins = [torch.full((cap, W), float("nan"), device="cuda") for _ in range(G)]
    for r, plan in enumerate(plans):
        olo, ohi = plan.rows
        halo_rows_fused(dev(img[olo:ohi]), p, plan, lambda q: wins[q])
    got = np.concatenate([host(halo_cols_fused(p, plans[r], lambda q: wins[q])) for r in range(G)])
    assert np.array_equal(got, want)


def test_symmetric_windows_fused_rc(tmp_path):
    """The fused halo path end to end through torch symmetric memory
    (rendezvous, peer-buffer views, device barrier) under torchrun with one
    rank -- the setup bench.py --c5-dist fused runs at N > 1."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "symm.py"
    script.write_text(
        "import sys, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {root!r})\n"
        "torch.cuda.set_device(0)\n"
        "dist.init_process_group('nccl', device_id=torch.device('cuda', 0))\n"
        "import paper_1407_2343_b200 as pl\n"
        "from paper_1407_2343_b200 import workloads\n"
        "from paper_1407_2343_b200.distributed import HaloPlan, symmetric_windows, halo_rc_fused\n"
        "p = (25, 7, 136.9)\n"
        "plan = HaloPlan(4096, 256, 1, 0, p)\n"
        "windows, barrier = symmetric_windows(plan, torch.device('cuda', 0))\n"
        "img = torch.from_numpy(workloads.make_image(4096, 256, 20, 25.0, seed=3)).cuda()\n"
        "got = halo_rc_fused(img, p, plan, windows, barrier)\n"
        "assert torch.equal(got, pl.snlm_2d_row_col(img, p))\n"
        "print('SYMM_OK')\n"
        "dist.destroy_process_group()\n")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29561", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "SYMM_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_image_metrics_vs_oracle(dtype):
    """Device MSE / PSNR / SSIM (metrics.cpp:98-158) against the oracle on the
    same inputs: per-pixel quantities are evaluated in the reference's order,
    only the final sums differ in association (rel 1e-12)."""
    from oracle import Oracle
    orc = Oracle.get()
    rng = np.random.default_rng(61)
    for (b, r, c) in [(1, 11, 11), (2, 16, 20), (3, 37, 45), (1, 300, 257), (2, 5, 7)]:
        a = rng.uniform(0, 255, (b, r, c))
        y = np.clip(a + rng.normal(0, 15, (b, r, c)), 0, 255)
        if dtype == torch.float32:
            a, y = a.astype(np.float32).astype(np.float64), y.astype(np.float32).astype(np.float64)
        got = host(pl.image_metrics(dev(a, dtype), dev(y, dtype)))
        for k in range(b):
            if r < 11 or c < 11:
                want_mse = float(np.mean((a[k] - y[k]) ** 2))
                assert abs(got[k, 0] - want_mse) <= 1e-12 * want_mse and np.isnan(got[k, 2])
                continue
            want = orc.metrics(a[k], y[k])
            assert np.allclose(got[k], want, rtol=1e-12, atol=0), (b, r, c, got[k], want)
    x = dev(rng.uniform(0, 255, (2, 30, 40)), dtype)
    m = host(pl.image_metrics(x, x))
    assert (m[:, 0] == 0).all() and np.isinf(m[:, 1]).all() and (m[:, 2] == 1.0).all()


@pytest.mark.parametrize("shape,p", [((3, 300, 256), (10, 3, 60.0)), ((1, 200, 130), (15, 5, 90.0)),
                                     ((1, 96, 64), (25, 7, 99.0)), ((2, 70, 90), (4, 2, 50.0)),
                                     ((1, 33, 20), (6, 9, 52.0)), ((1, 40, 7), (40, 1, 52.0))])
def test_transposed_intermediate_bitwise(shape, p):
    """pl_snlm_2d_row_col runs the row pass into a transposed intermediate
    (walk3 io=2: row staging + column flush on both passes); it must equal the
    plain row pass -> column pass pair bit for bit, and the strided entry point
    must reproduce both passes."""
    b, r, c = shape
    x = dev(np.random.default_rng(r + c).uniform(0, 255, shape).astype(np.float32))
    row = pl.nlm_row_pass(x, p)
    want = host(pl.nlm_col_pass(row, p))
    assert np.array_equal(host(pl.snlm_2d_row_col(x, p)), want)
    mid = torch.empty_like(x)
    pl.nlm_pass_strided(x, mid, b, r, c, c, 1, 1, r, r * c, p)
    assert np.array_equal(host(mid).reshape(b, c, r).transpose(0, 2, 1), host(row))
    out = torch.empty_like(x)
    pl.nlm_pass_strided(mid, out, b, c, r, r, 1, 1, c, r * c, p)
    assert np.array_equal(host(out), want)
    # plain layouts through the strided entry = the row / column pass APIs
    pl.nlm_pass_strided(x, out, b, r, c, c, 1, c, 1, r * c, p)
    assert np.array_equal(host(out), host(row))


def test_guard_bands_no_stray_access():
    """Stand-in for compute-sanitizer (closed on this pool): every kernel path runs on
    inputs/outputs embedded in NaN guard bands.  A stray read poisons an output with
    NaN; a stray write changes the output guard."""
    rng = np.random.default_rng(77)
    G = 4096
    for (b, r, c) in [(1, 1, 1), (1, 5, 7), (2, 33, 70), (1, 70, 300), (3, 130, 97),
                      (1, 600, 520), (1, 64, 2048),
                      (1, 3, 40000), (2, 5, 9000)]:  # few long rows: the folded 1D pass
        for (S, K) in [(0, 0), (1, 0), (4, 2), (10, 3), (15, 5), (25, 7), (10, 9), (40, 1)]:
            if K > min(r, c):
                continue
            n = b * r * c
            src = torch.full((n + 2 * G,), float("nan"), device="cuda")
            dst = torch.full((n + 2 * G,), -7.0, device="cuda")
            x = src[G:G + n].view(b, r, c)
            x.copy_(torch.from_numpy(rng.uniform(0, 255, (b, r, c)).astype(np.float32)))
            y = dst[G:G + n].view(b, r, c)
            p = (S, K, 60.0)
            for fn in (pl.nlm_row_pass, pl.nlm_col_pass, pl.snlm_2d_row_col, pl.snlm_2d):
                fn(x, p, out=y)
                torch.cuda.synchronize()
                assert torch.isfinite(y).all(), (b, r, c, S, K, fn.__name__)
                assert (dst[:G] == -7.0).all() and (dst[G + n:] == -7.0).all(), (b, r, c, S, K)
            if c % 16 == 0:
                pl.nlm_row_pass_blocked(x, p, 16, out=y)
                torch.cuda.synchronize()
                assert torch.isfinite(y).all()
                assert (dst[:G] == -7.0).all() and (dst[G + n:] == -7.0).all()
            line = x[0, 0]
            out1 = dst[G:G + c]
            pl.nlm_1d_patchlift(line.contiguous(), p, out=out1)
            torch.cuda.synchronize()
            assert torch.isfinite(out1).all() and (dst[:G] == -7.0).all()


def test_f64_route_matches_reference_library(ref):
    """The fp64 route (plgpu_walk64.cuh; the C++ drop-in's default) against the
    UNMODIFIED reference library on the same double inputs: every filter
    within 1e-9 on [0, 255] data (the reference's own filter-equivalence
    tolerance, acceptance_main.cpp:87-122), including edges, S > 32 (direct
    route) and S = 0."""
    rng = np.random.default_rng(64)
    for (r, c, S, K, h) in [(40, 57, 5, 2, 30.0), (33, 70, 10, 3, 74.8), (64, 48, 16, 5, 15.0),
                            (20, 90, 25, 7, 136.9), (12, 100, 40, 1, 50.0), (9, 30, 0, 2, 20.0),
                            (50, 50, 7, 0, 8.0)]:
        img = rng.uniform(0, 255, (r, c))
        x = torch.from_numpy(img).cuda()
        for op in ("row", "col", "rc", "cr", "snlm", "nlm2d"):
            got = pl.filter_f64(op, x, (S, K, h)).cpu().numpy()
            want = ref.filter(op if op != "nlm2d" else "nlm2d", img, S, K, h)
            err = float(np.abs(got - want).max())
            assert err <= 1e-9, (op, r, c, S, K, h, err)
    for (n, S, K, h) in [(300, 10, 3, 60.0), (77, 5, 8, 15.0), (1000, 32, 7, 200.0)]:
        f = rng.uniform(0, 255, (3, n))
        x = torch.from_numpy(f).cuda()
        for op, naive in (("lines", False), ("lines_naive", True)):
            got = pl.filter_f64(op, x, (S, K, h)).cpu().numpy()
            for row in range(3):
                want = ref.nlm_1d(f[row], S, K, h, naive=naive)
                assert float(np.abs(got[row] - want).max()) <= 1e-9, (op, n, S, K)


def test_small_h_f64_route_strict(ref):
    """Small h (5..25 on 8-bit data), where the fp32 running sums lose
    accuracy (test_small_h_fast_policy_bounds): the fp64 route holds the reference
    to 1e-9 -- far inside T2 -- for single passes and composites alike."""
    rng = np.random.default_rng(55)
    for t in range(8):
        r, c = int(rng.integers(20, 120)), int(rng.integers(20, 120))
        S, K = int(rng.integers(2, 26)), int(rng.integers(0, 4))
        h = float(rng.uniform(5.0, 25.0))
        img = rng.uniform(0, 255, (r, c))
        x = torch.from_numpy(img).cuda()
        for op in ("row", "col", "rc", "cr", "snlm"):
            got = pl.filter_f64(op, x, (S, K, h)).cpu().numpy()
            want = ref.filter(op, img, S, K, h)
            assert float(np.abs(got - want).max()) <= 1e-9, (op, r, c, S, K, h)

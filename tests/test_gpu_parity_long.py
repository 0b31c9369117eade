"""Parity of the long-line configurations against the oracle.

c5 (16384^2, K=7, S=25) runs the hot kernel ``nlm_pass3_kernel<25, 7, 1, io, 8>``
in its INTERIOR instantiation (MODE 1: no mirrored staging, no masked body) on
30 of every line's 32 segments.  Lines of at most a few hundred samples are a
single edge segment, so these tests use lines of the real c5 length:

* the RC / row pass / column pass of 512-row stripes of the c5 image itself
  (``workloads.make_image(..., row_range=...)`` builds exactly those rows), and
  of their transposes (16384-sample columns), against the oracle at T2;
* the full 16384^2 RC on the GPU, checked on bands of output rows (top edge,
  interior, bottom edge) whose oracle reference is the row pass of the band's
  rows followed by the column pass over the band (rows more than S+K from a
  band edge depend only on rows inside it);
* c1's distances (one 65,536-sample float signal) against the reference's
  direct O(NSK) sum (``patch_distance_sq_naive``, banded_kernel.cpp:86-108),
  tier T1.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1407_2343_b200 as pl  # noqa: E402
from paper_1407_2343_b200 import workloads  # noqa: E402

T2 = 1e-3
C5 = workloads.CONFIGS["c5"]
C5_SEED = 1 * 1000003  # image 0 of the c5 construction (bench.py / make_config)


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    pl.lib()
    yield


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def c5_rows(r0, r1):
    return workloads.make_image(C5["rows"], C5["cols"], C5["shapes"], C5["sigma"], seed=C5_SEED,
                                row_range=(r0, r1))


def test_c5_segments_reach_interior_mode():
    """The geometry these tests rely on: 16384-sample lines are cut into 32
    segments, 30 of which are interior (no clipping, no mirror)."""
    S, K, _ = workloads.params("c5")
    C = pl.segment_length(16384, S)
    nseg = -(-16384 // C)
    assert nseg == 32, nseg
    interior = [s for s in range(nseg)
                if s * C - S - K - 1 >= 0 and min(16384, (s + 1) * C) - 1 + 2 * S + K <= 16383]
    assert len(interior) >= 30, interior


@pytest.mark.parametrize("stripe", [(0, 512), (8000, 8512)])
def test_c5_long_rows_vs_oracle(orc, stripe):
    """512 x 16384 stripes of the c5 image: the row pass runs 16384-sample
    lines (interior MODE 1 on 30 of 32 segments) -- row pass alone and the RC
    composite (transposed intermediate, io = 2) against the oracle."""
    S, K, h = workloads.params("c5")
    img = c5_rows(*stripe)
    x = dev(img)
    img64 = img.astype(np.float64)
    want_row = orc.row_pass(img64, S, K, h, threads=16)
    got_row = host(pl.nlm_row_pass(x, (S, K, h))).astype(np.float64)
    assert np.abs(got_row - want_row).max() <= T2
    want_rc = orc.col_pass(want_row, S, K, h, threads=16)
    got_rc = host(pl.snlm_2d_row_col(x, (S, K, h))).astype(np.float64)
    err = np.abs(got_rc - want_rc).max()
    assert err <= T2, err


def test_c5_long_columns_vs_oracle(orc):
    """The transposed stripe (16384 x 512): the column pass runs the
    16384-sample lines -- column pass alone (io = 0) and RC (its column pass
    reads the transposed intermediate, io = 2) against the oracle."""
    S, K, h = workloads.params("c5")
    img = np.ascontiguousarray(c5_rows(4096, 4608).T)
    x = dev(img)
    img64 = img.astype(np.float64)
    want_col = orc.col_pass(img64, S, K, h, threads=16)
    got_col = host(pl.nlm_col_pass(x, (S, K, h))).astype(np.float64)
    assert np.abs(got_col - want_col).max() <= T2
    want_rc = orc.snlm_rc(img64, S, K, h, threads=16)
    got_rc = host(pl.snlm_2d_row_col(x, (S, K, h))).astype(np.float64)
    err = np.abs(got_rc - want_rc).max()
    assert err <= T2, err


@pytest.mark.slow
def test_c5_full_image_rc_bands_vs_oracle(orc):
    """The full c5 RC (one 16384^2 image, 1 GPU) against the oracle on bands of
    output rows: top edge, three interior bands, bottom edge."""
    S, K, h = workloads.params("c5")
    H, W = C5["rows"], C5["cols"]
    img = workloads.make_config("c5")[0]
    got = pl.snlm_2d_row_col(dev(img), (S, K, h))
    halo = S + K
    for a, b in [(0, 48), (4000, 4048), (8191, 8239), (12345, 12393), (H - 48, H)]:
        lo, hi = max(0, a - halo), min(H, b + halo)
        rows = orc.row_pass(img[lo:hi].astype(np.float64), S, K, h, threads=16)
        # output row i reads input rows [i-S-K, i+S+K] only: the band keeps
        # S+K rows of margin on each side that is not an image edge, so the
        # oracle's column pass over the band is exact on rows [a, b)
        want = orc.col_pass(rows, S, K, h, threads=16)[a - lo:b - lo]
        g = host(got[a:b]).astype(np.float64)
        err = np.abs(g - want).max()
        assert err <= T2, (a, b, err)


def test_c1_distances_vs_direct_sum(orc):
    """c1: the GPU's distances over the whole 65,536-sample float signal
    against the reference's direct O(NSK) sum (banded_kernel.cpp:86-108 over
    one extend_symmetric), tier T1 (relative to patch energy plus the running
    sum's rounding scale)."""
    S, K, _ = workloads.params("c1")
    f = workloads.make_config("c1").astype(np.float64)
    n = f.size
    got = host(pl.distance_band(dev(f), S, K))[0].astype(np.float64)
    want = orc.distance_band_direct(f, S, K)
    ok = ~np.isnan(want)
    assert np.array_equal(np.isnan(got), ~ok)
    ext = orc.extend_symmetric(f, K)
    energy = np.convolve(ext * ext, np.ones(2 * K + 1), mode="valid")  # F(i, i)
    i = np.arange(n)[:, None]
    j = np.clip(i + np.arange(-S, S + 1)[None, :], 0, n - 1)
    steps = pl.segment_length(n, S) + S
    walk = 4 * math.sqrt(steps) * 2.0 ** -24 * (2 * K + 1) * float(np.abs(f).max()) ** 2
    tol = 1e-5 * (1 + energy[i] + energy[j]) + walk
    err = np.abs(got - want)
    assert np.all(err[ok] <= tol[ok]), float((err[ok] / tol[ok]).max())

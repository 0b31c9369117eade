"""C-ABI behaviour on the device: the hot kernel's own distances (T0), the
kernel routes the composites take, and re-entrancy across streams/threads.

* T0 on the code that runs: ``pl_debug_hot_distance_band`` runs the hot filter
  kernel (``nlm_pass3_kernel``, the instantiation the configs use, interior
  MODE 1 and edge MODE 2 included for S = 25) with the sample prescale set to
  1 and exports every distance its running-sum recurrence produces; on
  integer-valued lines they equal the reference's
  ``kernel_distance_sq(compute_banded_kernel(...))`` bit for bit
  (banded_kernel.cpp:25-84).
* ``pl_snlm_2d``'s final pass (RC with the fused S-NLM average) runs the hot
  kernel's AVG instantiation (not the portable walker).
* Concurrent calls with ``work = NULL`` on two streams / two host threads give
  the serial results bit for bit (per-call stream-ordered scratch).
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1407_2343_b200 as pl  # noqa: E402
from paper_1407_2343_b200 import workloads  # noqa: E402


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


def quantize(x):
    return np.clip(np.sign(x) * np.floor(np.abs(x) + 0.5), 0, 255).astype(np.float32)


def _check_hot_band(orc, lines, S, K, check_rows):
    got = host(pl.debug_hot_distance_band(dev(lines), S, K))
    assert pl.last_route().startswith(f"hot<S={S},K={K},"), pl.last_route()
    for r in check_rows:
        want = orc.distance_band(lines[r].astype(np.float64), S, K)
        off = np.ones(2 * S + 1, bool)
        off[S] = False
        w, g = want[:, off], got[r][:, off].astype(np.float64)
        assert np.array_equal(np.isnan(w), np.isnan(g)), r
        ok = ~np.isnan(w)
        assert np.array_equal(w[ok], g[ok]), (r, float(np.abs(w[ok] - g[ok]).max()))


def test_hot_kernel_distances_bit_exact_c4(orc):
    """c4 (K=3, S=10, 2048-sample integer rows, 2 lines per lane)."""
    S, K, _ = workloads.params("c4")
    img = workloads.make_config("c4", batch=1)[0]
    _check_hot_band(orc, img[:64], S, K, range(0, 64, 3))


def test_hot_kernel_distances_bit_exact_c3(orc):
    """K=5, S=15 on quantised 4096-sample rows of the c3 construction."""
    S, K, _ = workloads.params("c3")
    img = quantize(workloads.make_image(64, 4096, 20, 30.0, seed=5))
    _check_hot_band(orc, img[:40], S, K, range(0, 40, 3))


def test_hot_kernel_distances_bit_exact_c5(orc):
    """K=7, S=25 on quantised 16384-sample rows (interior MODE 1 on 30 of 32
    segments, edge MODE 2 on the rest), plus short lines (one edge segment)."""
    S, K, _ = workloads.params("c5")
    c = workloads.CONFIGS["c5"]
    rows = quantize(workloads.make_image(c["rows"], c["cols"], c["shapes"], c["sigma"],
                                         seed=1000003, row_range=(100, 132)))
    _check_hot_band(orc, rows, S, K, [0, 7, 31])
    rng = np.random.default_rng(3)
    short = rng.integers(0, 256, (33, 300)).astype(np.float32)
    _check_hot_band(orc, short, S, K, [0, 32])


def test_hot_distance_export_rejects_non_hot():
    x = dev(np.zeros((32, 100), np.float32))
    with pytest.raises(RuntimeError):
        pl.debug_hot_distance_band(x, 9, 3)
    with pytest.raises(RuntimeError):
        pl.debug_hot_distance_band(dev(np.zeros((8, 100), np.float32)), 10, 3)


@pytest.mark.parametrize("S,K", [(10, 3), (15, 5), (25, 7)])
def test_composite_routes(S, K):
    """RC's passes and S-NLM's averaged final pass run the hot kernel with the
    transposed intermediate (io = 2); the S-NLM one with the fused average."""
    x = dev(np.random.default_rng(S).uniform(0, 255, (2, 256, 192)))
    p = (S, K, 70.0)
    pl.snlm_2d_row_col(x, p)
    assert pl.last_route().startswith(f"hot<S={S},K={K},") and ",io=2," in pl.last_route(), \
        pl.last_route()
    pl.snlm_2d(x, p)
    r = pl.last_route()
    assert r.startswith(f"hot<S={S},K={K},") and ",io=2," in r and ",avg=1" in r, r
    pl.nlm_row_pass(x, p)
    assert ",io=1," in pl.last_route()
    pl.nlm_col_pass(x, p)
    assert ",io=0," in pl.last_route()


def test_concurrent_streams_bitwise():
    """pl_snlm_2d_row_col / pl_snlm_2d with work = NULL on two streams at once,
    interleaved, equal the serial results bit for bit."""
    rng = np.random.default_rng(17)
    p = (10, 3, 60.0)
    xs = [dev(rng.uniform(0, 255, (3, 384, 512))) for _ in range(2)]
    want_rc = [host(pl.snlm_2d_row_col(x, p)) for x in xs]
    want_s = [host(pl.snlm_2d(x, p)) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    outs = [[], []]
    for it in range(6):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                outs[k].append(pl.snlm_2d_row_col(xs[k], p) if it % 2 == 0 else pl.snlm_2d(xs[k], p))
    torch.cuda.synchronize()
    for k in range(2):
        for it, o in enumerate(outs[k]):
            want = want_rc[k] if it % 2 == 0 else want_s[k]
            assert np.array_equal(o.cpu().numpy(), want), (k, it)


def test_concurrent_threads_bitwise():
    """Two host threads, each with its own stream, calling the composites with
    work = NULL concurrently (growing sizes, so the scratch changes size
    under the other thread's feet): results equal the serial ones."""
    rng = np.random.default_rng(19)
    p = (15, 5, 90.0)
    shapes = [(1, 200, 256), (2, 300, 320), (1, 512, 640), (3, 256, 256)]
    inputs = [[dev(rng.uniform(0, 255, s)) for s in shapes] for _ in range(2)]
    want = [[host(pl.snlm_2d_row_col(x, p)) for x in xs] for xs in inputs]
    got = [[None] * len(shapes) for _ in range(2)]
    errors = []

    def run(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rep in range(3):
                    for i, x in enumerate(inputs[k]):
                        got[k][i] = pl.snlm_2d_row_col(x, p)
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for k in range(2):
        for i in range(len(shapes)):
            assert np.array_equal(host(got[k][i]), want[k][i]), (k, i)


def test_out_argument_checked():
    x = dev(np.zeros((2, 64, 64), np.float32))
    with pytest.raises(ValueError):
        pl.snlm_2d_row_col(x, (10, 3, 50.0), out=torch.empty((2, 64, 63), device="cuda"))
    with pytest.raises(TypeError):
        pl.nlm_row_pass(x, (10, 3, 50.0), out=torch.empty((2, 64, 64), device="cuda",
                                                          dtype=torch.float64))
    with pytest.raises(ValueError):
        pl.snlm_2d(x, (10, 3, 50.0), work=torch.empty(10, device="cuda"))


def test_host_pipeline_reports_errors():
    """pl_snlm_2d_row_col_host validates before touching the device and
    returns the reference's message."""
    with pytest.raises(pl.ValidationError):
        pl.snlm_2d_row_col_host(np.zeros((4, 4), np.float32), (10, 9, 50.0))


def test_rc_graph_replay_bitwise():
    """pl_graph_rc_create / pl_graph_launch: the captured RC replays to the same
    bits as the direct call, and sees new input values written in place."""
    rng = np.random.default_rng(77)
    x = dev(rng.uniform(0, 255, (2, 96, 160)))
    p = (10, 3, 60.0)
    g = pl.RCGraph(x, p)
    torch.cuda.synchronize()
    for t in range(3):
        x.copy_(dev(rng.uniform(0, 255, (2, 96, 160))))
        y = g.launch()
        want = pl.snlm_2d_row_col(x, p)
        torch.cuda.synchronize()
        assert torch.equal(y, want), t


@pytest.mark.slow
def test_bench_multi_rank_logic_gloo(tmp_path):
    """bench.py's N > 1 path (c4 sharded strong + weak, the three c5 forms with
    the bitwise check against the single-GPU RC) with 2 ranks over gloo, both
    on cuda:0: a functional check of the multi-rank logic (timings meaningless,
    the line says so); the fused form needs symmetric memory, which gloo lacks."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--dist-backend", "gloo",
           "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 64 and line["e2e"]["matches_device_result"]
    assert line["weak"]["images_per_rank"] == 64
    forms = line["c5_forms"]
    assert forms["slab"]["bitwise_equal_single_gpu_rc"] is True
    assert forms["halo"]["bitwise_equal_single_gpu_rc"] is True
    assert "unavailable" in forms["fused"]


@pytest.mark.parametrize("lines,n,S,K", [
    (1, 65536, 10, 3),   # config c1's shape
    (3, 40000, 15, 5),
    (2, 70001, 25, 7),   # interior-only / edge-only bodies (S > 16)
    (1, 5000, 10, 3),    # ~480-sample segments: 8 folded + 3 edge segments
    (5, 9000, 15, 5),
    (31, 33000, 10, 3),  # just under one lane per line
])
def test_folded_1d_lines_bitwise(lines, n, S, K):
    """Few long lines (1D signals) run the hot kernel with the interior
    SEGMENTS of a line folded onto the lanes (route "hot-fold<...>",
    plgpu_walk3.cuh Pass3FoldDesc).  Same per-segment arithmetic: bitwise equal
    to the unfolded routes (walker 3 = folding off: one warp per segment from 16
    lines, the portable walker below) and to the portable walker,
    and within T2 of the oracle (nlm_1d_patchlift, nlm.cpp:144-166)."""
    from oracle import Oracle
    rng = np.random.default_rng(lines * 1000 + S)
    x = rng.uniform(0, 255, (lines, n)).astype(np.float32)
    p = (S, K, 60.0)
    xd = dev(x)
    y = host(pl.nlm_1d_patchlift(xd, p))
    assert pl.last_route().startswith(f"hot-fold<S={S},K={K},"), pl.last_route()
    with pl.debug_route(3):
        y_unfolded = host(pl.nlm_1d_patchlift(xd, p))  # hot kernel from 16 lines, else portable
        assert pl.last_route().startswith("hot<" if lines >= 16 else "portable<"), pl.last_route()
    with pl.debug_route(1):
        y_portable = host(pl.nlm_1d_patchlift(xd, p))
    assert np.array_equal(y, y_unfolded)
    assert np.array_equal(y, y_portable)
    want = Oracle.get().nlm_1d(x[lines - 1].astype(np.float64), S, K, 60.0)
    assert np.abs(y[lines - 1].astype(np.float64) - want).max() <= 1e-3


def test_folded_image_rows_with_few_rows():
    """A row pass over images of a few very long rows folds too (each row is
    its own virtual image); many rows do not."""
    rng = np.random.default_rng(77)
    x = rng.uniform(0, 255, (2, 6, 36000)).astype(np.float32)
    p = (10, 3, 70.0)
    y = host(pl.nlm_row_pass(dev(x), p))
    assert pl.last_route().startswith("hot-fold<"), pl.last_route()
    with pl.debug_route(3):
        assert np.array_equal(y, host(pl.nlm_row_pass(dev(x), p)))
    pl.nlm_row_pass(dev(rng.uniform(0, 255, (1, 64, 4000)).astype(np.float32)), p)
    assert pl.last_route().startswith("hot<"), pl.last_route()

"""Multi-process (gloo, world_size 2 and 4) tests of the partitioning host logic.

The CUDA passes are replaced by the oracle's CPU passes (test infrastructure)
so the slab plan, the all-to-all send layout and the exchange itself run on
CPU; the GPU tests pin the kernels' blocked layout separately
(test_gpu_parity.py::test_blocked_row_pass_layout)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_2343_b200.distributed import (HaloPlan, SlabPlan, blocked_layout, halo_rc,
                                              halo_rc_fused, shard, slab_rc)


def test_shard_covers_batch():
    for n in (1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            spans = [shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_slab_plan_bytes():
    p = SlabPlan(16384, 16384, 8, 3)
    assert p.rows == (6144, 8192) and p.cols == (6144, 8192)
    assert p.nvlink_bytes() == 7 * 2048 * 2048 * 4  # 112 MiB, SURVEY.md sec. 8(e)
    with pytest.raises(ValueError):
        SlabPlan(100, 30, 8, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, params, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_1407_2343_b200 import workloads

        orc = Oracle.get()
        img = workloads.make_image(H, W, 12, 20.0, seed=9).astype(np.float64)
        plan = SlabPlan(H, W, world, rank)
        r0, r1 = plan.rows
        S, K, h = params

        def row_pass_blocked(x, p, cb):
            y = orc.row_pass(x.numpy(), S, K, h)
            return torch.from_numpy(blocked_layout(y, cb))

        def col_pass(x, p):
            return torch.from_numpy(orc.col_pass(x.numpy(), S, K, h))

        got = slab_rc(torch.from_numpy(img[r0:r1].copy()), params, plan,
                      row_pass_blocked=row_pass_blocked, col_pass=col_pass)
        want = orc.snlm_rc(img, S, K, h)
        c0, c1 = plan.cols
        out_q.put((rank, bool(np.array_equal(got.numpy(), want[:, c0:c1]))))
        # batch sharding: each rank filters its images, results gathered == full batch
        imgs = np.stack([workloads.make_image(24, 20, 3, 20.0, seed=s) for s in range(5)])
        lo, hi = shard(5, world, rank)
        mine = torch.from_numpy(np.stack([orc.snlm_rc(imgs[b].astype(np.float64), S, K, h)
                                          for b in range(lo, hi)]) if hi > lo else
                                np.zeros((0, 24, 20)))
        sizes = [shard(5, world, r)[1] - shard(5, world, r)[0] for r in range(world)]
        pad = torch.zeros((max(sizes), 24, 20), dtype=torch.float64)
        pad[:hi - lo] = mine
        gathered = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(gathered, pad)
        full = np.concatenate([g.numpy()[:n] for g, n in zip(gathered, sizes)])
        want_b = np.stack([orc.snlm_rc(imgs[b].astype(np.float64), S, K, h) for b in range(5)])
        out_q.put((rank + 100, bool(np.array_equal(full, want_b))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_slab_all_to_all_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    H, W = 48, 64
    params = (10, 3, 74.8)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, params, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(2 * world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(results.values()), results


def test_halo_plan_c5():
    """c5 (16384^2, S=25, K=7) over 8 ranks: whole segments per rank, rows
    tile the image, halos come from the neighbours only."""
    p = (25, 7, 25.0)
    plans = [HaloPlan(16384, 16384, 8, r, p) for r in range(8)]
    assert plans[0].nseg % 8 == 0
    rows = [pl.rows for pl in plans]
    assert rows[0][0] == 0 and rows[-1][1] == 16384
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 600
    for r, pl in enumerate(plans):
        lo, hi = pl.window_rows
        assert lo <= pl.rows[0] and hi >= pl.rows[1]
        srcs = {s for s, d, _, _ in pl.transfers() if d == r}
        assert srcs <= {r - 1, r + 1}
        assert pl.halo_bytes() < 16 * 2**20  # vs 117 MB for the all-to-all
    # the plan is symmetric: every rank derives the same transfer list
    assert all(pl.transfers() == plans[0].transfers() for pl in plans)


def _halo_worker(rank, world, port, H, W, params, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_1407_2343_b200 import col_window, workloads

        orc = Oracle.get()
        S, K, h = params
        img = workloads.make_image(H, W, 12, 20.0, seed=11).astype(np.float64)
        plan = HaloPlan(H, W, world, rank, params)

        def row_pass(x, p, out):
            out.copy_(torch.from_numpy(orc.row_pass(x.numpy(), S, K, h)))

        def naive_cols(full):
            return np.stack([orc.nlm_1d(full[:, c], S, K, h, naive=True)
                             for c in range(full.shape[1])], axis=1)

        def col_pass_window(y, in_lo, H_, a, b, p):
            # Only the window is real; anything read outside it poisons the
            # result with NaN (the direct oracle reads exactly what it uses).
            full = np.full((H_, W), np.nan)
            full[in_lo:in_lo + y.shape[0]] = y.numpy()
            _, _, out_lo, out_hi = col_window(H_, a, b, p)
            return torch.from_numpy(naive_cols(full)[out_lo:out_hi])

        r0, r1 = plan.rows
        got = halo_rc(torch.from_numpy(img[r0:r1].copy()), params, plan, row_pass=row_pass,
                      col_pass_window=col_pass_window,
                      new_buffer=lambda shape: torch.zeros(shape, dtype=torch.float64))
        want = naive_cols(orc.row_pass(img, S, K, h))[r0:r1]
        ok = got.shape == want.shape and bool(np.array_equal(got.numpy(), want))
        out_q.put((rank, ok, len({s for s, d, _, _ in plan.transfers() if d == rank})))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    H, W = 3900, 12  # 9 column-pass segments of ~434 rows
    params = (4, 1, 30.0)
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, H, W, params, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in results), results
    if world >= 4:
        assert max(n for _, _, n in results) >= 2  # some window spans several owners


@pytest.mark.parametrize("H,W,world,p", [(16384, 16384, 2, (25, 7, 25.0)), (16384, 16384, 4, (25, 7, 25.0)),
                                         (16384, 16384, 8, (25, 7, 25.0)), (160, 24, 4, (4, 1, 30.0)),
                                         (4096, 64, 3, (15, 5, 50.0))])
def test_halo_fanout_plan(H, W, world, p):
    """The fused exchange's targets (HaloPlan.fanout) are exactly the plan's
    transfers, land inside the destination's window, and together with the
    destination's own rows cover its whole window; c5 needs <= 2 (the kernel's
    PL_MAX_FANOUT) targets per rank."""
    import paper_1407_2343_b200 as pl
    plans = [HaloPlan(H, W, world, r, p) for r in range(world)]
    for r, plan in enumerate(plans):
        fan = plan.fanout()
        assert [(r, d, lo, hi) for d, lo, hi, _ in fan] == [t for t in plan.transfers() if t[0] == r]
        for d, lo, hi, row in fan:
            wlo, whi = plans[d].window_rows
            assert row == lo - wlo and 0 <= row and row + (hi - lo) <= whi - wlo
            assert whi - wlo <= plan.window_capacity
        if H == 16384:
            assert len(fan) <= pl.PL_MAX_FANOUT
    for d, plan in enumerate(plans):
        wlo, whi = plan.window_rows
        have = np.zeros(whi - wlo, bool)
        olo, ohi = plan.rows
        have[olo - wlo:ohi - wlo] = True
        for s_, other in enumerate(plans):
            for dd, lo, hi, row in other.fanout():
                if dd == d:
                    have[row:row + hi - lo] = True
        assert have.all() or ohi <= olo


def _fused_worker(rank, world, port, H, W, params, wins, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_1407_2343_b200 import col_window, workloads

        orc = Oracle.get()
        S, K, h = params
        img = workloads.make_image(H, W, 12, 20.0, seed=12).astype(np.float64)
        plan = HaloPlan(H, W, world, rank, params)

        def row_pass_fanout(x, p, out, extras):
            # CPU stand-in for pl_nlm_row_pass_fanout: every produced row goes
            # to my window and straight into the peers' (shared-memory) windows
            y = torch.from_numpy(orc.row_pass(x.numpy(), S, K, h))
            out.copy_(y)
            for dst, lo, hi in extras:
                dst.copy_(y[lo:hi])

        def naive_cols(full):
            return np.stack([orc.nlm_1d(full[:, c], S, K, h, naive=True)
                             for c in range(full.shape[1])], axis=1)

        def col_pass_window(y, in_lo, H_, a, b, p):
            full = np.full((H_, W), np.nan)  # reads outside the window poison the result
            full[in_lo:in_lo + y.shape[0]] = y.numpy()
            _, _, out_lo, out_hi = col_window(H_, a, b, p)
            return torch.from_numpy(naive_cols(full)[out_lo:out_hi])

        r0, r1 = plan.rows
        got = halo_rc_fused(torch.from_numpy(img[r0:r1].copy()), params, plan, lambda r: wins[r],
                            dist.barrier, row_pass_fanout=row_pass_fanout,
                            col_pass_window=col_pass_window)
        want = naive_cols(orc.row_pass(img, S, K, h))[r0:r1]
        ok = got.shape == want.shape and bool(np.array_equal(got.numpy(), want))
        out_q.put((rank, ok, len(plan.fanout())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_fused_halo_matches_single_process(world):
    """The fused halo path's host logic (fan-out targets, peer windows, barrier,
    windowed column pass) across gloo processes; peer windows are shared-memory
    tensors standing in for NVLink-mapped symmetric memory."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    H, W = 3900, 12  # 9 column-pass segments of ~434 rows
    params = (4, 1, 30.0)
    wins = [torch.full((H, W), float("nan"), dtype=torch.float64).share_memory_()
            for _ in range(world)]
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, H, W, params, wins, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in results), results
    # segments are >= ~240 rows (or a whole line) and a halo is <= 2S+2K+81 <= 159
    # rows, so every rank's rows reach at most its two neighbours' windows
    assert max(n for _, _, n in results) <= 2

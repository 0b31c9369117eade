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

from paper_1407_2343_b200.distributed import SlabPlan, blocked_layout, shard, slab_rc


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

"""Multi-GPU partitioning of the separable filter.

One process per GPU (``torch.distributed``; NCCL over NVLink on the B200 box,
gloo for the CPU tests).  Two partitionings, both bitwise identical to the
single-GPU result because every line is filtered by the same per-line
arithmetic whatever the partition (segment boundaries depend only on the
line length):

* **Batch sharding** (config c4): contiguous image ranges per rank, no
  communication at all.
* **Slab transpose** (config c5, one large H x W image): rank g holds row slab
  g (H/G rows).  It runs the row pass writing its output directly in the
  all-to-all *send* layout (``pl_nlm_row_pass_blocked``: G column blocks of
  W/G, each [H/G][W/G] row-major), one ``all_to_all_single`` moves block p to
  rank p, and the received blocks stacked by source rank ARE the row-major
  [H][W/G] column slab, which the column pass consumes in place.  Output stays
  as column slabs.

The pass and exchange callables are injectable so the host logic (slab plan,
layouts, exchange) is tested on CPU with gloo and the oracle's passes
(tests/test_distributed.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


def shard(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n_items for rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return n_items * rank // world, n_items * (rank + 1) // world


@dataclass
class SlabPlan:
    """Row-slab -> column-slab plan for one H x W image over G ranks."""

    H: int
    W: int
    world: int
    rank: int

    def __post_init__(self):
        if self.H % self.world or self.W % self.world:
            raise ValueError("H and W must be divisible by the number of ranks")

    @property
    def rows(self) -> tuple[int, int]:  # my row slab [r0, r1)
        h = self.H // self.world
        return self.rank * h, (self.rank + 1) * h

    @property
    def cols(self) -> tuple[int, int]:  # my column slab [c0, c1)
        w = self.W // self.world
        return self.rank * w, (self.rank + 1) * w

    @property
    def block_elems(self) -> int:  # elements sent to each peer
        return (self.H // self.world) * (self.W // self.world)

    def nvlink_bytes(self, itemsize: int = 4) -> int:
        """Bytes this rank sends over NVLink (to the G-1 other ranks)."""
        return (self.world - 1) * self.block_elems * itemsize


def slab_rc(x_rowslab, params, plan: SlabPlan, *, row_pass_blocked: Callable | None = None,
            col_pass: Callable | None = None, all_to_all: Callable | None = None,
            new_buffer: Callable | None = None):
    """Row pass on my row slab -> all-to-all -> column pass on my column slab.

    x_rowslab: [H/G, W] of this rank.  Returns my [H, W/G] column slab of
    snlm_2d_row_col(image).  Defaults use the CUDA library and the default
    process group (NCCL)."""
    import torch
    if row_pass_blocked is None:
        import paper_1407_2343_b200 as pl
        row_pass_blocked = lambda x, p, cb: pl.nlm_row_pass_blocked(x, p, cb)  # noqa: E731
        col_pass = col_pass or (lambda x, p: pl.nlm_col_pass(x, p))
    if all_to_all is None:
        import torch.distributed as dist
        all_to_all = dist.all_to_all_single
    new_buffer = new_buffer or torch.empty_like
    cb = plan.W // plan.world
    send = row_pass_blocked(x_rowslab, params, cb)  # [G blocks][H/G][W/G], flat
    recv = new_buffer(send)
    all_to_all(recv.reshape(-1), send.reshape(-1))
    colslab = recv.reshape(plan.H, cb)  # blocks stacked by source rank = rows
    return col_pass(colslab, params)


def blocked_layout(x, col_block: int):
    """Reference (host) version of pl_nlm_row_pass_blocked's output layout:
    element (r, c) -> block c // cb, [r][c % cb] within the block."""
    rows, cols = x.shape[-2], x.shape[-1]
    return x.reshape(rows, cols // col_block, col_block).transpose(1, 0, 2).copy()

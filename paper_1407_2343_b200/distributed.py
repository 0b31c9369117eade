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

* **Halo exchange** (config c5, the alternative of SURVEY.md sec. 8(f)):
  ranks own contiguous runs of whole column-pass segments, i.e. contiguous
  row ranges.  Rank g runs the row pass on its own rows straight into a
  window buffer covering the rows its column segments read
  (``pl_col_window``), receives the missing rows (a few dozen above and a
  few hundred below, from the neighbours that own them) by point-to-point
  sends, and runs the windowed column pass (``pl_nlm_col_pass_window``).
  Output stays as row slabs; NVLink traffic per rank is the halo only
  (~13 MB for c5 on 8 GPUs, against 117 MB for the all-to-all).

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


@dataclass
class HaloPlan:
    """Row-partitioned plan for one H x W image over G ranks: rank q owns the
    column-pass segments [seg[q], seg[q+1]) (whole segments, so the column
    pass is bitwise the single-GPU one) and the rows they produce.

    ``window(H, seg_begin, seg_end, params) -> (in_lo, in_hi, out_lo, out_hi)``
    defaults to the library's ``pl_col_window``."""

    H: int
    W: int
    world: int
    rank: int
    params: tuple
    window: Callable | None = None

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError("bad world/rank")
        import paper_1407_2343_b200 as pl
        win = self.window or pl.col_window
        self.nseg = pl.col_segments(self.H, self.params)
        self.seg = [self.nseg * q // self.world for q in range(self.world + 1)]
        self.own, self.need = [], []
        for q in range(self.world):
            a, b = self.seg[q], self.seg[q + 1]
            if b > a:
                in_lo, in_hi, out_lo, out_hi = win(self.H, a, b, self.params)
            else:  # more ranks than segments: nothing to do
                in_lo = in_hi = out_lo = out_hi = 0
            self.own.append((out_lo, out_hi))
            self.need.append((in_lo, in_hi))

    @property
    def segments(self) -> tuple[int, int]:
        return self.seg[self.rank], self.seg[self.rank + 1]

    @property
    def rows(self) -> tuple[int, int]:  # rows this rank owns (input and output)
        return self.own[self.rank]

    @property
    def window_rows(self) -> tuple[int, int]:  # rows of the column-pass input window
        return self.need[self.rank]

    def transfers(self) -> list[tuple[int, int, int, int]]:
        """Every (src_rank, dst_rank, lo, hi): rows [lo, hi) of src's row-pass
        output that dst's window needs."""
        out = []
        for d in range(self.world):
            nlo, nhi = self.need[d]
            for s in range(self.world):
                olo, ohi = self.own[s]
                lo, hi = max(nlo, olo), min(nhi, ohi)
                if s != d and hi > lo:
                    out.append((s, d, lo, hi))
        return out

    def fanout(self) -> list[tuple[int, int, int, int]]:
        """Targets of the FUSED exchange (pl_nlm_row_pass_fanout): every
        (dst_rank, lo, hi, dst_row) -- my row-pass output rows [lo, hi) are
        stored straight into dst_rank's window, starting at its row dst_row."""
        return [(d, lo, hi, lo - self.need[d][0]) for s, d, lo, hi in self.transfers()
                if s == self.rank]

    @property
    def window_capacity(self) -> int:
        """Rows of the largest window (symmetric buffers are equal-sized)."""
        return max([hi - lo for lo, hi in self.need] + [1])

    def halo_bytes(self, itemsize: int = 4) -> int:
        """Bytes this rank receives over NVLink."""
        return sum((hi - lo) * self.W * itemsize for s, d, lo, hi in self.transfers()
                   if d == self.rank)


def halo_rc(x_rows, params, plan: HaloPlan, *, row_pass: Callable | None = None,
            col_pass_window: Callable | None = None, exchange: Callable | None = None,
            new_buffer: Callable | None = None):
    """Row pass on my rows -> halo exchange -> windowed column pass.

    x_rows: [out_hi - out_lo, W], my rows ``plan.rows`` of the image.  Returns
    the same rows of snlm_2d_row_col(image).  ``exchange(ops)`` gets a list of
    ("send"|"recv", peer, tensor) and must complete them all (default:
    ``torch.distributed.batch_isend_irecv``)."""
    import torch
    if row_pass is None:
        import paper_1407_2343_b200 as pl
        row_pass = lambda x, p, out: pl.nlm_row_pass(x, p, out=out)  # noqa: E731
        col_pass_window = col_pass_window or (
            lambda y, in_lo, H, a, b, p: pl.nlm_col_pass_window(y, in_lo, H, a, b, p))
    if exchange is None:
        exchange = _p2p_exchange
    olo, ohi = plan.rows
    wlo, whi = plan.window_rows
    if ohi <= olo:
        return x_rows[:0]
    if new_buffer is None:
        new_buffer = lambda shape: torch.empty(shape, dtype=x_rows.dtype,  # noqa: E731
                                               device=x_rows.device)
    y = new_buffer((whi - wlo, plan.W))
    row_pass(x_rows, params, y[olo - wlo:ohi - wlo])
    ops = []
    for s, d, lo, hi in plan.transfers():
        if s == plan.rank:
            ops.append(("send", d, y[lo - wlo:hi - wlo]))
        elif d == plan.rank:
            ops.append(("recv", s, y[lo - wlo:hi - wlo]))
    if ops:
        exchange(ops)
    a, b = plan.segments
    return col_pass_window(y, wlo, plan.H, a, b, params)


def halo_rows_fused(x_rows, params, plan: HaloPlan, windows: Callable, *,
                    row_pass_fanout: Callable | None = None):
    """Phase 1 of the fused halo path: the row pass on my rows writes its output
    into my window AND, in the same kernel, the rows my neighbours need into
    their windows (peer memory over NVLink; pl_nlm_row_pass_fanout).

    ``windows(rank)`` -> that rank's window buffer [>= window rows, W] as seen
    from this process (torch symmetric memory ``get_buffer``, or plain device
    tensors when G ranks are emulated on one GPU).  Targets beyond the kernel's
    PL_MAX_FANOUT are copied after the pass."""
    import paper_1407_2343_b200 as pl
    if row_pass_fanout is None:
        row_pass_fanout = pl.nlm_row_pass_fanout
    olo, ohi = plan.rows
    wlo, _ = plan.window_rows
    if ohi <= olo:
        return
    y = windows(plan.rank)
    targets = plan.fanout()
    fused = [(windows(d)[row:row + (hi - lo)], lo - olo, hi - olo)
             for d, lo, hi, row in targets[:pl.PL_MAX_FANOUT]]
    mine = y[olo - wlo:ohi - wlo]
    row_pass_fanout(x_rows, params, out=mine, extras=fused)
    for d, lo, hi, row in targets[pl.PL_MAX_FANOUT:]:
        windows(d)[row:row + (hi - lo)].copy_(mine[lo - olo:hi - olo])


def halo_cols_fused(params, plan: HaloPlan, windows: Callable, *,
                    col_pass_window: Callable | None = None):
    """Phase 2: the windowed column pass on my (now complete) window."""
    if col_pass_window is None:
        import paper_1407_2343_b200 as pl
        col_pass_window = pl.nlm_col_pass_window
    wlo, whi = plan.window_rows
    a, b = plan.segments
    if plan.rows[1] <= plan.rows[0]:
        return None
    return col_pass_window(windows(plan.rank)[:whi - wlo], wlo, plan.H, a, b, params)


def halo_rc_fused(x_rows, params, plan: HaloPlan, windows: Callable, barrier: Callable, *,
                  row_pass_fanout: Callable | None = None, col_pass_window: Callable | None = None):
    """barrier -> row pass with fused halo stores -> barrier -> windowed column
    pass.  ``barrier()`` (e.g. the symmetric-memory handle's device barrier on
    the current stream) orders every rank's row pass and its peer stores
    before any column pass, and -- the first one -- every peer's previous
    column pass (still reading its window) before this call's stores into it."""
    barrier()
    halo_rows_fused(x_rows, params, plan, windows, row_pass_fanout=row_pass_fanout)
    barrier()
    return halo_cols_fused(params, plan, windows, col_pass_window=col_pass_window)


def symmetric_windows(plan: HaloPlan, device, group=None):
    """Equal-sized window buffers in torch symmetric memory (one per rank,
    peer-mapped over NVLink).  Returns (windows, barrier) for halo_rc_fused."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    shape = (plan.window_capacity, plan.W)
    buf = symm.empty(*shape, dtype=torch.float32, device=device)
    hdl = symm.rendezvous(buf, group or dist.group.WORLD)
    views = {}

    def windows(r):  # every rank's buffer through the handle (own one included)
        if r not in views:
            views[r] = hdl.get_buffer(r, shape, torch.float32)
        return views[r]

    windows.keepalive = buf

    return windows, (lambda: hdl.barrier(channel=0))


def _p2p_exchange(ops):
    import torch.distributed as dist
    p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer)
           for kind, peer, t in ops]
    for req in dist.batch_isend_irecv(p2p):
        req.wait()

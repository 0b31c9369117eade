"""Per-rank kernel time of the c5 slab form at G ranks, measured on ONE GPU
(no collective): the row pass on an [H/G, W] row slab into the all-to-all
send layout, then the column pass on an [H, W/G] column slab; against the
1-GPU RC's passes per pixel.  python tools/time_slab.py [G ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_2343_b200 as pl  # noqa: E402
from paper_1407_2343_b200 import workloads as W  # noqa: E402

S, K, h = W.params("c5")
H = Wd = 16384
rng = np.random.default_rng(2)


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for G in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
    xs = torch.from_numpy(rng.uniform(0, 255, (H // G, Wd)).astype(np.float32)).cuda()
    mid = torch.empty_like(xs)
    cs = torch.from_numpy(rng.uniform(0, 255, (H, Wd // G)).astype(np.float32)).cuda()
    y = torch.empty_like(cs)
    t_row = timeit(lambda: pl.nlm_row_pass_blocked(xs, (S, K, h), Wd // G, out=mid))
    r_row = pl.last_route()
    t_col = timeit(lambda: pl.nlm_col_pass(cs, (S, K, h), out=y))
    r_col = pl.last_route()
    px = H * Wd // G
    print(f"G={G}: row pass {t_row:.3f} ms ({r_row}), column pass {t_col:.3f} ms ({r_col}); "
          f"{px / ((t_row + t_col) * 1e-3) / 1e6:.0f} Mpx/s per rank of kernel time")

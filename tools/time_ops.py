"""Time the composite entry points on device-resident inputs (CUDA events)."""
import sys

import torch

import paper_1407_2343_b200 as pl

b, n = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 2048
x = torch.rand(b, n, n, device="cuda") * 255
p = (10, 3, 74.83)
for f in (pl.nlm_row_pass, pl.nlm_col_pass, pl.snlm_2d_row_col, pl.snlm_2d_col_row, pl.snlm_2d):
    y = f(x, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f(x, p, out=y)
    e1.record()
    torch.cuda.synchronize()
    print(f"{f.__name__:18s} {e0.elapsed_time(e1) / 5:.3f} ms")

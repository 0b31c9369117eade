"""A/B timing of one config's RC passes for a given kernel route (test/tuning
tool): python tools/time_route.py c4 [lines] [wpc] [images].  Uses
pl_debug_set_route (code selection only; results are bitwise identical) and
prints the mean per-pass CUDA-event time and Mpx/s."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_2343_b200 as pl  # noqa: E402
from paper_1407_2343_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
lines = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wpc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = W.CONFIGS[cfg]
S, K, h = W.params(cfg)
nimg = int(sys.argv[4]) if len(sys.argv) > 4 else c.get("batch", 1)
rng = np.random.default_rng(3)
x = torch.from_numpy(rng.uniform(0, 255, (nimg, c["rows"], c["cols"])).astype(np.float32)).cuda()
mid, y = torch.empty_like(x), torch.empty_like(x)
R_, C_ = c["rows"], c["cols"]
with pl.debug_route(0, lines, wpc):
    def step():
        pl.nlm_pass_strided(x, mid, nimg, R_, C_, C_, 1, 1, R_, R_ * C_, (S, K, h))
        pl.nlm_pass_strided(mid, y, nimg, C_, R_, R_, 1, 1, C_, R_ * C_, (S, K, h))
    for _ in range(3):
        step()
    route = pl.last_route()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{cfg} lines={lines} wpc={wpc} route={route}: {ms / 2:.4f} ms/pass, "
      f"{nimg * R_ * C_ / (ms * 1e-3) / 1e6:.0f} Mpx/s")

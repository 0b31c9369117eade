"""Small cases exercising every kernel path, for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_2343_b200 as pl  # noqa: E402

rng = np.random.default_rng(0)
for (b, r, c) in [(1, 1, 1), (1, 5, 7), (2, 33, 70), (1, 70, 300), (3, 130, 97), (1, 600, 520)]:
    for (S, K) in [(0, 0), (1, 0), (4, 2), (10, 3), (15, 5), (25, 7), (10, 9), (40, 1)]:
        if K > min(r, c):
            continue
        x = torch.from_numpy(rng.uniform(0, 255, (b, r, c)).astype(np.float32)).cuda()
        p = (S, K, 60.0)
        for fn in (pl.nlm_row_pass, pl.nlm_col_pass, pl.snlm_2d_row_col, pl.snlm_2d):
            fn(x, p)
        if c % 4 == 0 and c >= 16:
            pl.nlm_row_pass_blocked(x, p, 4)
        pl.distance_band(x[0], S, K, dtype=torch.int32)
        pl.nlm_1d_patchlift(x[0], p)
torch.cuda.synchronize()
print("sanitize cases done")

"""Debug helper: compare the portable (1) and v2 (2) walkers on lines, for
library variants given on the command line (PLGPU_LIB)."""
import os, sys, subprocess, numpy as np
code = r'''
import sys, numpy as np, torch
import paper_1407_2343_b200 as pl
rng = np.random.default_rng(5)
outs = {}
for (L, n, S, K, h) in [(64, 517, 10, 3, 150.0), (64, 517, 10, 0, 150.0), (64, 517, 4, 2, 150.0)]:
    x = torch.from_numpy(rng.uniform(0, 255, (L, n)).astype(np.float32)).cuda()
    outs[f"{L}_{n}_{S}_{K}_{h}"] = pl.nlm_1d_patchlift(x, (S, K, h)).cpu().numpy()
np.savez(sys.argv[1], **outs)
'''
for var in sys.argv[1:]:
    res = []
    for f in "12":
        out = f"/tmp/o{f}.npz"
        env = dict(os.environ, PLGPU_FORCE_WALKER=f)
        if var != "base":
            env["PLGPU_LIB"] = f"paper_1407_2343_b200/lib/var_{var}/libplgpu.so"
        subprocess.run([sys.executable, "-c", code, out], env=env, check=True)
        res.append(np.load(out))
    for k in res[0].files:
        b, c = res[0][k], res[1][k]
        lines = np.nonzero((b != c).any(axis=1))[0]
        print(var, k, "1v2", int((b != c).sum()), "max", float(np.abs(b - c).max()), "lines", lines[:20])
        if len(lines):
            l = lines[0]
            bad = np.nonzero(b[l] != c[l])[0]
            print("   line", l, "pos", bad[:30], b[l, bad[:4]], c[l, bad[:4]])

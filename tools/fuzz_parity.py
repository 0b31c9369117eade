"""Randomised parity sweep on the GPU (test infrastructure: uses oracle/).

Each case draws a shape (batch, rows, cols), (S, K, h), data kind (uniform,
integer-valued, the configs' synthetic image, near-constant) and checks every
single pass and composite against the oracle at the strict T2 = 1e-3 (on the
[0, 255] scale, scaled with the data range) under the default precision
policy (--policy auto: h below 48/255 of the data range runs in double on the
device), or, with --policy fast (fp32 kernels only), at T2 * max(1, (25/h)^2)
for single passes and T2 * max(1, (36/h)^2) for composites (the fp32 running
sums' and the second pass's conditioning); and the
bitwise invariants
(transpose equivariance, batch invariance, snlm = (RC + CR) / 2).  Hot (K, S)
pairs are drawn often so the specialised kernel's edge / masked / partial-
group paths get covered.

    python tools/fuzz_parity.py --seconds 300 [--seed 1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1407_2343_b200 as pl
    from paper_1407_2343_b200 import workloads
    from oracle import Oracle

    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--long-frac", type=float, default=0.15,
                    help="fraction of cases with one 1,500-20,000-sample axis")
    ap.add_argument("--policy", choices=("auto", "fast"), default="auto")
    a = ap.parse_args()
    pl.lib().pl_set_precision_policy(1 if a.policy == "fast" else 0)
    rng = np.random.default_rng(a.seed)
    orc = Oracle.get()
    hot = [(10, 3), (15, 5), (25, 7)]
    t0, n, worst, fails, nf64 = time.time(), 0, 0.0, [], 0
    while time.time() - t0 < a.seconds:
        if rng.uniform() < 0.6:
            S, K = hot[rng.integers(0, 3)]
        else:
            S, K = int(rng.integers(0, 33)), int(rng.integers(0, 9))
        b = int(rng.integers(1, 4))
        r, c = int(rng.integers(1, 420)), int(rng.integers(1, 420))
        if rng.uniform() < a.long_frac:  # long lines: interior segments of the hot kernel
            b = 1
            long_n, short_n = int(rng.integers(1500, 20000)), int(rng.integers(1, 100))
            r, c = (long_n, short_n) if rng.uniform() < 0.5 else (short_n, long_n)
        if K > min(r, c):
            continue
        kind = rng.integers(0, 4)
        if kind == 0:
            x = rng.uniform(0, 255, (b, r, c))
        elif kind == 1:
            x = rng.integers(0, 256, (b, r, c)).astype(np.float64)
        elif kind == 2:
            x = np.stack([workloads.make_image(r, c, 8, 20.0, seed=int(rng.integers(1 << 30)))
                          for _ in range(b)]).astype(np.float64)
        else:
            x = 100.0 + rng.uniform(0, 1e-3, (b, r, c))
        h = float(np.exp(rng.uniform(np.log(5.0), np.log(2000.0))))
        p = (S, K, h)
        x32 = x.astype(np.float32)
        xd = torch.from_numpy(x32).cuda()
        scale = max(1.0, float(np.abs(x32).max()) / 255.0)
        try:
            out, route = {}, {}
            for op, fn in (("rc", pl.snlm_2d_row_col), ("cr", pl.snlm_2d_col_row),
                           ("snlm", pl.snlm_2d), ("row", pl.nlm_row_pass), ("col", pl.nlm_col_pass)):
                out[op] = fn(xd, p).cpu().numpy()
                route[op] = pl.last_route()
            f64 = route["rc"].startswith("f64")
            assert all(r.startswith("f64") == f64 for r in route.values()), route
            nf64 += f64
            for op, v in out.items():
                h0 = 25.0 if op in ("row", "col") else 36.0
                tol = 1e-3 * scale * (max(1.0, (h0 / h) ** 2) if a.policy == "fast" else 1.0)
                for i in range(b):
                    want = orc.filter(op, x32[i].astype(np.float64), S, K, h, threads=8)
                    err = float(np.abs(v[i].astype(np.float64) - want).max())
                    worst = max(worst, err / tol)
                    assert err <= tol, (op, i, err)
            xt = torch.from_numpy(np.ascontiguousarray(x32.transpose(0, 2, 1))).cuda()
            assert np.array_equal(pl.snlm_2d_col_row(xt, p).cpu().numpy(),
                                  out["rc"].transpose(0, 2, 1)), "transpose equivariance"
            mean = (out["rc"] + out["cr"]) / np.float32(2)
            if f64:  # averaged in double before the one rounding to fp32 (vs three roundings)
                assert np.abs(out["snlm"] - mean).max() <= 4e-5 * scale, "snlm mean"
            else:
                assert np.array_equal(out["snlm"], mean), "snlm mean"
            one = pl.snlm_2d_row_col(xd[b - 1:b].contiguous(), p).cpu().numpy()
            if pl.last_route().startswith("f64") == f64:  # the route is chosen per call
                assert np.array_equal(one[0], out["rc"][b - 1]), "batch invariance"
        except AssertionError as e:
            fails.append(((b, r, c), p, int(kind), str(e)))
            print("FAIL", fails[-1], flush=True)
        n += 1
    print(f"fuzz ({a.policy}): {n} cases in {time.time() - t0:.0f} s ({nf64} on the fp64 route), "
          f"{len(fails)} failures, worst error / tolerance {worst:.3g}")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

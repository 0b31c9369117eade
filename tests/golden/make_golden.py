"""Regenerate tests/golden/golden.npz from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libpatchlift_ref.so, the
unmodified reference sources compiled by oracle/Makefile).  The fixtures pin
the oracle (and through it the CUDA path) to the reference's outputs wherever
the reference library is not available.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Reference, build  # noqa: E402
from paper_1407_2343_b200 import workloads  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    build(with_reference=True)
    ref = Reference.get()
    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20241019)

    # 1D distance bands and filters over random (n, S, K, h), integer and uniform.
    cases = []
    for t in range(40):
        n = int(rng.integers(1, 97))
        K = int(rng.integers(0, min(n, 8) + 1))
        S = int(rng.integers(0, 20))
        h = float(np.exp(rng.uniform(np.log(15.0), np.log(1000.0))))
        integer = t % 2 == 0
        f = rng.integers(0, 256, n).astype(np.float64) if integer else rng.uniform(0, 255, n)
        f = f.astype(np.float32).astype(np.float64)  # fp32-representable inputs
        cases.append((n, S, K, h, int(integer)))
        g[f"l{t}_f"] = f
        g[f"l{t}_dist"] = ref.distance_band(f, S, K)
        g[f"l{t}_nlm"] = ref.nlm_1d(f, S, K, h)
    g["line_cases"] = np.array(cases, dtype=np.float64)

    # Images: every separable composite.
    icases = [(24, 17, 5, 2, 40.0), (13, 19, 4, 1, 25.0), (33, 40, 10, 3, 74.8331), (9, 64, 15, 5, 140.0)]
    for t, (r, c, S, K, h) in enumerate(icases):
        img = rng.uniform(0, 255, (r, c)).astype(np.float32).astype(np.float64)
        g[f"i{t}_img"] = img
        for op in ("row", "col", "rc", "cr", "snlm"):
            g[f"i{t}_{op}"] = ref.filter(op, img, S, K, h)
    g["image_cases"] = np.array(icases, dtype=np.float64)

    # Config 1 at full size (N = 65536): reference output, fp32.
    S, K, h = workloads.params("c1")
    f = workloads.make_config("c1").astype(np.float64)
    g["c1_input_sum"] = np.array([f.sum(), (f * f).sum()])
    g["c1_nlm"] = ref.nlm_1d(f, S, K, h).astype(np.float32)
    # distances at a few sampled rows of the band
    band = ref.distance_band(f[:4096], S, K)
    g["c1_dist_head"] = band.astype(np.float64)

    # Fidelity metrics (metrics.cpp:98-158): noisy / filtered image pairs.
    mrng = np.random.default_rng(77)
    mcases = [(11, 11), (16, 23), (40, 33), (64, 64)]
    for t, (r, c) in enumerate(mcases):
        a = mrng.uniform(0, 255, (r, c)).astype(np.float32).astype(np.float64)
        b = (a + mrng.normal(0, 12.0, (r, c))).astype(np.float32).astype(np.float64)
        g[f"m{t}_a"], g[f"m{t}_b"] = a, b
        g[f"m{t}_metrics"] = np.array(ref.metrics(a, b))
    g["metric_cases"] = np.array(mcases, dtype=np.float64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()

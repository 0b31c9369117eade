"""Seeded synthetic workloads for the five BASELINE.json configs.

The reference benchmarks on standard test images that are not redistributed
 and on iid uniform inputs (bench.cpp:98-116); BASELINE.json
names synthetic constructions instead, restated here with numpy's PCG64
(deterministic across machines for a given seed):

* signal (c1): 64 piecewise-constant segments (63 distinct cut points uniform
  in [1, N-1]), levels U[0,255], plus iid N(0, sigma^2).
* image (c2-c5): linear gradient background 32 + 192 (r+c)/(H+W-2); n_shapes
  axis-aligned rectangles or disks (probability 1/2 each), centres uniform,
  half-size / radius U[H/64, H/8], intensity U[0,255], painted in order; a
  sinusoidal texture 10 sin(2 pi c/17) cos(2 pi r/23); then iid N(0, sigma^2).
  ``quantize=True`` rounds half away from zero and clamps to [0,255]
  (quantize_u8, image_io.cpp:54-63) -- the integer-valued c4 images.

Throughput is data-independent (no early exits anywhere in the filter), so the
content matters only for parity.
"""
from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    # name: (kind, shape, S, K, sigma, shapes, quantize)
    "c1": dict(kind="signal", n=65536, S=10, K=3, sigma=20.0),
    "c2": dict(kind="image", batch=1, rows=512, cols=512, S=10, K=3, sigma=20.0, shapes=40),
    "c3": dict(kind="image", batch=1, rows=4096, cols=4096, S=15, K=5, sigma=30.0, shapes=200),
    "c4": dict(kind="image", batch=64, rows=2048, cols=2048, S=10, K=3, sigma=20.0,
               shapes=100, quantize=True),
    "c5": dict(kind="image", batch=1, rows=16384, cols=16384, S=25, K=7, sigma=25.0, shapes=2000),
}


def h_rule(sigma: float, K: int) -> float:
    """h = sqrt(2(2K+1)) * sigma (BASELINE.json configs)."""
    return math.sqrt(2 * (2 * K + 1)) * sigma


def params(name: str):
    c = CONFIGS[name]
    return c["S"], c["K"], h_rule(c["sigma"], c["K"])


def make_signal(n: int = 65536, sigma: float = 20.0, seed: int = 1, segments: int = 64) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    cuts = np.sort(rng.choice(np.arange(1, n), size=segments - 1, replace=False)) if n > segments else \
        np.arange(1, min(segments, n))
    levels = rng.uniform(0.0, 255.0, size=len(cuts) + 1)
    idx = np.searchsorted(cuts, np.arange(n), side="right")
    x = levels[idx] + rng.normal(0.0, sigma, size=n)
    return x.astype(np.float32)


NOISE_BLOCK = 256  # rows per independently seeded noise block


def make_image(rows: int, cols: int, shapes: int, sigma: float, seed: int = 1,
               quantize: bool = False, row_range: tuple[int, int] | None = None) -> np.ndarray:
    """Synthetic image (or only its rows [r0, r1) -- identical values either way,
    so a rank can build just its row slab)."""
    r0, r1 = row_range if row_range is not None else (0, rows)
    rng = np.random.Generator(np.random.PCG64(seed))
    r = np.arange(r0, r1, dtype=np.float32)[:, None]
    c = np.arange(cols, dtype=np.float32)[None, :]
    img = (32.0 + 192.0 * (r + c) / max(1, rows + cols - 2)).astype(np.float32)
    img = np.broadcast_to(img, (r1 - r0, cols)).copy()
    lo, hi = max(1.0, rows / 64.0), max(1.0, rows / 8.0)
    for _ in range(shapes):
        cy, cx = rng.uniform(0, rows), rng.uniform(0, cols)
        size = rng.uniform(lo, hi)
        val = np.float32(rng.uniform(0.0, 255.0))
        disk = rng.uniform() < 0.5
        y0, y1 = max(r0, int(cy - size)), min(r1, int(math.ceil(cy + size)) + 1)
        x0, x1 = max(0, int(cx - size)), min(cols, int(math.ceil(cx + size)) + 1)
        if y0 >= y1 or x0 >= x1:
            continue
        if disk:
            yy = np.arange(y0, y1, dtype=np.float32)[:, None] - cy
            xx = np.arange(x0, x1, dtype=np.float32)[None, :] - cx
            m = (yy * yy + xx * xx) <= size * size
            img[y0 - r0:y1 - r0, x0:x1][m] = val
        else:
            img[y0 - r0:y1 - r0, x0:x1] = val
    img += (10.0 * np.sin(2 * np.pi * c / 17.0) * np.cos(2 * np.pi * r / 23.0)).astype(np.float32)
    # noise: one PCG64 stream per block of NOISE_BLOCK rows (seeded from (seed, block))
    for b in range(r0 // NOISE_BLOCK, (r1 + NOISE_BLOCK - 1) // NOISE_BLOCK):
        nrng = np.random.Generator(np.random.PCG64([seed, b]))
        blk = nrng.standard_normal((NOISE_BLOCK, cols), dtype=np.float32)
        a, z = max(r0, b * NOISE_BLOCK), min(r1, (b + 1) * NOISE_BLOCK)
        img[a - r0:z - r0] += blk[a - b * NOISE_BLOCK:z - b * NOISE_BLOCK] * np.float32(sigma)
    if quantize:  # round half away from zero, clamp (quantize_u8, image_io.cpp:54-63)
        img = np.clip(np.sign(img) * np.floor(np.abs(img) + 0.5), 0.0, 255.0).astype(np.float32)
    return img


def make_batch(batch: int, rows: int, cols: int, shapes: int, sigma: float, seed: int = 1,
               quantize: bool = False) -> np.ndarray:
    out = np.empty((batch, rows, cols), dtype=np.float32)
    for b in range(batch):
        out[b] = make_image(rows, cols, shapes, sigma, seed=seed * 1000003 + b, quantize=quantize)
    return out


def make_config(name: str, seed: int = 1, batch: int | None = None) -> np.ndarray:
    c = CONFIGS[name]
    if c["kind"] == "signal":
        return make_signal(c["n"], c["sigma"], seed)
    b = c["batch"] if batch is None else batch
    return make_batch(b, c["rows"], c["cols"], c["shapes"], c["sigma"], seed,
                      c.get("quantize", False))

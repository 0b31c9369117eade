"""Pinned host<->device copy bandwidth on the box: H2D, D2H, and both at once."""
import time

import torch

n = 1 << 28  # 1 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device="cuda")
d_b = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


gb = n * 4 / 1e9
t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t_both = timed(both)
chunk = 1 << 22  # 16 MiB pieces, as the pipeline issues them


def both_chunked():
    for o in range(0, n, chunk):
        with torch.cuda.stream(s1):
            d_a[o:o + chunk].copy_(h_in[o:o + chunk], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[o:o + chunk].copy_(d_b[o:o + chunk], non_blocking=True)


t_bc = timed(both_chunked)
print(f"H2D {gb / t_h2d:.1f} GB/s  D2H {gb / t_d2h:.1f} GB/s  both: {2 * gb / t_both:.1f} GB/s total "
      f"({t_both * 1e3:.1f} ms for {gb:.2f} GB each way); chunked 16 MiB: {t_bc * 1e3:.1f} ms")

#!/usr/bin/env python
"""Benchmark of the separable PatchLift-NLM hot path (row pass -> column pass).

Default workload (BASELINE.json configs[3], the config the metric is quoted on
at 1/2/4/8 B200): c4 = a batch of 64 independent 2048x2048 integer-valued
images, K=3, S=10, h=sqrt(14)*20, RC order.  With N GPUs the 64 images are
sharded contiguously over the ranks with no communication (BASELINE's config,
"scaling": "strong"); the same line carries the weak form (every rank its own
64 images) and, at N > 1, the north-star single-image config c5 in all three
partition forms (slab all-to-all, NCCL halo, fused NVLink halo), each checked
bitwise against the single-GPU RC.  ``--config c3|c2|c1`` select the other
single-GPU workloads; ``--config c5`` at N > 1 makes the c5 form chosen by
``--c5-dist`` (default slab) the line.

One "step" = one RC over the whole (per-rank) batch, inputs resident in HBM.
``value`` = all ranks' pixels / max-over-ranks device time (CUDA events).
``roofline.frac`` = unique pairs per launch of the dominant pass kernel / its
event time, over the NOMINAL 16 EX2 per clock per SM;
``frac_measured_peak`` uses this GPU's live MUFU / FP32 microbenchmarks.
``e2e`` = the same metric through the C-ABI host entry point
(pl_snlm_2d_row_col_host) with pinned host buffers, H2D + D2H inside.
``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference library, all host threads) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "separable PatchLift-NLM Mpixel/s at 1/2/4/8 B200; % of exp/FP32/HBM roofline"
UNIT = "Mpixel/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-graph", action="store_true",
                    help="c1/c2: time eager launches instead of one CUDA graph of the K steps")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--c5-dist", default="slab", choices=["slab", "halo", "fused"],
                    help="c5 at N>1: row slabs -> NCCL all-to-all -> column slabs (slab, the "
                         "north-star design, default), row partition + NCCL halo send/recv "
                         "(halo), or the same partition with the halo rows stored into the "
                         "neighbours' symmetric-memory windows by the row-pass kernel (fused); "
                         "the other two forms are reported as fields of the same line")
    ap.add_argument("--no-c5-forms", action="store_true",
                    help="default c4 run at N>1: skip the c5 forms riding along")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the N>1 logic with every rank on cuda:0 "
                         "(timings meaningless)")
    return ap.parse_args()


# --------------------------------------------------------------------------- dist
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(cfg_name: str):
    from paper_1407_2343_b200 import workloads as W
    c = W.CONFIGS[cfg_name]
    S, K, h = W.params(cfg_name)
    return c, S, K, h


def dist_mode(cfg_name, world, how="halo"):
    """c5 at N > 1 (one image): "halo" (row partition + NCCL halo exchange),
    "fused" (the same partition, halo rows stored into the neighbours'
    symmetric-memory windows by the row-pass kernel itself) or "slab" (row
    slabs -> all-to-all -> column slabs); else None."""
    return how if cfg_name == "c5" and world > 1 else None


def make_inputs(cfg_name, lo, hi, row_range=None):
    from paper_1407_2343_b200 import workloads as W
    c = W.CONFIGS[cfg_name]
    if c["kind"] == "signal":
        return W.make_signal(c["n"], c["sigma"], seed=1)[None, :]
    if row_range is not None:
        return W.make_image(c["rows"], c["cols"], c["shapes"], c["sigma"], seed=1 * 1000003,
                            quantize=c.get("quantize", False), row_range=row_range)[None]
    out = np.empty((hi - lo, c["rows"], c["cols"]), np.float32)
    for k, b in enumerate(range(lo, hi)):
        out[k] = W.make_image(c["rows"], c["cols"], c["shapes"], c["sigma"], seed=1 * 1000003 + b,
                              quantize=c.get("quantize", False))
    return out


def describe(cfg_name, c, S, K, h, n_items):
    if c["kind"] == "signal":
        wl = f"{cfg_name}: 1D PatchLift NLM, N={c['n']} fp32 piecewise-constant+noise"
        return {"workload": wl, "n": c["n"], "S": S, "K": K, "h": round(h, 4), "order": "1d"}
    wl = (f"{cfg_name}: {c['batch']} x {c['rows']}x{c['cols']} "
          f"{'integer-valued (quantised) ' if c.get('quantize') else ''}fp32 synthetic images, "
          f"{c['shapes']} shapes, sigma={c['sigma']}")
    return {"workload": wl, "images": n_items, "rows": c["rows"], "cols": c["cols"], "S": S, "K": K,
            "h": round(h, 4), "order": "row->col (snlm_2d_row_col)"}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- peaks
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


def mufu_peak():
    """Live MUFU.EX2 throughput (exps/s) from lib/libplubench.so, full chip."""
    import ctypes as C
    so = os.path.join(ROOT, "paper_1407_2343_b200", "lib", "libplubench.so")
    if not os.path.exists(so):
        return None, None
    L = C.CDLL(so)
    L.plub_rate.restype = C.c_double
    L.plub_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    ms = C.c_double(0)
    ex2 = L.plub_rate(0, 8, 256, 4096, C.byref(ms))
    ffma = L.plub_rate(1, 8, 256, 4096, C.byref(ms))
    ffma2 = L.plub_rate(2, 8, 256, 4096, C.byref(ms))
    mufu_peak.ffma2 = ffma2 if ffma2 > 0 else None
    return (ex2 if ex2 > 0 else None), (ffma if ffma > 0 else None)


def ncu_traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                return json.load(f).get(cfg_name)
        except (OSError, ValueError):
            return None
    return None


# --------------------------------------------------------------------------- cpu
def cpu_reference_rate(cfg_name, imgs_host, S, K, h, seconds, max_items=None):
    """Reference library (oracle/_ref) RC on the host, all hardware threads.
    Returns (Mpx/s, cores, sample description, kind)."""
    from oracle import Oracle, Reference
    if Reference.available():
        eng, kind = Reference.get(), "reference"
        cores = eng.hardware_concurrency()
    else:
        eng, kind = Oracle.get(), "port"
        cores = os.cpu_count() or 1
    c, *_ = workload(cfg_name)
    done_px, t_total, n = 0, 0.0, 0
    limit = max_items or imgs_host.shape[0]
    while n < limit and (t_total < seconds or n == 0):
        img = imgs_host[n % imgs_host.shape[0]].astype(np.float64)
        t0 = time.perf_counter()
        if c["kind"] == "signal":
            eng.nlm_1d(img, S, K, h)
        elif kind == "reference":
            eng.filter("rc", img, S, K, h, threads=0)
        else:
            eng.snlm_rc(img, S, K, h, threads=cores)
        t_total += time.perf_counter() - t0
        done_px += img.size
        n += 1
    sample = (f"{n} of the workload's {c.get('batch', 1)} item(s) ({imgs_host.shape[-2] if imgs_host.ndim > 1 else 1}"
              f"x{imgs_host.shape[-1]}), snlm_2d_row_col(threads=0) of the reference library, "
              f"{t_total:.1f} s")
    return done_px / t_total / 1e6, cores, sample, kind


def run_reference_arm(args):
    world, rank, local = dist_env()
    c, S, K, h = workload(args.config)
    cfg = arm_config(args.config, world)
    if rank != 0:
        return
    sample_imgs = make_inputs(args.config, 0, 1)
    # each step: RC of one image of the workload (a bounded sample), all host threads
    for _ in range(args.warmup):
        cpu_reference_rate(args.config, sample_imgs, S, K, h, 0.0, max_items=1)
    rates, cores, sample, kind = [], None, "", ""
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, cores, sample, kind = cpu_reference_rate(args.config, sample_imgs, S, K, h, 0.0,
                                                    max_items=1)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = float(np.median(rates))
    px = sample_imgs[0].size
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": px / value / 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded PCG64, see paper_1407_2343_b200/workloads.py)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": "each step: " + sample.split(",", 1)[1].strip()
                         if "," in sample else sample,
                         "images_per_step": 1, "cpu_model": cpu_model()},
        "sample": "a bounded sample of the workload: each step filters ONE of its images "
                  "(Mpixel/s is per pixel, so the rate compares with the full batch)",
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ours
class Dist:
    """Process-group plumbing.  ``nccl`` (the product: one rank per GPU) or
    ``gloo`` (functional check of the N > 1 logic with every rank on cuda:0;
    its timings mean nothing): gloo has no device collectives beyond
    all-reduce / broadcast, so the exchanges stage through host memory."""

    def __init__(self, backend: str):
        import torch
        self.world, self.rank, self.local = dist_env()
        self.backend = backend
        self.d = None
        if self.world > 1:
            import torch.distributed as dist
            self.d = dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                torch.cuda.set_device(0)
                dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(0)
        self.dev = torch.device("cuda", torch.cuda.current_device())

    def _red(self, v: float, op) -> float:
        import torch
        if not self.d:
            return float(v)
        dev = self.dev if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        self.d.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return self._red(v, self.d.ReduceOp.MAX if self.d else None)

    def min(self, v: float) -> float:
        return self._red(v, self.d.ReduceOp.MIN if self.d else None)

    def barrier(self):
        if self.d:
            self.d.barrier()

    def all_to_all(self, recv, send):
        if self.backend == "nccl":
            self.d.all_to_all_single(recv, send)
        else:
            r = recv.cpu()
            self.d.all_to_all_single(r, send.cpu())
            recv.copy_(r)

    def p2p(self, ops):
        """ops: [("send"|"recv", peer, tensor)], all completed on return."""
        if not ops:
            return
        if self.backend == "nccl":
            p2p = [self.d.P2POp(self.d.isend if k == "send" else self.d.irecv, t, peer)
                   for k, peer, t in ops]
            for req in self.d.batch_isend_irecv(p2p):
                req.wait()
            return
        reqs, back = [], []
        for k, peer, t in ops:
            h = t.cpu() if k == "send" else torch_empty_like_cpu(t)
            reqs.append((self.d.isend if k == "send" else self.d.irecv)(h, peer))
            if k == "recv":
                back.append((t, h))
        for r in reqs:
            r.wait()
        for t, h in back:
            t.copy_(h)

    def gather_rows(self, full, part):
        """Rank 0: full = rows of every rank's equal-sized part, in rank order."""
        if not self.d:
            full.copy_(part)
            return
        if self.backend == "nccl":
            self.d.all_gather_into_tensor(full, part)
        else:
            parts = [torch_empty_like_cpu(part) for _ in range(self.world)]
            self.d.all_gather(parts, part.cpu())
            if full is not None:
                full.copy_(torch_cat(parts))

    def broadcast(self, t, src=0):
        if not self.d:
            return
        if self.backend == "nccl":
            self.d.broadcast(t, src)
        else:
            h = t.cpu()
            self.d.broadcast(h, src)
            t.copy_(h)

    def close(self):
        if self.d:
            self.d.barrier()
            self.d.destroy_process_group()


def torch_empty_like_cpu(t):
    import torch
    return torch.empty(tuple(t.shape), dtype=t.dtype)


def torch_cat(parts):
    import torch
    return torch.cat(parts, 0)


def timed_graph(D, first_pass, second_pass, steps, warmup, has_second=True):
    """Launch-bound configs (c1: one ~10 us kernel per step; c2: two): the K
    timed steps are captured into ONE CUDA graph and replayed with a single
    launch, so the events bracket device time and not the Python/ctypes launch
    path.  Per-pass times come from two more graphs (K first passes, K second
    passes).  The eager per-step time is reported beside it."""
    import torch

    def capture(fns):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(steps):
                for fn in fns:
                    fn()
        return g

    def replay_ms(g):
        s = torch.cuda.current_stream()
        for _ in range(max(3, warmup) // steps + 2):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.barrier()
        torch.cuda.synchronize()
        a.record(s)
        g.replay()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    eager = timed(D, first_pass, second_pass, steps, warmup, clocks=False)
    g_all, g_row = capture([first_pass, second_pass]), capture([first_pass])
    g_col = capture([second_pass]) if has_second else None
    sampler = ClockSampler(D.dev.index)
    sampler.__enter__()
    try:
        ms_step = D.max(replay_ms(g_all))
        row_ms, col_ms = replay_ms(g_row), (replay_ms(g_col) if g_col else 0.0)
        if len(sampler.lines) < 3:
            time.sleep(0.35)
    finally:
        sampler.__exit__(None, None, None)
    return {"ms_step": ms_step, "row_ms": row_ms, "col_ms": col_ms, "clocks": sampler.summary(),
            "eager_ms_step": eager["ms_step"],
            "launch": f"CUDA graph: the {steps} timed steps captured once, one launch"}


def timed(D, first_pass, second_pass, steps, warmup, clocks=True):
    """W warm-up steps, then K steps between two events on the launching
    stream (per-pass events inside), barrier + synchronize on both sides;
    the step time is the max over ranks."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(max(3, warmup)):
        first_pass()
        second_pass()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    D.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(D.dev.index) if clocks else None
    if sampler:
        sampler.__enter__()
    try:
        start.record(stream)
        for k in range(steps):
            ev[k][0].record(stream)
            first_pass()
            ev[k][1].record(stream)
            second_pass()
            ev[k][2].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
        if sampler and len(sampler.lines) < 3:
            time.sleep(0.35)  # very short regions still get clock samples
    finally:
        if sampler:
            sampler.__exit__(None, None, None)
    D.barrier()
    ms_step = D.max(start.elapsed_time(end)) / steps
    return {"ms_step": ms_step,
            "row_ms": float(np.mean([e[0].elapsed_time(e[1]) for e in ev])),
            "col_ms": float(np.mean([e[1].elapsed_time(e[2]) for e in ev])),
            "clocks": sampler.summary() if sampler else None}


def roofline(D, u_row, u_col, t, px_local, cfg_name, sms, f_max, live_peaks):
    """Roofline of SURVEY.md sec. 8(d) for the dominant pass kernel: per unique
    pair 1 MUFU.EX2 + 8 FP32 lane-ops, per pass 8 HBM bytes per pixel.
    ``frac`` is against the NOMINAL peak (16 EX2 = 128/8 FP32 lanes per clock
    per SM at the maximum SM clock); the live-measured
    MUFU / FP32 peaks of this GPU are a secondary denominator."""
    row_avg, col_avg = t["row_ms"], t["col_ms"]
    dom = "row" if row_avg >= col_avg else "col"
    u_dom, t_dom = (u_row, row_avg) if dom == "row" else (u_col, col_avg)
    nominal = 16 * sms * f_max  # pairs/s
    ex2_peak, ffma_peak = live_peaks
    live = min(ex2_peak or nominal, (ffma_peak or 8 * nominal) / 8.0)
    achieved = u_dom / (t_dom * 1e-3)
    hbm_bytes = 8 * px_local
    hbm_gbs = measured_peaks().get("hbm_gbs", 6541.5)
    return {
        "bound": "sfu+fp32 (tie: 1 EX2 and 8 FP32 lane-ops per pair)",
        "achieved": achieved / 1e9, "peak": nominal / 1e9, "unit": "Gpair/s",
        "frac": achieved / nominal, "traffic": ncu_traffic(cfg_name),
        "peak_kind": "nominal: 16 MUFU.EX2 (= 128 FP32 lanes / 8 ops) per clock per SM "
                     f"x {sms} SMs x {f_max / 1e6:.0f} MHz",
        "kernel": f"nlm_pass3_kernel ({dom} pass)",
        "definition": "unique in-band pairs U per launch / CUDA-event launch time",
        "frac_measured_peak": achieved / live, "measured_peak_gpair_s": live / 1e9,
        "ex2_peak_gexp_s": (ex2_peak or 0) / 1e9, "fp32_peak_glaneops_s": (ffma_peak or 0) / 1e9,
        "algorithmic_per_launch": {"pairs": u_dom, "exps": u_dom, "fp32_ops": 8 * u_dom,
                                   "hbm_bytes": hbm_bytes},
        "row_pass_ms": row_avg, "col_pass_ms": col_avg,
        "step_frac": (u_row + u_col) / (t["ms_step"] * 1e-3) / nominal,
        "hbm": {"achieved_gbs": hbm_bytes / (t_dom * 1e-3) / 1e9, "peak_gbs": hbm_gbs,
                "t_hbm_ms": hbm_bytes / (hbm_gbs * 1e9) * 1e3},
    }


class BatchRun:
    """Independent images (c2-c4) or the c1 signal: images [lo, hi) of the
    workload on this rank, no communication.  One step = the row pass into
    the transposed intermediate + the column pass (what pl_snlm_2d_row_col
    runs)."""

    def __init__(self, D, pl, cfg_name, lo, hi, params):
        import torch
        self.pl, self.params, self.cfg_name = pl, params, cfg_name
        c = W_CONFIGS()[cfg_name]
        self.c = c
        self.signal = c["kind"] == "signal"
        self.imgs_host = make_inputs(cfg_name, lo, hi)
        self.n_local = hi - lo
        self.x = torch.from_numpy(self.imgs_host).to(D.dev)
        self.y = torch.empty_like(self.x)
        self.mid = torch.empty_like(self.x)
        S = params[0]
        if self.signal:
            self.px_local = c["n"]
            self.u_row, self.u_col = pl.unique_pairs(c["n"], S), 0
        else:
            self.px_local = self.n_local * c["rows"] * c["cols"]
            self.u_row = self.n_local * c["rows"] * pl.unique_pairs(c["cols"], S)
            self.u_col = self.n_local * c["cols"] * pl.unique_pairs(c["rows"], S)

    def first_pass(self):
        if self.signal:
            self.pl.nlm_1d_patchlift(self.x, self.params, out=self.y)
            return
        R_, C_ = self.c["rows"], self.c["cols"]
        if self.n_local:
            self.pl.nlm_pass_strided(self.x, self.mid, self.n_local, R_, C_, C_, 1, 1, R_, R_ * C_,
                                     self.params)

    def second_pass(self):
        if self.signal or not self.n_local:
            return
        R_, C_ = self.c["rows"], self.c["cols"]
        self.pl.nlm_pass_strided(self.mid, self.y, self.n_local, C_, R_, R_, 1, 1, C_, R_ * C_,
                                 self.params)

    def e2e(self, D, steps):
        """Through the C-ABI host entry point (pinned host buffers, H2D + D2H
        inside); max over ranks.  Returns (seconds per step, bytes in, out, ok)."""
        import torch
        hin = torch.from_numpy(self.imgs_host).pin_memory()
        if self.signal:
            t0 = time.perf_counter()
            for _ in range(steps):
                yh = self.pl.nlm_1d_patchlift(hin.to(D.dev, non_blocking=True), self.params).cpu()
            return (time.perf_counter() - t0) / steps, hin.numel() * 4, yh.numel() * 4, None
        hout = torch.empty_like(hin).pin_memory()
        if self.n_local:
            self.pl.snlm_2d_row_col_host(hin, self.params, hout)  # warm-up
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            if self.n_local:
                self.pl.snlm_2d_row_col_host(hin, self.params, hout)
        e2e_s = D.max((time.perf_counter() - t0) / steps)
        ok = bool(torch.equal(hout, self.y.cpu()))
        return e2e_s, hin.numel() * 4, hout.numel() * 4, D.min(1.0 if ok else 0.0) > 0


def W_CONFIGS():
    from paper_1407_2343_b200 import workloads as W
    return W.CONFIGS


class C5Run:
    """One 16384^2 image over G ranks (north_star config c5), three forms:
    ``slab`` (row slabs -> row pass into the all-to-all send layout -> NCCL
    all-to-all -> column pass on the column slab, the north-star design),
    ``halo`` (row partition by whole column segments + NCCL halo send/recv +
    windowed column pass) and ``fused`` (the same partition, halo rows stored
    into the neighbours' symmetric-memory windows by the row-pass kernel)."""

    def __init__(self, D, pl, form, params, cfg_name="c5"):
        import torch
        self.D, self.pl, self.form, self.params = D, pl, form, params
        c = W_CONFIGS()[cfg_name]
        self.c = c
        H, Wd = c["rows"], c["cols"]
        world, rank = D.world, D.rank
        S = params[0]
        dev = D.dev
        if form == "slab":
            from paper_1407_2343_b200.distributed import SlabPlan
            self.plan = plan = SlabPlan(H, Wd, world, rank)
            self.imgs_host = make_inputs(cfg_name, 0, 1, row_range=plan.rows)
            self.cb = Wd // world
            self.x = torch.from_numpy(self.imgs_host).to(dev)
            self.mid = torch.empty_like(self.x)
            self.recv = torch.empty_like(self.x)
            self.y = torch.empty((H, self.cb), dtype=torch.float32, device=dev)
            self.region = ("cols",) + plan.cols
            self.nvlink_bytes = plan.nvlink_bytes()
            self.parallelism = f"row slabs -> NCCL all-to-all -> column slabs x{world}"
            self.u_row = (H // world) * pl.unique_pairs(Wd, S)
            self.u_col = self.cb * pl.unique_pairs(H, S)
            self.px_local = H * Wd // world
            return
        from paper_1407_2343_b200.distributed import HaloPlan
        self.plan = plan = HaloPlan(H, Wd, world, rank, params)
        (olo, ohi), (wlo, whi) = plan.rows, plan.window_rows
        self.olo, self.ohi, self.wlo, self.whi = olo, ohi, wlo, whi
        self.seg = plan.segments
        self.imgs_host = make_inputs(cfg_name, 0, 1, row_range=plan.rows)
        self.x = torch.from_numpy(self.imgs_host).to(dev)
        self.y = torch.empty((ohi - olo, Wd), dtype=torch.float32, device=dev)
        self.region = ("rows", olo, ohi)
        self.nvlink_bytes = plan.halo_bytes()
        self.u_row = (ohi - olo) * pl.unique_pairs(Wd, S)
        self.u_col = Wd * sum(min(S, H - 1 - i) for i in range(olo, ohi))
        self.px_local = (ohi - olo) * Wd
        if form == "fused":
            self._setup_fused()
            self.parallelism = f"row partition (whole column segments) + fused NVLink halo stores x{world}"
        else:
            self.win = torch.empty((whi - wlo, Wd), dtype=torch.float32, device=dev)
            self.parallelism = f"row partition (whole column segments) + NCCL halo send/recv x{world}"
        self.ops = []
        if form == "halo":
            for s_, d_, lo_, hi_ in plan.transfers():
                if s_ == rank:
                    self.ops.append(("send", d_, self.win[lo_ - wlo:hi_ - wlo]))
                elif d_ == rank:
                    self.ops.append(("recv", s_, self.win[lo_ - wlo:hi_ - wlo]))

    def _setup_fused(self):
        """Symmetric-memory windows, probed without any collective first so a
        rank that cannot allocate them never leaves its peers in a rendezvous
        (every rank agrees, then all rendezvous or none does)."""
        import torch
        D, plan = self.D, self.plan
        ok = 1.0
        if D.backend != "nccl":
            ok = 0.0
        else:
            try:
                import torch.distributed._symmetric_memory as symm
                symm.empty(1, dtype=torch.float32, device=D.dev)
            except Exception as e:  # noqa: BLE001 -- reported, then every rank agrees
                print(f"rank {D.rank}: symmetric memory unavailable ({e})", file=sys.stderr)
                ok = 0.0
        if D.min(ok) <= 0:
            raise RuntimeError("symmetric memory unavailable on some rank")
        from paper_1407_2343_b200.distributed import symmetric_windows
        self.windows, self.sym_barrier = symmetric_windows(plan, D.dev)
        self.fan = [(self.windows(d_)[row_:row_ + (hi_ - lo_)], lo_ - self.olo, hi_ - self.olo)
                    for d_, lo_, hi_, row_ in plan.fanout()]
        if len(self.fan) > self.pl.PL_MAX_FANOUT:
            raise RuntimeError("more than PL_MAX_FANOUT neighbours")
        self.win = self.windows(D.rank)[:self.whi - self.wlo]

    def first_pass(self):
        pl, p = self.pl, self.params
        if self.form == "slab":
            pl.nlm_row_pass_blocked(self.x, p, self.cb, out=self.mid)
            self.D.all_to_all(self.recv.reshape(-1), self.mid.reshape(-1))
        elif self.form == "fused":
            self.sym_barrier()  # peers done reading their windows (previous column pass)
            pl.nlm_row_pass_fanout(self.x[0], p, out=self.win[self.olo - self.wlo:self.ohi - self.wlo],
                                   extras=self.fan)
            self.sym_barrier()  # every halo row delivered
        else:
            pl.nlm_row_pass(self.x[0], p, out=self.win[self.olo - self.wlo:self.ohi - self.wlo])
            self.D.p2p(self.ops)

    def second_pass(self):
        pl, p = self.pl, self.params
        if self.form == "slab":
            pl.nlm_col_pass(self.recv.reshape(self.c["rows"], self.cb), p, out=self.y)
        else:
            pl.nlm_col_pass_window(self.win, self.wlo, self.c["rows"], self.seg[0], self.seg[1], p,
                                   out=self.y)

    def matches(self, ref):
        """Bitwise equal to the single-GPU RC (ref: the whole image)."""
        import torch
        kind, a, b = self.region
        want = ref[:, a:b] if kind == "cols" else ref[a:b]
        ok = bool(torch.equal(self.y, want))
        return self.D.min(1.0 if ok else 0.0) > 0

    def e2e(self, steps):
        import torch
        hin = torch.from_numpy(self.imgs_host).pin_memory()
        hout = torch.empty(tuple(self.y.shape), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        self.D.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            self.x.copy_(hin, non_blocking=True)
            self.first_pass()
            self.second_pass()
            hout.copy_(self.y, non_blocking=True)
            torch.cuda.synchronize()
        return (self.D.max((time.perf_counter() - t0) / steps), hin.numel() * 4 * self.D.world,
                hout.numel() * 4 * self.D.world)


def c5_reference(D, pl, params, slab_input):
    """Single-GPU RC of the whole c5 image on rank 0 (its rows gathered from
    the slab form's row slabs), broadcast to every rank for the bitwise check."""
    import torch
    c = W_CONFIGS()["c5"]
    full = torch.empty((c["rows"], c["cols"]), dtype=torch.float32, device=D.dev)
    D.gather_rows(full, slab_input.reshape(-1, c["cols"]))
    if D.rank == 0:
        ref = pl.snlm_2d_row_col(full, params)
    else:
        ref = torch.empty_like(full)
    del full
    D.broadcast(ref, 0)
    return ref


def c5_forms(D, pl, params, args, forms):
    """Time each c5 form (device, max over ranks) and check it bitwise against
    the single-GPU RC.  Returns {form: {...}} (unavailable forms say why)."""
    import torch
    out = {}
    ref = None
    for form in forms:
        try:
            run = C5Run(D, pl, form, params)
        except RuntimeError as e:
            out[form] = {"unavailable": str(e)}
            continue
        t = timed(D, run.first_pass, run.second_pass, args.steps, args.warmup, clocks=False)
        if ref is None:
            slab = run.x if form == "slab" else None
            if slab is None:
                from paper_1407_2343_b200.distributed import SlabPlan
                sp = SlabPlan(run.c["rows"], run.c["cols"], D.world, D.rank)
                slab = torch.from_numpy(make_inputs("c5", 0, 1, row_range=sp.rows)).to(D.dev)
            ref = c5_reference(D, pl, params, slab)
        px = run.c["rows"] * run.c["cols"]
        out[form] = {"value": px / (t["ms_step"] * 1e-3) / 1e6, "unit": UNIT,
                     "ms_per_step": t["ms_step"], "row_pass_ms": t["row_ms"],
                     "col_pass_ms": t["col_ms"], "nvlink_bytes_per_rank": run.nvlink_bytes,
                     "parallelism": run.parallelism,
                     "bitwise_equal_single_gpu_rc": run.matches(ref)}
        del run
        torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import paper_1407_2343_b200 as pl

    D = Dist(args.dist_backend)
    world, rank = D.world, D.rank
    c, S, K, h = workload(args.config)
    params = (S, K, h)
    n_items = c.get("batch", 1)
    f_max = measured_peaks().get("sm_max_mhz", 1965.0) * 1e6
    sms = torch.cuda.get_device_properties(D.dev).multi_processor_count
    live_peaks = mufu_peak() if rank == 0 else (None, None)
    cfg = arm_config(args.config, world)
    c5_main = args.config == "c5" and world > 1

    if c5_main:
        # the chosen form is the line; the other two ride along as fields
        run = C5Run(D, pl, args.c5_dist, params)
        t = timed(D, run.first_pass, run.second_pass, args.steps, args.warmup)
        px_total = c["rows"] * c["cols"]
        roof = roofline(D, run.u_row, run.u_col, t, run.px_local, args.config, sms, f_max, live_peaks)
        e2e_s, bi, bo = run.e2e(args.e2e_steps)
        e2e = {"value": px_total / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo,
               "api": f"pinned H2D + c5 {args.c5_dist} path (row pass, exchange, column pass) + D2H"}
        cfg["parallelism"] = run.parallelism
        cfg["nvlink_bytes_per_rank"] = run.nvlink_bytes
        launches = args.steps * 2
        del run
        torch.cuda.empty_cache()
        extra = {"c5_forms": c5_forms(D, pl, params, args, ["slab", "halo", "fused"])}
        scaling = "strong"
    else:
        if c["kind"] == "signal":
            lo, hi = 0, 1
        else:  # BASELINE's batch sharded across the ranks (contiguous shares)
            from paper_1407_2343_b200.distributed import shard
            lo, hi = shard(n_items, world, rank)
        run = BatchRun(D, pl, args.config, lo, hi, params)
        if args.config in ("c1", "c2") and world == 1 and not args.no_graph:
            t = timed_graph(D, run.first_pass, run.second_pass, args.steps, args.warmup,
                            has_second=not run.signal)
        else:
            t = timed(D, run.first_pass, run.second_pass, args.steps, args.warmup)
        px_total = c["n"] if run.signal else n_items * c["rows"] * c["cols"]
        roof = roofline(D, run.u_row, run.u_col, t, run.px_local, args.config, sms, f_max, live_peaks)
        e2e_s, bi, bo, ok = run.e2e(D, args.e2e_steps)
        e2e = {"value": px_total / e2e_s / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(D.max(bi) * world) if world > 1 else bi,
               "d2h_bytes_per_step": int(D.max(bo) * world) if world > 1 else bo}
        if not run.signal:
            e2e["api"] = "pl_snlm_2d_row_col_host (pinned host buffers)"
            e2e["matches_device_result"] = ok
        launches = args.steps * (1 if run.signal else 2)
        scaling = "strong"
        extra = {}
        if world > 1 and not run.signal:
            # weak form: every rank its own full batch (images 64r .. 64r+63)
            del run
            torch.cuda.empty_cache()
            wk = BatchRun(D, pl, args.config, rank * n_items, (rank + 1) * n_items, params)
            tw = timed(D, wk.first_pass, wk.second_pass, args.steps, args.warmup, clocks=False)
            extra["weak"] = {"value": world * n_items * c["rows"] * c["cols"] / (tw["ms_step"] * 1e-3) / 1e6,
                             "unit": UNIT, "ms_per_step": tw["ms_step"], "images_per_rank": n_items,
                             "scaling": "weak"}
            del wk
            torch.cuda.empty_cache()
        if world > 1 and args.config == "c4" and not args.no_c5_forms:
            # the north-star single-image path rides along at N > 1 (all three forms)
            extra["c5_forms"] = c5_forms(D, pl, workload("c5")[1:], args,
                                         ["slab", "halo", "fused"])

    value = px_total / (t["ms_step"] * 1e-3) / 1e6
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t["ms_step"], "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded PCG64 constructions of BASELINE.json, "
                    "paper_1407_2343_b200/workloads.py)",
            "config": cfg, "roofline": roof, "clocks": t["clocks"], "gpu_launches": launches,
            "e2e": e2e,
        }
        if D.backend != "nccl":
            line["functional_check_only"] = "gloo backend, all ranks on cuda:0: timings meaningless"
        line.update(extra)
        if "launch" in t:
            line["launch"] = t["launch"]
            line["eager_ms_per_step"] = t["eager_ms_step"]
        if world == 1 and not c5_main and not run.signal:
            line["snlm_2d"] = snlm_extra(pl, run, px_total, max(3, args.steps // 4))
        if world == 1 and not c5_main and not run.signal:
            line["e2e_dropin"] = dropin_e2e(run.imgs_host[0], S, K, h, args.e2e_steps)
        if world == 1 and not args.no_cpu_baseline:
            v, cores, sample, kind = cpu_reference_rate(args.config, run.imgs_host, S, K, h,
                                                        args.cpu_seconds)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                    "sample": sample, "cpu_model": cpu_model()}
        print(json.dumps(line), flush=True)
    D.close()


def snlm_extra(pl, run, px_total, steps):
    """The paper's averaged S-NLM (snlm_2d = (RC + CR) / 2, nlm.cpp:248-253) on
    the same resident batch: four passes, the average fused into the last
    store.  An extra beside the judged RC metric."""
    import torch
    out = torch.empty_like(run.x)
    work = torch.empty((2,) + tuple(run.x.shape), dtype=torch.float32, device=run.x.device)
    for _ in range(2):
        pl.snlm_2d(run.x, run.params, out=out, work=work)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        pl.snlm_2d(run.x, run.params, out=out, work=work)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    del out, work
    return {"value": px_total / (ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "api": "pl_snlm_2d (RC and CR, four passes, average fused into the last store)"}


def dropin_e2e(img, S, K, h, calls):
    """Mpixel/s through the C++ drop-in a reference caller links
    (patchlift::snlm_2d_row_col on a double Image2D, threads=0: copies and both
    passes per call), one image of the workload per call: its default
    reference-precision fp64 route, and the fp32 route (conversions included)."""
    import tempfile
    exe = os.path.join(ROOT, "paper_1407_2343_b200", "lib", "dropin_bench")
    if not os.path.exists(exe):
        return {"unavailable": "lib/dropin_bench not built"}
    res = {}
    with tempfile.NamedTemporaryFile(suffix=".f32") as f:
        np.ascontiguousarray(img, dtype=np.float32).tofile(f.name)
        for prec in ("fp64", "fp32"):
            r = subprocess.run([exe, f.name, str(img.shape[0]), str(img.shape[1]), str(S), str(K),
                                repr(float(h)), str(max(1, calls)), "0", prec],
                               capture_output=True, text=True, timeout=600)
            if r.returncode != 0:
                res[prec] = {"unavailable": (r.stderr or r.stdout).strip()[-300:]}
                continue
            out = json.loads(r.stdout.strip().splitlines()[-1])
            res[prec] = {"value": out["mpx_s"], "s_per_call": out["s_per_call"]}
    line = {"value": res.get("fp64", {}).get("value"), "unit": UNIT, "calls": max(1, calls),
            "images_per_call": 1, "precision": "fp64 (drop-in default)",
            "fp32_route": res.get("fp32"),
            "api": "patchlift::snlm_2d_row_col (C++ drop-in, double Image2D in and out, "
                   "threads=0; tests/cpp/dropin_bench.cpp)"}
    if "unavailable" in res.get("fp64", {}):
        line["unavailable"] = res["fp64"]["unavailable"]
    return line


def arm_config(cfg_name, world):
    """The `config` object both arms print (identical, so the driver compares
    like with like)."""
    c, S, K, h = workload(cfg_name)
    n_items = c.get("batch", 1)
    cfg = describe(cfg_name, c, S, K, h, n_items)
    if c["kind"] == "image":
        px_total = n_items * c["rows"] * c["cols"]
        cfg["l2"] = ("inputs + intermediate exceed the 126 MB L2" if px_total * 4 > 126e6
                     else "working set fits L2 (flush not applied; compute-bound kernel)")
        cfg["global_batch"] = n_items
    cfg["parallelism"] = ("1 GPU" if world == 1 else
                          f"{n_items} images sharded over {world} ranks (contiguous, no communication)"
                          if c["kind"] == "image" and n_items > 1 else f"{world} ranks")
    return cfg


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        info = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                info[k.strip()] = v.strip()
        return {"model": info.get("Model name"), "cpus": info.get("CPU(s)"),
                "sockets": info.get("Socket(s)"), "cores_per_socket": info.get("Core(s) per socket"),
                "threads_per_core": info.get("Thread(s) per core")}
    except (OSError, subprocess.SubprocessError):
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

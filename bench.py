#!/usr/bin/env python
"""Benchmark of the separable PatchLift-NLM hot path (row pass -> column pass).

Default workload (BASELINE.json configs[3], the config the metric is quoted on
at 1/2/4/8 B200): c4 = 64 independent 2048x2048 integer-valued images, K=3,
S=10, h=sqrt(14)*20, RC order.  With N GPUs every rank filters its own batch
of 64 such images (images 64r .. 64r+63 of the seeded construction) with no
communication: the path partitions into independent images, so the per-GPU
work is fixed and the line reports weak scaling (value = all ranks' pixels /
max-over-ranks time).  ``--config c3|c2|c1`` select the other single-GPU
workloads; ``--config c5`` at N > 1 partitions ONE 16384^2 image (strong
scaling, ``--c5-dist halo|fused|slab``).

One "step" = one RC over the whole (per-rank) batch, inputs resident in HBM.
``value`` = all ranks' pixels / max-over-ranks device time (CUDA events).
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
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--c5-dist", default="fused", choices=["fused", "halo", "slab"],
                    help="c5 at N>1: row partition with the halo rows stored into the "
                         "neighbours' symmetric-memory windows by the row-pass kernel (fused, "
                         "default), the same with NCCL send/recv (halo), or the row-slab -> "
                         "all-to-all -> column-slab transpose (slab)")
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
    n_items = c.get("batch", 1)
    cfg = describe(args.config, c, S, K, h, n_items)
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
        "higher_is_better": True, "scaling": "weak" if c["kind"] == "image" and c.get("batch", 1) > 1
        else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded PCG64, see paper_1407_2343_b200/workloads.py)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": "each step: " + sample.split(",", 1)[1].strip()
                         if "," in sample else sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import paper_1407_2343_b200 as pl

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    c, S, K, h = workload(args.config)
    params = (S, K, h)
    n_items = c.get("batch", 1)
    mode = dist_mode(args.config, world, args.c5_dist)
    slab, halo, fused = mode == "slab", mode in ("halo", "fused"), mode == "fused"
    if c["kind"] == "signal" or mode:
        lo, hi = 0, 1
    else:  # weak scaling: every rank its own batch of n_items images
        lo, hi = rank * n_items, (rank + 1) * n_items
    if slab:
        from paper_1407_2343_b200.distributed import SlabPlan
        plan = SlabPlan(c["rows"], c["cols"], world, rank)
        imgs_host = make_inputs(args.config, 0, 1, row_range=plan.rows)
    elif halo:
        from paper_1407_2343_b200.distributed import HaloPlan
        plan = HaloPlan(c["rows"], c["cols"], world, rank, params)
        imgs_host = make_inputs(args.config, 0, 1, row_range=plan.rows)
    else:
        imgs_host = make_inputs(args.config, lo, hi)
    x = torch.from_numpy(imgs_host).to(dev)
    y = torch.empty_like(x)
    mid = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    signal = c["kind"] == "signal"
    if slab:
        cb = c["cols"] // world
        recv = torch.empty_like(x)
        y = torch.empty((c["rows"], cb), dtype=x.dtype, device=dev)
    if halo:
        (olo, ohi), (wlo, whi) = plan.rows, plan.window_rows
        seg_a, seg_b = plan.segments
        win = torch.empty((whi - wlo, c["cols"]), dtype=x.dtype, device=dev)
        y = torch.empty((ohi - olo, c["cols"]), dtype=x.dtype, device=dev)
        p2p = []
        if fused:
            from paper_1407_2343_b200.distributed import symmetric_windows
            ok = torch.ones(1, device=dev)
            try:
                windows, sym_barrier = symmetric_windows(plan, dev)
                fan = [(windows(d_)[row_:row_ + (hi_ - lo_)], lo_ - olo, hi_ - olo)
                       for d_, lo_, hi_, row_ in plan.fanout()]
                if len(fan) > pl.PL_MAX_FANOUT:
                    raise RuntimeError("more than PL_MAX_FANOUT neighbours")
            except Exception as e:  # no symmetric memory here: NCCL halo exchange instead
                print(f"rank {rank}: fused halo unavailable ({e}); using NCCL send/recv",
                      file=sys.stderr)
                ok.zero_()
            torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
            if ok.item() > 0:
                win = windows(rank)[:whi - wlo]
            else:
                fused = False
        for s_, d_, lo_, hi_ in ([] if fused else plan.transfers()):
            if s_ == rank:
                p2p.append(torch.distributed.P2POp(torch.distributed.isend,
                                                   win[lo_ - wlo:hi_ - wlo], d_))
            elif d_ == rank:
                p2p.append(torch.distributed.P2POp(torch.distributed.irecv,
                                                   win[lo_ - wlo:hi_ - wlo], s_))

    def first_pass():
        if signal:
            pl.nlm_1d_patchlift(x, params, out=y)
        elif slab:
            pl.nlm_row_pass_blocked(x, params, cb, out=mid)
            torch.distributed.all_to_all_single(recv.reshape(-1), mid.reshape(-1))
        elif fused:
            sym_barrier()  # peers done reading their windows (previous column pass)
            pl.nlm_row_pass_fanout(x[0], params, out=win[olo - wlo:ohi - wlo], extras=fan)
            sym_barrier()  # every halo row delivered
        elif halo:
            pl.nlm_row_pass(x[0], params, out=win[olo - wlo:ohi - wlo])
            if p2p:
                for req in torch.distributed.batch_isend_irecv(p2p):
                    req.wait()
        else:  # row pass into the transposed intermediate (what pl_snlm_2d_row_col runs)
            R_, C_ = c["rows"], c["cols"]
            pl.nlm_pass_strided(x, mid, x.shape[0], R_, C_, C_, 1, 1, R_, R_ * C_, params)

    def second_pass():
        if signal:
            return
        if slab:
            pl.nlm_col_pass(recv.reshape(c["rows"], cb), params, out=y)
        elif halo:
            pl.nlm_col_pass_window(win, wlo, c["rows"], seg_a, seg_b, params, out=y)
        else:  # column pass reading the transposed intermediate
            R_, C_ = c["rows"], c["cols"]
            pl.nlm_pass_strided(mid, y, x.shape[0], C_, R_, R_, 1, 1, C_, R_ * C_, params)

    def step():
        first_pass()
        second_pass()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # per-launch timing of the two pass kernels (events on the launching stream)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        start.record(stream)
        for k in range(args.steps):
            ev[k][0].record(stream)
            first_pass()
            ev[k][1].record(stream)
            second_pass()
            ev[k][2].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
        # keep sampling a short moment so very short regions still get clock samples
        if len(clocks.lines) < 3:
            time.sleep(0.35)
    if world > 1:
        torch.distributed.barrier()
    ms_local = start.elapsed_time(end)
    t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    row_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    col_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]

    if signal:
        px_local = c["n"]
        px_total = px_local
    elif mode:
        px_local = x.numel() if halo else c["rows"] * c["cols"] // world
        px_total = c["rows"] * c["cols"]
    else:
        px_local = (hi - lo) * c["rows"] * c["cols"]
        px_total = world * n_items * c["rows"] * c["cols"]
    value = px_total / (ms_step * 1e-3) / 1e6

    # ---- roofline (dominant kernel): unique pairs = exps per launch ----------
    if signal:
        u_row = pl.unique_pairs(c["n"], S)
        u_col = 0
    elif slab:
        u_row = (c["rows"] // world) * pl.unique_pairs(c["cols"], S)
        u_col = (c["cols"] // world) * pl.unique_pairs(c["rows"], S)
    elif halo:  # pairs counted at their left endpoint, which my rows own
        u_row = (ohi - olo) * pl.unique_pairs(c["cols"], S)
        u_col = c["cols"] * sum(min(S, c["rows"] - 1 - i) for i in range(olo, ohi))
    else:
        u_row = (hi - lo) * c["rows"] * pl.unique_pairs(c["cols"], S)
        u_col = (hi - lo) * c["cols"] * pl.unique_pairs(c["rows"], S)
    row_avg = float(np.mean(row_ms))
    col_avg = float(np.mean(col_ms)) if not signal else 0.0
    dom = "row" if row_avg * 1.0 >= col_avg else "col"
    u_dom, t_dom = (u_row, row_avg) if dom == "row" else (u_col, col_avg)
    peaks = measured_peaks()
    ex2_peak, ffma_peak = (mufu_peak() if rank == 0 else (None, None))
    f_max = peaks.get("sm_max_mhz", 1965.0) * 1e6
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # Roofline of SURVEY.md sec. 8(d): per unique pair 1 MUFU.EX2 + 8 FP32 lane-ops,
    # per pass 8 HBM bytes per pixel.  Peaks measured live on this GPU
    # (lib/libplubench.so); nominal: 16 ex2 and 128 FP32 lanes per clock per SM.
    ex2_rate = ex2_peak or 16 * sms * f_max
    fp32_rate = ffma_peak or 128 * sms * f_max
    pair_peak = min(ex2_rate, fp32_rate / 8.0)  # pairs/s
    achieved = u_dom / (t_dom * 1e-3)
    hbm_bytes = 8 * px_local  # per pass: fp32 read + write
    hbm_gbs = peaks.get("hbm_gbs", 6541.5)
    roof = {
        "bound": "fp32" if fp32_rate / 8.0 < ex2_rate else "sfu",
        "achieved": achieved / 1e9, "peak": pair_peak / 1e9, "unit": "Gpair/s",
        "frac": achieved / pair_peak, "traffic": ncu_traffic(args.config),
        "kernel": f"nlm_pass3_kernel ({dom} pass)",
        "definition": "unique in-band pairs U per launch / CUDA-event launch time; peak = "
                      "min(MUFU.EX2 rate, FP32 lane-op rate / 8), both measured live",
        "ex2_peak_gexp_s": ex2_rate / 1e9, "fp32_peak_glaneops_s": fp32_rate / 1e9,
        "frac_of_ex2": achieved / ex2_rate,
        "peak_nominal_gpair_s": 16 * sms * f_max / 1e9,
        "algorithmic_per_launch": {"pairs": u_dom, "exps": u_dom, "fp32_ops": 8 * u_dom,
                                   "hbm_bytes": hbm_bytes},
        "row_pass_ms": row_avg, "col_pass_ms": col_avg,
        "step_frac": (u_row + u_col) / (ms_step * 1e-3) / pair_peak,
        "hbm": {"achieved_gbs": hbm_bytes / (t_dom * 1e-3) / 1e9, "peak_gbs": hbm_gbs,
                "t_hbm_ms": hbm_bytes / (hbm_gbs * 1e9) * 1e3},
    }

    line = None
    if rank == 0:
        cfg = describe(args.config, c, S, K, h, n_items)
        cfg["l2"] = ("inputs + intermediate exceed the 126 MB L2" if px_total * 4 > 126e6
                     else "working set fits L2 (flush not applied; compute-bound kernel)")
        cfg["parallelism"] = (f"{world} ranks x {n_items} images each (no communication)"
                              if world > 1 else "1 GPU")
        if not (mode or signal):
            cfg["global_batch"] = world * n_items
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (mode or signal) else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded PCG64 constructions of BASELINE.json, "
                    "paper_1407_2343_b200/workloads.py)",
            "config": cfg, "roofline": roof, "clocks": clocks.summary(),
            "gpu_launches": args.steps * (1 if signal else 2),
        }

    # ---- e2e through the C-ABI host entry point (N GPUs: each rank its shard) --
    if mode:
        hin = torch.from_numpy(imgs_host).pin_memory()
        hout = torch.empty(tuple(y.shape), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            x.copy_(hin, non_blocking=True)
            step()
            hout.copy_(y, non_blocking=True)
            torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        te = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        if rank == 0:
            line["e2e"] = {"value": px_total / float(te.item()) / 1e6, "unit": UNIT,
                           "h2d_bytes_per_step": int(hin.numel() * 4) * world,
                           "d2h_bytes_per_step": int(hout.numel() * 4) * world}
            if slab:
                line["e2e"]["api"] = "pinned H2D + row pass + NCCL all-to-all + column pass + D2H"
                line["config"]["nvlink_bytes_per_rank"] = plan.nvlink_bytes()
                line["config"]["parallelism"] = f"row slabs -> all-to-all -> column slabs x{world}"
            else:
                line["e2e"]["api"] = ("pinned H2D + row pass + " +
                                      ("fused NVLink halo stores (symmetric memory) + barrier"
                                       if fused else "NCCL halo send/recv") +
                                      " + windowed column pass + D2H")
                line["config"]["nvlink_bytes_per_rank"] = plan.halo_bytes()
                line["config"]["parallelism"] = (f"row partition (whole column segments) + "
                                                 f"{'fused NVLink halo stores' if fused else 'halo exchange'} x{world}")
    elif not signal:
        hin = torch.from_numpy(imgs_host).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        pl.snlm_2d_row_col_host(hin, params, hout)  # warm-up
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            pl.snlm_2d_row_col_host(hin, params, hout)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        te = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(te.item())
        ok = torch.equal(hout, y.cpu())
        if rank == 0:
            line["e2e"] = {"value": px_total / e2e_s / 1e6, "unit": UNIT,
                           "h2d_bytes_per_step": int(hin.numel() * 4) * world,
                           "d2h_bytes_per_step": int(hout.numel() * 4) * world,
                           "api": "pl_snlm_2d_row_col_host (pinned host buffers)",
                           "matches_device_result": bool(ok)}
    elif rank == 0:
        hin = torch.from_numpy(imgs_host).pin_memory()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            xd = hin.to(dev, non_blocking=True)
            yd = pl.nlm_1d_patchlift(xd, params)
            yh = yd.cpu()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        line["e2e"] = {"value": px_total / e2e_s / 1e6, "unit": UNIT,
                       "h2d_bytes_per_step": int(hin.numel() * 4),
                       "d2h_bytes_per_step": int(yh.numel() * 4)}

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, kind = cpu_reference_rate(args.config, imgs_host, S, K, h,
                                                    args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

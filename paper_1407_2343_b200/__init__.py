"""paper_1407_2343_b200 -- B200-native PatchLift separable-NLM hot path.

Python face of the C ABI in ``include/plgpu.h`` (``lib/libplgpu.so``), used by
the tests and by ``bench.py``.  Device buffers are torch CUDA tensors (torch is
plumbing here: allocation, streams, ``torch.distributed``); every filter runs
in the hand-written sm_100a kernels behind the C ABI.  There is no CPU route:
if the native library is missing, :func:`lib` raises.

Names mirror the reference API (``proj/include/patchlift/nlm.hpp``):
``nlm_1d_patchlift`` (batched lines), ``nlm_row_pass``, ``nlm_col_pass``,
``snlm_2d_row_col``, ``snlm_2d_col_row``, ``snlm_2d``, plus the distance-band
and F-bar exports of ``banded_kernel.hpp``.  Errors raise :class:`ValidationError`
with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

PKG = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(PKG, "lib")
LIBPLGPU = os.environ.get("PLGPU_LIB") or os.path.join(LIBDIR, "libplgpu.so")  # override: experiments
LIBDROPIN = os.path.join(LIBDIR, "libpatchlift_b200.so")

PL_OK, PL_ERR_VALIDATION, PL_ERR_RANGE, PL_ERR_CUDA, PL_ERR_UNSUPPORTED, PL_ERR_ARG = range(6)

# Every symbol include/plgpu.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "pl_abi_version", "pl_last_error", "pl_device_name", "pl_validate_params",
    "pl_validate_geometry", "pl_op_counts_1d", "pl_unique_pairs", "pl_segment_length",
    "pl_nlm_lines", "pl_nlm_lines_naive", "pl_nlm_row_pass", "pl_nlm_col_pass",
    "pl_nlm_row_pass_blocked", "pl_workspace_bytes", "pl_snlm_2d_row_col",
    "pl_snlm_2d_col_row", "pl_snlm_2d", "pl_snlm_2d_row_col_host", "pl_nlm_2d_naive",
    "pl_device_alloc", "pl_device_free", "pl_copy_to_device", "pl_copy_to_host",
    "pl_synchronize", "pl_distance_band_f32", "pl_distance_band_i32", "pl_banded_kernel_f64",
    "pl_col_window", "pl_nlm_col_pass_window", "pl_image_metrics_f32", "pl_image_metrics_f64",
    "pl_nlm_pass_strided", "pl_nlm_row_pass_fanout", "pl_last_route",
    "pl_debug_hot_distance_band", "pl_host_alloc", "pl_host_free", "pl_stream_create",
    "pl_stream_destroy", "pl_stream_synchronize", "pl_copy_to_device_async",
    "pl_copy_to_host_async", "pl_debug_set_route", "pl_graph_rc_create", "pl_graph_launch",
    "pl_graph_destroy", "pl_nlm_lines_f64", "pl_nlm_lines_naive_f64", "pl_nlm_row_pass_f64",
    "pl_nlm_col_pass_f64", "pl_snlm_2d_row_col_f64", "pl_snlm_2d_col_row_f64", "pl_snlm_2d_f64",
    "pl_nlm_2d_naive_f64", "pl_set_precision_policy", "pl_precision_policy", "pl_fast_h_threshold",
]
PL_PRECISION_AUTO, PL_PRECISION_FAST = 0, 1
PL_MAX_FANOUT = 2


class ValidationError(ValueError):
    """The reference's ``patchlift::ValidationError`` (a std::invalid_argument)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the native library."""


class _Params(C.Structure):
    _fields_ = [("search_radius", C.c_int32), ("patch_radius", C.c_int32), ("h", C.c_double)]


class _OpCounts(C.Structure):
    _fields_ = [("adds", C.c_uint64), ("muls", C.c_uint64), ("exps", C.c_uint64),
                ("clamps", C.c_uint64)]


@dataclass
class NlmParams:
    """``NlmParams`` (core_types.hpp:45-49)."""

    search_radius: int = 10
    patch_radius: int = 3
    h: float = 0.0

    def c(self) -> _Params:
        return _Params(int(self.search_radius), int(self.patch_radius), float(self.h))


_LIB = None


def lib() -> C.CDLL:
    """Load ``lib/libplgpu.so`` (build it with ``__graft_entry__.build()``)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIBPLGPU):
            raise ImportError(f"native library missing: {LIBPLGPU}; run __graft_entry__.build()")
        L = C.CDLL(LIBPLGPU)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        P = _Params
        sig = {
            "pl_abi_version": ([], C.c_int),
            "pl_last_error": ([], C.c_char_p),
            "pl_last_route": ([], C.c_char_p),
            "pl_debug_set_route": ([i32, i32, i32], C.c_int),
            "pl_set_precision_policy": ([i32], C.c_int),
            "pl_precision_policy": ([], i32),
            "pl_fast_h_threshold": ([], C.c_double),
            "pl_graph_rc_create": ([vp, vp, vp, i32, i32, i32, P, C.POINTER(vp)], C.c_int),
            "pl_graph_launch": ([vp, vp], C.c_int),
            "pl_graph_destroy": ([vp], C.c_int),
            "pl_nlm_lines_f64": ([vp, vp, i64, i32, i64, P, vp], C.c_int),
            "pl_nlm_lines_naive_f64": ([vp, vp, i64, i32, i64, P, vp], C.c_int),
            "pl_nlm_row_pass_f64": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_col_pass_f64": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d_row_col_f64": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d_col_row_f64": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d_f64": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_2d_naive_f64": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_debug_hot_distance_band": ([vp, vp, i32, i32, i32, i32, vp], C.c_int),
            "pl_device_name": ([], C.c_char_p),
            "pl_validate_params": ([P, i32], C.c_int),
            "pl_validate_geometry": ([i32, i32, i32], C.c_int),
            "pl_op_counts_1d": ([i32, P, C.POINTER(_OpCounts)], C.c_int),
            "pl_unique_pairs": ([i32, i32], C.c_uint64),
            "pl_segment_length": ([i32, i32], i32),
            "pl_nlm_lines": ([vp, vp, i64, i32, i64, P, vp], C.c_int),
            "pl_nlm_lines_naive": ([vp, vp, i64, i32, i64, P, vp], C.c_int),
            "pl_nlm_row_pass": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_col_pass": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_row_pass_blocked": ([vp, vp, i32, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_row_pass_fanout": ([vp, vp, i32, i32, P, i32, C.POINTER(vp), C.POINTER(i32),
                                        C.POINTER(i32), vp], C.c_int),
            "pl_col_window": ([i32, i32, i32, P] + [C.POINTER(i32)] * 4, C.c_int),
            "pl_image_metrics_f32": ([vp, vp, i32, i32, i32, vp, vp], C.c_int),
            "pl_nlm_pass_strided": ([vp, vp, i32, i32, i32, i64, i64, i64, i64, i64, P, vp],
                                    C.c_int),
            "pl_image_metrics_f64": ([vp, vp, i32, i32, i32, vp, vp], C.c_int),
            "pl_nlm_col_pass_window": ([vp, i32, i32, vp, i32, i32, i32, i32, i32, P, vp],
                                       C.c_int),
            "pl_workspace_bytes": ([i32, i32, i32, i32], C.c_size_t),
            "pl_snlm_2d_row_col": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d_col_row": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d": ([vp, vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_snlm_2d_row_col_host": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_nlm_2d_naive": ([vp, vp, i32, i32, i32, P, vp], C.c_int),
            "pl_distance_band_f32": ([vp, vp, i64, i32, i64, i32, i32, vp], C.c_int),
            "pl_distance_band_i32": ([vp, vp, i64, i32, i64, i32, i32, vp], C.c_int),
            "pl_banded_kernel_f64": ([vp, vp, i64, i32, i64, i32, i32, vp], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc == PL_OK:
        return
    msg = (lib().pl_last_error() or b"").decode()
    if rc == PL_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == PL_ERR_RANGE:
        raise IndexError(msg)
    if rc == PL_ERR_CUDA:
        raise DeviceError(msg)
    raise RuntimeError(f"plgpu error {rc}: {msg}")


def _params(p) -> _Params:
    if isinstance(p, NlmParams):
        return p.c()
    S, K, h = p
    return _Params(int(S), int(K), float(h))


def _stream(t) -> int:
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _dev(t, dtype=None):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError("expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t


def _out(out, like, shape=None):
    """A caller-supplied output: float32, contiguous, on like's device, with
    exactly the expected number of elements (shape defaults to like's)."""
    import torch
    shape = tuple(like.shape) if shape is None else tuple(shape)
    if out is None:
        return torch.empty(shape, dtype=torch.float32, device=like.device)
    _dev(out, torch.float32)
    if out.device != like.device:
        raise ValueError(f"out is on {out.device}, input on {like.device}")
    if out.numel() != math.prod(shape):
        raise ValueError(f"out has {out.numel()} elements, expected {math.prod(shape)} {shape}")
    return out


class debug_route:
    """Context manager pinning the kernel route (pl_debug_set_route): walker 0
    default / 1 portable only / 2 no hot kernel; lines, wpc of the hot kernel
    (0 = default).  Results are bitwise identical on every route."""

    def __init__(self, walker: int = 0, lines: int = 0, wpc: int = 0):
        self.args = (int(walker), int(lines), int(wpc))

    def __enter__(self):
        _check(lib().pl_debug_set_route(*self.args))
        return self

    def __exit__(self, *a):
        lib().pl_debug_set_route(0, 0, 0)


class precision_policy:
    """Context manager for ``pl_set_precision_policy``: ``"auto"`` (default:
    calls whose h is below ``fast_h_threshold()``/255 of the data range run in
    double on the device) or ``"fast"`` (always the fp32 kernels)."""

    def __init__(self, policy: str):
        self.policy = {"auto": PL_PRECISION_AUTO, "fast": PL_PRECISION_FAST}[policy]

    def __enter__(self):
        self.prev = lib().pl_precision_policy()
        _check(lib().pl_set_precision_policy(self.policy))
        return self

    def __exit__(self, *a):
        _check(lib().pl_set_precision_policy(self.prev))
        return False


def fast_h_threshold() -> float:
    """h (per 255 of data range) from which the fp32 kernels are used unconditionally."""
    return float(lib().pl_fast_h_threshold())


def last_route() -> str:
    """Kernel route of the last pass launched on this thread (diagnostic)."""
    return (lib().pl_last_route() or b"").decode()


# ---------------------------------------------------------------------------
# host-side helpers (no device)
def validate_params(p, n: int) -> None:
    _check(lib().pl_validate_params(_params(p), int(n)))


def validate_geometry(S: int, K: int, n: int) -> None:
    _check(lib().pl_validate_geometry(int(S), int(K), int(n)))


def op_counts_1d(n: int, p) -> dict:
    o = _OpCounts(0, 0, 0, 0)
    _check(lib().pl_op_counts_1d(int(n), _params(p), C.byref(o)))
    return {"adds": o.adds, "muls": o.muls, "exps": o.exps, "clamps": o.clamps}


def unique_pairs(n: int, S: int) -> int:
    return int(lib().pl_unique_pairs(int(n), int(S)))


def segment_length(n: int, S: int) -> int:
    return int(lib().pl_segment_length(int(n), int(S)))


def weight_coef(h: float) -> float:
    """c = -log2(e)/h^2 as the device uses it (w = 2^(c d))."""
    return -1.4426950408889634 / (h * h)


# ---------------------------------------------------------------------------
# device filters over torch CUDA tensors (float32, contiguous)
def _image_dims(x):
    if x.dim() == 2:
        return 1, x.shape[0], x.shape[1]
    if x.dim() == 3:
        return x.shape[0], x.shape[1], x.shape[2]
    raise ValueError("expected [rows, cols] or [batch, rows, cols]")


def nlm_1d_patchlift(x, p, out=None):
    """1D PatchLift NLM on every line of ``x`` ([n] or [lines, n])."""
    import torch
    _dev(x, torch.float32)
    n = x.shape[-1]
    lines = x.numel() // n if n else 0
    out = _out(out, x)
    _check(lib().pl_nlm_lines(x.data_ptr(), out.data_ptr(), lines, n, n, _params(p), _stream(x)))
    return out


def nlm_1d_naive(x, p, out=None):
    import torch
    _dev(x, torch.float32)
    n = x.shape[-1]
    out = _out(out, x)
    _check(lib().pl_nlm_lines_naive(x.data_ptr(), out.data_ptr(), x.numel() // n, n, n,
                                    _params(p), _stream(x)))
    return out


def _image_op(name, x, p, out=None, work=None):
    import torch
    _dev(x, torch.float32)
    b, r, c = _image_dims(x)
    out = _out(out, x)
    if work is not None:
        _dev(work, torch.float32)
        op = {"pl_snlm_2d_row_col": 0, "pl_snlm_2d_col_row": 1, "pl_snlm_2d": 2}[name]
        if work.numel() * 4 < workspace_bytes(op, b, r, c) or work.device != x.device:
            raise ValueError("work is smaller than pl_workspace_bytes or on another device")
    fn = getattr(lib(), name)
    if name in ("pl_nlm_row_pass", "pl_nlm_col_pass", "pl_nlm_2d_naive"):
        rc = fn(x.data_ptr(), out.data_ptr(), b, r, c, _params(p), _stream(x))
    else:
        rc = fn(x.data_ptr(), out.data_ptr(), None if work is None else work.data_ptr(), b, r, c,
                _params(p), _stream(x))
    _check(rc)
    return out


def nlm_row_pass(x, p, out=None):
    return _image_op("pl_nlm_row_pass", x, p, out)


def nlm_col_pass(x, p, out=None):
    return _image_op("pl_nlm_col_pass", x, p, out)


def snlm_2d_row_col(x, p, out=None, work=None):
    return _image_op("pl_snlm_2d_row_col", x, p, out, work)


def snlm_2d_col_row(x, p, out=None, work=None):
    return _image_op("pl_snlm_2d_col_row", x, p, out, work)


def snlm_2d(x, p, out=None, work=None):
    return _image_op("pl_snlm_2d", x, p, out, work)


def nlm_2d_naive(x, p, out=None):
    return _image_op("pl_nlm_2d_naive", x, p, out)


def nlm_row_pass_blocked(x, p, col_block: int, out=None):
    """Row pass writing [col_block]-wide column blocks (the all-to-all send layout)."""
    import torch
    _dev(x, torch.float32)
    b, r, c = _image_dims(x)
    out = _out(out, x)
    _check(lib().pl_nlm_row_pass_blocked(x.data_ptr(), out.data_ptr(), b, r, c, int(col_block),
                                         _params(p), _stream(x)))
    return out


def nlm_row_pass_fanout(x, p, out=None, extras=()):
    """Row pass of one image [rows, cols] that also stores output rows
    [lo, hi) into each extra destination as it produces them.

    ``extras``: up to PL_MAX_FANOUT (dst, lo, hi); dst is a device pointer
    (int) or a tensor of >= (hi - lo) * cols floats, row pitch cols -- e.g. a
    peer GPU's window buffer (torch symmetric memory): the fused halo
    exchange of the row-partitioned multi-GPU path."""
    import torch
    _dev(x, torch.float32)
    if x.dim() != 2:
        raise ValueError("expected one image [rows, cols]")
    r, c = x.shape
    out = _out(out, x)
    n = len(extras)
    ptrs = (C.c_void_p * max(1, n))(*[e[0] if isinstance(e[0], int) else e[0].data_ptr()
                                      for e in extras])
    lo = (C.c_int32 * max(1, n))(*[int(e[1]) for e in extras])
    hi = (C.c_int32 * max(1, n))(*[int(e[2]) for e in extras])
    _check(lib().pl_nlm_row_pass_fanout(x.data_ptr(), out.data_ptr(), r, c, _params(p), n, ptrs,
                                        lo, hi, _stream(x)))
    return out


def col_window(rows_total: int, seg_begin: int, seg_end: int, p):
    """(in_lo, in_hi, out_lo, out_hi): input rows the windowed column pass over
    segments [seg_begin, seg_end) reads, and the output rows it produces."""
    v = [C.c_int32() for _ in range(4)]
    _check(lib().pl_col_window(int(rows_total), int(seg_begin), int(seg_end), _params(p),
                               *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def col_segments(rows_total: int, p) -> int:
    """Number of column-pass segments of a rows_total-row image."""
    S = min(int(_params(p).search_radius), rows_total - 1)
    C_ = segment_length(rows_total, S)
    return (rows_total + C_ - 1) // C_


def nlm_col_pass_window(x_win, in_lo: int, rows_total: int, seg_begin: int, seg_end: int, p,
                        out=None):
    """Column pass of segments [seg_begin, seg_end) from input rows
    [in_lo, in_lo + x_win.shape[-2]); returns rows [out_lo, out_hi)."""
    import torch
    _dev(x_win, torch.float32)
    b, r, c = _image_dims(x_win)
    _, _, out_lo, out_hi = col_window(rows_total, seg_begin, seg_end, p)
    shape = (out_hi - out_lo, c) if x_win.dim() == 2 else (b, out_hi - out_lo, c)
    out = _out(out, x_win, shape)
    _check(lib().pl_nlm_col_pass_window(x_win.data_ptr(), int(in_lo), r, out.data_ptr(), b,
                                        int(rows_total), c, int(seg_begin), int(seg_end),
                                        _params(p), _stream(x_win)))
    return out


def nlm_pass_strided(src, dst, batch: int, lines: int, n: int, src_line_stride: int,
                     src_pos_stride: int, dst_line_stride: int, dst_pos_stride: int,
                     img_stride: int, p):
    """One pass over arbitrarily strided lines of device tensors (see plgpu.h)."""
    import torch
    _dev(src, torch.float32)
    _dev(dst, torch.float32)
    if dst.device != src.device:
        raise ValueError("src and dst on different devices")
    # the last element each side addresses must lie inside the tensor
    last_pos = int(batch - 1) * int(img_stride) + (int(n) - 1)
    if (last_pos + (int(lines) - 1) * int(src_line_stride) + (int(n) - 1) * (int(src_pos_stride) - 1)
            >= src.numel() or
            last_pos + (int(lines) - 1) * int(dst_line_stride) + (int(n) - 1) * (int(dst_pos_stride) - 1)
            >= dst.numel()):
        raise ValueError("strides address past the end of src or dst")
    _check(lib().pl_nlm_pass_strided(src.data_ptr(), dst.data_ptr(), int(batch), int(lines), int(n),
                                     int(src_line_stride), int(src_pos_stride),
                                     int(dst_line_stride), int(dst_pos_stride), int(img_stride),
                                     _params(p), _stream(src)))
    return dst


def workspace_bytes(op: int, batch: int, rows: int, cols: int) -> int:
    return int(lib().pl_workspace_bytes(op, batch, rows, cols))


def filter_f64(op: str, x, p):
    """The fp64 reference-precision route on a float64 device tensor: op in
    lines, lines_naive (x [..., n]), row, col, rc, cr, snlm, nlm2d (x [rows,
    cols] or [batch, rows, cols])."""
    import torch
    _dev(x, torch.float64)
    out = torch.empty_like(x)
    L = lib()
    if op in ("lines", "lines_naive"):
        n = x.shape[-1]
        fn = L.pl_nlm_lines_f64 if op == "lines" else L.pl_nlm_lines_naive_f64
        _check(fn(x.data_ptr(), out.data_ptr(), x.numel() // n, n, n, _params(p), _stream(x)))
        return out
    b, r, c = _image_dims(x)
    if op in ("rc", "cr", "snlm"):
        fn = {"rc": L.pl_snlm_2d_row_col_f64, "cr": L.pl_snlm_2d_col_row_f64,
              "snlm": L.pl_snlm_2d_f64}[op]
        _check(fn(x.data_ptr(), out.data_ptr(), None, b, r, c, _params(p), _stream(x)))
    else:
        fn = {"row": L.pl_nlm_row_pass_f64, "col": L.pl_nlm_col_pass_f64,
              "nlm2d": L.pl_nlm_2d_naive_f64}[op]
        _check(fn(x.data_ptr(), out.data_ptr(), b, r, c, _params(p), _stream(x)))
    return out


class RCGraph:
    """pl_snlm_2d_row_col captured as a CUDA Graph on fixed device buffers x ->
    out; ``launch()`` replays both passes with one launch on the current
    stream."""

    def __init__(self, x, p, out=None):
        import torch
        _dev(x, torch.float32)
        b, r, c = _image_dims(x)
        self.x, self.out = x, _out(out, x)
        h = C.c_void_p()
        _check(lib().pl_graph_rc_create(x.data_ptr(), self.out.data_ptr(), None, b, r, c,
                                        _params(p), C.byref(h)))
        self._h = h

    def launch(self):
        _check(lib().pl_graph_launch(self._h, _stream(self.x)))
        return self.out

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.pl_graph_destroy(self._h)
            self._h = None


def snlm_2d_row_col_host(x_host, p, out_host=None):
    """End-to-end RC over HOST float32 arrays/tensors (copies inside)."""
    import numpy as np
    import torch
    if isinstance(x_host, torch.Tensor):
        assert not x_host.is_cuda and x_host.dtype == torch.float32 and x_host.is_contiguous()
        src = x_host.data_ptr()
        out_host = torch.empty_like(x_host) if out_host is None else out_host
        dst = out_host.data_ptr()
        shape = tuple(x_host.shape)
    else:
        x_host = np.ascontiguousarray(x_host, dtype=np.float32)
        out_host = np.empty_like(x_host) if out_host is None else out_host
        src, dst, shape = x_host.ctypes.data, out_host.ctypes.data, x_host.shape
    b, r, c = (1,) + shape if len(shape) == 2 else shape
    stream = torch.cuda.current_stream().cuda_stream
    _check(lib().pl_snlm_2d_row_col_host(src, dst, b, r, c, _params(p), stream))
    return out_host


def distance_band(x, S: int, K: int, dtype=None):
    """Distance band [lines, n, 2S+1] (NaN / -1 outside the line), int32 or fp32."""
    import torch
    _dev(x, torch.float32)
    dtype = dtype or torch.float32
    n = x.shape[-1]
    lines = x.numel() // n
    band = torch.empty((lines, n, 2 * S + 1), dtype=dtype, device=x.device)
    fn = lib().pl_distance_band_i32 if dtype == torch.int32 else lib().pl_distance_band_f32
    _check(fn(x.data_ptr(), band.data_ptr(), lines, n, n, int(S), int(K), _stream(x)))
    return band


def debug_hot_distance_band(x, S: int, K: int):
    """Distances the HOT filter kernel computes (prescale 1) for the lines of
    x ([lines, n], >= 16 lines, hot (K, S)): [lines, n, 2S+1] fp32, NaN where
    not written (diagonal included).  Exact on integer-valued inputs."""
    import torch
    _dev(x, torch.float32)
    lines, n = x.shape
    band = torch.empty((lines, n, 2 * S + 1), dtype=torch.float32, device=x.device)
    _check(lib().pl_debug_hot_distance_band(x.data_ptr(), band.data_ptr(), lines, n, int(S),
                                            int(K), _stream(x)))
    return band


def banded_kernel_f64(x, S: int, K: int):
    """F-bar band [lines, n, 2S+1] in fp64 (compute_banded_kernel)."""
    import torch
    _dev(x, torch.float64)
    n = x.shape[-1]
    lines = x.numel() // n
    band = torch.empty((lines, n, 2 * S + 1), dtype=torch.float64, device=x.device)
    _check(lib().pl_banded_kernel_f64(x.data_ptr(), band.data_ptr(), lines, n, n, int(S), int(K),
                                      _stream(x)))
    return band


def image_metrics(a, b):
    """(mse, psnr_db, ssim) per image pair of device tensors [rows, cols] or
    [batch, rows, cols] (float32 or float64): a [batch, 3] float64 tensor."""
    import torch
    _dev(a)
    _dev(b, a.dtype)
    if a.shape != b.shape:
        raise ValidationError("image dimensions do not match")
    bt, r, c = _image_dims(a)
    out = torch.empty((bt, 3), dtype=torch.float64, device=a.device)
    fn = {torch.float32: lib().pl_image_metrics_f32,
          torch.float64: lib().pl_image_metrics_f64}.get(a.dtype)
    if fn is None:
        raise TypeError("expected float32 or float64 images")
    _check(fn(a.data_ptr(), b.data_ptr(), bt, r, c, out.data_ptr(), _stream(a)))
    return out


def h_for(sigma: float, K: int) -> float:
    """The configs' rule h = sqrt(2(2K+1)) * sigma."""
    return math.sqrt(2 * (2 * K + 1)) * sigma

"""Parity checkers -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and its ``--impl reference`` arm) may import this
package.  The product path (``paper_1407_2343_b200``) never does.

Two checkers share one numpy-facing API:

* :class:`Oracle` -- ``_build/liboracle.so``, my plain-C restatement of the
  reference algorithm (``patchlift_oracle.c``; each function cites the
  reference file:line it follows).
* :class:`Reference` -- ``_ref/libpatchlift_ref.so``, the unmodified reference
  sources compiled in place by ``oracle/Makefile`` behind ``ref_shim.cpp``.
  It exists wherever it was built (here, and on the GPU box because built
  files travel with the gpurun snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpatchlift_ref.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)

FILTER_OPS = {"row": 0, "col": 1, "rc": 2, "cr": 3, "snlm": 4, "nlm2d": 5}


class OracleError(Exception):
    """Raised with the checker's status code (1 validation, 2 out-of-range)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(with_reference: bool | None = None) -> None:
    """Compile the checkers (``make -C oracle``).  The reference build runs
    only where ``/root/reference`` exists (this container)."""
    targets = ["oracle"]
    if with_reference is None:
        with_reference = os.path.isdir(REF_SRC)
    if with_reference:
        targets += ["ref", "acceptance"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class _Base:
    _prefix = ""
    _lock = threading.Lock()

    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = getattr(self.lib, self._prefix + "last_error")()
            raise OracleError(rc, msg.decode() if msg else "")


def _metrics(obj, fn, a, b):
    a, b = _f64(a), _f64(b)
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError("expected two images of equal [rows, cols] shape")
    out = np.empty(3)
    obj._check(fn(_ptr(a), _ptr(b), C.c_int(a.shape[0]), C.c_int(a.shape[1]), _ptr(out)))
    return float(out[0]), float(out[1]), float(out[2])


class Oracle(_Base):
    """My C restatement (double precision)."""

    _prefix = "orc_"
    _inst = None

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(with_reference=False)
        lib = C.CDLL(path)
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_weight.restype = C.c_double
        lib.orc_weight.argtypes = [C.c_double, C.c_double]
        self.lib = lib

    @classmethod
    def get(cls) -> "Oracle":
        with cls._lock:
            if cls._inst is None:
                cls._inst = cls()
            return cls._inst

    # -- validation ---------------------------------------------------------
    def validate_params(self, S, K, h, n) -> None:
        self._check(self.lib.orc_validate_params(C.c_int(S), C.c_int(K), C.c_double(h), C.c_int(n)))

    def validate_geometry(self, S, K, n) -> None:
        self._check(self.lib.orc_validate_geometry(C.c_int(S), C.c_int(K), C.c_int(n)))

    # -- 1D -------------------------------------------------------------------
    def extend_symmetric(self, f, pad):
        f = _f64(f)
        out = np.empty(f.size + 2 * max(pad, 0))
        self._check(self.lib.orc_extend_symmetric(_ptr(f), C.c_int(f.size), C.c_int(pad), _ptr(out)))
        return out

    def banded_kernel(self, f, S, K):
        f = _f64(f)
        band = np.empty((f.size, 2 * S + 1))
        adds, muls = C.c_uint64(0), C.c_uint64(0)
        self._check(self.lib.orc_banded_kernel(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                               _ptr(band), C.byref(adds), C.byref(muls)))
        return band, (adds.value, muls.value)

    def distance_band(self, f, S, K):
        f = _f64(f)
        band = np.empty((f.size, 2 * S + 1))
        clamps = C.c_uint64(0)
        self._check(self.lib.orc_distance_band(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                               _ptr(band), C.byref(clamps)))
        return band

    def distance_band_direct(self, f, S, K):
        f = _f64(f)
        band = np.empty((f.size, 2 * S + 1))
        self._check(self.lib.orc_distance_band_direct(_ptr(f), C.c_int(f.size), C.c_int(S),
                                                      C.c_int(K), _ptr(band)))
        return band

    def patch_distance(self, f, i, j, K):
        f = _f64(f)
        out = C.c_double(0)
        self._check(self.lib.orc_patch_distance(_ptr(f), C.c_int(f.size), C.c_int(i), C.c_int(j),
                                                C.c_int(K), C.byref(out)))
        return out.value

    def weight(self, rho_sq, h):
        return self.lib.orc_weight(rho_sq, h)

    def metrics(self, a, b):
        """(mse, psnr_db, ssim) of two [rows, cols] images (metrics.cpp:98-158)."""
        return _metrics(self, getattr(self.lib, self._prefix + "metrics"), a, b)

    def nlm_1d(self, f, S, K, h, naive=False, ops=None):
        f = _f64(f)
        out = np.empty_like(f)
        o4 = (C.c_uint64 * 4)()
        fn = self.lib.orc_nlm_1d_naive if naive else self.lib.orc_nlm_1d_patchlift
        self._check(fn(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K), C.c_double(h), _ptr(out),
                       C.cast(o4, _u64p)))
        if ops is not None:
            ops[:] = list(o4)
        return out

    # -- 2D -------------------------------------------------------------------
    def row_pass(self, img, S, K, h, threads: int = 1):
        img = _f64(img)
        rows, cols = img.shape
        out = np.empty_like(img)
        self.validate_params(S, K, h, cols)
        bounds = np.linspace(0, rows, max(1, min(threads, rows)) + 1).astype(int)

        def run(a, b):
            self._check(self.lib.orc_row_pass_rows(_ptr(img), rows, cols, S, K, C.c_double(h),
                                                   int(a), int(b), _ptr(out), None))

        if len(bounds) == 2:
            run(0, rows)
        else:  # ctypes drops the GIL; row ranges are independent (nlm.cpp:13-17)
            with ThreadPoolExecutor(len(bounds) - 1) as ex:
                list(ex.map(lambda ab: run(*ab), zip(bounds[:-1], bounds[1:])))
        return out

    def col_pass(self, img, S, K, h, threads: int = 1):
        return np.ascontiguousarray(self.row_pass(_f64(img).T, S, K, h, threads).T)

    def snlm_rc(self, img, S, K, h, threads: int = 1):
        img = _f64(img)
        self.validate_params(S, K, h, img.shape[0])
        self.validate_params(S, K, h, img.shape[1])
        return self.col_pass(self.row_pass(img, S, K, h, threads), S, K, h, threads)

    def snlm_cr(self, img, S, K, h, threads: int = 1):
        img = _f64(img)
        self.validate_params(S, K, h, img.shape[0])
        self.validate_params(S, K, h, img.shape[1])
        return self.row_pass(self.col_pass(img, S, K, h, threads), S, K, h, threads)

    def snlm(self, img, S, K, h, threads: int = 1):
        return (self.snlm_rc(img, S, K, h, threads) + self.snlm_cr(img, S, K, h, threads)) / 2.0

    def filter(self, op: str, img, S, K, h, threads: int = 1):
        return {"row": self.row_pass, "col": self.col_pass, "rc": self.snlm_rc,
                "cr": self.snlm_cr, "snlm": self.snlm}[op](img, S, K, h, threads)


class Reference(_Base):
    """The reference library itself (oracle/_ref), through ref_shim.cpp."""

    _prefix = "ref_"
    _inst = None

    def __init__(self, path: str = REF_SO):
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_weight.restype = C.c_double
        lib.ref_weight.argtypes = [C.c_double, C.c_double]
        self.lib = lib

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def get(cls) -> "Reference":
        with cls._lock:
            if cls._inst is None:
                cls._inst = cls()
            return cls._inst

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def extend_symmetric(self, f, pad):
        f = _f64(f)
        out = np.empty(f.size + 2 * max(pad, 0))
        self._check(self.lib.ref_extend_symmetric(_ptr(f), C.c_int(f.size), C.c_int(pad), _ptr(out)))
        return out

    def banded_kernel(self, f, S, K):
        f = _f64(f)
        band = np.empty((f.size, 2 * S + 1))
        o4 = (C.c_uint64 * 4)()
        self._check(self.lib.ref_banded_kernel(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                               _ptr(band), C.cast(o4, _u64p)))
        return band, (o4[0], o4[1])

    def distance_band(self, f, S, K):
        f = _f64(f)
        band = np.empty((f.size, 2 * S + 1))
        clamps = C.c_uint64(0)
        self._check(self.lib.ref_distance_band(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                               _ptr(band), C.byref(clamps)))
        return band

    def patch_distance(self, f, i, j, K):
        f = _f64(f)
        out = C.c_double(0)
        self._check(self.lib.ref_patch_distance(_ptr(f), C.c_int(f.size), C.c_int(i), C.c_int(j),
                                                C.c_int(K), C.byref(out)))
        return out.value

    def weight(self, rho_sq, h):
        return self.lib.ref_weight(rho_sq, h)

    def metrics(self, a, b):
        """(mse, psnr_db, ssim) of two [rows, cols] images (metrics.cpp:98-158)."""
        return _metrics(self, getattr(self.lib, self._prefix + "metrics"), a, b)

    def nlm_1d(self, f, S, K, h, naive=False, ops=None):
        f = _f64(f)
        out = np.empty_like(f)
        o4 = (C.c_uint64 * 4)()
        self._check(self.lib.ref_nlm_1d(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                        C.c_double(h), C.c_int(1 if naive else 0), _ptr(out),
                                        C.cast(o4, _u64p)))
        if ops is not None:
            ops[:] = list(o4)
        return out

    def filter(self, op: str, img, S, K, h, threads: int = 1, ops=None):
        img = _f64(img)
        rows, cols = img.shape
        out = np.empty_like(img)
        o4 = (C.c_uint64 * 4)()
        self._check(self.lib.ref_image_filter(C.c_int(FILTER_OPS[op]), _ptr(img), C.c_int(rows),
                                              C.c_int(cols), C.c_int(S), C.c_int(K), C.c_double(h),
                                              C.c_int(threads), _ptr(out),
                                              C.cast(o4, _u64p) if ops is not None else None))
        if ops is not None:
            ops[:] = list(o4)
        return out

    def dump_kernel_csv(self, f, S, K) -> str:
        f = _f64(f)
        need = C.c_size_t(0)
        self._check(self.lib.ref_dump_kernel_csv(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                                 None, C.c_size_t(0), C.byref(need)))
        buf = C.create_string_buffer(need.value + 1)
        self._check(self.lib.ref_dump_kernel_csv(_ptr(f), C.c_int(f.size), C.c_int(S), C.c_int(K),
                                                 buf, C.c_size_t(need.value + 1), C.byref(need)))
        return buf.value.decode()

"""C-ABI boundary checks that need no GPU: the libraries load, export every
symbol their headers declare, and the host-side logic (validation with the
reference's messages, op-count closed forms, pair counts) is right."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1407_2343_b200 as pl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "plgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pl_[a-z0-9_]+)\s*\(", text)))


def dynsyms(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_lib_exports_every_header_symbol():
    syms = dynsyms(pl.LIBPLGPU)
    declared = header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if s not in syms]
    assert not missing, missing
    assert sorted(pl.EXPORTS) == declared


def test_dropin_exports_reference_api():
    syms = dynsyms(pl.LIBDROPIN)
    demangled = subprocess.run(["c++filt"], input="\n".join(sorted(syms)), capture_output=True,
                               text=True).stdout
    for fn in ["patchlift::snlm_2d_row_col(", "patchlift::snlm_2d_col_row(", "patchlift::snlm_2d(",
               "patchlift::nlm_row_pass(", "patchlift::nlm_col_pass(", "patchlift::nlm_1d_patchlift(",
               "patchlift::nlm_1d_naive(", "patchlift::nlm_2d_naive(",
               "patchlift::compute_banded_kernel(", "patchlift::kernel_distance_sq(",
               "patchlift::patch_distance_sq_naive(", "patchlift::dump_kernel_csv(",
               "patchlift::extend_symmetric(", "patchlift::transpose(", "patchlift::validate_params(",
               "patchlift::validate_geometry(", "patchlift::weight(", "patchlift::lift_value(",
               "patchlift::Signal1D::Signal1D(", "patchlift::Image2D::Image2D(",
               "patchlift::BandedKernel::at(", "patchlift::mse(", "patchlift::psnr(",
               "patchlift::ssim(", "patchlift::compare_images(", "patchlift::add_awgn(",
               "patchlift::MetricReport::to_line"]:
        assert fn in demangled, fn


def test_abi_version_and_geometry():
    assert pl.lib().pl_abi_version() == 1
    for n in (1, 5, 127, 128, 129, 4096, 65536):
        C = pl.segment_length(n, 10)
        assert 1 <= C <= n


def test_validation_messages_match_reference():
    cases = [((-1, 0, 1.0), 8, "search radius must be nonnegative"),
             ((0, -1, 1.0), 8, "patch radius must be nonnegative"),
             ((0, 9, 1.0), 8, "patch radius exceeds signal length"),
             ((1, 1, 0.0), 8, "smoothing parameter h must be positive"),
             ((1, 1, -2.0), 8, "smoothing parameter h must be positive"),
             ((1, 1, 1.0), 0, "signal length must be at least 1")]
    for p, n, msg in cases:
        with pytest.raises(pl.ValidationError, match=msg):
            pl.validate_params(p, n)
    pl.validate_params((0, 0, 1.0), 1)
    pl.validate_geometry(100, 8, 8)


def test_op_counts_match_reference(ref):
    rng = np.random.default_rng(29)
    for _ in range(30):
        n = int(rng.integers(1, 150))
        S = int(rng.integers(0, 20))
        K = int(rng.integers(0, min(n, 6) + 1))
        ops = [0] * 4
        ref.nlm_1d(rng.uniform(0, 255, n), S, K, 40.0, ops=ops)
        got = pl.op_counts_1d(n, (S, K, 40.0))
        assert [got["adds"], got["muls"], got["exps"]] == ops[:3]


def test_op_counts_image_match_reference(ref):
    img = np.random.default_rng(30).uniform(0, 255, (23, 17))
    ops = [0] * 4
    ref.filter("snlm", img, 4, 1, 35.0, ops=ops)
    row = pl.op_counts_1d(17, (4, 1, 35.0))
    col = pl.op_counts_1d(23, (4, 1, 35.0))
    for k, key in enumerate(["adds", "muls", "exps"]):
        assert ops[k] == 2 * (23 * row[key] + 17 * col[key])


def test_unique_pairs():
    assert pl.unique_pairs(65536, 10) == 655305
    assert 4096 * pl.unique_pairs(4096, 15) * 2 == 502333440  # c3 RC
    assert pl.unique_pairs(5, 99) == 10
    assert pl.unique_pairs(1, 3) == 0


def test_product_has_no_oracle_dependency():
    """The product package must never import or link the checkers."""
    pkg = os.path.join(ROOT, "paper_1407_2343_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "patchlift_ref" not in text, f
    for so in (pl.LIBPLGPU, pl.LIBDROPIN):
        needed = subprocess.run(["readelf", "-d", so], capture_output=True, text=True).stdout
        assert "oracle" not in needed and "patchlift_ref" not in needed


def test_bench_reference_arm_runs_on_cpu(tmp_path):
    """`bench.py --impl reference` needs no GPU: it times the reference library
    (oracle/_ref) on host cores and prints the contract's JSON line."""
    import json
    import sys
    from oracle import Reference
    if not Reference.available():
        pytest.skip("reference library not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "c2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["unit"] == "Mpixel/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_precision_policy_api_host_only():
    """pl_set_precision_policy / pl_precision_policy / pl_fast_h_threshold touch
    no device: default AUTO, FAST round-trips, anything else is PL_ERR_ARG."""
    L = pl.lib()
    assert L.pl_precision_policy() == pl.PL_PRECISION_AUTO
    assert L.pl_fast_h_threshold() == 48.0
    with pl.precision_policy("fast"):
        assert L.pl_precision_policy() == pl.PL_PRECISION_FAST
    assert L.pl_precision_policy() == pl.PL_PRECISION_AUTO
    assert L.pl_set_precision_policy(7) == pl.PL_ERR_ARG
    assert b"precision policy" in L.pl_last_error()
    assert L.pl_debug_set_route(3, 0, 0) == pl.PL_OK  # walker 3: 1D lines never folded
    assert L.pl_debug_set_route(4, 0, 0) == pl.PL_ERR_ARG
    assert L.pl_debug_set_route(0, 0, 0) == pl.PL_OK

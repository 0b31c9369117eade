/* plgpu.h -- C ABI of the B200 PatchLift separable-NLM hot path.
 *
 * The reference (arXiv 1407.2343 artifact, C++20 library `patchlift`) has no
 * FFI; its boundary is the C++ function API in proj/include/patchlift/.  This
 * header is the flat, exception-free face of that API over DEVICE fp32
 * buffers, one entry point per reference function it replaces:
 *
 *   pl_nlm_lines           nlm_1d_patchlift            nlm.hpp:30, nlm.cpp:144-166
 *   pl_nlm_row_pass        nlm_row_pass                nlm.hpp:39-40, nlm.cpp:215-227
 *   pl_nlm_col_pass        nlm_col_pass                nlm.hpp:41-42, nlm.cpp:229-232
 *   pl_nlm_col_pass_window nlm_col_pass on a row window (multi-GPU halo form of the same)
 *   pl_nlm_row_pass_fanout nlm_row_pass + fused halo stores into peers' windows (multi-GPU)
 *   pl_snlm_2d_row_col     snlm_2d_row_col             nlm.hpp:45-46, nlm.cpp:234-239
 *   pl_snlm_2d_col_row     snlm_2d_col_row             nlm.hpp:47-48, nlm.cpp:241-246
 *   pl_snlm_2d             snlm_2d (RC+CR)/2           nlm.hpp:51-52, nlm.cpp:248-253
 *   pl_distance_band_f32   compute_banded_kernel + kernel_distance_sq over the
 *   pl_distance_band_i32     band (BandedKernel cell layout)  banded_kernel.cpp:25-84
 *   pl_banded_kernel_f64   compute_banded_kernel (F-bar values)  banded_kernel.cpp:25-72
 *   pl_nlm_lines_naive     nlm_1d_naive (direct O(K) distances)  nlm.cpp:120-142
 *   pl_validate_params     validate_params             core_types.cpp:49-69
 *   pl_op_counts_1d        OpCounter closed forms      nlm.cpp:154-164, banded_kernel.cpp:49-66
 *
 * Conventions
 *  - Buffers are caller-owned device pointers (fp32 unless stated); images
 *    are batches of row-major [batch][rows][cols] planes.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and returns immediately; re-entrant: concurrent calls on
 *    different streams or host threads share no device state (library
 *    scratch is allocated per call, stream-ordered, from a per-device pool).
 *  - Return value: PL_OK or an error code; the message of the last failure on
 *    the calling thread is pl_last_error().  Validation failures reuse the
 *    reference's exact ValidationError messages (core_types.cpp:13-77).
 *  - Boundary convention: half-sample mirror for patch content
 *    (core_types.cpp:71-88), search windows clipped to the line
 *    (nlm.cpp:71-73).  S larger than line-1 behaves as line-1.
 *  - Arithmetic: fp32 (double for calls the precision policy routes there).
 *    Weights exp(-d/h^2) are ex2(-d') with d' the patch distance of samples
 *    prescaled by sqrt(log2 e)/h (computed in double on the host); quotients
 *    num/den by rcp, clamped into the range of the walked samples (constant
 *    inputs are exact fixpoints, outputs stay in the convex hull).  The distance-band exports are exact (bit-equal to
 *    the reference) on integer-valued inputs.
 *  - Results are bitwise independent of batch size, line count, GPU count and
 *    of which axis a line lies on (row and column passes run identical per-
 *    line arithmetic), so transpose equivariance holds bit for bit -- within
 *    one arithmetic route: under PL_PRECISION_AUTO a call with h < 48 picks
 *    fp32 or double from its own data range (pl_set_precision_policy below).
 */
#ifndef PLGPU_H_
#define PLGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLGPU_ABI_VERSION 1

enum pl_status {
  PL_OK = 0,
  PL_ERR_VALIDATION = 1, /* reference ValidationError (std::invalid_argument) */
  PL_ERR_RANGE = 2,      /* reference std::out_of_range */
  PL_ERR_CUDA = 3,       /* CUDA runtime / launch failure */
  PL_ERR_UNSUPPORTED = 4,
  PL_ERR_ARG = 5 /* null pointer or malformed descriptor */
};

/* NlmParams (core_types.hpp:45-49): S, K, h. */
typedef struct pl_params {
  int32_t search_radius;
  int32_t patch_radius;
  double h;
} pl_params;

/* OpCounter (op_counter.hpp:9-24). */
typedef struct pl_op_counts {
  uint64_t adds;
  uint64_t muls;
  uint64_t exps;
  uint64_t clamps;
} pl_op_counts;

int pl_abi_version(void);
const char* pl_last_error(void);
/* Diagnostic: the kernel route the last pass launched on the calling thread
 * ("hot<S=..,K=..,lines=..,io=..,wpc=..,avg=..>", "staged<...>",
 * "portable<...>", "direct", "none"); for composites, their last pass. */
const char* pl_last_route(void);
/* Debug / test hook: pin the kernel route process-wide.  walker 0 = default,
 * 1 = portable walker only, 2 = no hot-configuration kernel, 3 = default
 * walkers but few-line 1D calls are not folded onto lanes; lines 0/1/2 and
 * wpc 0/2/8 pin the hot kernel's lines per lane and warps per CTA (0 =
 * default).  Every route computes the same bits; this only selects code for
 * coverage and A/B timing.  (0, 0, 0) restores the defaults. */
int pl_debug_set_route(int32_t walker, int32_t lines, int32_t wpc);
/* Precision policy of the reference-API entry points (pl_nlm_lines,
 * pl_nlm_row_pass, pl_nlm_col_pass, pl_snlm_2d_row_col, pl_snlm_2d_col_row,
 * pl_snlm_2d, pl_snlm_2d_row_col_host).  The fp32 kernels hold the output
 * bound (max abs error 1e-3 on a [0, 255] scale against the reference's
 * double arithmetic) while h >= pl_fast_h_threshold() / 255 of the data range
 * (48: every setting of the configs).  PL_PRECISION_AUTO
 * (default): calls with h >= the threshold run the fp32 kernels directly;
 * below it the input's range is measured (one reduction, the call then
 * synchronises `stream`) and, if h is under threshold/255 of it, the call runs
 * in double on the device (fp32 in, fp64 arithmetic and intermediates, fp32
 * out: plgpu_walk64.cuh), slower but within the bound at any h.
 * PL_PRECISION_FAST: always the fp32 kernels.  Process-wide.  The partition-
 * level entry points (strided / blocked / window / fan-out passes, graphs)
 * are fp32 only: under PL_PRECISION_AUTO they return PL_ERR_UNSUPPORTED for
 * h below the threshold instead of silently exceeding the bound. */
enum pl_precision_policy { PL_PRECISION_AUTO = 0, PL_PRECISION_FAST = 1 };
int pl_set_precision_policy(int32_t policy);
int32_t pl_precision_policy(void);
double pl_fast_h_threshold(void);
/* Name of the device the library will launch on, or "" if none. */
const char* pl_device_name(void);

/* Host-only checks with the reference's messages; no device is touched. */
int pl_validate_params(pl_params p, int32_t n);
int pl_validate_geometry(int32_t search_radius, int32_t patch_radius, int32_t n);

/* Reference op-count closed forms for one 1D PatchLift filter of length n
 * (kernel build + 4 adds, 2 muls, 1 exp per ordered window; clamps 0 because
 * the squared-difference route is nonnegative by construction).  Added to
 * *out. */
int pl_op_counts_1d(int32_t n, pl_params p, pl_op_counts* out);

/* Unique in-band pairs U(n,S) = n*S' - S'(S'+1)/2, S' = min(S, n-1): the exps
 * the device evaluates per line (w_ij = w_ji, w_ii = 1). */
uint64_t pl_unique_pairs(int32_t n, int32_t search_radius);

/* Segment length the device uses for lines of length n (a function of n
 * only, so results never depend on the launch shape). */
int32_t pl_segment_length(int32_t n, int32_t search_radius);

/* ---- 1D: n_lines lines of n samples, line l starts at src + l*ld ----- */
int pl_nlm_lines(const float* src, float* dst, int64_t n_lines, int32_t n, int64_t ld,
                 pl_params p, void* stream);
int pl_nlm_lines_naive(const float* src, float* dst, int64_t n_lines, int32_t n, int64_t ld,
                       pl_params p, void* stream);

/* ---- 2D separable passes on [batch][rows][cols] ------------------------- */
int pl_nlm_row_pass(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream);
int pl_nlm_col_pass(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream);

/* Windowed column pass (row-partitioned multi-GPU, halo exchange; SURVEY.md
 * sec. 8(f)).  The column pass of an image with rows_total rows is cut into
 * segments of pl_segment_length(rows_total, min(S, rows_total-1)) rows; this
 * produces segments [seg_begin, seg_end), i.e. output rows [out_lo, out_hi),
 * bit-identical to the same rows of pl_nlm_col_pass on the whole image.
 *   pl_col_window: the input rows [in_lo, in_hi) the pass may read for that
 *     segment range (walker over-fetch included) and the output rows.
 *   pl_nlm_col_pass_window: src holds input rows [in_lo, in_lo + in_rows)
 *     (must cover pl_col_window's range), per image [in_rows][cols];
 *     dst holds output rows [out_lo, out_hi), per image [out_hi-out_lo][cols].
 *     Needs 1 <= min(S, rows_total-1) <= 32. */
int pl_col_window(int32_t rows_total, int32_t seg_begin, int32_t seg_end, pl_params p,
                  int32_t* in_lo, int32_t* in_hi, int32_t* out_lo, int32_t* out_hi);
int pl_nlm_col_pass_window(const float* src, int32_t in_lo, int32_t in_rows, float* dst,
                           int32_t batch, int32_t rows_total, int32_t cols, int32_t seg_begin,
                           int32_t seg_end, pl_params p, void* stream);

/* One pass over `lines` lines of n samples per image, any layout:
 * element (b, line, pos) of src at b*img_stride + line*src_line_stride +
 * pos*src_pos_stride, of dst likewise with the dst strides.  Row pass:
 * (cols, 1, cols, 1); column pass: (1, cols, 1, cols); the RC composite's
 * transposed intermediate: row pass (cols, 1, 1, rows) then column pass
 * (rows, 1, 1, cols) -- what pl_snlm_2d_row_col runs internally. */
int pl_nlm_pass_strided(const float* src, float* dst, int32_t batch, int32_t lines, int32_t n,
                        int64_t src_line_stride, int64_t src_pos_stride, int64_t dst_line_stride,
                        int64_t dst_pos_stride, int64_t img_stride, pl_params p, void* stream);

/* Row pass whose output is written in column blocks of width col_block:
 * element (b, r, c) lands at dst + b*rows*cols + (c / col_block)*rows*col_block
 * + r*col_block + (c % col_block).  With one image per rank this is exactly
 * the send layout of the row-slab -> column-slab all-to-all (cols must be a
 * multiple of col_block). */
int pl_nlm_row_pass_blocked(const float* src, float* dst, int32_t batch, int32_t rows,
                            int32_t cols, int32_t col_block, pl_params p, void* stream);

/* Row pass of ONE image whose output rows are also stored, as each tile is
 * flushed, into up to PL_MAX_FANOUT extra destinations: rows [lo[x], hi[x])
 * of the pass land at extra[x] + (r - lo[x]) * cols (row pitch cols).  With
 * extra[x] a peer GPU's buffer mapped into this process (CUDA IPC / torch
 * symmetric memory over NVLink), the halo exchange of the row-partitioned
 * multi-GPU S-NLM is fused into the row pass: the neighbours' halo rows are
 * written over NVLink by the same stores that write the local window, no
 * separate collective.  dst is bit-identical to pl_nlm_row_pass and every
 * extra row to the corresponding dst row.  Replaces the send/recv pair of the
 * halo exchange (no reference counterpart: nlm_col_pass's transpose,
 * core_types.cpp:90-98, is its single-node analogue). */
#define PL_MAX_FANOUT 2
int pl_nlm_row_pass_fanout(const float* src, float* dst, int32_t rows, int32_t cols, pl_params p,
                           int32_t n_extra, float* const* extra, const int32_t* lo, const int32_t* hi,
                           void* stream);

/* Bytes of device workspace the composites need (0 for single passes). */
size_t pl_workspace_bytes(int32_t op, int32_t batch, int32_t rows, int32_t cols);

/* Composites.  `work` is caller-provided device scratch of
 * pl_workspace_bytes(...) bytes, or NULL: the call then allocates its own
 * scratch on `stream` (cudaMallocFromPoolAsync from a per-device pool that
 * keeps its memory) and frees it in stream order after its last kernel. */
int pl_snlm_2d_row_col(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, void* stream);
int pl_snlm_2d_col_row(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, void* stream);
int pl_snlm_2d(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
               int32_t cols, pl_params p, void* stream);

/* End-to-end form of pl_snlm_2d_row_col over HOST buffers (pinned or
 * pageable): H2D copies, both passes and D2H copies are pipelined on `stream`
 * and two copy streams -- over groups of images for batches of small images,
 * and INSIDE the image for images of 32 MiB and more (rows go up in chunks,
 * each chunk's row pass runs as it lands, each block of whole column-pass
 * segments runs as soon as the rows it reads are there and its output rows go
 * down at once), so a single 16384^2 image moves at the PCIe full-duplex rate.
 * Results are bitwise those of pl_snlm_2d_row_col.  Blocks until done. */
int pl_snlm_2d_row_col_host(const float* host_src, float* host_dst, int32_t batch, int32_t rows,
                            int32_t cols, pl_params p, void* stream);

/* CUDA Graph of pl_snlm_2d_row_col on fixed buffers: both passes are captured
 * once (the intermediate is owned by the graph when `work` is NULL) and each
 * pl_graph_launch replays them with one launch on `stream`.  For repeated
 * calls on small images, where launch latency is the cost. */
typedef struct pl_graph pl_graph;
int pl_graph_rc_create(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, pl_graph** out);
int pl_graph_launch(pl_graph* graph, void* stream);
int pl_graph_destroy(pl_graph* graph);

/* ---- classical 2D NLM (nlm_2d_naive, nlm.cpp:168-213): the baseline the
 * separable filter is compared against (per-pixel (2S+1)^2 window, direct
 * (2K+1)^2 patch distances, 2D half-sample mirror).  Not the hot path. */
int pl_nlm_2d_naive(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream);

/* ---- fp64 reference-precision route (plgpu_walk64.cuh): the same filters on
 * device DOUBLE buffers, in double arithmetic with exp(-d/(h*h)) -- outputs
 * match the reference library (all-double, core_types.hpp:23,35) to rounding
 * rather than to the fp32 tiers.  The C++ drop-in uses this route by default.
 * `work` (or NULL for stream-ordered scratch) holds 2 * pl_workspace_bytes(op,
 * ...) bytes (doubles). */
int pl_nlm_lines_f64(const double* src, double* dst, int64_t n_lines, int32_t n, int64_t ld,
                     pl_params p, void* stream);
int pl_nlm_lines_naive_f64(const double* src, double* dst, int64_t n_lines, int32_t n, int64_t ld,
                           pl_params p, void* stream);
int pl_nlm_row_pass_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream);
int pl_nlm_col_pass_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream);
int pl_snlm_2d_row_col_f64(const double* src, double* dst, double* work, int32_t batch,
                           int32_t rows, int32_t cols, pl_params p, void* stream);
int pl_snlm_2d_col_row_f64(const double* src, double* dst, double* work, int32_t batch,
                           int32_t rows, int32_t cols, pl_params p, void* stream);
int pl_snlm_2d_f64(const double* src, double* dst, double* work, int32_t batch, int32_t rows,
                   int32_t cols, pl_params p, void* stream);
int pl_nlm_2d_naive_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream);

/* ---- device memory helpers so host layers need no CUDA runtime of their own */
int pl_device_alloc(void** ptr, size_t bytes);
int pl_device_free(void* ptr);
int pl_copy_to_device(void* dst, const void* src, size_t bytes);
int pl_copy_to_host(void* dst, const void* src, size_t bytes);
int pl_synchronize(void);
/* Pinned (page-locked) host staging memory, streams and stream-ordered
 * copies: what a host layer needs to keep a call's H2D, kernels and D2H on
 * one stream (the C++ drop-in's per-thread staging context). */
int pl_host_alloc(void** ptr, size_t bytes);
int pl_host_free(void* ptr);
int pl_stream_create(void** stream);
int pl_stream_destroy(void* stream);
int pl_stream_synchronize(void* stream);
int pl_copy_to_device_async(void* dst, const void* src, size_t bytes, void* stream);
int pl_copy_to_host_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---- distance / kernel bands (BandedKernel layout, banded_kernel.hpp:11-38)
 * band[l][i][o] for pair (i, i+o-S), o in [0, 2S+1); cells whose partner is
 * outside [0,n) hold the sentinel NaN (f32/f64) or -1 (i32). */
int pl_distance_band_f32(const float* src, float* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t search_radius, int32_t patch_radius, void* stream);
/* Integer distances; src must hold integer values (|x| <= 2^24 / ...).  The
 * device computes them exactly in the same running-sum recurrence as the
 * filter and converts to int32. */
int pl_distance_band_i32(const float* src, int32_t* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t search_radius, int32_t patch_radius, void* stream);
/* Debug: the distances the HOT filter kernel itself computes.  Runs the row
 * pass of n_lines lines of n samples (row-major, ld = n) through the hot
 * kernel's distance-export instantiation with the sample prescale set to 1,
 * so its running-sum recurrence works on the raw samples, and stores every
 * distance d(i, i+k) of the pixels it owns into band (layout as above, NaN
 * elsewhere, diagonal cells not written).  Exact (bit-equal to the
 * reference) on integer-valued inputs.  Needs n_lines >= 16 and a hot
 * (K, S) pair: (3, 10), (5, 15), (7, 25), with S <= n - 1. */
int pl_debug_hot_distance_band(const float* src, float* band, int32_t n_lines, int32_t n,
                               int32_t search_radius, int32_t patch_radius, void* stream);

/* F-bar cells of compute_banded_kernel in fp64, same diagonal recursion and
 * evaluation order as the reference (bit-equal to it). src is fp64. */
int pl_banded_kernel_f64(const double* src, double* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t search_radius, int32_t patch_radius, void* stream);

/* ---- fidelity metrics (metrics.cpp:98-158) ---
 * For each of `batch` image pairs [rows][cols] (device buffers, fp32 or fp64):
 * out[3*b + 0] = mse, out[3*b + 1] = psnr_db (+inf for identical images),
 * out[3*b + 2] = ssim (11x11 Gaussian window, sigma 1.5, valid positions).
 * `out` is a device buffer of 3*batch doubles.  Images smaller than 11x11
 * have no SSIM (the reference throws "image smaller than the 11x11
 * structural window"): their ssim is NaN, mse and psnr are still valid. */
int pl_image_metrics_f32(const float* a, const float* b, int32_t batch, int32_t rows, int32_t cols,
                         double* out, void* stream);
int pl_image_metrics_f64(const double* a, const double* b, int32_t batch, int32_t rows,
                         int32_t cols, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PLGPU_H_ */

/* oracle/patchlift_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (double precision) restatement of the reference PatchLift /
 * separable-NLM path, used as the parity CHECKER for the CUDA product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * it.  It is never called by the product library (paper_1407_2343_b200/),
 * which fails loudly when its CUDA library is missing.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference's proj/).  Arithmetic is written in the reference's evaluation
 * order and built with -ffp-contract=off (the reference build has no -march,
 * hence no FMA contraction), so on the same glibc the results are expected to
 * be BIT-IDENTICAL to the reference; tests/test_oracle.py pins that against
 * oracle/_ref (the reference itself) and tests/golden/ fixtures.
 *
 * Status codes: 0 ok, 1 validation error (reference ValidationError),
 * 2 out-of-range index (reference std::out_of_range).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local const char* g_err = "";

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

/* validate_geometry: core_types.cpp:49-62 (messages verbatim: they are the
 * reference's user-facing error contract). */
int orc_validate_geometry(int S, int K, int n) {
  if (n < 1) return fail(1, "signal length must be at least 1");
  if (S < 0) return fail(1, "search radius must be nonnegative");
  if (K < 0) return fail(1, "patch radius must be nonnegative");
  if (K > n) return fail(1, "patch radius exceeds signal length");
  return 0;
}

/* validate_params: core_types.cpp:64-69 */
int orc_validate_params(int S, int K, double h, int n) {
  int rc = orc_validate_geometry(S, K, n);
  if (rc) return rc;
  if (!(h > 0.0)) return fail(1, "smoothing parameter h must be positive");
  return 0;
}

/* extend_symmetric: core_types.cpp:71-88.  ext has n + 2*pad cells;
 * ext[pad + t] = f[t]; position -1-t mirrors t; position n+t mirrors n-1-t. */
int orc_extend_symmetric(const double* f, int n, int pad, double* ext) {
  if (pad < 0) return fail(1, "pad must be nonnegative");
  if (pad > n) return fail(1, "insufficient signal for symmetric extension");
  for (int t = 0; t < pad; ++t) {
    ext[pad - 1 - t] = f[t];
    ext[pad + n + t] = f[n - 1 - t];
  }
  for (int i = 0; i < n; ++i) ext[pad + i] = f[i];
  return 0;
}

/* compute_banded_kernel: banded_kernel.cpp:25-72.  band holds n*(2S+1) cells,
 * cell (i,o) <-> pair (i, i+o-S), NaN outside [0,n) (banded_kernel.hpp:11-15).
 * One direct (2K+1)-term sum starts each diagonal d, then the two-term
 * moving-sum recursion runs along it and the value is mirrored to (j,i). */
int orc_banded_kernel(const double* f, int n, int S, int K, double* band, uint64_t* adds_out,
                      uint64_t* muls_out) {
  int rc = orc_validate_geometry(S, K, n);
  if (rc) return rc;
  const int bw = 2 * S + 1;
  double* e = (double*)malloc(sizeof(double) * (size_t)(n + 2 * K));
  if (!e) return fail(3, "out of memory");
  orc_extend_symmetric(f, n, K, e);
  for (size_t c = 0; c < (size_t)n * bw; ++c) band[c] = NAN;
  uint64_t adds = 0, muls = 0;
  const int max_offset = S < n - 1 ? S : n - 1;
  for (int d = 0; d <= max_offset; ++d) {
    double sum = 0.0;
    for (int k = -K; k <= K; ++k) sum += e[k + K] * e[d + k + K];
    muls += (uint64_t)(2 * K + 1);
    adds += (uint64_t)(2 * K);
    band[(size_t)0 * bw + (d + S)] = sum;   /* slot(0, d) */
    band[(size_t)d * bw + (S - d)] = sum;   /* slot(d, 0) */
    const int len = n - d;
    for (int i = 1; i < len; ++i) {
      const int j = i + d;
      sum = sum + e[i + 2 * K] * e[j + 2 * K] - e[i - 1] * e[j - 1];
      band[(size_t)i * bw + (j - i + S)] = sum;
      band[(size_t)j * bw + (i - j + S)] = sum;
    }
    adds += 2 * (uint64_t)(len - 1);
    muls += 2 * (uint64_t)(len - 1);
  }
  free(e);
  if (adds_out) *adds_out += adds;
  if (muls_out) *muls_out += muls;
  return 0;
}

/* kernel_distance_sq: banded_kernel.cpp:74-84 (three band lookups, clamp <0). */
static double band_at(const double* band, int S, int i, int j) {
  return band[(size_t)i * (2 * S + 1) + (j - i + S)];
}

double orc_kernel_distance_sq(const double* band, int n, int S, int i, int j, uint64_t* clamps) {
  (void)n;
  const double d = band_at(band, S, i, i) + band_at(band, S, j, j) - 2.0 * band_at(band, S, i, j);
  if (d < 0.0) {
    if (clamps) ++*clamps;
    return 0.0;
  }
  return d;
}

/* Distance band (same cell layout) from the banded kernel: the distances the
 * reference's 1D PatchLift filter consumes (nlm.cpp:150-152). */
int orc_distance_band(const double* f, int n, int S, int K, double* dist, uint64_t* clamps) {
  const int bw = 2 * S + 1;
  double* band = (double*)malloc(sizeof(double) * (size_t)n * bw);
  if (!band) return fail(3, "out of memory");
  int rc = orc_banded_kernel(f, n, S, K, band, NULL, NULL);
  if (rc) {
    free(band);
    return rc;
  }
  for (int i = 0; i < n; ++i)
    for (int o = 0; o < bw; ++o) {
      const int j = i + o - S;
      dist[(size_t)i * bw + o] =
          (j < 0 || j >= n) ? NAN : orc_kernel_distance_sq(band, n, S, i, j, clamps);
    }
  free(band);
  return 0;
}

/* Direct O(K) distance, patch_distance_sq_naive: banded_kernel.cpp:86-108 and
 * its per-call extension (:95) hoisted out (patch_distance_sq_ext, nlm.cpp:56-63). */
static double dist_ext(const double* e, int i, int j, int K) {
  double acc = 0.0;
  for (int k = -K; k <= K; ++k) {
    const double diff = e[i + k + K] - e[j + k + K];
    acc += diff * diff;
  }
  return acc;
}

int orc_patch_distance(const double* f, int n, int i, int j, int K, double* out) {
  int rc = orc_validate_geometry(0, K, n);
  if (rc) return rc;
  if (i < 0 || i >= n || j < 0 || j >= n) return fail(2, "patch index out of range");
  double* e = (double*)malloc(sizeof(double) * (size_t)(n + 2 * K));
  if (!e) return fail(3, "out of memory");
  orc_extend_symmetric(f, n, K, e);
  *out = dist_ext(e, i, j, K);
  free(e);
  return 0;
}

/* Direct-sum distance band (no recursion): an independent second route, as
 * the reference tests' reference_kernel does (banded_kernel_test.cpp:19-41). */
int orc_distance_band_direct(const double* f, int n, int S, int K, double* dist) {
  int rc = orc_validate_geometry(S, K, n);
  if (rc) return rc;
  const int bw = 2 * S + 1;
  double* e = (double*)malloc(sizeof(double) * (size_t)(n + 2 * K));
  if (!e) return fail(3, "out of memory");
  orc_extend_symmetric(f, n, K, e);
  for (int i = 0; i < n; ++i)
    for (int o = 0; o < bw; ++o) {
      const int j = i + o - S;
      dist[(size_t)i * bw + o] = (j < 0 || j >= n) ? NAN : dist_ext(e, i, j, K);
    }
  free(e);
  return 0;
}

/* weight: nlm.cpp:116-118 */
double orc_weight(double rho_sq, double h) { return exp(-rho_sq / (h * h)); }

/* Window count per line (nlm.cpp:155-159): sum over i of the clipped window. */
static uint64_t window_count(int n, int S) {
  uint64_t w = 0;
  for (int i = 0; i < n; ++i) {
    const int lo = i - S > 0 ? i - S : 0;
    const int hi = i + S < n - 1 ? i + S : n - 1;
    w += (uint64_t)(hi - lo + 1);
  }
  return w;
}

/* nlm_1d_patchlift (nlm.cpp:144-166) via nlm_1d_impl's clipped, ascending
 * window loop (nlm.cpp:66-81) and WeightAccumulator (nlm.hpp:11-20).
 * ops4 = {adds, muls, exps, clamps} accumulated (may be NULL). */
int orc_nlm_1d_patchlift(const double* f, int n, int S, int K, double h, double* out,
                         uint64_t* ops4) {
  int rc = orc_validate_params(S, K, h, n);
  if (rc) return rc;
  const int bw = 2 * S + 1;
  double* band = (double*)malloc(sizeof(double) * (size_t)n * bw);
  if (!band) return fail(3, "out of memory");
  uint64_t adds = 0, muls = 0, clamps = 0;
  orc_banded_kernel(f, n, S, K, band, &adds, &muls);
  for (int i = 0; i < n; ++i) {
    const int lo = i - S > 0 ? i - S : 0;
    const int hi = i + S < n - 1 ? i + S : n - 1;
    double num = 0.0, den = 0.0;
    for (int j = lo; j <= hi; ++j) {
      const double w = orc_weight(orc_kernel_distance_sq(band, n, S, i, j, &clamps), h);
      num += w * f[j];
      den += w;
    }
    out[i] = num / den;
  }
  free(band);
  if (ops4) {
    const uint64_t win = window_count(n, S);
    ops4[0] += adds + win * 4;
    ops4[1] += muls + win * 2;
    ops4[2] += win;
    ops4[3] += clamps;
  }
  return 0;
}

/* nlm_1d_naive: nlm.cpp:120-142 */
int orc_nlm_1d_naive(const double* f, int n, int S, int K, double h, double* out,
                     uint64_t* ops4) {
  int rc = orc_validate_params(S, K, h, n);
  if (rc) return rc;
  double* e = (double*)malloc(sizeof(double) * (size_t)(n + 2 * K));
  if (!e) return fail(3, "out of memory");
  orc_extend_symmetric(f, n, K, e);
  for (int i = 0; i < n; ++i) {
    const int lo = i - S > 0 ? i - S : 0;
    const int hi = i + S < n - 1 ? i + S : n - 1;
    double num = 0.0, den = 0.0;
    for (int j = lo; j <= hi; ++j) {
      const double w = orc_weight(dist_ext(e, i, j, K), h);
      num += w * f[j];
      den += w;
    }
    out[i] = num / den;
  }
  free(e);
  if (ops4) {
    const uint64_t win = window_count(n, S);
    ops4[0] += win * (2 * (uint64_t)(2 * K + 1) + 2);
    ops4[1] += win * ((uint64_t)(2 * K + 1) + 1);
    ops4[2] += win;
  }
  return 0;
}

/* transpose: core_types.cpp:90-98 */
void orc_transpose(const double* in, int rows, int cols, double* out) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) out[(size_t)c * rows + r] = in[(size_t)r * cols + c];
}

/* nlm_row_pass on a row range [r0, r1): nlm.cpp:215-227.  The reference's
 * parallel_for (nlm.cpp:18-54) only splits rows, so any row split is
 * bit-identical; callers may fan row ranges out over threads. */
int orc_row_pass_rows(const double* img, int rows, int cols, int S, int K, double h, int r0,
                      int r1, double* out, uint64_t* ops4) {
  int rc = orc_validate_params(S, K, h, cols);
  if (rc) return rc;
  (void)rows;
  for (int r = r0; r < r1; ++r) {
    rc = orc_nlm_1d_patchlift(img + (size_t)r * cols, cols, S, K, h, out + (size_t)r * cols, ops4);
    if (rc) return rc;
  }
  return 0;
}

int orc_row_pass(const double* img, int rows, int cols, int S, int K, double h, double* out,
                 uint64_t* ops4) {
  if (rows < 1 || cols < 1) return fail(1, "image dimensions must be at least 1x1");
  return orc_row_pass_rows(img, rows, cols, S, K, h, 0, rows, out, ops4);
}

/* nlm_col_pass = transpose . row_pass . transpose: nlm.cpp:229-232 */
int orc_col_pass(const double* img, int rows, int cols, int S, int K, double h, double* out,
                 uint64_t* ops4) {
  if (rows < 1 || cols < 1) return fail(1, "image dimensions must be at least 1x1");
  const size_t cnt = (size_t)rows * cols;
  double* t = (double*)malloc(sizeof(double) * cnt);
  double* u = (double*)malloc(sizeof(double) * cnt);
  if (!t || !u) {
    free(t);
    free(u);
    return fail(3, "out of memory");
  }
  orc_transpose(img, rows, cols, t);
  int rc = orc_row_pass(t, cols, rows, S, K, h, u, ops4);
  if (!rc) orc_transpose(u, cols, rows, out);
  free(t);
  free(u);
  return rc;
}

/* snlm_2d_row_col (nlm.cpp:234-239) and snlm_2d_col_row (nlm.cpp:241-246). */
int orc_snlm_order(int row_first, const double* img, int rows, int cols, int S, int K, double h,
                   double* out, uint64_t* ops4) {
  int rc = orc_validate_params(S, K, h, rows);
  if (!rc) rc = orc_validate_params(S, K, h, cols);
  if (rc) return rc;
  double* mid = (double*)malloc(sizeof(double) * (size_t)rows * cols);
  if (!mid) return fail(3, "out of memory");
  if (row_first) {
    rc = orc_row_pass(img, rows, cols, S, K, h, mid, ops4);
    if (!rc) rc = orc_col_pass(mid, rows, cols, S, K, h, out, ops4);
  } else {
    rc = orc_col_pass(img, rows, cols, S, K, h, mid, ops4);
    if (!rc) rc = orc_row_pass(mid, rows, cols, S, K, h, out, ops4);
  }
  free(mid);
  return rc;
}

/* snlm_2d = average(RC, CR), average = (a+b)/2.0: nlm.cpp:248-253, 106-112 */
int orc_snlm(const double* img, int rows, int cols, int S, int K, double h, double* out,
             uint64_t* ops4) {
  const size_t cnt = (size_t)rows * cols;
  double* rc_img = (double*)malloc(sizeof(double) * cnt);
  double* cr_img = (double*)malloc(sizeof(double) * cnt);
  if (!rc_img || !cr_img) {
    free(rc_img);
    free(cr_img);
    return fail(3, "out of memory");
  }
  int rc = orc_snlm_order(1, img, rows, cols, S, K, h, rc_img, ops4);
  if (!rc) rc = orc_snlm_order(0, img, rows, cols, S, K, h, cr_img, ops4);
  if (!rc)
    for (size_t k = 0; k < cnt; ++k) out[k] = (rc_img[k] + cr_img[k]) / 2.0;
  free(rc_img);
  free(cr_img);
  return rc;
}

/* ---- image fidelity metrics (metrics.cpp:12-150) ------------------------ */
/* 11-tap Gaussian window, sigma 1.5, normalised: metrics.cpp:14-17,25-37 */
static void ssim_kernel(double k[11]) {
  double total = 0.0;
  for (int t = 0; t < 11; ++t) {
    const double x = t - (11 - 1) / 2;
    k[t] = exp(-x * x / (2.0 * 1.5 * 1.5));
    total += k[t];
  }
  for (int t = 0; t < 11; ++t) k[t] /= total;
}

/* valid-mode separable correlation, rows then columns: metrics.cpp:39-64 */
static void ssim_blur(const double* src, int h, int w, const double k[11], double* tmp,
                      double* out) {
  const int wo = w - 11 + 1, ho = h - 11 + 1;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < wo; ++c) {
      double s = 0.0;
      for (int t = 0; t < 11; ++t) s += k[t] * src[(size_t)r * w + c + t];
      tmp[(size_t)r * wo + c] = s;
    }
  for (int r = 0; r < ho; ++r)
    for (int c = 0; c < wo; ++c) {
      double s = 0.0;
      for (int t = 0; t < 11; ++t) s += k[t] * tmp[(size_t)(r + t) * wo + c];
      out[(size_t)r * wo + c] = s;
    }
}

/* mse (metrics.cpp:98-106), psnr (:108-114), ssim (:116-150) of one image
 * pair; out[0..2] = mse, psnr_db, ssim.  psnr is +inf for identical images. */
int orc_metrics(const double* a, const double* b, int rows, int cols, double* out) {
  if (rows < 11 || cols < 11) return fail(1, "image smaller than the 11x11 structural window");
  const size_t n = (size_t)rows * cols;
  double acc = 0.0;
  for (size_t k = 0; k < n; ++k) {
    const double diff = a[k] - b[k];
    acc += diff * diff;
  }
  const double m = acc / (double)n;
  out[0] = m;
  out[1] = m == 0.0 ? INFINITY : 10.0 * log10(255.0 * 255.0 / m);
  const int wo = cols - 10, ho = rows - 10;
  const size_t no = (size_t)ho * wo;
  double* buf = (double*)malloc(sizeof(double) * (3 * n + (size_t)rows * wo + 5 * no));
  if (!buf) return fail(3, "out of memory");
  double *xx = buf, *yy = xx + n, *xy = yy + n, *tmp = xy + n, *mu_x = tmp + (size_t)rows * wo;
  double *mu_y = mu_x + no, *e_xx = mu_y + no, *e_yy = e_xx + no, *e_xy = e_yy + no;
  for (size_t k = 0; k < n; ++k) {
    xx[k] = a[k] * a[k];
    yy[k] = b[k] * b[k];
    xy[k] = a[k] * b[k];
  }
  double kern[11];
  ssim_kernel(kern);
  ssim_blur(a, rows, cols, kern, tmp, mu_x);
  ssim_blur(b, rows, cols, kern, tmp, mu_y);
  ssim_blur(xx, rows, cols, kern, tmp, e_xx);
  ssim_blur(yy, rows, cols, kern, tmp, e_yy);
  ssim_blur(xy, rows, cols, kern, tmp, e_xy);
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  double total = 0.0;
  for (size_t k = 0; k < no; ++k) {
    const double mx = mu_x[k], my = mu_y[k];
    const double var_x = e_xx[k] - mx * mx;
    const double var_y = e_yy[k] - my * my;
    const double cov = e_xy[k] - mx * my;
    total += ((2.0 * mx * my + C1) * (2.0 * cov + C2)) /
             ((mx * mx + my * my + C1) * (var_x + var_y + C2));
  }
  out[2] = total / (double)no;
  free(buf);
  return 0;
}

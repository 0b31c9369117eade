// plgpu_metrics.cuh -- image fidelity metrics on the device (sm_100a).
//
// MSE, PSNR and SSIM of image pairs (metrics.cpp:98-158), the quality loop
// around the filter.  FP64 throughout, and every
// per-pixel quantity is evaluated in the reference's operation order with
// explicit round-to-nearest intrinsics (no contraction: the reference build
// has no FMA), so the SSIM map and the squared differences are bit-equal to
// the reference's on the same inputs; only the final sums run as fixed-shape
// tree reductions (deterministic, ~1 ulp from the reference's serial sums).
#pragma once

#include <cstdint>

namespace plgpu {

constexpr int kSsimWin = 11;    // metrics.cpp:14
constexpr int kSsimTW = 32;     // output tile: 32 columns x 8 rows per CTA
constexpr int kSsimTH = 8;
constexpr int kMetricThreads = 256;
constexpr int kMseBlocks = 64;  // partial sums per image for the MSE

struct SsimWindow {
  double k[kSsimWin];  // normalised Gaussian taps (metrics.cpp:25-37), host-computed
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
#pragma unroll
  for (int s = kMetricThreads / 2; s > 0; s >>= 1) {
    if (t < s) red[t] = __dadd_rn(red[t], red[t + s]);
    __syncthreads();
  }
  return red[0];
}

// Squared differences (metrics.cpp:98-106): partial[img * kMseBlocks + blk].
template <typename T>
__global__ void __launch_bounds__(kMetricThreads) mse_partial_kernel(const T* a, const T* b,
                                                                     int64_t n, double* partial) {
  __shared__ double red[kMetricThreads];
  const int64_t img = blockIdx.y;
  const T* pa = a + img * n;
  const T* pb = b + img * n;
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * kMetricThreads + threadIdx.x; k < n;
       k += (int64_t)kMseBlocks * kMetricThreads) {
    const double diff = __dsub_rn((double)pa[k], (double)pb[k]);
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[img * kMseBlocks + blockIdx.x] = s;
}

// SSIM map (metrics.cpp:116-150) over one 8 x 32 tile of valid window
// positions; partial[img * tiles + tile] = sum of the tile's SSIM values.
template <typename T>
__global__ void __launch_bounds__(kMetricThreads) ssim_partial_kernel(const T* a, const T* b,
                                                                      int rows, int cols,
                                                                      SsimWindow win,
                                                                      double* partial) {
  constexpr int IH = kSsimTH + kSsimWin - 1, IW = kSsimTW + kSsimWin - 1;
  __shared__ double sa[IH][IW], sb[IH][IW];
  __shared__ double hs[5][IH][kSsimTW];  // row-blurred x, y, xx, yy, xy
  __shared__ double red[kMetricThreads];
  const int wo = cols - kSsimWin + 1, ho = rows - kSsimWin + 1;
  const int c0 = blockIdx.x * kSsimTW, r0 = blockIdx.y * kSsimTH;
  const int64_t img = blockIdx.z;
  const T* pa = a + img * (int64_t)rows * cols;
  const T* pb = b + img * (int64_t)rows * cols;
  for (int e = threadIdx.x; e < IH * IW; e += kMetricThreads) {
    const int r = e / IW, c = e % IW;
    const int gr = min(r0 + r, rows - 1), gc = min(c0 + c, cols - 1);  // clamp: unused lanes
    sa[r][c] = (double)pa[(int64_t)gr * cols + gc];
    sb[r][c] = (double)pb[(int64_t)gr * cols + gc];
  }
  __syncthreads();
  // Row pass of the separable correlation: s = 0; s += k[t] * v, t ascending
  // (metrics.cpp:44-52), on x, y and the rounded products xx, yy, xy (:127-131).
  for (int e = threadIdx.x; e < IH * kSsimTW; e += kMetricThreads) {
    const int r = e / kSsimTW, c = e % kSsimTW;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
    for (int t = 0; t < kSsimWin; ++t) {
      const double x = sa[r][c + t], y = sb[r][c + t], k = win.k[t];
      s0 = __dadd_rn(s0, __dmul_rn(k, x));
      s1 = __dadd_rn(s1, __dmul_rn(k, y));
      s2 = __dadd_rn(s2, __dmul_rn(k, __dmul_rn(x, x)));
      s3 = __dadd_rn(s3, __dmul_rn(k, __dmul_rn(y, y)));
      s4 = __dadd_rn(s4, __dmul_rn(k, __dmul_rn(x, y)));
    }
    hs[0][r][c] = s0;
    hs[1][r][c] = s1;
    hs[2][r][c] = s2;
    hs[3][r][c] = s3;
    hs[4][r][c] = s4;
  }
  __syncthreads();
  // Column pass (metrics.cpp:54-62) and the per-position SSIM (:140-148).
  const int r = threadIdx.x / kSsimTW, c = threadIdx.x % kSsimTW;
  double v = 0.0;
  if (r0 + r < ho && c0 + c < wo) {
    double m[5];
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < kSsimWin; ++t) s = __dadd_rn(s, __dmul_rn(win.k[t], hs[f][r + t][c]));
      m[f] = s;
    }
    const double mx = m[0], my = m[1];
    const double var_x = __dsub_rn(m[2], __dmul_rn(mx, mx));
    const double var_y = __dsub_rn(m[3], __dmul_rn(my, my));
    const double cov = __dsub_rn(m[4], __dmul_rn(mx, my));
    constexpr double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
    const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mx), my), C1),
                                 __dadd_rn(__dmul_rn(2.0, cov), C2));
    const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), C1),
                                 __dadd_rn(__dadd_rn(var_x, var_y), C2));
    v = __ddiv_rn(num, den);
  }
  const double s = block_sum(v, red);
  if (threadIdx.x == 0)
    partial[img * (int64_t)gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = s;
}

// out[3 img + {0,1,2}] = mse, psnr_db (metrics.cpp:108-114), ssim.
__global__ void __launch_bounds__(kMetricThreads) metrics_finish_kernel(
    const double* mse_part, const double* ssim_part, int64_t tiles, int64_t n, int64_t n_valid,
    double* out) {
  __shared__ double red[kMetricThreads];
  const int64_t img = blockIdx.x;
  double v = threadIdx.x < kMseBlocks ? mse_part[img * kMseBlocks + threadIdx.x] : 0.0;
  const double se = block_sum(v, red);
  __syncthreads();
  double w = 0.0;
  for (int64_t t = threadIdx.x; t < tiles; t += kMetricThreads)
    w = __dadd_rn(w, ssim_part[img * tiles + t]);
  const double ss = block_sum(w, red);
  if (threadIdx.x == 0) {
    const double m = se / (double)n;
    out[3 * img + 0] = m;
    out[3 * img + 1] = m == 0.0 ? __longlong_as_double(0x7ff0000000000000ll)
                                : 10.0 * log10(255.0 * 255.0 / m);
    out[3 * img + 2] = n_valid > 0 ? ss / (double)n_valid : __longlong_as_double(0x7ff8000000000000ll);
  }
}

}  // namespace plgpu

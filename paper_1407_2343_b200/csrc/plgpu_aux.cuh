// plgpu_aux.cuh -- secondary device kernels behind the C ABI:
//   * banded_kernel_f64: F-bar cells (compute_banded_kernel, banded_kernel.cpp:25-72)
//     with the reference's own diagonal recursion and evaluation order in
//     fp64 (explicit _rn intrinsics: no FMA contraction), so cells are
//     bit-equal to the reference's.  Not on the filter's hot path.
//   * nlm_direct_kernel: the direct O(K)-per-window route of nlm_1d_naive
//     (nlm.cpp:120-142); also serves radii above the walker's instantiations.
#pragma once

#include <cstring>

#include <cstdint>

#include "plgpu_walk.cuh"
#include "plgpu_walk64.cuh"

namespace plgpu {

struct KernelBandDesc {
  const double* src;
  double* band;
  int64_t n_lines, ld;
  int32_t n, S, S_band, K;
};

// One thread per (line, diagonal d).  e[q] = extended sample at q - K.
__global__ void banded_kernel_f64(KernelBandDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nd = g.S + 1;
  if (w >= g.n_lines * nd) return;
  const int64_t line = w / nd;
  const int d = (int)(w % nd);
  const int n = g.n, K = g.K;
  const double* f = g.src + line * g.ld;
  const int bw = 2 * g.S_band + 1;
  double* band = g.band + line * (int64_t)n * bw;
  auto e = [&](int q) -> double { return f[mirror_pos(q - K, n)]; };
  double sum = 0.0;
  for (int k = -K; k <= K; ++k) sum = __dadd_rn(sum, __dmul_rn(e(k + K), e(d + k + K)));
  band[(int64_t)0 * bw + (d + g.S_band)] = sum;
  band[(int64_t)d * bw + (g.S_band - d)] = sum;
  for (int i = 1; i < n - d; ++i) {
    const int j = i + d;
    sum = __dsub_rn(__dadd_rn(sum, __dmul_rn(e(i + 2 * K), e(j + 2 * K))),
                    __dmul_rn(e(i - 1), e(j - 1)));
    band[(int64_t)i * bw + (j - i + g.S_band)] = sum;
    band[(int64_t)j * bw + (i - j + g.S_band)] = sum;
  }
}

struct DirectDesc {
  const float* src;
  float* dst;
  int64_t n_lines, ld;
  int32_t n, S, K;
  float coef;
};

// One thread per pixel; clipped window ascending, direct distances.
__global__ void __launch_bounds__(128) nlm_direct_kernel(DirectDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.n) return;
  const int64_t line = w / g.n;
  const int i = (int)(w % g.n);
  const float* f = g.src + line * g.ld;
  const int n = g.n, K = g.K;
  const int lo = max(0, i - g.S), hi = min(n - 1, i + g.S);
  float num = 0.f, den = 0.f, vmin = 3.402823466e38f, vmax = -3.402823466e38f;
  for (int j = lo; j <= hi; ++j) {
    float dsq = 0.f;
    for (int t = -K; t <= K; ++t) {
      const float df = __ldg(f + mirror_pos(i + t, n)) - __ldg(f + mirror_pos(j + t, n));
      dsq = fmaf(df, df, dsq);
    }
    const float wt = ex2_approx(g.coef * dsq);
    const float fj = __ldg(f + j);
    num = fmaf(wt, fj, num);
    den += wt;
    vmin = fminf(vmin, fj);
    vmax = fmaxf(vmax, fj);
  }
  g.dst[line * g.ld + i] = fminf(fmaxf(num / den, vmin), vmax);
}

// (a + b) / 2 elementwise: average(), nlm.cpp:106-112.
__global__ void average_kernel(const float* __restrict__ a, const float* __restrict__ b,
                               float* __restrict__ out, int64_t count) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (a[k] + b[k]) / 2.0f;
}

}  // namespace plgpu

namespace plgpu {

struct Naive2DDesc {
  const float* src;
  float* dst;
  int32_t batch, rows, cols, S, K;
  float coef;
};

// Classical 2D NLM (nlm_2d_naive, nlm.cpp:168-213): one thread per pixel,
// clipped (2S+1)^2 window, (2K+1)^2 patches over the per-axis half-sample
// mirror (extend_symmetric_2d, nlm.cpp:84-104).  Baseline only.
__global__ void __launch_bounds__(128) nlm_2d_naive_kernel(Naive2DDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t plane = (int64_t)g.rows * g.cols;
  if (w >= plane * g.batch) return;
  const int64_t b = w / plane;
  const int r = (int)((w % plane) / g.cols), c = (int)(w % g.cols);
  const float* img = g.src + b * plane;
  const int H = g.rows, W = g.cols, S = g.S, K = g.K;
  auto px = [&](int y, int x) { return __ldg(img + (int64_t)mirror_pos(y, H) * W + mirror_pos(x, W)); };
  float num = 0.f, den = 0.f, vmin = 3.402823466e38f, vmax = -3.402823466e38f;
  for (int r2 = max(0, r - S); r2 <= min(H - 1, r + S); ++r2)
    for (int c2 = max(0, c - S); c2 <= min(W - 1, c + S); ++c2) {
      float dsq = 0.f;
      for (int py = -K; py <= K; ++py)
        for (int qx = -K; qx <= K; ++qx) {
          const float df = px(r + py, c + qx) - px(r2 + py, c2 + qx);
          dsq = fmaf(df, df, dsq);
        }
      const float wt = (r2 == r && c2 == c) ? 1.f : ex2_approx(g.coef * dsq);
      const float v = __ldg(img + (int64_t)r2 * W + c2);
      num = fmaf(wt, v, num);
      den += wt;
      vmin = fminf(vmin, v);
      vmax = fmaxf(vmax, v);
    }
  g.dst[w] = fminf(fmaxf(num / den, vmin), vmax);
}

}  // namespace plgpu

namespace plgpu {

// Direct-sum distance band for radii above the walker instantiations: one
// thread per (line, i), (2K+1)-term sums in t-ascending order (exact on
// integer inputs, like the walker).
template <typename T>
__global__ void __launch_bounds__(128) distance_band_direct_kernel(BandDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.n) return;
  const int64_t line = w / g.n;
  const int i = (int)(w % g.n);
  const float* f = g.src + line * g.ld;
  const int n = g.n, K = g.K, bw = 2 * g.S_band + 1;
  T* band = reinterpret_cast<T*>(g.band) + (line * (int64_t)n + i) * bw;
  for (int j = max(0, i - g.S); j <= min(n - 1, i + g.S); ++j) {
    float dsq = 0.f;
    for (int t = -K; t <= K; ++t) {
      const float df = __ldg(f + mirror_pos(i + t, n)) - __ldg(f + mirror_pos(j + t, n));
      dsq = fmaf(df, df, dsq);
    }
    band[j - i + g.S_band] = band_cast<T>(dsq);
  }
}

}  // namespace plgpu

namespace plgpu {

// Direct route in double (S = 0 or S above the walker range): every window
// of pixel i summed from scratch, ascending j (nlm.cpp:66-81).
__global__ void __launch_bounds__(128) direct_pass64_kernel(Pass64Desc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.n) return;
  const int64_t line = w % g.n_lines;
  const int i = (int)(w / g.n_lines);
  const int64_t img = line / g.lines_per_img;
  const int64_t li = line - img * g.lines_per_img;
  const double* f = g.src + img * g.src_img_stride + li * g.src_line_stride;
  const int64_t ps = g.src_pos_stride;
  const int n = g.n, K = g.K;
  const int lo = max(0, i - g.S), hi = min(n - 1, i + g.S);
  double num = 0.0, den = 0.0, vmin = 1.7976931348623157e308, vmax = -vmin;
  for (int j = lo; j <= hi; ++j) {
    double dsq = 0.0;
    for (int t = -K; t <= K; ++t) {
      const double df = __ldg(f + mirror_pos(i + t, n) * ps) - __ldg(f + mirror_pos(j + t, n) * ps);
      dsq = fma(df, df, dsq);
    }
    const double wt = (j == i) ? 1.0 : exp(-dsq * g.inv_h2);
    const double fj = __ldg(f + (int64_t)j * ps);
    num = fma(wt, fj, num);
    den += wt;
    vmin = fmin(vmin, fj);
    vmax = fmax(vmax, fj);
  }
  double* dst = g.dst + img * g.dst_img_stride + li * g.dst_line_stride + (int64_t)i * g.dst_pos_stride;
  double v = fmin(fmax(num / den, vmin), vmax);
  if (g.avg) v = (g.avg[dst - g.dst] + v) / 2.0;
  *dst = v;
}

}  // namespace plgpu

namespace plgpu {

struct Naive2D64Desc {
  const double* src;
  double* dst;
  int32_t batch, rows, cols, S, K;
  double inv_h2;
};

// Classical 2D NLM in double (nlm_2d_naive, nlm.cpp:168-213), the drop-in's
// reference-precision baseline: clipped (2S+1)^2 window, (2K+1)^2 patches
// over the per-axis half-sample mirror, exp(-d / (h h)).
__global__ void __launch_bounds__(128) nlm_2d_naive64_kernel(Naive2D64Desc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t plane = (int64_t)g.rows * g.cols;
  if (w >= plane * g.batch) return;
  const int64_t b = w / plane;
  const int r = (int)((w % plane) / g.cols), c = (int)(w % g.cols);
  const double* img = g.src + b * plane;
  const int H = g.rows, W = g.cols, S = g.S, K = g.K;
  auto px = [&](int y, int x) { return __ldg(img + (int64_t)mirror_pos(y, H) * W + mirror_pos(x, W)); };
  double num = 0.0, den = 0.0, vmin = 1.7976931348623157e308, vmax = -vmin;
  for (int r2 = max(0, r - S); r2 <= min(H - 1, r + S); ++r2)
    for (int c2 = max(0, c - S); c2 <= min(W - 1, c + S); ++c2) {
      double dsq = 0.0;
      for (int py = -K; py <= K; ++py)
        for (int qx = -K; qx <= K; ++qx) {
          const double df = px(r + py, c + qx) - px(r2 + py, c2 + qx);
          dsq = fma(df, df, dsq);
        }
      const double wt = (r2 == r && c2 == c) ? 1.0 : exp(-dsq * g.inv_h2);
      const double v = __ldg(img + (int64_t)r2 * W + c2);
      num = fma(wt, v, num);
      den += wt;
      vmin = fmin(vmin, v);
      vmax = fmax(vmax, v);
    }
  g.dst[w] = fmin(fmax(num / den, vmin), vmax);
}


// ---- precision policy helpers (plgpu.cu: choose_precise / precise_*) --------
// Order-preserving map float -> uint32 so atomicMin / atomicMax give the
// range of a buffer (NaNs are skipped).
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float ordered_value(uint32_t o) {
  const uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
#endif
}

// Range of `lines` lines of n samples (line l at src + l * ld) into
// out[0] = ordered min, out[1] = ordered max (preset to ~0u / 0u).
__global__ void __launch_bounds__(256) range_kernel(const float* __restrict__ src, int64_t lines,
                                                    int32_t n, int64_t ld, uint32_t* out) {
  const int64_t total = lines * n;
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = ld == n ? src[i] : src[(i / n) * ld + (i % n)];
    if (v == v) {
      const uint32_t o = ordered_bits(v);
      lo = min(lo, o);
      hi = max(hi, o);
    }
  }
  lo = __reduce_min_sync(0xFFFFFFFFu, lo);
  hi = __reduce_max_sync(0xFFFFFFFFu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

// fp32 lines (stride ld) -> compact fp64 lines (stride n) and back.
__global__ void __launch_bounds__(256) widen_kernel(const float* __restrict__ src,
                                                    double* __restrict__ dst, int64_t lines,
                                                    int32_t n, int64_t ld) {
  const int64_t total = lines * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (double)(ld == n ? src[i] : src[(i / n) * ld + (i % n)]);
}
__global__ void __launch_bounds__(256) narrow_kernel(const double* __restrict__ src,
                                                     float* __restrict__ dst, int64_t lines,
                                                     int32_t n, int64_t ld) {
  const int64_t total = lines * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = (float)src[i];
    if (ld == n) dst[i] = v;
    else dst[(i / n) * ld + (i % n)] = v;
  }
}

}  // namespace plgpu

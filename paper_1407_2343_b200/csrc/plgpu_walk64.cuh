// plgpu_walk64.cuh -- the fp64 line filter: the reference-precision route.
//
// Same algorithm as the fp32 walkers (plgpu_walk.cuh: moving-sum distances
// along the lifted image's diagonals, one weight per unique pair feeding both
// endpoints, centre term first) carried out in double, with the reference's
// weight exp(-d / (h h)) (nlm.cpp:116-118) from CUDA's double exp -- so the
// outputs agree with the reference library (double throughout,
// core_types.hpp:23,35) to rounding, not only to the fp32 tolerance tiers.
// The C++ drop-in routes every filter here by default; the fp32 kernels stay
// the throughput path of the C ABI.  B200 keeps a full-rate FP64 pipe (half
// the FP32 lane rate), so this route costs ~a few x the fp32 one, not orders
// of magnitude.
//
// One thread per (line, segment), global loads (the lines are re-read from
// L1/L2), S-specialised register rings exactly as the portable walker.
#pragma once

#include <cstdint>

#include "plgpu_walk.cuh"

namespace plgpu {

struct Pass64Desc {
  const double* src;
  double* dst;
  const double* avg;  // optional, dst layout: store (avg + out) / 2 (snlm_2d's average)
  int64_t n_lines;
  int64_t src_img_stride, src_line_stride, src_pos_stride;
  int64_t dst_img_stride, dst_line_stride, dst_pos_stride;
  int32_t lines_per_img;
  int32_t n, seg_len, nseg;
  int32_t S, K;     // effective radius (<= template, <= n - 1), patch radius
  double inv_h2;    // 1 / (h h)
};

template <int ST, bool EDGE>
__device__ __forceinline__ void walk64_segment(const Pass64Desc& g, const double* __restrict__ src,
                                               double* __restrict__ dst, int s0, int s1) {
  constexpr int R = ST + 1;
  const int n = g.n;
  const int S = EDGE ? g.S : ST;
  const int K = g.K;
  const int i0 = max(0, s0 - S);
  const int T = s1 - i0;
  const int64_t ps = g.src_pos_stride, dps = g.dst_pos_stride;
  auto ld = [&](int p) -> double {
    if (EDGE) p = mirror_pos(p, n);
    return __ldg(src + (int64_t)p * ps);
  };
  double fr[R], nr[R], orr[R], d[R], an[R], ad[R];
  double lo = 1.7976931348623157e308, hi = -1.7976931348623157e308;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    fr[q] = ld(i0 + q);
    lo = fmin(lo, fr[q]);
    hi = fmax(hi, fr[q]);
    nr[q] = ld(i0 + K + q);
    orr[q] = ld(i0 - 1 - K + q);
    an[q] = fr[q];  // centre sample (w = 1) first
    ad[q] = 1.0;
    d[q] = 0.0;
  }
  for (int t = -K; t <= K; ++t) {  // anchor d_k(i0 - 1)
    const double a = ld(i0 - 1 + t);
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const double df = a - ld(i0 - 1 + t + k);
      d[k] = fma(df, df, d[k]);
    }
  }
  double* op = dst + (int64_t)s0 * dps;
  const double* ap = g.avg ? g.avg + (dst - g.dst) + (int64_t)s0 * dps : nullptr;
  for (int sb = 0; sb < T; sb += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = sb + r;
      if (s >= T) break;
      const int i = i0 + s;
      const double tf = ld(i + 1 + ST);
      const double tn = ld(i + 1 + K + ST);
      const double to = ld(i - K + ST);
      const double an_ = nr[r], ao = orr[r], fi = fr[r];
      const int kmax = EDGE ? min(S, n - 1 - i) : ST;
      double num = an[r], den = ad[r];
#pragma unroll
      for (int k = 1; k <= ST; ++k) {
        const int rk = (r + k) % R;
        const double dn = an_ - nr[rk];
        double dk = fma(dn, dn, d[k]);
        const double dq = ao - orr[rk];
        dk = fma(-dq, dq, dk);
        d[k] = dk;
        double w = exp(-dk * g.inv_h2);
        if (EDGE) w = (k <= kmax) ? w : 0.0;
        num = fma(w, fr[rk], num);
        den += w;
        an[rk] = fma(w, fi, an[rk]);
        ad[rk] += w;
      }
      if (i >= s0) {
        double v = fmin(fmax(num / den, lo), hi);
        if (ap) {
          v = (*ap + v) / 2.0;
          ap += dps;
        }
        *op = v;
        op += dps;
      }
      an[r] = tf;
      ad[r] = 1.0;
      lo = fmin(lo, tf);
      hi = fmax(hi, tf);
      fr[r] = tf;
      nr[r] = tn;
      orr[r] = to;
    }
  }
}

template <int ST>
__global__ void __launch_bounds__(128) nlm_pass64_kernel(Pass64Desc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.nseg) return;
  const int64_t line = w % g.n_lines;
  const int seg = (int)(w / g.n_lines);
  const int64_t img = line / g.lines_per_img;
  const int64_t li = line - img * g.lines_per_img;
  const double* src = g.src + img * g.src_img_stride + li * g.src_line_stride;
  double* dst = g.dst + img * g.dst_img_stride + li * g.dst_line_stride;
  const int s0 = seg * g.seg_len;
  const int s1 = min(g.n, s0 + g.seg_len);
  const int i0 = max(0, s0 - g.S);
  const bool interior = (g.S == ST) && (i0 - 1 - g.K >= 0) && (s1 + g.K + g.S < g.n);
  if (interior) walk64_segment<ST, false>(g, src, dst, s0, s1);
  else walk64_segment<ST, true>(g, src, dst, s0, s1);
}

template <int ST>
void launch_pass64(const Pass64Desc& g, cudaStream_t st) {
  const int64_t work = g.n_lines * g.nseg;
  nlm_pass64_kernel<ST><<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
}

}  // namespace plgpu


// plgpu_walk.cuh -- the fused PatchLift-NLM line walker (sm_100a).
//
// One thread owns one (line, segment).  It walks the segment's positions in
// order, carrying for every offset k = 1..S the running patch distance
//
//     d_k(i) = sum_{|t|<=K} (e[i+t] - e[i+k+t])^2                (1)
//
// updated by the moving-sum recurrence of the lifted kernel's k-th diagonal
//
//     d_k(i) = d_k(i-1) + (e[i+K]-e[i+K+k])^2 - (e[i-1-K]-e[i-1-K+k])^2   (2)
//
// (PatchLift: banded_kernel.cpp:46-62 runs the same recursion on F-bar and
// forms d = F(i,i)+F(j,j)-2F(i,j) at :74-84; here the recursion runs directly
// on the squared differences, so d >= 0 by construction).  The filter runs
// it on PRESCALED samples e' = s e, s = sqrt(log2 e)/h (fp32, from double on
// the host), so d' = d log2(e)/h^2 up to rounding and the weight
// w = exp(-d/h^2) (weight(), nlm.cpp:116-118) is one MUFU.EX2 of -d' -- no
// per-pair multiply.  The distance exports (distance_band_kernel) run the
// recurrence on the raw samples, where integer inputs give exact integer
// distances (every partial sum < 2^24 for K <= 127).
// Each unique pair (i, i+k) is weighted ONCE and feeds both endpoints:
//
//     num[i] += w f[i+k]; den[i] += w;  num[i+k] += w f[i]; den[i+k] += w
//
// (WeightAccumulator, nlm.hpp:11-20; the centre sample weighs exactly 1 and
// seeds the pixel's sums when it enters the rings).
// Nothing of the N x (2S+1) band is materialised: the samples live in three
// register rings of S+1 (partners of the entering term, of the leaving term,
// and the f values), the S distances in registers, and the pending
// numerators/denominators of the next S+1 pixels in a fourth ring.  With the
// walk unrolled by S+1 steps every ring index is a compile-time constant, so
// the rings are plain registers and the recurrence costs O(1) in K.
//
// Segments.  A line of n samples is cut into segments of C samples (C a
// function of n only: pl_segment_length).  A segment [s0, s1) is walked from
// i0 = max(0, s0 - S): the S "pre-walk" steps deliver the contributions of
// pairs (i, i+k), i < s0 <= i+k, to the segment's first pixels.  Running sums
// are anchored by a direct sum at i0-1, so every segment is independent and
// results are bitwise independent of how segments/lines are scheduled.  Row
// and column passes call the same walker (only strides differ): identical
// per-line arithmetic, hence exact transpose equivariance
// (nlm_test.cpp:186-215, acceptance_main.cpp:292-300).
#pragma once

#include <cstdint>

namespace plgpu {

// One pass over a set of lines.  Line l = img * lines_per_img + li.
struct PassDesc {
  const float* src;
  float* dst;
  int64_t n_lines;
  int64_t src_img_stride, src_line_stride, src_pos_stride;
  int64_t dst_img_stride, dst_line_stride, dst_pos_stride;
  int64_t dst_block_stride;  // blocked output along the line (row-slab send layout)
  int32_t dst_pos_block;     // positions per output block (== n when unblocked)
  int32_t lines_per_img;
  int32_t n;        // line length
  int32_t seg_len;  // C
  int32_t nseg;     // segments processed (ceil(n / C) unless windowed)
  int32_t seg_begin;  // index of the first processed segment (windowed passes)
  float scale;        // s = sqrt(log2 e) / h: sample prescale
  float inv_scale;    // 1 / s (double division, rounded once): acc_prescaled output unscale
  const float* avg;   // optional, dst layout: store (avg + out) / 2 (snlm_2d's average)
  int32_t S;        // effective search radius, <= template S, <= n-1
  int32_t K;        // patch radius
  float coef;       // -log2(e) / h^2
  // Fan-out (pl_nlm_row_pass_fanout, batch 1): output lines [xlo[x], xhi[x])
  // are also stored at xdst[x] + (line - xlo[x]) * dst_line_stride + pos *
  // dst_pos_stride as they are produced -- e.g. into a peer GPU's window.
  float* xdst[2];
  int32_t xlo[2], xhi[2];
  int32_t nx;
  // Debug (pl_debug_hot_distance_band): the hot kernel also stores every
  // distance it computes into this band ([line][n][2S+1]); NULL otherwise.
  float* dexp;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Output epilogue: plain store, or the S-NLM average (a + b) / 2 with the
// other order's result (average(), nlm.cpp:106-112) fused into the store.
__device__ __forceinline__ float epi(const float* avg, const float* dst, const float* p, float v) {
  return avg ? (__ldg(avg + (p - dst)) + v) / 2.0f : v;
}

// num / den for the filter output: one MUFU.RCP and a multiply (within ~2 ulp
// of the IEEE quotient).  Every walker clamps the quotient into the range of
// the samples it walked, which is what makes constant inputs exact fixpoints
// and keeps outputs inside the convex hull (acceptance_main.cpp:256-283); a
// Newton/Markstein correction step bought nothing on top of the clamp and
// cost ~2%.  All walkers use it, so their outputs stay
// bitwise equal.
__device__ __forceinline__ float div_fix(float num, float den) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(den));
  return num * r;
}

// Accumulation form (shared rule of all walkers, a function of the template
// radius ST alone, like the clamp range below).  For ST <= 10 the filters
// accumulate PRESCALED samples: num = sum of w x' with x' = s f, the values the
// distance rings already hold, so the 2-line hot kernel keeps no separate f
// ring (22 registers and one LDS.64 per step less: c4 +1.5 %); den = sum of w
// as before and the output is num * (rcp(den) * (1 / s)).  Larger radii (the
// 1-line packed kernels, where the extra multiplies cost c3 2.3 %) accumulate
// the raw samples: num * rcp(den).
__host__ __device__ constexpr bool acc_prescaled(int ST) { return ST <= 10; }
__device__ __forceinline__ float div_unscale(float num, float den, float inv_s) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(den));
  return __fmul_rn(num, __fmul_rn(r, inv_s));
}

// Three-input min / max (FMNMX3).  The clamp range of every walker is built
// from the same sequence of these ops, so all walkers agree bit for bit.
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Clamp range (shared rule of all walkers).  Outputs are clamped into the
// range of samples the walk has read, so fp32 rounding of num/den can never
// leave the input range (acceptance_main.cpp:256-283) and constant inputs are
// exact fixpoints.  Two forms, chosen by (K, template radius ST) alone:
//  * paired (K >= 1, ST <= 16): the range grows by the raw sample x_s
//    entering the distance ring at step s (position i + K + ST + 1), in pairs:
//    with r = s mod (ST + 1), odd r adds {x_(s-1), x_s} with one FMNMX3 per
//    bound, an even last step r = ST adds x_s alone, other even steps add
//    nothing (x_s waits for the next step).  At the clamp of step s the range
//    covers every position up to i + K + ST - 1 >= i + S, the window's right
//    end.  It starts as the positions [i0, i0 + K + ST] in ascending order.
//    Half the min/max instructions of the per-step form (c4 +1.2 %).
//  * per step (K = 0, where pairs would miss the window end, and ST > 16,
//    where the extra live value cost the S = 25 kernel 13 %): every step adds
//    the sample entering the f ring (position i + ST + 1); the range starts as
//    the positions [i0, i0 + ST].
__host__ __device__ constexpr bool clamp_pairs(int K, int ST) { return K >= 1 && ST <= 16; }

// Half-sample mirror (core_types.cpp:71-88) extended by a clamp: positions
// beyond the extension only ever feed pairs that are masked out.
__device__ __forceinline__ int mirror_pos(int p, int n) {
  p = p < 0 ? -1 - p : p;
  p = p >= n ? 2 * n - 1 - p : p;
  return min(max(p, 0), n - 1);
}

// EDGE: the segment touches a line end (mirrored loads, clipped windows) or
// the template radius exceeds the effective one (pairs with k > S masked).
template <int ST, bool EDGE>
__device__ __forceinline__ void walk_segment(const PassDesc& g, const float* __restrict__ src,
                                             int64_t ps, float* __restrict__ dst, int64_t dps,
                                             int s0, int s1, float* x0 = nullptr, float* x1 = nullptr) {
  constexpr int R = ST + 1;
  constexpr bool AP = acc_prescaled(ST);
  const int n = g.n;
  const int S = EDGE ? g.S : ST;
  const int K = g.K;
  const float sc = g.scale;  // distance-side samples are prescaled: d' = -c d
  const int i0 = max(0, s0 - S);
  const int T = s1 - i0;

  auto ld = [&](int p) -> float {
    if (EDGE) p = mirror_pos(p, n);
    return __ldg(src + (int64_t)p * ps);
  };
  // __fmul_rn: the scaled sample is rounded once, never contracted into the
  // difference that consumes it (all walkers must round identically).
  auto lds = [&](int p) -> float { return __fmul_rn(ld(p), sc); };

  float fr[R], nr[R], orr[R];  // rings: f[i+q], e[i+K+q], e[i-1-K+q]
  float d[R];                  // d[k], k = 1..ST (d[0] unused)
  float an[R], ad[R];          // pending num/den of pixel i+q
  // Range of every sample the segment's windows can touch: outputs are
  // clamped into it, so fp32 rounding of num/den can never leave the input
  // range (the convex-combination guarantee, acceptance_main.cpp:256-283).
  float lo = 3.402823466e38f, hi = -3.402823466e38f;
  float xprev = 0.f;  // x of the previous (even) step, tracked at the next

#pragma unroll
  for (int q = 0; q < R; ++q) {
    const float f0 = ld(i0 + q);
    lo = fminf(lo, f0);
    hi = fmaxf(hi, f0);
    fr[q] = AP ? __fmul_rn(f0, sc) : f0;
    nr[q] = lds(i0 + K + q);
    orr[q] = lds(i0 - 1 - K + q);
    an[q] = fr[q];  // the centre sample (w = 1) starts each pixel's sums
    ad[q] = 1.f;
    d[q] = 0.f;
  }
  const bool pairs = clamp_pairs(K, ST);
  if (pairs) {
    for (int q = R - K; q < R; ++q) {  // the rest of [i0, i0 + K + ST]
      const float x = ld(i0 + K + q);
      lo = fminf(lo, x);
      hi = fmaxf(hi, x);
    }
  }
  // Anchor: d_k(i0-1) by a direct (2K+1)-term sum, t ascending.
  for (int t = -K; t <= K; ++t) {
    const float a = lds(i0 - 1 + t);
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const float df = a - lds(i0 - 1 + t + k);
      d[k] = fmaf(df, df, d[k]);
    }
  }

  // Output cursor (supports the blocked layout of pl_nlm_row_pass_blocked).
  const int blk = g.dst_pos_block;
  int orem = blk - (s0 % blk);
  float* op = dst + (int64_t)(s0 / blk) * g.dst_block_stride + (int64_t)(s0 % blk) * dps;

  for (int sb = 0; sb < T; sb += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = sb + r;
      if (s >= T) break;
      const int i = i0 + s;
      // Entering samples for step s+1 (prefetched one step ahead): the ring
      // slot r advances by R = ST+1 positions.
      const float tf = ld(i + 1 + ST);
      const float tx = ld(i + 1 + K + ST);  // raw x_s (clamp range)
      const float tn = __fmul_rn(tx, sc);
      const float to = lds(i - K + ST);
      const float an_ = nr[r], ao = orr[r], fi = fr[r];
      const int kmax = EDGE ? min(S, n - 1 - i) : ST;
      float num = an[r];  // centre + j-side contributions so far
      float den = ad[r];
#pragma unroll
      for (int k = 1; k <= ST; ++k) {
        const int rk = (r + k) % R;
        const float dn = an_ - nr[rk];
        float dk = fmaf(dn, dn, d[k]);
        const float dq = ao - orr[rk];
        dk = fmaf(-dq, dq, dk);
        d[k] = dk;
        float w = ex2_approx(-dk);
        if (EDGE) w = (k <= kmax) ? w : 0.f;
        num = fmaf(w, fr[rk], num);
        den += w;
        an[rk] = fmaf(w, fi, an[rk]);
        ad[rk] += w;
      }
      if (i >= s0) {
        const float q = AP ? div_unscale(num, den, g.inv_scale) : div_fix(num, den);
        const float v = epi(g.avg, g.dst, op, fminf(fmaxf(q, lo), hi));
        *op = v;
        if (x0) x0[(int64_t)i * dps] = v;  // fan-out (unblocked layout only)
        if (x1) x1[(int64_t)i * dps] = v;
        op += dps;
        if (--orem == 0) {
          op += g.dst_block_stride - (int64_t)blk * dps;
          orem = blk;
        }
      }
      const float tfs = AP ? __fmul_rn(tf, sc) : tf;
      an[r] = tfs;  // pixel i + R enters slot r: centre term first
      ad[r] = 1.f;
      if (!pairs) {
        lo = fminf(lo, tf);
        hi = fmaxf(hi, tf);
      } else if (r & 1) {
        lo = min3f(lo, xprev, tx);
        hi = max3f(hi, xprev, tx);
      } else if (r == R - 1) {
        lo = fminf(lo, tx);
        hi = fmaxf(hi, tx);
      } else {
        xprev = tx;
      }
      fr[r] = tfs;
      nr[r] = tn;
      orr[r] = to;
    }
  }
}

template <int ST>
__global__ void __launch_bounds__(128) nlm_pass_kernel(PassDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.nseg) return;
  const int64_t line = w % g.n_lines;
  const int seg = g.seg_begin + (int)(w / g.n_lines);
  const int64_t img = line / g.lines_per_img;
  const int64_t li = line - img * g.lines_per_img;
  const float* src = g.src + img * g.src_img_stride + li * g.src_line_stride;
  float* dst = g.dst + img * g.dst_img_stride + li * g.dst_line_stride;
  const int s0 = seg * g.seg_len;
  const int s1 = min(g.n, s0 + g.seg_len);
  const int i0 = max(0, s0 - g.S);
  float* x[2] = {nullptr, nullptr};
  for (int k = 0; k < g.nx; ++k)
    if (li >= g.xlo[k] && li < g.xhi[k]) x[k] = g.xdst[k] + (li - g.xlo[k]) * g.dst_line_stride;
  const bool interior = (g.S == ST) && (i0 - 1 - g.K >= 0) && (s1 + g.K + g.S < g.n);
  if (interior)
    walk_segment<ST, false>(g, src, g.src_pos_stride, dst, g.dst_pos_stride, s0, s1, x[0], x[1]);
  else
    walk_segment<ST, true>(g, src, g.src_pos_stride, dst, g.dst_pos_stride, s0, s1, x[0], x[1]);
}

// ---------------------------------------------------------------------------
// Distance-band export: the SAME recurrence (anchor at i0-1, update (2)),
// writing d_k(i) into the BandedKernel cell layout instead of weighting it.
template <typename T>
__device__ __forceinline__ T band_cast(float v);
template <>
__device__ __forceinline__ float band_cast<float>(float v) { return v; }
template <>
__device__ __forceinline__ int32_t band_cast<int32_t>(float v) { return __float2int_rn(v); }

struct BandDesc {
  const float* src;
  void* band;
  int64_t n_lines, ld;
  int32_t n, seg_len, nseg;
  int32_t S;       // effective radius actually computed (<= template, <= n-1)
  int32_t S_band;  // radius of the band layout (requested S)
  int32_t K;
};

template <int ST, typename T>
__global__ void __launch_bounds__(128) distance_band_kernel(BandDesc g) {
  constexpr int R = ST + 1;
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.nseg) return;
  const int64_t line = w % g.n_lines;
  const int seg = (int)(w / g.n_lines);
  const float* src = g.src + line * g.ld;
  const int bw = 2 * g.S_band + 1;
  T* band = reinterpret_cast<T*>(g.band) + line * (int64_t)g.n * bw;
  const int n = g.n, S = g.S, K = g.K;
  const int s0 = seg * g.seg_len;
  const int s1 = min(n, s0 + g.seg_len);
  const int i0 = max(0, s0 - S);
  auto ld = [&](int p) -> float { return __ldg(src + mirror_pos(p, n)); };

  float nr[R], orr[R], d[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    nr[q] = ld(i0 + K + q);
    orr[q] = ld(i0 - 1 - K + q);
    d[q] = 0.f;
  }
  for (int t = -K; t <= K; ++t) {
    const float a = ld(i0 - 1 + t);
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const float df = a - ld(i0 - 1 + t + k);
      d[k] = fmaf(df, df, d[k]);
    }
  }
  for (int sb = 0; sb < s1 - i0; sb += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = sb + r;
      if (s >= s1 - i0) break;
      const int i = i0 + s;
      const float tn = ld(i + 1 + K + ST);
      const float to = ld(i - K + ST);
      const float an_ = nr[r], ao = orr[r];
      if (i >= s0) band[(int64_t)i * bw + g.S_band] = band_cast<T>(0.f);
#pragma unroll
      for (int k = 1; k <= ST; ++k) {
        const int rk = (r + k) % R;
        const float dn = an_ - nr[rk];
        float dk = fmaf(dn, dn, d[k]);
        const float dq = ao - orr[rk];
        dk = fmaf(-dq, dq, dk);
        d[k] = dk;
        if (k <= S && i + k < n) {
          if (i >= s0) band[(int64_t)i * bw + g.S_band + k] = band_cast<T>(dk);
          if (i + k >= s0 && i + k < s1) band[(int64_t)(i + k) * bw + g.S_band - k] = band_cast<T>(dk);
        }
      }
      nr[r] = tn;
      orr[r] = to;
    }
  }
}

}  // namespace plgpu

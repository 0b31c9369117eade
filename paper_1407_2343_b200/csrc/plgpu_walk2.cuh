// plgpu_walk2.cuh -- the production PatchLift-NLM pass kernel (sm_100a).
//
// Same per-line arithmetic as plgpu_walk.cuh (prescaled samples, anchor at
// i0-1, moving-sum update (2), one ex2 per unique pair, both endpoints
// accumulated, rcp division, range clamp) -- the two kernels give bitwise-identical outputs --
// but organised for the B200:
//
//  * A warp owns LW = 32*LINES lines x one segment.  With LINES = 2 every lane
//    carries two lines in lock-step and all FP32 work is packed f32x2
//    (FADD2 / FFMA2 / FMUL2: half the issue slots); the two MUFU.EX2 of a
//    pair-of-pairs write the halves of one register pair directly.
//  * Samples reach the register rings through a per-warp shared-memory ring
//    of SR positions x LW lines, filled by cp.async in chunks of CH positions,
//    NS chunks in flight, synchronised with __syncwarp only (no CTA barrier).
//    Column pass: rows of LW consecutive columns, 16-byte copies.  Row pass:
//    4-byte copies that TRANSPOSE on the fly into [position][line] with an
//    XOR swizzle (line ^ 2*(pos mod 16)) that makes both the scattered writes
//    and the LDS.64 reads bank-conflict-free.  Mirror extension happens in
//    the copy addressing, so the compute loop never branches on borders.
//  * Row-pass outputs go through a CH x LW shared ring and leave as 64-byte
//    row segments; column-pass outputs are one coalesced STG per step.
//
// Requirements (checked on the host): K <= 7 (2K < CH), template radius <= 32.
#pragma once

#include <cstdint>

#include "plgpu_walk.cuh"

namespace plgpu {

// ---------------------------------------------------------------- f32 / f32x2
struct F2 {
  unsigned long long r;
};

__device__ __forceinline__ F2 f2_make(float a, float b) {
  F2 o;
  asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(a), "f"(b));
  return o;
}
__device__ __forceinline__ void f2_split(F2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v.r));
}
// {a, v.hi}: the high half flows from v, so a ring slot whose high half is a
// constant keeps it in place instead of re-materialising it on every refill.
__device__ __forceinline__ F2 f2_set_lo(F2 v, float a) {
  F2 o;
  asm("{.reg .f32 l, h; mov.b64 {l, h}, %1; mov.b64 %0, {%2, h};}" : "=l"(o.r) : "l"(v.r), "f"(a));
  return o;
}

template <int LINES>
struct VecOps;

template <>
struct VecOps<1> {
  using V = float;
  static __device__ __forceinline__ V splat(float x) { return x; }
  static __device__ __forceinline__ V add(V a, V b) { return a + b; }
  static __device__ __forceinline__ V sub(V a, V b) { return a - b; }
  static __device__ __forceinline__ V mul(V a, V b) { return __fmul_rn(a, b); }  // never contracted
  static __device__ __forceinline__ V scale(V a, float s) { return __fmul_rn(a, s); }
  static __device__ __forceinline__ V fma(V a, V b, V c) { return fmaf(a, b, c); }
  static __device__ __forceinline__ V fms(V a, V b, V c) { return fmaf(-a, b, c); }  // c - a*b
  static __device__ __forceinline__ V ex2(V a) { return ex2_approx(a); }
  static __device__ __forceinline__ V ex2n(V a) { return ex2_approx(-a); }
  static __device__ __forceinline__ V zero_if(bool z, V a) { return z ? 0.f : a; }
  static __device__ __forceinline__ float lo(V a) { return a; }
  static __device__ __forceinline__ float hi(V a) { return a; }
  static __device__ __forceinline__ V div(V n, V d) { return div_fix(n, d); }
  static __device__ __forceinline__ V div_unscale(V n, V d, float inv_s) {
    return plgpu::div_unscale(n, d, inv_s);
  }
  static __device__ __forceinline__ V rcp(V a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
  }
  static __device__ __forceinline__ V lds(const float* p) { return *p; }
};

template <>
struct VecOps<2> {
  using V = F2;
  static __device__ __forceinline__ V splat(float x) { return f2_make(x, x); }
  static __device__ __forceinline__ V add(V a, V b) {
    V o;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
    return o;
  }
  static __device__ __forceinline__ V sub(V a, V b) {
    V o;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
    return o;
  }
  static __device__ __forceinline__ V mul(V a, V b) {
    V o;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
    return o;
  }
  static __device__ __forceinline__ V fma(V a, V b, V c) {
    V o;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
    return o;
  }
  // c - a*b: the scalar negations fold into FFMA2's operand-negate bit.
  static __device__ __forceinline__ V fms(V a, V b, V c) {
    V o;
    asm("{.reg .f32 l, h; .reg .b64 n; mov.b64 {l, h}, %1; neg.f32 l, l; neg.f32 h, h;"
        " mov.b64 n, {l, h}; fma.rn.f32x2 %0, n, %2, %3;}"
        : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
    return o;
  }
  static __device__ __forceinline__ V ex2(V a) {
    float x, y;
    f2_split(a, x, y);
    return f2_make(ex2_approx(x), ex2_approx(y));
  }
  // Sample prescale as two scalar mul.rn: ptxas contracts a packed
  // mul.rn.f32x2 into a following sub.rn.f32x2 (one FFMA2, one rounding less)
  // whenever the product has a single use, which would make the rounding of
  // a walker depend on its schedule.  Scalar mul.rn is never contracted.
  static __device__ __forceinline__ V scale(V a, float s) {
    float x, y;
    f2_split(a, x, y);
    return f2_make(__fmul_rn(x, s), __fmul_rn(y, s));
  }
  static __device__ __forceinline__ V ex2n(V a) {  // 2^-a (negation folds into MUFU)
    float x, y;
    f2_split(a, x, y);
    return f2_make(ex2_approx(-x), ex2_approx(-y));
  }
  static __device__ __forceinline__ V zero_if(bool z, V a) {
    V o;
    o.r = z ? 0ull : a.r;
    return o;
  }
  static __device__ __forceinline__ float lo(V a) {
    float x, y;
    f2_split(a, x, y);
    return x;
  }
  static __device__ __forceinline__ float hi(V a) {
    float x, y;
    f2_split(a, x, y);
    return y;
  }
  static __device__ __forceinline__ V rcp(V a) {
    float x, y, rx, ry;
    f2_split(a, x, y);
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rx) : "f"(x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ry) : "f"(y));
    return f2_make(rx, ry);
  }
  // packed div_fix (same arithmetic per half)
  static __device__ __forceinline__ V div(V n, V d) {
    const V r = rcp(d);
    return mul(n, r);
  }
  // num * (rcp(den) * (1/s)): plgpu_walk.cuh div_unscale per half
  static __device__ __forceinline__ V div_unscale(V n, V d, float inv_s) {
    return mul(n, mul(rcp(d), splat(inv_s)));
  }

  static __device__ __forceinline__ V lds(const float* p) {
    V o;
    o.r = *reinterpret_cast<const unsigned long long*>(p);
    return o;
  }
};

// ---------------------------------------------------------------- async copy
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct Pass2Desc {
  const float* src;
  float* dst;
  int64_t src_img_stride, src_line_stride, src_pos_stride;
  int64_t dst_img_stride, dst_line_stride, dst_pos_stride, dst_block_stride;
  int32_t dst_pos_block;
  int32_t lines_per_img;
  int32_t groups_per_img;
  int32_t n, seg_len, nseg, S, K;
  int32_t seg_begin;  // first processed segment (windowed passes; nseg counts from it)
  float scale;        // s = sqrt(log2 e) / h: sample prescale
  float inv_scale;    // 1 / s: output unscale where acc_prescaled(ST) (plgpu_walk.cuh)
  const float* avg;   // optional, dst layout (column passes): store (avg + out) / 2
  int32_t vec16;  // column pass: 16-byte copies legal (aligned, full line groups)
  int64_t total_warps;
  float coef;
  // Fan-out (pl_nlm_row_pass_fanout, batch 1): output lines [xlo[x], xhi[x])
  // are also stored at xdst[x] + (line - xlo[x]) * dst_line_stride + pos *
  // dst_pos_stride as they are produced -- e.g. into a peer GPU's window.
  float* xdst[2];
  int32_t xlo[2], xhi[2];
  int32_t nx;
  float* dexp;  // debug distance export (hot kernel only, see PassDesc)
};

constexpr int kCH = 16;  // positions per chunk
constexpr int kNS = 4;   // chunks in the ring
constexpr int kSR = kCH * kNS;
constexpr int kWarpsPerCta = 2;

template <int LINES, bool ROWS>
__host__ __device__ constexpr int pass2_smem_floats_per_warp() {
  return kSR * 32 * LINES + (ROWS ? 2 * kCH * 32 * LINES : 0);
}

// Swizzled slot of line l (0..LW-1) at ring position u (row pass only): the
// 16 positions of a chunk map line l to 16 distinct banks.
template <bool ROWS>
__device__ __forceinline__ int swz(int l, int u) {
  return ROWS ? (l ^ ((u & 15) << 1)) : l;
}

// Staging schedule (per warp, no CTA barrier).  Positions are ring
// coordinates u = p - pos0.  With base = ST + 2K + 2, chunk c holds
// u in [16c + base, 16c + base + 16); step s reads u in [s+1+ST, s+base], i.e.
// at most chunks floor(s/16)-1 and floor(s/16).  Step s copies piece s%16 of
// chunk floor(s/16)+2 (one cp.async group per step), so every chunk lands 17+
// steps before first use: wait_group(16) at the top of each step suffices,
// and the slot it overwrites (chunk floor(s/16)-2) was last read two chunks
// earlier (requires 2K < 16).
// KT >= 0: patch radius fixed at compile time; KT < 0: runtime K.  Three
// register rings of S+1 samples (f values, entering-term partners,
// leaving-term partners); three LDS per step.
template <int ST, int KT, int LINES, bool ROWS, bool EDGE>
__device__ __forceinline__ void walk2(const Pass2Desc& g, float* ring, const int lane,
                                      const int64_t wid) {
  using Ops = VecOps<LINES>;
  using V = typename Ops::V;
  constexpr int LW = 32 * LINES;
  constexpr int R = ST + 1;
  constexpr int P = R;  // body length (steps)
  float* oring = ring + kSR * LW;

  const int seg = g.seg_begin + (int)(wid % g.nseg);
  const int64_t grp = wid / g.nseg;
  const int64_t img = grp / g.groups_per_img;
  const int l0 = (int)(grp % g.groups_per_img) * LW;
  const int n = g.n;
  const int S = g.S;
  const int K = KT >= 0 ? KT : g.K;
  const int s0 = seg * g.seg_len;
  const int s1 = min(n, s0 + g.seg_len);
  const int i0 = max(0, s0 - S);
  const int T = s1 - i0;
  const int pos0 = i0 - 1 - K;   // ring coordinate u = p - pos0
  const int base = ST + 2 * K + 2;
  const float* src = g.src + img * g.src_img_stride;
  const int last_line = g.lines_per_img - 1;

  auto slot = [&](int u) -> float* { return ring + ((u - base) & (kSR - 1)) * LW; };

  // One piece (1/16) of chunk c; always commits one group.
  auto issue_piece = [&](int c, int j) {
    if constexpr (ROWS) {
      constexpr int LPP = LW / 16;  // lines per piece; 16 lanes (positions) per line
      const int u = 16 * c + base + (lane & 15);
      const float* col = src + (int64_t)(EDGE ? mirror_pos(pos0 + u, n) : pos0 + u) * g.src_pos_stride;
      float* row = slot(u);
#pragma unroll
      for (int h = 0; h < LPP / 2; ++h) {
        const int l = j * LPP + 2 * h + (lane >> 4);
        cp_async4(row + swz<true>(l, u), col + (int64_t)min(l0 + l, last_line) * g.src_line_stride);
      }
    } else {
      const int u = 16 * c + base + j;
      const float* rowp = src + (int64_t)(EDGE ? mirror_pos(pos0 + u, n) : pos0 + u) * g.src_pos_stride;
      float* dstrow = slot(u);
      if (g.vec16) {
        if (lane < LW / 4) cp_async16(dstrow + 4 * lane, rowp + l0 + 4 * lane);
      } else {
#pragma unroll
        for (int h = 0; h < LINES; ++h) {
          const int l = lane * LINES + h;
          cp_async4(dstrow + l, rowp + (int64_t)min(l0 + l, last_line) * g.src_line_stride);
        }
      }
    }
    cp_commit();
  };
  auto ld = [&](int u) -> V { return Ops::lds(slot(u) + swz<ROWS>(lane * LINES, u)); };

  // ---- prologue: chunks -m..0 (init window), then chunk 1
  const int m = (base + 15) / 16;
  for (int c = -m; c <= 0; ++c)
#pragma unroll 1
    for (int j = 0; j < 16; ++j) issue_piece(c, j);
  cp_wait<0>();
  __syncwarp();

  // Sample rings fr/nr/orr[(s+q) mod R] = samples at u = s+1+K+q, s+1+2K+q,
  // s+q; the distance-side rings nr/orr hold prescaled samples (plgpu_walk.cuh).
  constexpr bool AP = acc_prescaled(ST);
  V fr[R], nr[R], orr[R];
  V an[R], ad[R], d[R];
  const V zero = Ops::splat(0.f);
  auto lds = [&](int u) -> V { return Ops::scale(ld(u), g.scale); };
  float lo0 = 3.402823466e38f, hi0 = -3.402823466e38f, lo1 = lo0, hi1 = hi0;
  auto track = [&](V v) {
    lo0 = fminf(lo0, Ops::lo(v));
    hi0 = fmaxf(hi0, Ops::lo(v));
    lo1 = fminf(lo1, Ops::hi(v));
    hi1 = fmaxf(hi1, Ops::hi(v));
  };
  auto track2 = [&](V a, V b) {  // clamp-range rule: plgpu_walk.cuh
    lo0 = min3f(lo0, Ops::lo(a), Ops::lo(b));
    hi0 = max3f(hi0, Ops::lo(a), Ops::lo(b));
    lo1 = min3f(lo1, Ops::hi(a), Ops::hi(b));
    hi1 = max3f(hi1, Ops::hi(a), Ops::hi(b));
  };
  V xprev = zero;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    fr[q] = AP ? lds(q + 1 + K) : ld(q + 1 + K);  // accumulation side (plgpu_walk.cuh rule)
    nr[q] = lds(q + 1 + 2 * K);
    orr[q] = lds(q);
    d[q] = zero;
  }
  const V one = Ops::splat(1.f);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    track(ld(q + 1 + K));
    an[q] = fr[q];  // the centre sample (w = 1) starts each pixel's sums
    ad[q] = one;
  }
  const bool pairs = clamp_pairs(K, ST);  // clamp-range rule: plgpu_walk.cuh
  if (pairs)
    for (int q = R - K; q < R; ++q) track(ld(q + 1 + 2 * K));  // rest of [i0, i0 + K + ST]
#pragma unroll 1
  for (int t = 0; t <= 2 * K; ++t) {  // anchor d_k(i0-1), t ascending
    const V a = lds(t);
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const V df = Ops::sub(a, lds(t + k));
      d[k] = Ops::fma(df, df, d[k]);
    }
  }
  __syncwarp();
#pragma unroll 1
  for (int j = 0; j < 16; ++j) issue_piece(1, j);

  const int64_t dst_img = img * g.dst_img_stride;
  const int my_line = l0 + lane * LINES;
  float* op = g.dst + dst_img + (int64_t)my_line * g.dst_line_stride + (int64_t)s0 * g.dst_pos_stride;

  // Row pass: flush piece j (lines j*LW/16 ..) of output chunk k, positions < qend.
  auto flush_piece = [&](int k, int j, int qend) {
    constexpr int LPP = LW / 16;
    const int q = lane & 15;
    const int p = s0 + 16 * k + q;
    const int blk = g.dst_pos_block;
    const float* orow = oring + ((k & 1) * kCH + q) * LW;
    if (q < qend) {
      const int64_t pofs = (int64_t)(p / blk) * g.dst_block_stride + (int64_t)(p % blk) * g.dst_pos_stride;
#pragma unroll
      for (int h = 0; h < LPP / 2; ++h) {
        const int l = j * LPP + 2 * h + (lane >> 4);
        if (l0 + l <= last_line)
          g.dst[dst_img + (int64_t)(l0 + l) * g.dst_line_stride + pofs] = orow[swz<true>(l, q)];
      }
    }
  };

  for (int sb = 0; sb < T; sb += P) {
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int s = sb + r;
      if (s >= T) break;
      const int i = i0 + s;
      const int ra = r % R;  // accumulator ring slot of pixel i
      cp_wait<16>();
      __syncwarp();
      // ring refills (shared-memory latency hides behind the step)
      const V tf = ld(s + 2 + K + ST);
      const V tx = ld(s + base);  // raw x_s (clamp range)
      const V tn = Ops::scale(tx, g.scale);
      const V to = lds(s + 1 + ST);
      const V an_ = nr[ra], ao = orr[ra], fi = fr[ra];
      const int kmax = EDGE ? min(S, n - 1 - i) : ST;
      V num = an[ra];  // centre + j-side contributions so far
      V den = ad[ra];
#pragma unroll
      for (int k = 1; k <= ST; ++k) {
        const int rk = (ra + k) % R;
        const V pn = nr[rk], po = orr[rk], pf = fr[rk];
        const V dn = Ops::sub(an_, pn);
        V dk = Ops::fma(dn, dn, d[k]);
        const V dq = Ops::sub(ao, po);
        dk = Ops::fms(dq, dq, dk);
        d[k] = dk;
        V w = Ops::ex2n(dk);
        if constexpr (EDGE) w = Ops::zero_if(k > kmax, w);
        num = Ops::fma(w, pf, num);
        den = Ops::add(w, den);
        an[rk] = Ops::fma(w, fi, an[rk]);
        ad[rk] = Ops::add(w, ad[rk]);
      }
      const int o = i - s0;
      if (o >= 0) {
        const V qv = AP ? Ops::div_unscale(num, den, g.inv_scale) : Ops::div(num, den);
        const float o0 = fminf(fmaxf(Ops::lo(qv), lo0), hi0);
        float o1 = o0;
        if constexpr (LINES == 2) o1 = fminf(fmaxf(Ops::hi(qv), lo1), hi1);
        if constexpr (ROWS) {
          const int q = o & (kCH - 1);
          float* sl = oring + (((o >> 4) & 1) * kCH + q) * LW + swz<true>(lane * LINES, q);
          if constexpr (LINES == 2) *reinterpret_cast<float2*>(sl) = make_float2(o0, o1);
          else *sl = o0;
          if (o >= kCH) flush_piece((o >> 4) - 1, q, kCH);
        } else {
          if constexpr (LINES == 2) {
            if (g.vec16) {
              float2 v = make_float2(o0, o1);
              if (g.avg) {
                const float2 a = __ldg(reinterpret_cast<const float2*>(g.avg + (op - g.dst)));
                v = make_float2((a.x + o0) / 2.0f, (a.y + o1) / 2.0f);
              }
              *reinterpret_cast<float2*>(op) = v;
            } else {
              if (my_line <= last_line) op[0] = epi(g.avg, g.dst, op, o0);
              if (my_line + 1 <= last_line)
                op[g.dst_line_stride] = epi(g.avg, g.dst, op + g.dst_line_stride, o1);
            }
          } else {
            if (my_line <= last_line) *op = epi(g.avg, g.dst, op, o0);
          }
          op += g.dst_pos_stride;
        }
      }
      const V tfs = AP ? Ops::scale(tf, g.scale) : tf;
      an[ra] = tfs;  // pixel i + R enters slot ra: centre term first
      ad[ra] = one;
      if (!pairs) track(tf);
      else if (ra & 1) track2(xprev, tx);
      else if (ra == R - 1) track(tx);
      else xprev = tx;
      fr[ra] = tfs;
      nr[ra] = tn;
      orr[ra] = to;
      issue_piece((s >> 4) + 2, s & 15);
    }
  }
  if constexpr (ROWS) {  // tail of the output ring
    __syncwarp();
    const int olast = s1 - 1 - s0;
    const int kl = olast >> 4, jl = olast & 15;
    if (kl >= 1)
#pragma unroll 1
      for (int j = jl + 1; j < 16; ++j) flush_piece(kl - 1, j, kCH);
#pragma unroll 1
    for (int j = 0; j < 16; ++j) flush_piece(kl, j, jl + 1);
  }
  cp_wait<0>();
}

template <int ST, int KT, int LINES, bool ROWS>
__global__ void __launch_bounds__(32 * kWarpsPerCta) nlm_pass2_kernel(const Pass2Desc g) {
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * kWarpsPerCta + wib;
  if (wid >= g.total_warps) return;
  float* ring = smem + wib * pass2_smem_floats_per_warp<LINES, ROWS>();
  // Interior segments (the bulk) need neither mirrored staging nor pair
  // masking: everything the warp ever stages lies inside the line.
  const int seg = g.seg_begin + (int)(wid % g.nseg);
  const int s0 = seg * g.seg_len;
  const int s1 = min(g.n, s0 + g.seg_len);
  const int K = KT >= 0 ? KT : g.K;
  const int pos0 = max(0, s0 - g.S) - 1 - K;
  const bool interior = g.S == ST && pos0 >= 0 && s1 + 2 * ST + 2 * K + 80 <= g.n;
  if (interior)
    walk2<ST, KT, LINES, ROWS, false>(g, ring, lane, wid);
  else
    walk2<ST, KT, LINES, ROWS, true>(g, ring, lane, wid);
}

}  // namespace plgpu

// plgpu_walk3.cuh -- the hot-configuration PatchLift-NLM pass kernel (sm_100a).
//
// Same per-line arithmetic as plgpu_walk.cuh / plgpu_walk2.cuh (bitwise equal
// outputs), specialised for a compile-time patch radius KT so that the whole
// shared-memory traffic uses immediate offsets:
//
//  * staging chunks are exactly R = S+1 positions, i.e. one unrolled body
//    iteration (R steps) consumes one chunk.  Chunk c holds ring coordinates
//    u in [cR + BASE, cR + BASE + R), BASE = S + 2K + 2.  Iteration c reads
//    only chunks c-1 and c (needs 2K+2 <= R), so every sample load is
//    "row pointer of chunk c-1 or c + compile-time offset".
//  * NS = 4 chunk slots: at iteration c the warp copies chunk c+2 (cp.async,
//    one group) into the slot of chunk c-2 and waits for chunk c
//    (wait_group 2): a full iteration of latency hiding, no CTA barrier.
//  * Row pass: the copy transposes 64 lines x R positions into rows of
//    PITCH = LW + 2 floats; 16 lanes write 16 consecutive positions of one line
//    -> banks (2u + l) mod 32 are distinct, and the compute reads (LDS.64 of
//    lines 2l, 2l+1) are contiguous.  Outputs are staged the same way and
//    leave once per iteration as contiguous row pieces.
//  * Interior segments (no mirror, no clipped windows) run the EDGE = false
//    instantiation; the scheduler places all interior warps before the edge
//    warps so each SM's instruction cache holds one variant at a time.
#pragma once

#include <cstdint>

#include "plgpu_walk2.cuh"

namespace plgpu {

constexpr int kNS3 = 4;

template <int ST, int LINES, bool ROWS>
__host__ __device__ constexpr int pass3_smem_floats_per_warp() {
  return kNS3 * (ST + 1) * (32 * LINES + (ROWS ? 2 : 0)) +
         (ROWS ? (ST + 1) * (32 * LINES + 2) : 0);
}

struct Pass3Desc {
  Pass2Desc b;          // geometry (strides, lines, segments, coef, S, K)
  int32_t seg_lo, seg_hi;  // interior segment range [seg_lo, seg_hi]
  int64_t interior_warps;  // groups * (seg_hi - seg_lo + 1)
};

template <int ST, int KT, int LINES, bool ROWS, bool EDGE>
__device__ __forceinline__ void walk3(const Pass2Desc& g, float* ring, const int lane,
                                      const int64_t grp, const int seg) {
  using Ops = VecOps<LINES>;
  using V = typename Ops::V;
  constexpr int LW = 32 * LINES;
  constexpr int R = ST + 1;
  constexpr int BASE = ST + 2 * KT + 2;
  constexpr int PITCH = LW + (ROWS ? 2 : 0);
  constexpr int CHUNK = R * PITCH;  // floats per chunk slot
  constexpr int M = (BASE + R - 1) / R;  // chunks before chunk 0 (init window)
  static_assert(2 * KT + 2 <= R, "iteration must read at most two chunks");
  static_assert(M <= 2, "prologue must fit the ring");
  float* oring = ring + kNS3 * CHUNK;

  const int64_t img = grp / g.groups_per_img;
  const int l0 = (int)(grp % g.groups_per_img) * LW;
  const int n = g.n;
  const int S = EDGE ? g.S : ST;
  const int s0 = seg * g.seg_len;
  const int s1 = min(n, s0 + g.seg_len);
  const int i0 = max(0, s0 - S);
  const int T = s1 - i0;
  const int pos0 = i0 - 1 - KT;  // ring coordinate u = p - pos0
  const float* src = g.src + img * g.src_img_stride;
  const int last_line = g.lines_per_img - 1;
  const int nchunks = (T + R - 1) / R;  // body iterations

  auto slot = [&](int c) -> float* { return ring + (c & (kNS3 - 1)) * CHUNK; };
  // Copy chunk c (positions u = cR + BASE + q, q < R); always commits a group.
  // Positions with u < 0 (ahead of the anchor) are never read and not copied.
  auto issue_chunk = [&](int c) {
    if (c <= nchunks - 1) {
      float* dstc = slot(c);
      const int ubase = c * R + BASE;
      if constexpr (ROWS) {
        // lanes 0..15 -> 16 consecutive positions of line 2j, lanes 16..31 -> line 2j+1
#pragma unroll
        for (int qb = 0; qb < R; qb += 16) {
          const int q = qb + (lane & 15);
          if (q < R && ubase + q >= 0) {
            const int p = pos0 + ubase + q;
            const float* col = src + (int64_t)(EDGE ? mirror_pos(p, n) : p) * g.src_pos_stride;
            float* drow = dstc + q * PITCH;
#pragma unroll 4
            for (int j = 0; j < LW / 2; ++j) {
              const int l = 2 * j + (lane >> 4);
              const int line = min(l0 + l, last_line);  // partial line groups
              cp_async4(drow + l, col + (int64_t)line * g.src_line_stride);
            }
          }
        }
      } else {
#pragma unroll 4
        for (int q = 0; q < R; ++q) {
          if (ubase + q < 0) continue;
          const int p = pos0 + ubase + q;
          const float* rowp = src + (int64_t)(EDGE ? mirror_pos(p, n) : p) * g.src_pos_stride;
          if (g.vec16) {
            if (lane < LW / 4) cp_async16(dstc + q * PITCH + 4 * lane, rowp + l0 + 4 * lane);
          } else {
#pragma unroll
            for (int h = 0; h < LINES; ++h) {
              const int l = lane * LINES + h;
              cp_async4(dstc + q * PITCH + l, rowp + (int64_t)min(l0 + l, last_line) * g.src_line_stride);
            }
          }
        }
      }
    }
    cp_commit();
  };

  // ---- prologue: chunks -M..1; the init window u in [0, BASE) lies in -M..-1
  for (int c = -M; c <= 1; ++c) issue_chunk(c);
  cp_wait<1>();  // chunks -M..0 landed
  __syncwarp();
  // sample at ring coordinate u < BASE + R (chunks -M..0), compile-time u
  auto ld_init = [&](int u) -> V {
    const int c = (u - BASE + M * R) / R - M;  // floor((u - BASE) / R)
    return Ops::lds(slot(c) + (u - BASE - c * R) * PITCH + lane * LINES);
  };
  V fr[R], nr[R], orr[R], an[R], ad[R], d[R];
  const V zero = Ops::splat(0.f);
  float lo0 = 3.402823466e38f, hi0 = -3.402823466e38f, lo1 = lo0, hi1 = hi0;
  auto track = [&](V v) {
    lo0 = fminf(lo0, Ops::lo(v));
    hi0 = fmaxf(hi0, Ops::lo(v));
    lo1 = fminf(lo1, Ops::hi(v));
    hi1 = fmaxf(hi1, Ops::hi(v));
  };
#pragma unroll
  for (int q = 0; q < R; ++q) {
    fr[q] = ld_init(q + 1 + KT);
    nr[q] = ld_init(q + 1 + 2 * KT);
    orr[q] = ld_init(q);
    an[q] = zero;
    ad[q] = zero;
    d[q] = zero;
    track(fr[q]);
  }
#pragma unroll
  for (int t = 0; t <= 2 * KT; ++t) {  // anchor d_k(i0-1), t ascending
    const V a = ld_init(t);
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const V df = Ops::sub(a, ld_init(t + k));
      d[k] = Ops::fma(df, df, d[k]);
    }
  }

  const V coefv = Ops::splat(g.coef);
  const V one = Ops::splat(1.f);
  const int64_t dst_img = img * g.dst_img_stride;
  const int my_line = l0 + lane * LINES;
  float* op = g.dst + dst_img + (int64_t)my_line * g.dst_line_stride + (int64_t)i0 * g.dst_pos_stride;

  for (int c = 0; c < nchunks; ++c) {
    __syncwarp();       // all lanes done with chunk c-2 (iteration c-1)
    issue_chunk(c + 2);  // into the slot of chunk c-2
    cp_wait<2>();       // chunk c landed
    __syncwarp();
    const float* prv = slot(c - 1) + lane * LINES;
    const float* cur = slot(c) + lane * LINES;
    // sample at ring coordinate s + off for body step r (all compile-time but c)
    auto at = [&](int r, int off) -> V {
      const int q = r + off - BASE;  // relative to chunk c's first position
      return q >= 0 ? Ops::lds(cur + q * PITCH) : Ops::lds(prv + (q + R) * PITCH);
    };
    const int sb = c * R;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = sb + r;
      // Interior segments walk a whole number of iterations (the segment
      // length is chosen so that C + S is a multiple of S+1): no per-step exit,
      // so the scheduler overlaps consecutive steps.
      if (EDGE && s >= T) break;
      const int i = i0 + s;
      const V tf = at(r, 2 + KT + ST);
      const V tn = at(r, BASE);
      const V to = at(r, 1 + ST);
      const V an_ = nr[r], ao = orr[r], fi = fr[r];
      const int kmax = EDGE ? min(S, n - 1 - i) : ST;
      V num = Ops::add(an[r], fi);
      V den = Ops::add(ad[r], one);
#pragma unroll
      for (int k = 1; k <= ST; ++k) {
        const int rk = (r + k) % R;
        const V dn = Ops::sub(an_, nr[rk]);
        V dk = Ops::fma(dn, dn, d[k]);
        const V dq = Ops::sub(ao, orr[rk]);
        dk = Ops::fms(dq, dq, dk);
        d[k] = dk;
        V w = Ops::ex2(Ops::mul(dk, coefv));
        if constexpr (EDGE) w = Ops::zero_if(k > kmax, w);
        num = Ops::fma(w, fr[rk], num);
        den = Ops::add(w, den);
        an[rk] = Ops::fma(w, fi, an[rk]);
        ad[rk] = Ops::add(w, ad[rk]);
      }
      const V qv = Ops::div(num, den);
      const float o0 = fminf(fmaxf(Ops::lo(qv), lo0), hi0);
      float o1 = o0;
      if constexpr (LINES == 2) o1 = fminf(fmaxf(Ops::hi(qv), lo1), hi1);
      if constexpr (ROWS) {
        float* sl = oring + r * PITCH + lane * LINES;
        if constexpr (LINES == 2) *reinterpret_cast<float2*>(sl) = make_float2(o0, o1);
        else *sl = o0;
      } else if (i >= s0) {
        if constexpr (LINES == 2) {
          if (g.vec16) {
            *reinterpret_cast<float2*>(op) = make_float2(o0, o1);
          } else {
            if (my_line <= last_line) op[0] = o0;
            if (my_line + 1 <= last_line) op[g.dst_line_stride] = o1;
          }
        } else {
          if (my_line <= last_line) *op = o0;
        }
      }
      if constexpr (!ROWS) op += g.dst_pos_stride;
      an[r] = zero;
      ad[r] = zero;
      track(tf);
      fr[r] = tf;
      nr[r] = tn;
      orr[r] = to;
    }
    if constexpr (ROWS) {
      // flush this iteration's outputs: positions p = i0 + sb + q, q < R
      __syncwarp();
#pragma unroll
      for (int qb = 0; qb < R; qb += 16) {
        const int q = qb + (lane & 15);
        const int p = i0 + sb + q;
        if (q < R && p >= s0 && p < s1) {
          const int blk = g.dst_pos_block;
          const int64_t pofs =
              (int64_t)(p / blk) * g.dst_block_stride + (int64_t)(p % blk) * g.dst_pos_stride;
          float* dbase = g.dst + dst_img + pofs;
          const float* orow = oring + q * PITCH;
#pragma unroll 4
          for (int j = 0; j < LW / 2; ++j) {
            const int l = 2 * j + (lane >> 4);
            if (l0 + l <= last_line)
              dbase[(int64_t)(l0 + l) * g.dst_line_stride] = orow[l];
          }
        }
      }
    }
  }
  cp_wait<0>();
}

// Minimum resident CTAs per SM: caps registers so that three warps fit each
// SM sub-partition's 16K-register file (<= 168 regs) where the ring state allows.
template <int ST, int LINES>
constexpr int pass3_min_blocks() { return 1; }

template <int ST, int KT, int LINES, bool ROWS>
__global__ void __launch_bounds__(32 * kWarpsPerCta, (pass3_min_blocks<ST, LINES>()))
    nlm_pass3_kernel(const Pass3Desc d) {
  extern __shared__ __align__(16) float smem[];
  const Pass2Desc& g = d.b;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * kWarpsPerCta + wib;
  if (wid >= g.total_warps) return;
  float* ring = smem + wib * pass3_smem_floats_per_warp<ST, LINES, ROWS>();
  const int n_int = max(0, d.seg_hi - d.seg_lo + 1);
  if (wid < d.interior_warps) {  // interior segments first
    walk3<ST, KT, LINES, ROWS, false>(g, ring, lane, wid / n_int, d.seg_lo + (int)(wid % n_int));
  } else {
    const int n_edge = g.nseg - n_int;
    const int64_t e = wid - d.interior_warps;
    int sidx = (int)(e % n_edge);
    if (n_int > 0 && sidx >= d.seg_lo) sidx += n_int;
    walk3<ST, KT, LINES, ROWS, true>(g, ring, lane, e / n_edge, sidx);
  }
}

}  // namespace plgpu

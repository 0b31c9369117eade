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
//    leave once per iteration as contiguous row pieces.  The 2-line
//    transposed-intermediate passes (io 2) copy 4 positions x 8 lines per
//    instruction instead (immediate position offsets, one address add per
//    8 lines; pitch LW + 8).
//  * One instantiation per configuration: chunks inside the line take the fast
//    copy path, chunks touching a line end the mirrored one (per chunk, at run
//    time); every iteration that needs no window clipping runs the branch-free
//    unmasked body, only the last partial/clipped iteration of a line runs the
//    masked body (per-step exit, weight 0 for pairs beyond the line end).
#pragma once

#include <cstdint>
#include <type_traits>

#include "plgpu_walk2.cuh"


// Build-variant knobs (tools/build_variant.py -D...): compile-time A/B switches
// behind the measured tables of profiles/README.md.  The defaults are the
// shipped kernels; none is read at run time and none changes a result bit.
#ifndef PLGPU_PK1
#define PLGPU_PK1 1  // 1-line kernels: {num, den} packed (FFMA2); 0 = scalar accumulators
#endif

#ifndef PLGPU_PK_REFILL_RING
#define PLGPU_PK_REFILL_RING 1  // packed 1-line form with prescaled sums: refill {x', 1} from the nr ring (else LDS + scale)
#endif
// refill loads issued ahead of the step's pair loop, per template radius:
// bit 0 = entering f, bit 1 = leaving partner, bit 2 = entering x
#ifndef PLGPU_EARLY_S10
#define PLGPU_EARLY_S10 0
#endif
#ifndef PLGPU_EARLY_S15
#define PLGPU_EARLY_S15 7
#endif
#ifndef PLGPU_EARLY_S25
#define PLGPU_EARLY_S25 0
#endif
#ifndef PLGPU_LOCK_WPC
#define PLGPU_LOCK_WPC 8   // warps per lockstep CTA
#endif
#ifndef PLGPU_LOCK_MINB
#define PLGPU_LOCK_MINB 1  // resident lockstep CTAs per SM the register budget allows
#endif

namespace plgpu {

constexpr int kNS3 = 4;
constexpr int kLockWpc = PLGPU_LOCK_WPC;

// Per warp: NS staging chunks + one output chunk, R rows each; rounded up to
// 16 bytes so every warp's ring (and its 16-byte flush rows) stays aligned.
// 2-line io-2 staging copies 4 positions x 8 lines per instruction (c4:
// +2 %); with 1 line per lane it measured slower (c3 -2 %, c5 -11 %).
template <int LINES, int IO>
__host__ __device__ constexpr bool pass3_copy8x4() {
  return IO == 2 && LINES == 2;
}
// Row pitch of the staging ring: io 0 rows of LW lines; the transposing
// copies of 16 positions x 2 lines (io 1, 1-line io 2) and the row flush are
// conflict-free at LW + 2, the 4-positions x 8-lines copies at LW + 8.
template <int LINES, int IO>
__host__ __device__ constexpr int pass3_pitch() {
  return 32 * LINES + (pass3_copy8x4<LINES, IO>() ? 8 : IO != 0 ? 2 : 0);
}
// Output ring pitch: padded (conflict-free transposed reads) only for the
// row-mode flush; the column flushes read whole dense rows.
template <int LINES, int IO>
__host__ __device__ constexpr int pass3_opitch() {
  return IO == 1 ? pass3_pitch<LINES, IO>() : 32 * LINES;
}
template <int ST, int LINES, int IO>
__host__ __device__ constexpr int pass3_smem_floats_per_warp() {
  return ((kNS3 + 1) * (ST + 1) * pass3_pitch<LINES, IO>() + 3) / 4 * 4;
}

struct Pass3Desc {
  Pass2Desc b;          // geometry (strides, lines, segments, coef, S, K)
  int32_t lines;        // lines per lane (1 or 2); b.total_warps / groups follow it
  int32_t wpc;          // warps per CTA: 2 (independent) or 8 (lockstep)
  int32_t seg_lo, seg_hi;  // segments (relative to b.seg_begin) needing no clipping (S > 16)
  int64_t interior_warps;  // groups * (seg_hi - seg_lo + 1)
};

// Interior/edge split (two bodies in two instantiations) for radii whose
// unrolled body is large enough that carrying the masked copy in the same
// kernel costs instruction-cache hits.
__host__ __device__ constexpr bool pass3_split(int ST) { return ST > 16; }  // S=15 split measured slower

// MODE 0: unified (per-chunk mirror check, per-iteration masked/unmasked
// body).  MODE 1: interior segment only (no mirrored staging, no masked body
// compiled: smaller code for large S).  MODE 2: edge segment (always masked).
// IO: 0 = column staging + column flush (lines contiguous on both sides);
// 1 = row staging + row flush (positions contiguous on both sides);
// 2 = row staging + column flush (positions contiguous in the source, lines
// contiguous in the destination: the transposed-intermediate RC composite).
// EXP (debug instantiation, pl_debug_hot_distance_band): every distance the
// walk computes for a pixel of this segment is also stored into g.dexp, so
// the exactness of the code that actually runs can be checked (with the
// prescale set to 1 the recurrence runs on the raw samples).
// base + q * stride as one 32x32 -> 64-bit multiply-add (IMAD.WIDE.U32; with q
// a compile-time constant after unrolling ptxas takes it as an immediate).
template <typename T>
__device__ __forceinline__ T* mad_wide_u32(uint32_t q, uint32_t stride, T* base) {
  T* r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(q), "r"(stride), "l"(base));
  return r;
}

__device__ __forceinline__ void st_global_f2(void* p, float2 v) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

template <int ST, int KT, int LINES, int IO, int MODE = 0, bool AVG = false, bool EXP = false>
__device__ __forceinline__ void walk3(const Pass2Desc& g, float* ring, const int lane,
                                      const int64_t grp, const int seg, const int bar_threads = 0) {
  constexpr bool ROWS = IO != 0;   // transposing (row-mode) staging
  constexpr bool OROWS = IO == 1;  // row-mode output flush
  using Ops = VecOps<LINES>;
  using V = typename Ops::V;
  constexpr int LW = 32 * LINES;
  constexpr int R = ST + 1;
  constexpr int BASE = ST + 2 * KT + 2;
  constexpr int PITCH = pass3_pitch<LINES, IO>();
  constexpr int CHUNK = R * PITCH;  // floats per chunk slot
  constexpr int M = (BASE + R - 1) / R;  // chunks before chunk 0 (init window)
  static_assert(2 * KT + 2 <= R, "iteration must read at most two chunks");
  static_assert(M <= 2, "prologue must fit the ring");
  float* const oring = ring + kNS3 * CHUNK;
  constexpr int OPITCH = pass3_opitch<LINES, IO>();

  const int64_t img = grp / g.groups_per_img;
  const int l0 = (int)(grp % g.groups_per_img) * LW;
  const int n = g.n;
  const int S = g.S;  // effective radius (<= ST; pairs with k > S are masked)
  const int s0 = seg * g.seg_len;
  const int s1 = min(n, s0 + g.seg_len);
  const int i0 = max(0, s0 - S);
  const int T = s1 - i0;
  const int pos0 = i0 - 1 - KT;  // ring coordinate u = p - pos0
  const float* src = g.src + img * g.src_img_stride;
  const int last_line = g.lines_per_img - 1;
  const int nchunks = (T + R - 1) / R;  // body iterations
  const bool full_group = l0 + LW - 1 <= last_line;
  // fan-out lines in this group (warp-uniform; row flush only)
  bool fan = false;
  for (int x = 0; x < g.nx; ++x) fan |= l0 < g.xhi[x] && l0 + LW > g.xlo[x];
  // Column pass with 2 lines per lane: every lane stages (8-byte copies) and
  // flushes exactly the lines it computes -> no warp barriers around the ring.
  // (the host routes 2-line column-flush passes here only when they are
  // 16-byte aligned with whole line groups, g.vec16; otherwise to walk2)
  constexpr bool own = !ROWS && LINES == 2;
  // column-mode flush where each lane stores exactly the lines it computed
  // 2-line column flush: each lane stores its own two lines from registers
  // (no output ring, no warp barrier)
  constexpr bool oown = !OROWS && LINES == 2;

  auto slot = [&](int c) -> float* { return ring + (c & (kNS3 - 1)) * CHUNK; };
  // Copy chunk c (positions u = cR + BASE + q, q < R); always commits a group.
  // Positions with u < 0 (ahead of the anchor) are never read and not copied.
  // Chunks entirely inside the line take the fast path (incremental 64-bit
  // addresses); chunks touching a line end use the half-sample mirror.
  const int lane16 = lane & 15, half = lane >> 4;
  const int64_t ps = g.src_pos_stride, ls = g.src_line_stride;
  const float* rows_base = src + (int64_t)min(l0 + half, last_line) * ls;
  auto issue_chunk = [&](int c) {
    if (c <= nchunks - 1) {
      float* dstc = slot(c);
      const int ubase = c * R + BASE;
      const int pfirst = pos0 + ubase;
      const bool inside = MODE == 1 || (MODE == 0 && pfirst >= 0 && pfirst + R - 1 <= n - 1);
      if constexpr (ROWS) {
#pragma unroll
        for (int qb = 0; qb < R; qb += 16) {
          const int q = qb + lane16;
          if (q < R && ubase + q >= 0) {
            const int p = pfirst + q;
            float* drow = dstc + q * PITCH + half;
            if (inside && full_group && !pass3_copy8x4<LINES, IO>()) {
              const float* gp = rows_base + p;
#pragma unroll 8
              for (int j = 0; j < LW / 2; ++j) {
                cp_async4(drow + 2 * j, gp);
                gp += 2 * ls;
              }
            } else if (!(inside && full_group)) {
              const float* col = src + (int64_t)mirror_pos(p, n) * ps;
#pragma unroll 4
              for (int j = 0; j < LW / 2; ++j)
                cp_async4(drow + 2 * j, col + (int64_t)min(l0 + 2 * j + half, last_line) * ls);
            }
          }
        }
        if (pass3_copy8x4<LINES, IO>() && inside && full_group) {
          // 4 positions x 8 lines per copy instruction (pp = lane & 3,
          // lg = lane >> 2): the positions step by immediate offsets, the
          // lines by one 64-bit add per 8-line group; 8-16 L1 sectors per copy
          const int pp = lane & 3, lg = lane >> 2;
          const float* gl = src + (int64_t)(l0 + lg) * ls + pfirst + pp;
          float* dl = dstc + pp * PITCH + lg;
          const int64_t gstep = 8 * ls;
#pragma unroll
          for (int g8 = 0; g8 < LW / 8; ++g8) {
#pragma unroll
            for (int t = 0; t < (R + 3) / 4; ++t) {
              const int q = 4 * t + pp;
              if (q < R && ubase + q >= 0) cp_async4(dl + 4 * t * PITCH, gl + 4 * t);
            }
            gl += gstep;
            dl += 8;
          }
        }
      } else if (own) {
        float* dp = dstc + LINES * lane;
        if (inside) {
          const float* gp = src + (int64_t)pfirst * ps + l0 + LINES * lane;
#pragma unroll
          for (int q = 0; q < R; ++q) {
            if (ubase + q >= 0) cp_async8(dp, gp);
            gp += ps;
            dp += PITCH;
          }
        } else {
#pragma unroll 4
          for (int q = 0; q < R; ++q) {
            if (ubase + q >= 0)
              cp_async8(dp, src + (int64_t)mirror_pos(pfirst + q, n) * ps + l0 + LINES * lane);
            dp += PITCH;
          }
        }
      } else if (g.vec16) {
        // one line per lane: 16-byte copies, 32*16/(4*LW) position rows per instruction
        constexpr int LPR = LW / 4, RPI = 32 / LPR;
        const int qo = lane / LPR;
        float* dp = dstc + qo * PITCH + 4 * (lane % LPR);
#pragma unroll
        for (int qb = 0; qb < R; qb += RPI) {
          const int q = qb + qo;
          if (q < R && ubase + q >= 0) {
            const int p = inside ? pfirst + q : mirror_pos(pfirst + q, n);
            cp_async16(dp, src + (int64_t)p * ps + l0 + 4 * (lane % LPR));
          }
          dp += RPI * PITCH;
        }
      } else {
#pragma unroll 4
        for (int q = 0; q < R; ++q) {
          if (ubase + q < 0) continue;
          const float* rowp = src + (int64_t)mirror_pos(pfirst + q, n) * ps;
#pragma unroll
          for (int h = 0; h < LINES; ++h) {
            const int l = lane * LINES + h;
            cp_async4(dstc + q * PITCH + l, rowp + (int64_t)min(l0 + l, last_line) * ls);
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
  // LINES == 2: two lines per lane, all state packed line-wise (f32x2).
  // LINES == 1: one line per lane; the numerator/denominator pairs are packed
  // instead, {num, den} += w * {f, 1} being one FFMA2 (w broadcast), and the
  // f ring holds {f, 1} pairs.  Same per-line arithmetic either way.
  constexpr bool PK = LINES == 1 && PLGPU_PK1;
  // Accumulation form (plgpu_walk.cuh acc_prescaled, a function of ST): for
  // ST <= 10 the sums take the prescaled samples x' -- the sample at position
  // i + k is already in the distance rings, so the 2-line kernel keeps no
  // separate f ring (22 registers and one LDS.64 per step less, c4 +1.5 %) and
  // the packed 1-line form keeps {x', 1} pairs; larger radii keep the raw f.
  constexpr bool AP = acc_prescaled(ST);
  V fr[(PK || AP) ? 1 : R], an[PK ? 1 : R], ad[PK ? 1 : R];
  V nr[R], orr[R], d[R];
  F2 frp[PK ? R : 1], acc[PK ? R : 1];
  const V zero = Ops::splat(0.f);
  const float sv = g.scale;
  const V svv = Ops::splat(sv);
  auto sc = [&](V v) -> V { return Ops::scale(v, sv); };  // distance-side sample
  float lo0 = 3.402823466e38f, hi0 = -3.402823466e38f, lo1 = lo0, hi1 = hi0;
  auto track = [&](V v) {
    lo0 = fminf(lo0, Ops::lo(v));
    hi0 = fmaxf(hi0, Ops::lo(v));
    lo1 = fminf(lo1, Ops::hi(v));
    hi1 = fmaxf(hi1, Ops::hi(v));
  };
  // clamp-range rule (plgpu_walk.cuh): pairs of distance-ring samples for
  // K >= 1 and S <= 16, one f-ring sample per step otherwise
  constexpr bool PAIR = clamp_pairs(KT, ST);
  auto track2 = [&](V a, V b) {
    lo0 = min3f(lo0, Ops::lo(a), Ops::lo(b));
    hi0 = max3f(hi0, Ops::lo(a), Ops::lo(b));
    lo1 = min3f(lo1, Ops::hi(a), Ops::hi(b));
    hi1 = max3f(hi1, Ops::hi(a), Ops::hi(b));
  };
#pragma unroll
  for (int q = 0; q < R; ++q) {
    nr[q] = sc(ld_init(q + 1 + 2 * KT));
    orr[q] = sc(ld_init(q));
    d[q] = zero;
    const V f = ld_init(q + 1 + KT);
    V fa = f;  // accumulation-side sample
    if constexpr (AP) fa = sc(f);
    if constexpr (PK) {  // the centre sample (w = 1) starts each pixel's sums
      frp[q] = f2_make(Ops::lo(fa), 1.f);
      acc[q] = frp[q];
    } else {
      if constexpr (!AP) fr[q] = fa;
      an[q] = fa;
      ad[q] = Ops::splat(1.f);
    }
    track(f);
  }
  if constexpr (PAIR) {
#pragma unroll
    for (int q = R - KT; q < R; ++q) track(ld_init(q + 1 + 2 * KT));  // rest of [i0, i0 + K + ST]
  }
#pragma unroll
  for (int t = 0; t <= 2 * KT; ++t) {  // anchor d_k(i0-1), t ascending
    const V a = sc(ld_init(t));
#pragma unroll
    for (int k = 1; k <= ST; ++k) {
      const V df = Ops::sub(a, sc(ld_init(t + k)));
      d[k] = Ops::fma(df, df, d[k]);
    }
  }

  const V one = Ops::splat(1.f);
  const int64_t dst_img = img * g.dst_img_stride;
  const int my_line = l0 + lane * LINES;
  // debug distance export: pair (i, i+k) into cells (i, S+k) and (i+k, S-k)
  auto dexport = [&](int i, int k, int kmax, V dk) {
    if constexpr (EXP) {
      if (i < s0 || i >= s1 || k > kmax) return;
      const int64_t W = 2 * S + 1;
#pragma unroll
      for (int h = 0; h < LINES; ++h) {
        if (my_line + h > last_line) continue;
        float* b = g.dexp + ((int64_t)img * g.lines_per_img + my_line + h) * n * W;
        const float v = h == 0 ? Ops::lo(dk) : Ops::hi(dk);
        b[(int64_t)i * W + S + k] = v;
        b[(int64_t)(i + k) * W + S - k] = v;
      }
    }
  };

  // One chunk iteration (staging, R-step body, flush).  Clean iterations
  // (no masking) form a prefix of the loop and run in a loop of their own, so
  // the hot loop has a single body and no merge at its back edge.
  auto iteration = [&](const int c, auto mask_tag) {
    // Lockstep CTAs (large S): every warp of the CTA starts each iteration
    // together, so the SM's warps stream the (large) unrolled body through the
    // instruction cache once instead of once per warp.
    if (bar_threads) asm volatile("bar.sync 1, %0;" ::"r"(bar_threads) : "memory");
    // Row pass: lanes read positions staged by other lanes -> warp barriers.
    if (!own) __syncwarp();  // all lanes done with chunk c-2 (iteration c-1)
    issue_chunk(c + 2);      // into the slot of chunk c-2
    cp_wait<2>();            // chunk c landed
    if (!own) __syncwarp();
    const float* prv = slot(c - 1) + lane * LINES;
    const float* cur = slot(c) + lane * LINES;
    // sample at ring coordinate s + off for body step r (all compile-time but c)
    auto at = [&](int r, int off) -> V {
      const int q = r + off - BASE;  // relative to chunk c's first position
      return q >= 0 ? Ops::lds(cur + q * PITCH) : Ops::lds(prv + (q + R) * PITCH);
    };
    const int sb = c * R;
    // One iteration = R steps.  MASK = false: all R steps exist and no pair
    // leaves the line (the common case, branch-free); MASK = true: the last,
    // partial or clipped iteration(s) -- per-step exit, pairs beyond the line
    // end (or k > S) get weight exactly 0.
    float2 outv[oown ? R : 1];  // this iteration's outputs (2-line column flush)
    auto body = [&](auto mask_tag) {
      constexpr bool MASK = decltype(mask_tag)::value;
      V xprev;  // x of the previous (even) step, tracked with the next
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int s = sb + r;
        if (MASK && s >= T) break;
        const int i = i0 + s;
        const V an_ = nr[r], ao = orr[r];
        // Source order of the step's refill loads (positions fixed by the
        // step, not by the rings): ahead of the pair loop for the 1-line S = 15
        // kernel (c3 +0.9 %; S = 25, at 255 registers, -0.5 %).
        constexpr int EARLY = ST <= 10 ? PLGPU_EARLY_S10 : ST <= 16 ? (LINES == 1 ? PLGPU_EARLY_S15 : 0)
                                                                    : PLGPU_EARLY_S25;
        constexpr bool E_F = (EARLY & 1) && !AP, E_O = (EARLY & 2) != 0, E_X = (EARLY & 4) != 0;
        V e_fnew = zero, e_orr = zero, e_xr = zero;
        if constexpr (E_F) e_fnew = at(r, 2 + KT + ST);
        if constexpr (E_O && !(2 * KT < ST && ST <= 16 && LINES == 2)) e_orr = at(r, 1 + ST);
        if constexpr (E_X) e_xr = at(r, BASE);
        const int kmax = MASK ? min(S, n - 1 - i) : ST;
        V qv;
        if constexpr (PK) {
          using O2 = VecOps<2>;
          const F2 fip = frp[r];
          F2 nd = acc[r];  // {f_i + j-side num, 1 + j-side den}
#pragma unroll
          for (int k = 1; k <= ST; ++k) {
            const int rk = (r + k) % R;
            const float dn = an_ - nr[rk];
            float dk = fmaf(dn, dn, d[k]);
            const float dq = ao - orr[rk];
            dk = fmaf(-dq, dq, dk);
            d[k] = dk;
            dexport(i, k, MASK ? kmax : min(S, n - 1 - i), dk);
            float w = ex2_approx(-dk);
            if constexpr (MASK) w = k > kmax ? 0.f : w;
            const F2 ww = f2_make(w, w);
            nd = O2::fma(frp[rk], ww, nd);  // num += w f_{i+k}; den += w
            // first contribution to the slot recycled at step r-1: onto its
            // centre term {f, 1}
            acc[rk] = O2::fma(fip, ww, k == ST ? frp[rk] : acc[rk]);
          }
          float qn, qd;
          f2_split(nd, qn, qd);
          qv = AP ? div_unscale(qn, qd, g.inv_scale) : div_fix(qn, qd);
        } else {
          // accumulation-side sample at position i + k: the prescaled one sits
          // in the distance rings (AP), else the f ring
          auto fsc = [&](int k) -> V {
            if constexpr (AP) return k >= KT ? nr[(r + k - KT) % R] : orr[(r + k + KT + 1) % R];
            else return fr[AP ? 0 : (r + k) % R];
          };
          const V fi = fsc(0);
          V num = an[r];  // centre + j-side contributions so far
          V den = ad[r];
#pragma unroll
          for (int k = 1; k <= ST; ++k) {
            const int rk = (r + k) % R;
            const V fk = fsc(k);
            const V dn = Ops::sub(an_, nr[rk]);
            V dk = Ops::fma(dn, dn, d[k]);
            const V dq = Ops::sub(ao, orr[rk]);
            dk = Ops::fms(dq, dq, dk);
            d[k] = dk;
            dexport(i, k, MASK ? kmax : min(S, n - 1 - i), dk);
            V w = Ops::ex2n(dk);
            if constexpr (MASK) w = Ops::zero_if(k > kmax, w);
            num = Ops::fma(w, fk, num);
            den = Ops::add(w, den);
            if (k == ST) {  // first contribution to the slot recycled at step r-1,
              an[rk] = Ops::fma(w, fi, fk);  // onto its centre term: the portable
              ad[rk] = Ops::add(w, one);     // walker's fma(w, f_i, f) and 1 + w
            } else {
              an[rk] = Ops::fma(w, fi, an[rk]);
              ad[rk] = Ops::add(w, ad[rk]);
            }
          }
          qv = AP ? Ops::div_unscale(num, den, g.inv_scale) : Ops::div(num, den);
        }
        const float o0 = fminf(fmaxf(Ops::lo(qv), lo0), hi0);
        float o1 = o0;
        if constexpr (LINES == 2) o1 = fminf(fmaxf(Ops::hi(qv), lo1), hi1);
        if constexpr (oown) {
          outv[r] = make_float2(o0, o1);
        } else {  // every step lands in the output ring, filtered at the flush
          float* sl = oring + r * OPITCH + lane * LINES;
          if constexpr (LINES == 2) *reinterpret_cast<float2*>(sl) = make_float2(o0, o1);
          else *sl = o0;
        }
        // refill slot r in place (position i + ST + 1): first read at step r+1's last offset
        if constexpr (AP) {
          if constexpr (!PAIR) track(at(r, 2 + KT + ST));
          if constexpr (PK) {  // x' at position i + ST + 1: in the nr ring for K >= 1
            float fs1;
            if constexpr (KT >= 1 && PLGPU_PK_REFILL_RING) fs1 = Ops::lo(nr[(r + ST + 1 - KT) % R]);
            else fs1 = Ops::lo(sc(at(r, 2 + KT + ST)));
            frp[r] = f2_set_lo(frp[r], fs1);
          }
        } else {
          const V fnew = E_F ? e_fnew : at(r, 2 + KT + ST);
          if constexpr (!PAIR) track(fnew);
          // {f, 1}: keeping the 1.0 half in place measured c3 +1.4 %, c5 -22 % (register
          // allocation at 255 registers), so only for S <= 16
          if constexpr (PK && ST <= 16) frp[r] = f2_set_lo(frp[r], Ops::lo(fnew));
          else if constexpr (PK) frp[r] = f2_make(Ops::lo(fnew), 1.f);
          else fr[r] = fnew;
        }
        // The leaving-term partner entering now (coordinate s+1+ST) entered
        // the nr ring 2K+1 steps ago and is still there when 2K < S: it is
        // copied from the nr ring (2-line
        // kernel) or re-read from the staged chunk and scaled (1-line kernels:
        // the copy's register shuffles cost c3 2.5 %; S = 25 spills with it).
        if constexpr (2 * KT < ST && ST <= 16 && LINES == 2) orr[r] = nr[(r + R - 2 * KT - 1) % R];
        else orr[r] = sc(E_O ? e_orr : at(r, 1 + ST));
        // Packed prescale (one FMUL2 instead of two FMULs: c4 +2.3 %) where
        // the scaled sample feeds many subtractions (the nr ring doubles as
        // the orr ring), so ptxas has no single-use product it could contract
        // into a following subtraction; bitwise equal to the scalar form.
        const V xr = E_X ? e_xr : at(r, BASE);  // raw x_s: distance ring and clamp range
        if constexpr (LINES == 2 && 2 * KT < ST && ST <= 16) nr[r] = Ops::mul(xr, svv);
        else nr[r] = sc(xr);
        if constexpr (PAIR) {
          if (r & 1) track2(xprev, xr);
          else if (r == R - 1) track(xr);
          else xprev = xr;
        }
      }
    };
    body(mask_tag);

    if constexpr (!OROWS) {
      // flush this iteration's outputs (row q = position i0 + sb + q)
      if constexpr (oown) {  // each lane stores its own two lines, from registers
        // position q's address = base + q * pitch (one IMAD.WIDE with the
        // immediate q; the host keeps R * pitch < 2^32)
        const uint32_t pitch = (uint32_t)g.dst_pos_stride * (uint32_t)sizeof(float);
        char* const base = reinterpret_cast<char*>(g.dst + dst_img + (int64_t)(i0 + sb) * g.dst_pos_stride +
                                                   my_line);
        const bool whole = i0 + sb >= s0 && i0 + sb + R <= s1;
        if constexpr (AVG) {  // fused S-NLM average: all partner loads before any store
          const char* const abase = reinterpret_cast<const char*>(g.avg) +
                                    (base - reinterpret_cast<char*>(g.dst));
          float2 a[R];
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int p = i0 + sb + q;
            a[q] = (whole || (p >= s0 && p < s1))
                       ? __ldg(reinterpret_cast<const float2*>(mad_wide_u32(q, pitch, abase)))
                       : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int p = i0 + sb + q;
            if (whole || (p >= s0 && p < s1))
              st_global_f2(mad_wide_u32(q, pitch, base),
                           make_float2((a[q].x + outv[q].x) / 2.0f, (a[q].y + outv[q].y) / 2.0f));
          }
        } else if (whole) {
#pragma unroll
          for (int q = 0; q < R; ++q) st_global_f2(mad_wide_u32(q, pitch, base), outv[q]);
        } else {
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int p = i0 + sb + q;
            if (p >= s0 && p < s1) st_global_f2(mad_wide_u32(q, pitch, base), outv[q]);
          }
        }
      } else if (g.vec16) {
        __syncwarp();
        constexpr int LPR = LW / 4;  // lanes per row, 16 B each
#pragma unroll
        auto flush16 = [&](auto check_tag) {
          constexpr bool CHECK = decltype(check_tag)::value;
#pragma unroll
          for (int qb = 0; qb < R; qb += 32 / LPR) {
            const int q = qb + lane / LPR;
            const int p = i0 + sb + q;
            if (q < R && (!CHECK || (p >= s0 && p < s1))) {
              float4 v = *reinterpret_cast<const float4*>(oring + q * OPITCH + 4 * (lane % LPR));
              const int64_t off = dst_img + (int64_t)p * g.dst_pos_stride + l0 + 4 * (lane % LPR);
              if constexpr (AVG) {  // fused S-NLM average
                const float4 a = __ldg(reinterpret_cast<const float4*>(g.avg + off));
                v = make_float4((a.x + v.x) / 2.0f, (a.y + v.y) / 2.0f, (a.z + v.z) / 2.0f,
                                (a.w + v.w) / 2.0f);
              }
              *reinterpret_cast<float4*>(g.dst + off) = v;
            }
          }
        };
        if (i0 + sb >= s0 && i0 + sb + R <= s1) flush16(std::integral_constant<bool, false>{});
        else flush16(std::integral_constant<bool, true>{});
        __syncwarp();
      } else {
        __syncwarp();
#pragma unroll 2
        for (int q = 0; q < R; ++q) {
          const int p = i0 + sb + q;
          if (p >= s0 && p < s1) {
#pragma unroll
            for (int h = 0; h < LINES; ++h)
              if (my_line + h <= last_line) {
                float* dp = g.dst + dst_img + (int64_t)p * g.dst_pos_stride +
                            (int64_t)(my_line + h) * g.dst_line_stride;
                *dp = epi(AVG ? g.avg : nullptr, g.dst, dp, oring[q * OPITCH + lane * LINES + h]);
              }
          }
        }
        __syncwarp();
      }
    }
    if constexpr (OROWS) {
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
          const float* orow = oring + q * PITCH + half;
          if (full_group) {
            float* dp = g.dst + dst_img + pofs + (int64_t)(l0 + half) * g.dst_line_stride;
            const int64_t dstep = 2 * g.dst_line_stride;
#pragma unroll 8
            for (int j = 0; j < LW / 2; ++j) {
              *dp = orow[2 * j];
              dp += dstep;
            }
          } else {
            float* dbase = g.dst + dst_img + pofs;
#pragma unroll 4
            for (int j = 0; j < LW / 2; ++j) {
              const int l = 2 * j + half;
              if (l0 + l <= last_line) dbase[(int64_t)(l0 + l) * g.dst_line_stride] = orow[2 * j];
            }
          }
          if (fan) {  // the same values into the fan-out destinations
            for (int x = 0; x < g.nx; ++x) {
#pragma unroll 4
              for (int j = 0; j < LW / 2; ++j) {
                const int line = l0 + 2 * j + half;
                if (line <= last_line && line >= g.xlo[x] && line < g.xhi[x])
                  g.xdst[x][(int64_t)(line - g.xlo[x]) * g.dst_line_stride + pofs] = orow[2 * j];
              }
            }
          }
        }
      }
      __syncwarp();
    }
  };
  using Clean = std::integral_constant<bool, false>;
  using Masked = std::integral_constant<bool, true>;
  if constexpr (MODE == 1) {
    for (int c = 0; c < nchunks; ++c) iteration(c, Clean{});
  } else if constexpr (MODE == 2) {
    for (int c = 0; c < nchunks; ++c) iteration(c, Masked{});
  } else {
    // iteration c is clean iff S == ST, (c+1)R <= T and i0 + (c+1)R - 1 + ST <= n - 1
    const int nclean = S == ST ? min(T / R, max(0, (n - ST - i0) / R)) : 0;
    int c = 0;
    for (; c < nclean; ++c) iteration(c, Clean{});
    for (; c < nchunks; ++c) iteration(c, Masked{});
  }
  cp_wait<0>();
}

// WPC = warps per CTA.  WPC = 2: independent warps.  WPC = 8 ("lockstep"):
// the CTA's warps take 8 consecutive line groups of ONE segment and
// synchronise once per iteration (named barrier over the active warps).
template <int ST, int KT, int LINES, int IO, int WPC = kWarpsPerCta, bool AVG = false,
          bool EXP = false>
__global__ void __launch_bounds__(32 * WPC, (WPC == kLockWpc && LINES == 1 && ST <= 16) ? PLGPU_LOCK_MINB : 1)
    nlm_pass3_kernel(const Pass3Desc d) {
  extern __shared__ __align__(16) float smem[];
  const Pass2Desc& g = d.b;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* ring = smem + wib * pass3_smem_floats_per_warp<ST, LINES, IO>();
  if constexpr (WPC == kLockWpc) {
    const int bpi = (g.groups_per_img + WPC - 1) / WPC;  // WPC-group blocks per image
    const int64_t blocks_per_seg = (g.total_warps / g.nseg + 0) / g.groups_per_img * bpi;
    const int n_int = pass3_split(ST) ? max(0, d.seg_hi - d.seg_lo + 1) : 0;
    const int64_t int_ctas = (int64_t)n_int * blocks_per_seg;
    int seg;
    int64_t blk;
    bool interior;
    if ((int64_t)blockIdx.x < int_ctas) {
      seg = g.seg_begin + d.seg_lo + (int)(blockIdx.x % n_int);
      blk = blockIdx.x / n_int;
      interior = true;
    } else {
      const int64_t e = blockIdx.x - int_ctas;
      const int n_edge = g.nseg - n_int;
      int sidx = (int)(e % n_edge);
      if (n_int > 0 && sidx >= d.seg_lo) sidx += n_int;
      seg = g.seg_begin + sidx;
      blk = e / n_edge;
      interior = !pass3_split(ST);
    }
    const int64_t img = blk / bpi;
    const int gb = (int)(blk % bpi) * WPC;
    const int active = min(WPC, g.groups_per_img - gb);
    if (wib >= active) return;
    const int64_t grp = img * g.groups_per_img + gb + wib;
    const int bt = active * 32;
    if constexpr (!pass3_split(ST)) {
      walk3<ST, KT, LINES, IO, 0, AVG, EXP>(g, ring, lane, grp, seg, bt);
    } else if (interior) {
      walk3<ST, KT, LINES, IO, 1, AVG, EXP>(g, ring, lane, grp, seg, bt);
    } else {
      walk3<ST, KT, LINES, IO, 2, AVG, EXP>(g, ring, lane, grp, seg, bt);
    }
    return;
  }
  const int64_t wid = (int64_t)blockIdx.x * WPC + wib;
  if (wid >= g.total_warps) return;
  if constexpr (!pass3_split(ST)) {
    walk3<ST, KT, LINES, IO, 0, AVG, EXP>(g, ring, lane, wid / g.nseg, g.seg_begin + (int)(wid % g.nseg));
  } else {
    // large S: interior warps (segments needing no clipping) first, then edges
    const int n_int = max(0, d.seg_hi - d.seg_lo + 1);
    if (wid < d.interior_warps) {
      walk3<ST, KT, LINES, IO, 1, AVG, EXP>(g, ring, lane, wid / n_int,
                                            g.seg_begin + d.seg_lo + (int)(wid % n_int));
    } else {
      const int n_edge = g.nseg - n_int;
      const int64_t e = wid - d.interior_warps;
      int sidx = (int)(e % n_edge);
      if (n_int > 0 && sidx >= d.seg_lo) sidx += n_int;
      walk3<ST, KT, LINES, IO, 2, AVG, EXP>(g, ring, lane, e / n_edge, g.seg_begin + sidx);
    }
  }
}

// ---- folded 1D pass -----------------------------------------------------------
// Few, long lines (1D signals: c1 is ONE 65,536-sample line) leave the lane
// dimension empty when a lane is a line.  Here the lanes of a warp take
// consecutive SEGMENTS of one real line instead: the interior segments
// [jlo, jhi] of a line become the "lines" of a virtual image whose line l
// starts at sample (jlo - 1 + l) * C of the real line (line stride C, length
// 3C) and whose only processed segment is its second one -- exactly the real
// segment jlo + l with its pre-walk and halo, all inside the real line, so the
// walker runs the interior arithmetic unchanged (bitwise the same outputs as
// one warp per segment).  The segments that touch a line end (mirror, window
// clipping) run as warps of the same launch on the real lines (`edge`).
struct Pass3FoldDesc {
  Pass2Desc fold;     // virtual image per real line (seg_begin = 1, nseg = 1)
  Pass2Desc edge;     // the real lines; nseg / total_warps count all segments
  int32_t jlo, jhi;   // folded (interior) segments of every real line
  int32_t fold_ctas;  // CTAs [0, fold_ctas) run `fold`, the rest `edge`
  int64_t edge_warps; // real line groups x segments outside [jlo, jhi]
};

template <int ST, int KT, int LINES>
__global__ void __launch_bounds__(32 * kWarpsPerCta, 1)
    nlm_pass3_fold_kernel(const Pass3FoldDesc d) {
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* ring = smem + wib * pass3_smem_floats_per_warp<ST, LINES, 1>();
  constexpr int MI = pass3_split(ST) ? 1 : 0;  // interior-only body for large S
  constexpr int ME = pass3_split(ST) ? 2 : 0;
  if ((int)blockIdx.x < d.fold_ctas) {
    const int64_t wid = (int64_t)blockIdx.x * kWarpsPerCta + wib;
    if (wid >= d.fold.total_warps) return;
    walk3<ST, KT, LINES, 1, MI>(d.fold, ring, lane, wid, d.fold.seg_begin);
  } else {
    const int64_t e = ((int64_t)blockIdx.x - d.fold_ctas) * kWarpsPerCta + wib;
    if (e >= d.edge_warps) return;
    const int n_edge = d.edge.nseg - (d.jhi - d.jlo + 1);
    int sidx = (int)(e % n_edge);
    if (sidx >= d.jlo) sidx += d.jhi - d.jlo + 1;
    walk3<ST, KT, LINES, 1, ME>(d.edge, ring, lane, e / n_edge, d.edge.seg_begin + sidx);
  }
}


}  // namespace plgpu

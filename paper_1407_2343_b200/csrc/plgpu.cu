// plgpu.cu -- C ABI (include/plgpu.h) over the sm_100a PatchLift kernels.
// Host-side responsibilities: the reference's validation (core_types.cpp:49-69,
// same messages), effective radius clipping, segment geometry, dispatch onto
// the S-specialised walker instantiations, and composite sequencing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "plgpu.h"
#include "plgpu_aux.cuh"
#include "plgpu_launch.cuh"
#include "plgpu_metrics.cuh"
#include "plgpu_walk.cuh"

namespace {

thread_local std::string g_err;
// Diagnostic: which kernel route the last pass on this thread took.
thread_local std::string g_route;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define PL_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err(PL_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(PL_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return PL_OK;
}

// validate_geometry / validate_params (core_types.cpp:49-69).
int validate_geometry(int S, int K, int n) {
  if (n < 1) return set_err(PL_ERR_VALIDATION, "signal length must be at least 1");
  if (S < 0) return set_err(PL_ERR_VALIDATION, "search radius must be nonnegative");
  if (K < 0) return set_err(PL_ERR_VALIDATION, "patch radius must be nonnegative");
  if (K > n) return set_err(PL_ERR_VALIDATION, "patch radius exceeds signal length");
  return PL_OK;
}

int validate_params(const pl_params& p, int n) {
  int rc = validate_geometry(p.search_radius, p.patch_radius, n);
  if (rc) return rc;
  if (!(p.h > 0.0)) return set_err(PL_ERR_VALIDATION, "smoothing parameter h must be positive");
  return PL_OK;
}

int validate_image(int batch, int rows, int cols) {
  if (rows < 1 || cols < 1) return set_err(PL_ERR_VALIDATION, "image dimensions must be at least 1x1");
  if (batch < 1) return set_err(PL_ERR_ARG, "batch must be at least 1");
  return PL_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Segment length: a function of (n, S) only, identical for rows and columns
// (transpose equivariance) and for every launch shape or GPU count.  About
// 480 samples, rounded up so that an interior segment's walk (C + S steps, S
// of pre-walk) is a whole number of S+1-step iterations of the unrolled
// walker.  Lines of 8192+ samples use a multiple of 8 segments, so that the
// row-partitioned multi-GPU column pass (whole segments per rank) splits
// evenly over 2, 4 or 8 GPUs.  Signal-length lines (32768+ samples: 1D
// signals, processed one or a few at a time) use ~32-sample segments so a
// single line still spreads over enough lanes (the folded pass of
// plgpu_walk3.cuh puts one segment on each lane): c1 (one 65,536-sample
// line) 11.7 us per call vs 15.9 us at ~64, for S/32 extra pre-walk.  Short
// lines (<= 1024 samples: small images, a few hundred lines each) use
// ~64-sample segments, so a 512^2 image runs 64 warps instead of 16.
// (build-variant knobs for the segment-length sweeps of profiles/README.md;
// the shipped values are the defaults -- a different value changes result bits)
#ifndef PLGPU_SEG_MID
#define PLGPU_SEG_MID 480
#endif
#ifndef PLGPU_SEG_LONG
#define PLGPU_SEG_LONG 32
#endif
int32_t segment_length(int32_t n, int32_t S) {
  const int32_t R = std::max(1, S + 1);
  // long segments: pre-walk overhead S/C stays small
  // ~512 for lines up to 2048 samples: 4 segments of a 2048-sample line
  // instead of 5 (c4 +1.75 %; the per-GPU share of c4 at 8 GPUs, 8 images,
  // fits one wave: +18 %)
  const int32_t target = n >= 32768 ? PLGPU_SEG_LONG : n <= 1024 ? 64 : (n <= 2048 ? 512 : PLGPU_SEG_MID);
  int32_t nseg = std::max(1, (n + target - 1) / target);
  if (n >= 8192) nseg = std::max(8, (nseg + 4) / 8 * 8);
  int32_t C = (n + nseg - 1) / nseg;       // near-equal segments
  C += (R - (C + S) % R) % R;              // C + S: whole S+1-step iterations (round up,
                                           // so nseg segments still cover the line)
  return n < C ? n : C;
}

// Kernel selection: the hot-configuration kernel (plgpu_walk3.cuh) for the
// configs' (K, S), the production walker (plgpu_walk2.cuh) for K <= 7 on
// either axis, the portable walker (plgpu_walk.cuh) for larger patch radii;
// all run the same per-line arithmetic (bitwise-equal results).  The routing
// and the hot kernel's lines-per-lane / warps-per-CTA can be pinned for
// testing through pl_debug_set_route (process-wide; performance and coverage
// only -- no setting changes a result bit).  No environment variable is read.
std::atomic<int> g_dbg_walker{0};  // 0 default, 1 portable only, 2 no hot kernel
std::atomic<int> g_dbg_lines{0};   // 0 default, 1 or 2 lines per lane (S <= 16)
std::atomic<int> g_dbg_wpc{0};     // 0 default, 2 or 8 warps per CTA
std::atomic<int> g_dbg_fold{0};    // 0 default, 2 = never fold 1D lines onto lanes

bool force_portable() { return g_dbg_walker.load(std::memory_order_relaxed) == 1; }
bool force_portable_v2() { return g_dbg_walker.load(std::memory_order_relaxed) == 2; }
// Lines per lane of the hot-configuration kernel: 1 = one line per lane with
// {num, den} packed, 2 = two lines per lane packed line-wise.
int walk3_lines(int ST) {
  if (ST > 16) return 1;
  const int forced = g_dbg_lines.load(std::memory_order_relaxed);
  if (forced == 1 || forced == 2) return forced;
  return ST <= 10 ? 2 : 1;  // measured on B200: c4 (S=10) 2 lines, c3 (S=15) 1 line
}
int walk3_wpc(int ST) {
  const int forced = g_dbg_wpc.load(std::memory_order_relaxed);
  if (forced == 2) return 2;
  if (forced == 8) return plgpu::kLockWpc;
  return ST >= 15 ? plgpu::kLockWpc : 2;  // measured: lockstep helps S=15/25 (I-cache), hurts S=10
}

// Largest radius with a specialised walker; larger radii use the direct kernel.
constexpr int kMaxWalkS = 32;
// Instantiated template radii; an effective S runs on the smallest >= it
// (extra offsets are masked to weight exactly 0, which leaves every sum
// bitwise unchanged).
constexpr int kWalkS[] = {1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 15, 16, 20, 25, 32};

int template_radius(int S) {
  for (int t : kWalkS)
    if (t >= S) return t;
  return -1;
}

int dispatch_pass(const plgpu::PassDesc& g, cudaStream_t st) {
  g_route = "portable<S=" + std::to_string(template_radius(g.S)) + ">";
  switch (template_radius(g.S)) {
#define PL_CASE(v) \
  case v: plgpu::launch_pass<v>(g, st); break;
    PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
    default:
      return set_err(PL_ERR_UNSUPPORTED, "search radius above walker range");
  }
  return check_launch();
}

float weight_coef(double h) { return static_cast<float>(-1.4426950408889634 / (h * h)); }

// Generic direct-route pass over strided lines (used for S > kMaxWalkS and S == 0).
__global__ void direct_pass_kernel(plgpu::PassDesc g) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= g.n_lines * g.n) return;
  const int64_t line = w % g.n_lines;
  const int i = (int)(w / g.n_lines);
  const int64_t img = line / g.lines_per_img;
  const int64_t li = line - img * g.lines_per_img;
  const float* f = g.src + img * g.src_img_stride + li * g.src_line_stride;
  const int64_t ps = g.src_pos_stride;
  const int n = g.n, K = g.K;
  const int lo = max(0, i - g.S), hi = min(n - 1, i + g.S);
  float num = 0.f, den = 0.f, vmin = 3.402823466e38f, vmax = -3.402823466e38f;
  for (int j = lo; j <= hi; ++j) {
    float dsq = 0.f;
    for (int t = -K; t <= K; ++t) {
      const float df = __ldg(f + plgpu::mirror_pos(i + t, n) * ps) -
                       __ldg(f + plgpu::mirror_pos(j + t, n) * ps);
      dsq = fmaf(df, df, dsq);
    }
    const float wt = (j == i) ? 1.f : plgpu::ex2_approx(g.coef * dsq);
    const float fj = __ldg(f + (int64_t)j * ps);
    num = fmaf(wt, fj, num);
    den += wt;
    vmin = fminf(vmin, fj);
    vmax = fmaxf(vmax, fj);
  }
  const int blk = g.dst_pos_block;
  float* dst = g.dst + img * g.dst_img_stride + li * g.dst_line_stride +
               (int64_t)(i / blk) * g.dst_block_stride + (int64_t)(i % blk) * g.dst_pos_stride;
  *dst = plgpu::epi(g.avg, g.dst, dst, fminf(fmaxf(num / den, vmin), vmax));
}

// Production walker launch, if the geometry qualifies (returns -1 if not).
int try_pass2(const plgpu::PassDesc& g, cudaStream_t st) {
  if (g.avg && g.dst_pos_stride == 1) return -1;  // fused average: column-mode flushes only
  // A warp carries 32-64 lines: for a handful of lines the one-thread-per-
  // segment portable walker wastes less.
  // (unless the hot kernel can fold the lines' segments onto its lanes, below)
  if (force_portable() || g.K > 7 || g.S < 1 || g.S > kMaxWalkS) return -1;
  const int ST = template_radius(g.S);
  const bool few_lines = g.lines_per_img < 16;
  if (few_lines && (force_portable_v2() || plgpu::pass3_k_for(ST) != g.K || ST != g.S ||
                    g.src_pos_stride != 1 || g.dst_pos_stride != 1))
    return -1;
  // fan-out stores: hot kernel's row flush or the portable walker
  if (g.nx > 0 && (force_portable_v2() || plgpu::pass3_k_for(ST) != g.K || ST != g.S ||
                   g.src_pos_stride != 1 || g.dst_pos_stride != 1))
    return -1;
  const int LW = 32 * plgpu::pass2_lines(ST);
  const bool rows = g.src_pos_stride == 1 && g.dst_pos_stride == 1;
  const bool cols = g.src_line_stride == 1 && g.dst_line_stride == 1;
  // positions contiguous in the source, lines contiguous in the destination:
  // the transposed-intermediate RC composite (walk3 io = 2; walk2 treats it
  // as a column pass with general source strides)
  const bool mixed = !rows && g.src_pos_stride == 1 && g.dst_line_stride == 1;
  if (!rows && !cols && !mixed) return -1;
  if (rows && g.dst_pos_block != g.n && g.dst_pos_block % plgpu::kCH != 0) return -1;
  if (!rows && g.dst_pos_block != g.n) return -1;
  plgpu::Pass2Desc d{};
  d.src = g.src;
  d.dst = g.dst;
  d.src_img_stride = g.src_img_stride;
  d.src_line_stride = g.src_line_stride;
  d.src_pos_stride = g.src_pos_stride;
  d.dst_img_stride = g.dst_img_stride;
  d.dst_line_stride = g.dst_line_stride;
  d.dst_pos_stride = g.dst_pos_stride;
  d.dst_block_stride = g.dst_block_stride;
  d.dst_pos_block = g.dst_pos_block;
  d.lines_per_img = g.lines_per_img;
  d.groups_per_img = (g.lines_per_img + LW - 1) / LW;
  d.n = g.n;
  d.seg_len = g.seg_len;
  d.nseg = g.nseg;
  d.seg_begin = g.seg_begin;
  d.S = g.S;
  d.K = g.K;
  d.coef = g.coef;
  d.scale = g.scale;
  d.inv_scale = g.inv_scale;
  d.nx = g.nx;
  for (int x = 0; x < 2; ++x) {
    d.xdst[x] = g.xdst[x];
    d.xlo[x] = g.xlo[x];
    d.xhi[x] = g.xhi[x];
  }
  d.avg = g.avg;
  d.dexp = g.dexp;
  const int64_t images = g.n_lines / g.lines_per_img;
  d.total_warps = images * d.groups_per_img * d.nseg;
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  d.vec16 = !rows && g.lines_per_img % LW == 0 && g.src_pos_stride % 4 == 0 &&
            g.src_img_stride % 4 == 0 && g.dst_pos_stride % 4 == 0 && g.dst_img_stride % 4 == 0 &&
            a16(g.src) && a16(g.dst);
  if (!force_portable_v2()) {
    // hot (K, S) pairs: compile-time-K kernel with interior/edge warp ordering
    const int KT3 = plgpu::pass3_k_for(ST);
    if (KT3 == g.K && ST == g.S) {
      const int R = ST + 1, BASE = ST + 2 * KT3 + 2;
      plgpu::Pass3Desc d3{};
      d3.b = d;
      // lines per lane for the hot kernel (PLGPU_LINES=1|2 overrides)
      d3.lines = walk3_lines(ST);
      // Small calls (c2: one 512^2 image = 64 two-line warps on 148 SMs) are
      // latency-bound: one line per lane doubles the warps and shortens each
      // warp's step (c2 +17 %); routing only, same bits.
      if (d3.lines == 2 && g_dbg_lines.load(std::memory_order_relaxed) == 0 &&
          images * ((g.lines_per_img + 63) / 64) * d.nseg < 148 * 4)
        d3.lines = 1;
      d3.wpc = walk3_wpc(ST);
      const int LW3 = 32 * d3.lines;
      d3.b.groups_per_img = (g.lines_per_img + LW3 - 1) / LW3;
      d3.b.total_warps = images * d3.b.groups_per_img * d.nseg;
      const int io = rows ? 1 : (mixed ? 2 : 0);
      const bool dst16 = g.lines_per_img % LW3 == 0 && g.dst_line_stride == 1 &&
                         g.dst_pos_stride % 4 == 0 && g.dst_img_stride % 4 == 0 && a16(g.dst);
      const bool src16 = g.src_line_stride == 1 && g.src_pos_stride % 4 == 0 &&
                         g.src_img_stride % 4 == 0 && a16(g.src);
      // io 0: 16-byte staging copies and stores; io 2: 16-byte stores only
      d3.b.vec16 = io == 0 ? (dst16 && src16) : io == 2 ? dst16 : false;
      // The 2-line column flush stores from registers at base + q * pitch:
      // it needs the aligned layout and a 32-bit R * pitch; walk2 otherwise.
      const bool own_ok = d3.b.vec16 && (uint64_t)g.dst_pos_stride * sizeof(float) * R < (1ull << 32);
      if (d3.lines == 2 && io != 1 && !own_ok) goto staged;
      // Few long lines (1D signals): fold the interior segments onto the
      // lanes (plgpu_walk3.cuh, Pass3FoldDesc).  Whole lines only, plain
      // row layout, contiguous line stack, segments long enough that an
      // interior segment's halo stays inside its neighbours.
      if (io == 1 && g_dbg_fold.load(std::memory_order_relaxed) != 2 && d.seg_begin == 0 &&
          d.nseg == (d.n + d.seg_len - 1) / d.seg_len && d.nx == 0 && !d.avg && !d.dexp &&
          d.dst_pos_block == d.n && g.lines_per_img < 32 &&
          (images == 1 || (g.src_img_stride == g.src_line_stride * g.lines_per_img &&
                           g.dst_img_stride == g.dst_line_stride * g.lines_per_img))) {
        const int C = d.seg_len;
        // interior segments j: j C - S - K - 1 >= 0 and (j + 1) C + S + K <= n - 1
        const int jlo = 1;
        const int jhi = (int)std::min<int64_t>(d.nseg - 1, ((int64_t)d.n - 1 - ST - KT3) / C - 1);
        const int NL = jhi - jlo + 1;
        if (C >= ST + KT3 + 1 && (C + ST) % R == 0 && NL >= 8) {
          plgpu::Pass3FoldDesc f{};
          const int64_t real_lines = g.n_lines;
          // one line per lane unless that would exceed one wave of warps
          const int fl = (ST <= 16 && real_lines * ((NL + 31) / 32) > 148 * 8) ? 2 : 1;
          const int FLW = 32 * fl;
          f.edge = d;
          f.edge.groups_per_img = (g.lines_per_img + FLW - 1) / FLW;
          f.edge.vec16 = 0;
          f.jlo = jlo;
          f.jhi = jhi;
          f.edge_warps = images * f.edge.groups_per_img * (d.nseg - NL);
          f.edge.total_warps = f.edge_warps;
          f.fold = d;
          f.fold.src = g.src + (int64_t)(jlo - 1) * C;
          f.fold.dst = g.dst + (int64_t)(jlo - 1) * C;
          f.fold.src_img_stride = g.src_line_stride;  // one virtual image per real line
          f.fold.dst_img_stride = g.dst_line_stride;
          f.fold.src_line_stride = f.fold.dst_line_stride = C;
          f.fold.lines_per_img = NL;
          f.fold.groups_per_img = (NL + FLW - 1) / FLW;
          f.fold.n = 3 * C;
          f.fold.dst_pos_block = 3 * C;
          f.fold.seg_begin = 1;
          f.fold.nseg = 1;
          f.fold.vec16 = 0;
          f.fold.total_warps = real_lines * f.fold.groups_per_img;
          f.fold_ctas = (int32_t)((f.fold.total_warps + plgpu::kWarpsPerCta - 1) / plgpu::kWarpsPerCta);
          bool launched = false;
          switch (ST) {
#define PL_CASE(v) \
  case v: launched = plgpu::launch_pass3_fold<v>(f, fl, st); break;
            PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
          }
          if (launched) {
            g_route = "hot-fold<S=" + std::to_string(ST) + ",K=" + std::to_string(KT3) +
                      ",lines=" + std::to_string(fl) + ",folded=" + std::to_string(NL) + ">";
            return check_launch();
          }
        }
      }
      if (few_lines) return -1;  // not foldable: portable walker
      int lo = d.nseg, hi = -1;
      for (int sgi = 0; sgi < d.nseg; ++sgi) {
        const int s0 = (d.seg_begin + sgi) * d.seg_len, s1 = std::min(d.n, s0 + d.seg_len);
        const int i0 = std::max(0, s0 - d.S), T = s1 - i0, pos0 = i0 - 1 - d.K;
        const int nch = (T + R - 1) / R;
        const bool interior = pos0 >= 0 && pos0 + nch * R + BASE - 1 <= d.n - 1 && T % R == 0 &&
                              s1 - 1 + ST <= d.n - 1;
        if (interior) {
          lo = std::min(lo, sgi);
          hi = std::max(hi, sgi);
        }
      }
      if (hi < lo) {
        lo = 0;
        hi = -1;
      }
      d3.seg_lo = lo;
      d3.seg_hi = hi;
      const int64_t groups = d3.b.total_warps / d.nseg;
      d3.interior_warps = groups * std::max(0, hi - lo + 1);
      bool launched = false;
      switch (ST) {
#define PL_CASE(v) \
  case v: launched = plgpu::launch_pass3<v>(d3, io, st); break;
        PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
      }
      if (launched) {
        g_route = "hot<S=" + std::to_string(ST) + ",K=" + std::to_string(KT3) + ",lines=" +
                  std::to_string(d3.lines) + ",io=" + std::to_string(io) + ",wpc=" +
                  std::to_string(d3.wpc) + ",avg=" + std::to_string(d.avg ? 1 : 0) + ">";
        return check_launch();
      }
    }
  }
staged:
  g_route = "staged<S=" + std::to_string(ST) + ",rows=" + std::to_string(rows ? 1 : 0) + ">";
  if (g.dexp) return set_err(PL_ERR_UNSUPPORTED, "distance export needs the hot kernel's (K, S)");
  switch (ST) {
#define PL_CASE(v) \
  case v: plgpu::launch_pass2<v>(d, rows, st); break;
    PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
    default:
      return -1;
  }
  return check_launch();
}

int run_pass(plgpu::PassDesc g, const pl_params& p, cudaStream_t st) {
  g.S = std::min<int32_t>(p.search_radius, g.n - 1);
  g.K = p.patch_radius;
  g.coef = weight_coef(p.h);
  // debug distance export: the recurrence on raw samples (exact on integers)
  g.scale = g.dexp ? 1.0f : static_cast<float>(std::sqrt(1.4426950408889634) / p.h);
  g.inv_scale = static_cast<float>(1.0 / static_cast<double>(g.scale));  // acc_prescaled unscale
  g.seg_len = segment_length(g.n, g.S);
  if (g.nseg <= 0) {  // whole lines (windowed passes preset seg_begin / nseg)
    g.seg_begin = 0;
    g.nseg = (g.n + g.seg_len - 1) / g.seg_len;
  }
  if (g.dst_pos_block <= 0) g.dst_pos_block = g.n;
  g_route = "none";
  if (g.n_lines <= 0) return PL_OK;
  if (g.n_lines % g.lines_per_img == 0) {
    const int rc = try_pass2(g, st);
    if (rc >= 0) return rc;
  }
  if (g.dexp) return set_err(PL_ERR_UNSUPPORTED, "distance export needs the hot kernel");
  if (g.S >= 1 && g.S <= kMaxWalkS) return dispatch_pass(g, st);
  const int64_t work = g.n_lines * g.n;
  g_route = "direct";
  direct_pass_kernel<<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
  return check_launch();
}

plgpu::PassDesc row_desc(const float* src, float* dst, int batch, int rows, int cols) {
  plgpu::PassDesc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = (int64_t)batch * rows;
  g.lines_per_img = rows;
  g.src_img_stride = g.dst_img_stride = (int64_t)rows * cols;
  g.src_line_stride = g.dst_line_stride = cols;
  g.src_pos_stride = g.dst_pos_stride = 1;
  g.dst_block_stride = 0;
  g.dst_pos_block = cols;
  g.n = cols;
  return g;
}

plgpu::PassDesc col_desc(const float* src, float* dst, int batch, int rows, int cols) {
  plgpu::PassDesc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = (int64_t)batch * cols;
  g.lines_per_img = cols;
  g.src_img_stride = g.dst_img_stride = (int64_t)rows * cols;
  g.src_line_stride = g.dst_line_stride = 1;
  g.src_pos_stride = g.dst_pos_stride = cols;
  g.dst_block_stride = 0;
  g.dst_pos_block = rows;
  g.n = rows;
  return g;
}

// Row -> column composite with a TRANSPOSED intermediate: the row pass
// stores its lines as columns of `mid` ([cols][rows] per image), so both
// passes stage positions along contiguous memory and flush lines along
// contiguous memory (walk3 io = 2), instead of the row pass paying a
// transposing flush.  Same per-line arithmetic: bit-identical to the
// row_desc/col_desc pair.  `avg` (optional) fuses the S-NLM average.
int rc_passes(const float* src, float* dst, float* mid, int batch, int rows, int cols,
              const pl_params& p, cudaStream_t st, const float* avg = nullptr) {
  plgpu::PassDesc a = row_desc(src, mid, batch, rows, cols);
  a.dst_line_stride = 1;
  a.dst_pos_stride = rows;
  int rc = run_pass(a, p, st);
  if (rc) return rc;
  plgpu::PassDesc b = col_desc(mid, dst, batch, rows, cols);
  b.src_line_stride = rows;
  b.src_pos_stride = 1;
  b.avg = avg;
  return run_pass(b, p, st);
}

// Library-owned scratch (work = NULL): stream-ordered allocations from one
// memory pool per device (cudaMallocFromPoolAsync / cudaFreeAsync on the
// caller's stream).  Every call gets its own buffer, released in stream order
// after its last kernel, so concurrent calls on different streams (or host
// threads) never share an intermediate, and nothing is freed while a caller
// may still use it.  The pool keeps its memory (release threshold = max), so a
// steady stream of calls does not go back to the driver.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

int device_pool(cudaMemPool_t* out) {
  int dev = 0;
  PL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_pool_mu);
  cudaMemPool_t& pool = g_pool[dev & 63];
  if (!pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    PL_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t keep = UINT64_MAX;
    PL_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = pool;
  return PL_OK;
}

// Scratch owned by one call: allocated on `st`, freed on `st` when the
// object goes out of scope (after the call has enqueued its kernels).
class Scratch {
 public:
  explicit Scratch(cudaStream_t st) : st_(st) {}
  ~Scratch() {
    if (ptr_) cudaFreeAsync(ptr_, st_);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <typename T>
  int alloc(size_t bytes, T** out) {
    cudaMemPool_t pool;
    int rc = device_pool(&pool);
    if (rc) return rc;
    PL_CUDA(cudaMallocFromPoolAsync(&ptr_, bytes ? bytes : 16, pool, st_));
    *out = static_cast<T*>(ptr_);
    return PL_OK;
  }

 private:
  cudaStream_t st_;
  void* ptr_ = nullptr;
};

int check_ptrs(const void* a, const void* b) {
  if (!a || !b) return set_err(PL_ERR_ARG, "null buffer");
  return PL_OK;
}

// ---- precision policy --------------------------------------------------------
// The fp32 walkers hold the 1e-3 output bound (on a [0, 255] scale) while
// h >= ~0.16 x the data range (below that the moving sums
// carry rounding of ulp(d / h^2) and a composite's second pass amplifies the
// fp32 intermediate's quantisation by ~ 2 |df| |f - out| / h^2).  Under
// PL_PRECISION_AUTO (default) the reference-API entry points therefore run
// such calls in double on the device (plgpu_walk64.cuh: fp32 in, fp64
// arithmetic and intermediates, fp32 out).  h >= 48 -- every 8-bit-scale
// setting the fp32 kernels are bounded for -- goes straight to the fp32
// kernels; below that the input's range is measured first (one reduction and a
// stream synchronisation) and h is compared with 48/255 of it.  (The fp32 composites reach 1.03e-3 at
// h = 33 on 12,875-sample lines, K = 1, and scale like 1 / h^2: 0.5e-3 at 48.)
std::atomic<int> g_policy{PL_PRECISION_AUTO};
constexpr double kFastH = 48.0;  // per 255 of data range

int choose_precise(const float* src, int64_t lines, int32_t n, int64_t ld, double h,
                   cudaStream_t st, bool* precise) {
  *precise = false;
  if (g_policy.load(std::memory_order_relaxed) == PL_PRECISION_FAST || h >= kFastH) return PL_OK;
  if (lines <= 0 || n <= 0) return PL_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PL_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return set_err(PL_ERR_UNSUPPORTED,
                   "h below the fp32 kernels' bounded range cannot be decided inside a stream "
                   "capture (set PL_PRECISION_FAST or call outside the capture)");
  Scratch scratch(st);
  uint32_t* mm = nullptr;
  int rc = scratch.alloc(2 * sizeof(uint32_t), &mm);
  if (rc) return rc;
  const uint32_t init[2] = {0xFFFFFFFFu, 0u};
  uint32_t got[2] = {0, 0};
  PL_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
  const int64_t total = lines * n;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8);
  plgpu::range_kernel<<<blocks, 256, 0, st>>>(src, lines, n, ld, mm);
  if ((rc = check_launch())) return rc;
  PL_CUDA(cudaMemcpyAsync(got, mm, sizeof got, cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  if (got[0] > got[1]) return PL_OK;  // no finite sample
  const double range = (double)plgpu::ordered_value(got[1]) - (double)plgpu::ordered_value(got[0]);
  *precise = h < kFastH * range / 255.0;
  return PL_OK;
}

// The partition-level entry points (strided / blocked / window / fan-out
// passes) run the fp32 kernels only: under PL_PRECISION_AUTO they refuse an h
// the fp32 kernels are not bounded for instead of silently exceeding the
// output tolerance (the caller confirms with PL_PRECISION_FAST).
int require_fp32_bounded(double h) {
  if (g_policy.load(std::memory_order_relaxed) == PL_PRECISION_FAST || h >= kFastH) return PL_OK;
  return set_err(PL_ERR_UNSUPPORTED,
                 "this entry point runs the fp32 kernels only and h is below their bounded range "
                 "(pl_fast_h_threshold); use the whole-image entry points or PL_PRECISION_FAST");
}

// fp32 buffers through an fp64 entry point: widen into stream-ordered
// scratch, `call(src64, dst64, work64)`, narrow.  `work_doubles` = the fp64
// composite's own workspace.
template <typename Call>
int run_precise(const float* src, float* dst, int64_t lines, int32_t n, int64_t ld,
                size_t work_doubles, cudaStream_t st, Call&& call) {
  if (lines <= 0) return PL_OK;
  const int64_t cnt = lines * n;
  Scratch scratch(st);
  double* buf = nullptr;
  int rc = scratch.alloc((2 * (size_t)cnt + work_doubles) * sizeof(double), &buf);
  if (rc) return rc;
  const unsigned blocks = (unsigned)std::min<int64_t>((cnt + 255) / 256, 148 * 16);
  plgpu::widen_kernel<<<blocks, 256, 0, st>>>(src, buf, lines, n, ld);
  if ((rc = check_launch())) return rc;
  if ((rc = call(buf, buf + cnt, buf + 2 * cnt))) return rc;
  plgpu::narrow_kernel<<<blocks, 256, 0, st>>>(buf + cnt, dst, lines, n, ld);
  return check_launch();
}

// Image composites / passes in double: op 0 RC, 1 CR, 2 S-NLM, 3 row, 4 col.
int precise_image(int op, const float* src, float* dst, int batch, int rows, int cols,
                  const pl_params& p, cudaStream_t st) {
  const size_t img = (size_t)batch * rows * cols;
  const size_t work = op == 2 ? 2 * img : (op <= 1 ? img : 0);
  return run_precise(src, dst, (int64_t)batch * rows, cols, cols, work, st,
                     [&](double* s64, double* d64, double* w64) {
                       switch (op) {
                         case 0: return pl_snlm_2d_row_col_f64(s64, d64, w64, batch, rows, cols, p, st);
                         case 1: return pl_snlm_2d_col_row_f64(s64, d64, w64, batch, rows, cols, p, st);
                         case 2: return pl_snlm_2d_f64(s64, d64, w64, batch, rows, cols, p, st);
                         case 3: return pl_nlm_row_pass_f64(s64, d64, batch, rows, cols, p, st);
                         default: return pl_nlm_col_pass_f64(s64, d64, batch, rows, cols, p, st);
                       }
                     });
}

}  // namespace

namespace {
template <typename T>
int distance_band(const float* src, T* band, int64_t n_lines, int32_t n, int64_t ld, int32_t S,
                  int32_t K, cudaStream_t st) {
  int rc = validate_geometry(S, K, n);
  if (rc) return rc;
  if ((rc = check_ptrs(src, band))) return rc;
  if (n_lines <= 0) return PL_OK;
  const int64_t cells = n_lines * (int64_t)n * (2 * S + 1);
  PL_CUDA(cudaMemsetAsync(band, 0xFF, cells * sizeof(T), st));  // NaN / -1 sentinel
  plgpu::BandDesc g{};
  g.src = src;
  g.band = band;
  g.n_lines = n_lines;
  g.ld = ld;
  g.n = n;
  g.S = std::min<int32_t>(S, n - 1);
  g.S_band = S;
  g.K = K;
  g.seg_len = segment_length(n, g.S);
  g.nseg = (n + g.seg_len - 1) / g.seg_len;
  if (g.S > kMaxWalkS) {
    const int64_t work = n_lines * (int64_t)n;
    plgpu::distance_band_direct_kernel<T><<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
    return check_launch();
  }
  switch (template_radius(std::max(1, g.S))) {
#define PL_CASE(v) \
  case v: plgpu::launch_band<v, T>(g, st); break;
    PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
    default:
      return set_err(PL_ERR_UNSUPPORTED, "search radius above walker range");
  }
  return check_launch();
}
}  // namespace

extern "C" {

int pl_abi_version(void) { return PLGPU_ABI_VERSION; }

int pl_debug_set_route(int32_t walker, int32_t lines, int32_t wpc) {
  if (walker < 0 || walker > 3 || (lines != 0 && lines != 1 && lines != 2) ||
      (wpc != 0 && wpc != 2 && wpc != 8))
    return set_err(PL_ERR_ARG, "debug route: walker 0..3, lines 0/1/2, wpc 0/2/8");
  g_dbg_fold.store(walker == 3 ? 2 : 0);  // 3: default walkers, 1D lines never folded
  if (walker == 3) walker = 0;
  g_dbg_walker.store(walker);
  g_dbg_lines.store(lines);
  g_dbg_wpc.store(wpc);
  return PL_OK;
}

int pl_set_precision_policy(int32_t policy) {
  if (policy != PL_PRECISION_AUTO && policy != PL_PRECISION_FAST)
    return set_err(PL_ERR_ARG, "precision policy: PL_PRECISION_AUTO or PL_PRECISION_FAST");
  g_policy.store(policy);
  return PL_OK;
}

int32_t pl_precision_policy(void) { return g_policy.load(); }

double pl_fast_h_threshold(void) { return kFastH; }

const char* pl_last_error(void) { return g_err.c_str(); }

const char* pl_last_route(void) { return g_route.c_str(); }

const char* pl_device_name(void) {
  static thread_local char name[256];
  name[0] = 0;
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
    std::snprintf(name, sizeof(name), "%s", prop.name);
  else
    cudaGetLastError();
  return name;
}

int pl_validate_params(pl_params p, int32_t n) { return validate_params(p, n); }

int pl_validate_geometry(int32_t S, int32_t K, int32_t n) { return validate_geometry(S, K, n); }

int pl_op_counts_1d(int32_t n, pl_params p, pl_op_counts* out) {
  int rc = validate_params(p, n);
  if (rc) return rc;
  if (!out) return set_err(PL_ERR_ARG, "null op counter");
  const uint64_t S = (uint64_t)p.search_radius, K = (uint64_t)p.patch_radius;
  // compute_banded_kernel (banded_kernel.cpp:49-66): per diagonal d <= min(S, n-1)
  const int64_t maxd = std::min<int64_t>(p.search_radius, (int64_t)n - 1);
  uint64_t adds = 0, muls = 0, windows = 0;
  for (int64_t d = 0; d <= maxd; ++d) {
    adds += 2 * K + 2 * (uint64_t)(n - d - 1);
    muls += 2 * K + 1 + 2 * (uint64_t)(n - d - 1);
  }
  // window loop (nlm.cpp:155-162)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = std::max<int64_t>(0, i - (int64_t)S);
    const int64_t hi = std::min<int64_t>(n - 1, i + (int64_t)S);
    windows += (uint64_t)(hi - lo + 1);
  }
  out->adds += adds + windows * 4;
  out->muls += muls + windows * 2;
  out->exps += windows;
  return PL_OK;
}

uint64_t pl_unique_pairs(int32_t n, int32_t S) {
  if (n < 1 || S < 0) return 0;
  const uint64_t s = (uint64_t)std::min<int64_t>(S, (int64_t)n - 1);
  return (uint64_t)n * s - s * (s + 1) / 2;
}

int32_t pl_segment_length(int32_t n, int32_t S) { return segment_length(n, S); }

int pl_nlm_lines(const float* src, float* dst, int64_t n_lines, int32_t n, int64_t ld, pl_params p,
                 void* stream) {
  int rc = validate_params(p, n);
  if (rc) return rc;
  if ((rc = check_ptrs(src, dst))) return rc;
  bool precise = false;
  if ((rc = choose_precise(src, n_lines, n, ld, p.h, as_stream(stream), &precise))) return rc;
  if (precise)
    return run_precise(src, dst, n_lines, n, ld, 0, as_stream(stream),
                       [&](double* s64, double* d64, double*) {
                         return pl_nlm_lines_f64(s64, d64, n_lines, n, n, p, stream);
                       });
  plgpu::PassDesc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = n_lines;
  g.lines_per_img = (int32_t)std::max<int64_t>(1, std::min<int64_t>(n_lines, INT32_MAX));
  g.src_img_stride = g.dst_img_stride = ld * g.lines_per_img;
  g.src_line_stride = g.dst_line_stride = ld;
  g.src_pos_stride = g.dst_pos_stride = 1;
  g.dst_pos_block = n;
  g.n = n;
  return run_pass(g, p, as_stream(stream));
}

int pl_nlm_lines_naive(const float* src, float* dst, int64_t n_lines, int32_t n, int64_t ld,
                       pl_params p, void* stream) {
  int rc = validate_params(p, n);
  if (rc) return rc;
  if ((rc = check_ptrs(src, dst))) return rc;
  if (n_lines <= 0) return PL_OK;
  plgpu::DirectDesc g{src, dst, n_lines, ld, n, p.search_radius, p.patch_radius,
                      weight_coef(p.h)};
  const int64_t work = n_lines * n;
  plgpu::nlm_direct_kernel<<<(unsigned)((work + 127) / 128), 128, 0, as_stream(stream)>>>(g);
  return check_launch();
}

int pl_nlm_row_pass(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  bool precise = false;
  if ((rc = choose_precise(src, (int64_t)batch * rows, cols, cols, p.h, as_stream(stream), &precise)))
    return rc;
  if (precise) return precise_image(3, src, dst, batch, rows, cols, p, as_stream(stream));
  return run_pass(row_desc(src, dst, batch, rows, cols), p, as_stream(stream));
}

int pl_nlm_col_pass(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  bool precise = false;
  if ((rc = choose_precise(src, (int64_t)batch * rows, cols, cols, p.h, as_stream(stream), &precise)))
    return rc;
  if (precise) return precise_image(4, src, dst, batch, rows, cols, p, as_stream(stream));
  return run_pass(col_desc(src, dst, batch, rows, cols), p, as_stream(stream));
}

// Rows of the column-pass input that the walkers may read (loads, staging
// over-fetch included) while producing segments [seg_begin, seg_end): the
// exact recurrence needs [s0 - S - K - 1, s1 + 2S + K] (walk3 chunk ring);
// the chunked v2 walker stages up to 16 rows ahead of its anchor and
// 2K + 80 rows past the last window.  Positions past a line end are
// half-sample mirrored, exactly as the kernels do.
static void col_window(int32_t n, int32_t S, int32_t K, int32_t seg_begin, int32_t seg_end,
                       int32_t* in_lo, int32_t* in_hi, int32_t* out_lo, int32_t* out_hi) {
  const int32_t C = segment_length(n, S);
  const int32_t s0 = seg_begin * C, s1 = std::min(n, seg_end * C);
  const int64_t lo_raw = (int64_t)s0 - S - K - 1 - 16;
  const int64_t hi_raw = (int64_t)s1 + 2 * S + 2 * K + 81;  // exclusive
  auto mirror = [n](int64_t p) -> int32_t {
    p = p < 0 ? -1 - p : p;
    p = p >= n ? 2 * (int64_t)n - 1 - p : p;
    return (int32_t)std::min<int64_t>(std::max<int64_t>(p, 0), n - 1);
  };
  int32_t lo = (int32_t)std::max<int64_t>(0, std::min<int64_t>(lo_raw, n - 1));
  int32_t hi = (int32_t)std::min<int64_t>(n, std::max<int64_t>(hi_raw, 1));
  // Mirrored reads land within S+K+17 rows of a line end; widen to cover them.
  if (lo_raw < 0) hi = std::max(hi, mirror(lo_raw) + 1);
  if (hi_raw > n) lo = std::min(lo, mirror(hi_raw - 1));
  *in_lo = lo;
  *in_hi = hi;
  *out_lo = s0;
  *out_hi = s1;
}

int pl_col_window(int32_t rows_total, int32_t seg_begin, int32_t seg_end, pl_params p,
                  int32_t* in_lo, int32_t* in_hi, int32_t* out_lo, int32_t* out_hi) {
  int rc = validate_params(p, rows_total);
  if (rc) return rc;
  if (!in_lo || !in_hi || !out_lo || !out_hi) return set_err(PL_ERR_ARG, "null output pointer");
  const int32_t S = std::min<int32_t>(p.search_radius, rows_total - 1);
  const int32_t C = segment_length(rows_total, S);
  const int32_t nseg = (rows_total + C - 1) / C;
  if (seg_begin < 0 || seg_end > nseg || seg_begin >= seg_end)
    return set_err(PL_ERR_RANGE, "segment range out of range");
  col_window(rows_total, S, p.patch_radius, seg_begin, seg_end, in_lo, in_hi, out_lo, out_hi);
  return PL_OK;
}

int pl_nlm_col_pass_window(const float* src, int32_t in_lo, int32_t in_rows, float* dst,
                           int32_t batch, int32_t rows_total, int32_t cols, int32_t seg_begin,
                           int32_t seg_end, pl_params p, void* stream) {
  int rc = validate_image(batch, rows_total, cols);
  if (!rc) rc = validate_params(p, rows_total);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if ((rc = require_fp32_bounded(p.h))) return rc;
  int32_t need_lo, need_hi, out_lo, out_hi;
  if ((rc = pl_col_window(rows_total, seg_begin, seg_end, p, &need_lo, &need_hi, &out_lo,
                          &out_hi)))
    return rc;
  if (in_lo < 0 || in_rows < 1 || in_lo > need_lo || (int64_t)in_lo + in_rows < need_hi ||
      (int64_t)in_lo + in_rows > rows_total)
    return set_err(PL_ERR_RANGE, "input window does not cover the rows pl_col_window requires");
  const int32_t S = std::min<int32_t>(p.search_radius, rows_total - 1);
  if (S < 1 || S > kMaxWalkS)
    return set_err(PL_ERR_UNSUPPORTED, "windowed column pass needs 1 <= S <= 32");
  // Global row coordinates: the kernels address src/dst as if they held the
  // whole line (only rows inside the windows are ever touched).
  plgpu::PassDesc g = col_desc(nullptr, nullptr, batch, rows_total, cols);
  g.src = reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(src) -
                                         (uintptr_t)in_lo * cols * sizeof(float));
  g.dst = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(dst) -
                                   (uintptr_t)out_lo * cols * sizeof(float));
  g.src_img_stride = (int64_t)in_rows * cols;
  g.dst_img_stride = (int64_t)(out_hi - out_lo) * cols;
  g.seg_begin = seg_begin;
  g.nseg = seg_end - seg_begin;
  return run_pass(g, p, as_stream(stream));
}

int pl_nlm_pass_strided(const float* src, float* dst, int32_t batch, int32_t lines, int32_t n,
                        int64_t src_line_stride, int64_t src_pos_stride, int64_t dst_line_stride,
                        int64_t dst_pos_stride, int64_t img_stride, pl_params p, void* stream) {
  int rc = validate_image(batch, lines, n);
  if (!rc) rc = validate_params(p, n);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if ((rc = require_fp32_bounded(p.h))) return rc;
  if (src_line_stride < 0 || src_pos_stride < 1 || dst_line_stride < 0 || dst_pos_stride < 1 ||
      img_stride < 0)
    return set_err(PL_ERR_ARG, "strides must be nonnegative (position strides positive)");
  plgpu::PassDesc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = (int64_t)batch * lines;
  g.lines_per_img = lines;
  g.src_img_stride = g.dst_img_stride = img_stride;
  g.src_line_stride = src_line_stride;
  g.src_pos_stride = src_pos_stride;
  g.dst_line_stride = dst_line_stride;
  g.dst_pos_stride = dst_pos_stride;
  g.dst_pos_block = n;
  g.n = n;
  return run_pass(g, p, as_stream(stream));
}

int pl_nlm_row_pass_fanout(const float* src, float* dst, int32_t rows, int32_t cols, pl_params p,
                           int32_t n_extra, float* const* extra, const int32_t* lo, const int32_t* hi,
                           void* stream) {
  int rc = validate_image(1, rows, cols);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if ((rc = require_fp32_bounded(p.h))) return rc;
  if (n_extra < 0 || n_extra > PL_MAX_FANOUT || (n_extra > 0 && (!extra || !lo || !hi)))
    return set_err(PL_ERR_ARG, "n_extra must be 0..PL_MAX_FANOUT with extra/lo/hi arrays");
  for (int x = 0; x < n_extra; ++x)
    if (!extra[x] || lo[x] < 0 || lo[x] > hi[x] || hi[x] > rows)
      return set_err(PL_ERR_ARG, "fan-out rows must satisfy 0 <= lo <= hi <= rows, non-null extra");
  cudaStream_t st = as_stream(stream);
  plgpu::PassDesc g = row_desc(src, dst, 1, rows, cols);
  const int S_eff = std::min<int>(p.search_radius, cols - 1);
  if (S_eff < 1 || S_eff > kMaxWalkS) {  // direct route: pass, then copy the rows out
    if ((rc = run_pass(g, p, st))) return rc;
    for (int x = 0; x < n_extra; ++x)
      if (hi[x] > lo[x])
        PL_CUDA(cudaMemcpyAsync(extra[x], dst + (int64_t)lo[x] * cols,
                                sizeof(float) * (size_t)(hi[x] - lo[x]) * cols, cudaMemcpyDefault, st));
    return PL_OK;
  }
  g.nx = n_extra;
  for (int x = 0; x < n_extra; ++x) {
    g.xdst[x] = extra[x];
    g.xlo[x] = lo[x];
    g.xhi[x] = hi[x];
  }
  return run_pass(g, p, st);
}

int pl_nlm_row_pass_blocked(const float* src, float* dst, int32_t batch, int32_t rows,
                            int32_t cols, int32_t col_block, pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if ((rc = require_fp32_bounded(p.h))) return rc;
  if (col_block < 1 || cols % col_block != 0)
    return set_err(PL_ERR_ARG, "cols must be a positive multiple of col_block");
  plgpu::PassDesc g = row_desc(src, dst, batch, rows, cols);
  g.dst_line_stride = col_block;
  g.dst_pos_block = col_block;
  g.dst_block_stride = (int64_t)rows * col_block;
  return run_pass(g, p, as_stream(stream));
}

size_t pl_workspace_bytes(int32_t op, int32_t batch, int32_t rows, int32_t cols) {
  const size_t img = (size_t)std::max(batch, 0) * std::max(rows, 0) * std::max(cols, 0) * sizeof(float);
  return op == 2 ? 2 * img : img;  // op 2: snlm (CR, mid); else one intermediate
}

int pl_snlm_2d_row_col(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  bool precise = false;
  if ((rc = choose_precise(src, (int64_t)batch * rows, cols, cols, p.h, as_stream(stream), &precise)))
    return rc;
  if (precise) return precise_image(0, src, dst, batch, rows, cols, p, as_stream(stream));
  Scratch scratch(as_stream(stream));
  if (!work && (rc = scratch.alloc(pl_workspace_bytes(0, batch, rows, cols), &work))) return rc;
  return rc_passes(src, dst, work, batch, rows, cols, p, as_stream(stream));
}

// ---- CUDA Graph of the RC composite ----------------------------------------
// Both passes captured once on a private stream (the intermediate owned by the
// graph unless the caller passes `work`); each pl_graph_launch replays them
// with one launch call.  For repeated small calls (c2-sized images) the two
// kernel launches and the scratch allocation leave the per-call path.
struct pl_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  float* owned = nullptr;
};

int pl_graph_rc_create(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, pl_graph** out) {
  if (!out) return set_err(PL_ERR_ARG, "null graph handle");
  *out = nullptr;
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if (g_policy.load(std::memory_order_relaxed) != PL_PRECISION_FAST && p.h < kFastH)
    return set_err(PL_ERR_UNSUPPORTED,
                   "graph capture covers the fp32 kernels only: h is below their bounded range "
                   "(pl_fast_h_threshold); use pl_snlm_2d_row_col or PL_PRECISION_FAST");
  pl_graph* g = new pl_graph();
  auto fail = [&](int code) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->owned) cudaFree(g->owned);
    delete g;
    return code;
  };
  if (!work) {
    cudaError_t e = cudaMalloc(&g->owned, std::max<size_t>(16, pl_workspace_bytes(0, batch, rows, cols)));
    if (e != cudaSuccess) return fail(set_err(PL_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
    work = g->owned;
  }
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(set_err(PL_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e)));
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    rc = rc_passes(src, dst, work, batch, rows, cols, p, st);
    cudaGraph_t graph = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(st, &graph);
    g->graph = graph;
    if (!rc && e2 != cudaSuccess)
      rc = set_err(PL_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e2));
  } else {
    rc = set_err(PL_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
  }
  cudaStreamDestroy(st);
  if (rc) return fail(rc);
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess)
    return fail(set_err(PL_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e)));
  *out = g;
  return PL_OK;
}

int pl_graph_launch(pl_graph* g, void* stream) {
  if (!g || !g->exec) return set_err(PL_ERR_ARG, "null graph");
  PL_CUDA(cudaGraphLaunch(g->exec, as_stream(stream)));
  return PL_OK;
}

int pl_graph_destroy(pl_graph* g) {
  if (!g) return PL_OK;
  cudaError_t e = cudaSuccess;
  if (g->exec) e = cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  if (g->owned) cudaFree(g->owned);
  delete g;
  if (e != cudaSuccess) return set_err(PL_ERR_CUDA, std::string("cudaGraphExecDestroy: ") + cudaGetErrorString(e));
  return PL_OK;
}

int pl_snlm_2d_col_row(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
                       int32_t cols, pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  bool precise = false;
  if ((rc = choose_precise(src, (int64_t)batch * rows, cols, cols, p.h, as_stream(stream), &precise)))
    return rc;
  if (precise) return precise_image(1, src, dst, batch, rows, cols, p, as_stream(stream));
  Scratch scratch(st);
  if (!work && (rc = scratch.alloc(pl_workspace_bytes(1, batch, rows, cols), &work))) return rc;
  if ((rc = run_pass(col_desc(src, work, batch, rows, cols), p, st))) return rc;
  return run_pass(row_desc(work, dst, batch, rows, cols), p, st);
}

int pl_snlm_2d(const float* src, float* dst, float* work, int32_t batch, int32_t rows,
               int32_t cols, pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  bool precise = false;
  if ((rc = choose_precise(src, (int64_t)batch * rows, cols, cols, p.h, as_stream(stream), &precise)))
    return rc;
  if (precise) return precise_image(2, src, dst, batch, rows, cols, p, as_stream(stream));
  Scratch scratch(as_stream(stream));
  if (!work && (rc = scratch.alloc(pl_workspace_bytes(2, batch, rows, cols), &work))) return rc;
  const int64_t cnt = (int64_t)batch * rows * cols;
  float* cr_img = work;
  float* mid = work + cnt;
  // CR into the workspace, then RC with the average fused into the final
  // column pass's store: dst = (CR + RC) / 2 (average(), nlm.cpp:106-112).
  // (the fp32 route is decided: run CR's passes directly, not through its entry point)
  if ((rc = run_pass(col_desc(src, mid, batch, rows, cols), p, as_stream(stream)))) return rc;
  if ((rc = run_pass(row_desc(mid, cr_img, batch, rows, cols), p, as_stream(stream)))) return rc;
  return rc_passes(src, dst, mid, batch, rows, cols, p, as_stream(stream), cr_img);
}

namespace {

// Copy streams and events are kept per host thread and device between calls
// (the call blocks until its pipeline has drained, so they are idle again).
struct HostPipe {
  int dev = -1;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  void reset() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    s_in = s_out = nullptr;
  }
  ~HostPipe() { reset(); }
  int open() {
    int d = 0;
    PL_CUDA(cudaGetDevice(&d));
    if (d != dev) {
      reset();
      dev = d;
    }
    if (!s_in) PL_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    if (!s_out) PL_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    used = 0;
    return PL_OK;
  }
  int event(cudaEvent_t* out) {
    if (used == ev.size()) {
      cudaEvent_t e = nullptr;
      PL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    *out = ev[used++];
    return PL_OK;
  }
};
HostPipe& host_pipe() {
  thread_local HostPipe pipe;
  return pipe;
}

// Host-buffer RC of LARGE images, streamed inside the image: rows go up in
// chunks (H2D engine), each chunk's row pass runs as it lands, and as soon as
// the rows a block of column-pass segments reads are present
// (col_window: whole segments, so the result is bitwise the full pass's) that
// block's column pass runs and its output rows go down (D2H engine).  Upload,
// both passes and download of one image overlap; a 16384^2 image (1 GiB each
// way) takes ~max(H2D, D2H) instead of H2D + passes + D2H.
int host_rc_streamed(const float* host_src, float* host_dst, int32_t batch, int32_t rows,
                     int32_t cols, const pl_params& p, cudaStream_t st) {
  const size_t img = (size_t)rows * cols;
  const int32_t S_col = std::min<int32_t>(p.search_radius, rows - 1);
  const int32_t C = segment_length(rows, S_col);
  const int32_t nseg = (rows + C - 1) / C;
  const size_t row_bytes = (size_t)cols * sizeof(float);
  // Chunk sizes by WARPS, not bytes: a pass launch takes at least one segment
  // walk (c5: ~0.45 ms) however few lines it has, and the launches of one
  // image run back to back on `st`, so each should fill the GPU (~148 x 8
  // warps of 32 lines) -- capped at a quarter of the image so that uploads,
  // passes and downloads still overlap (c3: 4 row chunks, 5 column blocks).
  const int32_t S_row = std::min<int32_t>(p.search_radius, cols - 1);
  const int32_t C_row = segment_length(cols, S_row);
  const int32_t nseg_row = (cols + C_row - 1) / C_row;
  constexpr int64_t kWave = 148 * 8;
  auto up64 = [](int64_t v) { return (v + 63) / 64 * 64; };
  const int32_t chunk_rows = (int32_t)std::min<int64_t>(
      rows, std::max<int64_t>(64, std::min<int64_t>(up64((kWave + nseg_row - 1) / nseg_row * 32),
                                                    up64((rows + 3) / 4))));
  const int64_t warps_per_seg = std::max<int64_t>(1, cols / 32);
  const int32_t segs_per_block = (int32_t)std::max<int64_t>(
      1, std::min<int64_t>((kWave + warps_per_seg - 1) / warps_per_seg, nseg / 4));
  HostPipe& pipe = host_pipe();
  if (int r = pipe.open()) return r;
  Scratch scratch(st);
  float* buf = nullptr;
  int rc = scratch.alloc(3 * img * sizeof(float), &buf);
  if (rc) return rc;
  float* in = buf;
  float* mid = buf + img;  // transposed intermediate [cols][rows] (rc_passes)
  float* out = buf + 2 * img;
  cudaEvent_t start = nullptr, drained = nullptr;
  if ((rc = pipe.event(&start)) || (rc = pipe.event(&drained))) return rc;
  PL_CUDA(cudaEventRecord(start, st));  // after the caller's prior work and the allocation
  PL_CUDA(cudaStreamWaitEvent(pipe.s_in, start, 0));
  auto image = [&](int b) -> int {
    const float* hs = host_src + (size_t)b * img;
    float* hd = host_dst + (size_t)b * img;
    int32_t uploaded = 0;
    for (int32_t a = 0; a < nseg; a += segs_per_block) {
      const int32_t bb = std::min(nseg, a + segs_per_block);
      int32_t in_lo, in_hi, out_lo, out_hi;
      col_window(rows, S_col, p.patch_radius, a, bb, &in_lo, &in_hi, &out_lo, &out_hi);
      const int32_t need = std::min<int64_t>(rows, ((int64_t)in_hi + 63) / 64 * 64);
      while (uploaded < need) {
        const int32_t r0 = uploaded, r1 = std::min(rows, r0 + chunk_rows);
        cudaEvent_t up = nullptr;
        if (int r = pipe.event(&up)) return r;
        PL_CUDA(cudaMemcpyAsync(in + (size_t)r0 * cols, hs + (size_t)r0 * cols,
                                (size_t)(r1 - r0) * row_bytes, cudaMemcpyHostToDevice, pipe.s_in));
        PL_CUDA(cudaEventRecord(up, pipe.s_in));
        PL_CUDA(cudaStreamWaitEvent(st, up, 0));
        plgpu::PassDesc rp = row_desc(in + (size_t)r0 * cols, mid + r0, 1, r1 - r0, cols);
        rp.dst_line_stride = 1;  // row r becomes column r of the transposed intermediate
        rp.dst_pos_stride = rows;
        if (int r = run_pass(rp, p, st)) return r;
        uploaded = r1;
      }
      plgpu::PassDesc cp = col_desc(mid, out, 1, rows, cols);
      cp.src_line_stride = rows;
      cp.src_pos_stride = 1;
      cp.seg_begin = a;
      cp.nseg = bb - a;
      if (int r = run_pass(cp, p, st)) return r;
      cudaEvent_t done = nullptr;
      if (int r = pipe.event(&done)) return r;
      PL_CUDA(cudaEventRecord(done, st));
      PL_CUDA(cudaStreamWaitEvent(pipe.s_out, done, 0));
      PL_CUDA(cudaMemcpyAsync(hd + (size_t)out_lo * cols, out + (size_t)out_lo * cols,
                              (size_t)(out_hi - out_lo) * row_bytes, cudaMemcpyDeviceToHost,
                              pipe.s_out));
    }
    if (b + 1 < batch) {  // the next image reuses the three buffers
      cudaEvent_t passes = nullptr, down = nullptr;
      if (int r = pipe.event(&passes)) return r;
      if (int r = pipe.event(&down)) return r;
      PL_CUDA(cudaEventRecord(passes, st));
      PL_CUDA(cudaStreamWaitEvent(pipe.s_in, passes, 0));  // `in` is free once its row passes ran
      PL_CUDA(cudaEventRecord(down, pipe.s_out));
      PL_CUDA(cudaStreamWaitEvent(st, down, 0));  // `out` is free once it is downloaded
    }
    return PL_OK;
  };
  for (int b = 0; b < batch && !rc; ++b) rc = image(b);
  cudaError_t e0 = cudaEventRecord(drained, pipe.s_out);
  if (e0 == cudaSuccess) e0 = cudaStreamWaitEvent(st, drained, 0);  // scratch freed after the last download
  const cudaError_t e1 = cudaStreamSynchronize(pipe.s_out);
  const cudaError_t e2 = cudaStreamSynchronize(pipe.s_in);
  const cudaError_t e3 = cudaStreamSynchronize(st);
  if (rc) return rc;
  for (cudaError_t e : {e0, e1, e2, e3})
    if (e != cudaSuccess)
      return set_err(PL_ERR_CUDA, std::string("host pipeline: ") + cudaGetErrorString(e));
  return check_launch();
}

}  // namespace

int pl_snlm_2d_row_col_host(const float* host_src, float* host_dst, int32_t batch, int32_t rows,
                            int32_t cols, pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(host_src, host_dst);
  if (rc) return rc;
  // Three-stage pipeline over images: copy-in (H2D engine), filter (SMs),
  // copy-out (D2H engine) on three streams ordered by events, NSLOT device
  // slots of (in, mid, out) so image b+2's upload, image b+1's filter and
  // image b's download run concurrently.  Group images so each transfer is
  // >= ~8 MiB (fewer, larger copies).  Every CUDA call is checked; on an
  // error the pipeline drains (all three streams synchronised) before the
  // first error is returned.
  cudaStream_t st = as_stream(stream);
  const size_t img = (size_t)rows * cols;
  // precision policy on host data: the range is scanned on the host
  bool precise = false;
  if (g_policy.load(std::memory_order_relaxed) != PL_PRECISION_FAST && p.h < kFastH) {
    float lo = std::numeric_limits<float>::infinity(), hi = -lo;
    const size_t total = img * batch;
    for (size_t i = 0; i < total; ++i) {
      const float v = host_src[i];
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
    precise = hi >= lo && p.h < kFastH * ((double)hi - (double)lo) / 255.0;
  }
  // large images: stream rows / column-pass segments inside the image
  if (!precise && img * sizeof(float) >= (32u << 20) && rows >= 1024)
    return host_rc_streamed(host_src, host_dst, batch, rows, cols, p, st);
  const int per = (int)std::max<size_t>(1, std::min<size_t>(batch, (8u << 20) / (img * 4) + 1));
  const int ngroups = (batch + per - 1) / per;
  constexpr int NSLOT = 3;
  const size_t slot_elems = 3 * img * per;
  HostPipe& pipe = host_pipe();  // copy streams + events, kept per host thread
  if ((rc = pipe.open())) return rc;
  cudaEvent_t evs[3 * NSLOT + 2];
  for (cudaEvent_t& e : evs)
    if ((rc = pipe.event(&e))) return rc;
  cudaEvent_t* up = evs;
  cudaEvent_t* done = evs + NSLOT;
  cudaEvent_t* freed = evs + 2 * NSLOT;
  cudaEvent_t start = evs[3 * NSLOT], drained = evs[3 * NSLOT + 1];
  Scratch scratch(st);  // freed on st after `drained` (below)
  float* buf = nullptr;
  if ((rc = scratch.alloc(NSLOT * slot_elems * sizeof(float), &buf))) return rc;
  // the caller's stream orders the whole pipeline after prior work (and the allocation)
  PL_CUDA(cudaEventRecord(start, st));
  PL_CUDA(cudaStreamWaitEvent(pipe.s_in, start, 0));
  auto step = [&](int gi) -> int {
    const int k = gi % NSLOT;
    const int b0 = gi * per, nb = std::min(per, batch - b0);
    float* in = buf + k * slot_elems;
    float* mid = in + img * per;
    float* out = mid + img * per;
    if (gi >= NSLOT) PL_CUDA(cudaStreamWaitEvent(pipe.s_in, freed[k], 0));  // slot's download done
    PL_CUDA(cudaMemcpyAsync(in, host_src + (size_t)b0 * img, nb * img * sizeof(float),
                            cudaMemcpyHostToDevice, pipe.s_in));
    PL_CUDA(cudaEventRecord(up[k], pipe.s_in));
    PL_CUDA(cudaStreamWaitEvent(st, up[k], 0));
    int r = precise ? precise_image(0, in, out, nb, rows, cols, p, st)
                    : rc_passes(in, out, mid, nb, rows, cols, p, st);
    if (r) return r;
    PL_CUDA(cudaEventRecord(done[k], st));
    PL_CUDA(cudaStreamWaitEvent(pipe.s_out, done[k], 0));
    PL_CUDA(cudaMemcpyAsync(host_dst + (size_t)b0 * img, out, nb * img * sizeof(float),
                            cudaMemcpyDeviceToHost, pipe.s_out));
    PL_CUDA(cudaEventRecord(freed[k], pipe.s_out));
    return PL_OK;
  };
  for (int gi = 0; gi < ngroups && !rc; ++gi) rc = step(gi);
  // the scratch is released on st only after the last download
  cudaError_t e0 = cudaEventRecord(drained, pipe.s_out);
  if (e0 == cudaSuccess) e0 = cudaStreamWaitEvent(st, drained, 0);
  const cudaError_t e1 = cudaStreamSynchronize(pipe.s_out);
  const cudaError_t e2 = cudaStreamSynchronize(pipe.s_in);
  const cudaError_t e3 = cudaStreamSynchronize(st);
  if (rc) return rc;
  for (cudaError_t e : {e0, e1, e2, e3})
    if (e != cudaSuccess) return set_err(PL_ERR_CUDA, std::string("host pipeline: ") + cudaGetErrorString(e));
  return check_launch();
}


int pl_debug_hot_distance_band(const float* src, float* band, int32_t n_lines, int32_t n,
                               int32_t S, int32_t K, void* stream) {
  int rc = validate_image(1, n_lines, n);
  if (!rc) rc = validate_geometry(S, K, n);
  if (!rc) rc = check_ptrs(src, band);
  if (rc) return rc;
  if (n_lines < 16 || S > n - 1 || plgpu::pass3_k_for(template_radius(S)) != K ||
      template_radius(S) != S)
    return set_err(PL_ERR_UNSUPPORTED,
                   "hot distance export needs >= 16 lines, a hot (K, S) pair and S <= n - 1");
  cudaStream_t st = as_stream(stream);
  PL_CUDA(cudaMemsetAsync(band, 0xFF, sizeof(float) * (size_t)n_lines * n * (2 * S + 1), st));
  Scratch scratch(st);
  float* out = nullptr;
  if ((rc = scratch.alloc(sizeof(float) * (size_t)n_lines * n, &out))) return rc;
  plgpu::PassDesc g = row_desc(src, out, 1, n_lines, n);
  g.dexp = band;
  return run_pass(g, pl_params{S, K, 1.0}, st);
}

int pl_distance_band_f32(const float* src, float* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t S, int32_t K, void* stream) {
  return distance_band<float>(src, band, n_lines, n, ld, S, K, as_stream(stream));
}

int pl_distance_band_i32(const float* src, int32_t* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t S, int32_t K, void* stream) {
  return distance_band<int32_t>(src, band, n_lines, n, ld, S, K, as_stream(stream));
}

int pl_banded_kernel_f64(const double* src, double* band, int64_t n_lines, int32_t n, int64_t ld,
                         int32_t S, int32_t K, void* stream) {
  int rc = validate_geometry(S, K, n);
  if (rc) return rc;
  if ((rc = check_ptrs(src, band))) return rc;
  if (n_lines <= 0) return PL_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t cells = n_lines * (int64_t)n * (2 * S + 1);
  PL_CUDA(cudaMemsetAsync(band, 0xFF, cells * sizeof(double), st));  // NaN sentinel
  plgpu::KernelBandDesc g{src, band, n_lines, ld, n, std::min<int32_t>(S, n - 1), S, K};
  const int64_t work = n_lines * (g.S + 1);
  plgpu::banded_kernel_f64<<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
  return check_launch();
}

}  // extern "C"

extern "C" {

// ---- fp64 reference-precision route (plgpu_walk64.cuh) -----------------------
}  // extern "C"

namespace {

plgpu::Pass64Desc desc64(const double* src, double* dst, int batch, int rows, int cols, bool col) {
  plgpu::Pass64Desc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = (int64_t)batch * (col ? cols : rows);
  g.lines_per_img = col ? cols : rows;
  g.src_img_stride = g.dst_img_stride = (int64_t)rows * cols;
  g.src_line_stride = g.dst_line_stride = col ? 1 : cols;
  g.src_pos_stride = g.dst_pos_stride = col ? cols : 1;
  g.n = col ? rows : cols;
  return g;
}

int run_pass64(plgpu::Pass64Desc g, const pl_params& p, cudaStream_t st) {
  g.S = std::min<int32_t>(p.search_radius, g.n - 1);
  g.K = p.patch_radius;
  g.inv_h2 = 1.0 / (p.h * p.h);
  g.seg_len = segment_length(g.n, g.S);
  g.nseg = (g.n + g.seg_len - 1) / g.seg_len;
  if (g.n_lines <= 0) return PL_OK;
  if (g.S >= 1 && g.S <= kMaxWalkS) {
    g_route = "f64<S=" + std::to_string(template_radius(g.S)) + ">";
    switch (template_radius(g.S)) {
#define PL_CASE(v) \
  case v: plgpu::launch_pass64<v>(g, st); break;
      PLGPU_FOR_EACH_RADIUS(PL_CASE)
#undef PL_CASE
    }
    return check_launch();
  }
  g_route = "f64-direct";
  const int64_t work = g.n_lines * g.n;
  plgpu::direct_pass64_kernel<<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
  return check_launch();
}

int image_checks64(const double* src, const double* dst, int batch, int rows, int cols,
                   const pl_params& p) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  return rc;
}

}  // namespace

extern "C" {

int pl_nlm_lines_f64(const double* src, double* dst, int64_t n_lines, int32_t n, int64_t ld,
                     pl_params p, void* stream) {
  int rc = validate_params(p, n);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  plgpu::Pass64Desc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = n_lines;
  g.lines_per_img = (int32_t)std::max<int64_t>(1, std::min<int64_t>(n_lines, INT32_MAX));
  g.src_img_stride = g.dst_img_stride = ld * g.lines_per_img;
  g.src_line_stride = g.dst_line_stride = ld;
  g.src_pos_stride = g.dst_pos_stride = 1;
  g.n = n;
  return run_pass64(g, p, as_stream(stream));
}

int pl_nlm_lines_naive_f64(const double* src, double* dst, int64_t n_lines, int32_t n, int64_t ld,
                           pl_params p, void* stream) {
  int rc = validate_params(p, n);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  if (n_lines <= 0) return PL_OK;
  plgpu::Pass64Desc g{};
  g.src = src;
  g.dst = dst;
  g.n_lines = n_lines;
  g.lines_per_img = (int32_t)std::max<int64_t>(1, std::min<int64_t>(n_lines, INT32_MAX));
  g.src_img_stride = g.dst_img_stride = ld * g.lines_per_img;
  g.src_line_stride = g.dst_line_stride = ld;
  g.src_pos_stride = g.dst_pos_stride = 1;
  g.n = n;
  g.S = p.search_radius;  // the naive route does not clip S (windows are clipped per pixel)
  g.K = p.patch_radius;
  g.inv_h2 = 1.0 / (p.h * p.h);
  const int64_t work = n_lines * n;
  plgpu::direct_pass64_kernel<<<(unsigned)((work + 127) / 128), 128, 0, as_stream(stream)>>>(g);
  return check_launch();
}

int pl_nlm_row_pass_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, cols);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  return run_pass64(desc64(src, dst, batch, rows, cols, false), p, as_stream(stream));
}

int pl_nlm_col_pass_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, rows);
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  return run_pass64(desc64(src, dst, batch, rows, cols, true), p, as_stream(stream));
}

int pl_snlm_2d_row_col_f64(const double* src, double* dst, double* work, int32_t batch,
                           int32_t rows, int32_t cols, pl_params p, void* stream) {
  int rc = image_checks64(src, dst, batch, rows, cols, p);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  Scratch scratch(st);
  if (!work && (rc = scratch.alloc(2 * pl_workspace_bytes(0, batch, rows, cols), &work))) return rc;
  if ((rc = run_pass64(desc64(src, work, batch, rows, cols, false), p, st))) return rc;
  return run_pass64(desc64(work, dst, batch, rows, cols, true), p, st);
}

int pl_snlm_2d_col_row_f64(const double* src, double* dst, double* work, int32_t batch,
                           int32_t rows, int32_t cols, pl_params p, void* stream) {
  int rc = image_checks64(src, dst, batch, rows, cols, p);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  Scratch scratch(st);
  if (!work && (rc = scratch.alloc(2 * pl_workspace_bytes(1, batch, rows, cols), &work))) return rc;
  if ((rc = run_pass64(desc64(src, work, batch, rows, cols, true), p, st))) return rc;
  return run_pass64(desc64(work, dst, batch, rows, cols, false), p, st);
}

int pl_snlm_2d_f64(const double* src, double* dst, double* work, int32_t batch, int32_t rows,
                   int32_t cols, pl_params p, void* stream) {
  int rc = image_checks64(src, dst, batch, rows, cols, p);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  Scratch scratch(st);
  if (!work && (rc = scratch.alloc(2 * pl_workspace_bytes(2, batch, rows, cols), &work))) return rc;
  const int64_t cnt = (int64_t)batch * rows * cols;
  double* cr_img = work;
  double* mid = work + cnt;
  if ((rc = pl_snlm_2d_col_row_f64(src, cr_img, mid, batch, rows, cols, p, stream))) return rc;
  if ((rc = run_pass64(desc64(src, mid, batch, rows, cols, false), p, st))) return rc;
  plgpu::Pass64Desc g = desc64(mid, dst, batch, rows, cols, true);
  g.avg = cr_img;  // (CR + RC) / 2 fused into the final store (average(), nlm.cpp:106-112)
  return run_pass64(g, p, st);
}

int pl_nlm_2d_naive_f64(const double* src, double* dst, int32_t batch, int32_t rows, int32_t cols,
                        pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, std::min(rows, cols));
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  plgpu::Naive2D64Desc g{src, dst, batch, rows, cols, p.search_radius, p.patch_radius,
                         1.0 / (p.h * p.h)};
  const int64_t work = (int64_t)batch * rows * cols;
  plgpu::nlm_2d_naive64_kernel<<<(unsigned)((work + 127) / 128), 128, 0, as_stream(stream)>>>(g);
  return check_launch();
}

int pl_nlm_2d_naive(const float* src, float* dst, int32_t batch, int32_t rows, int32_t cols,
                    pl_params p, void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = validate_params(p, std::min(rows, cols));
  if (!rc) rc = check_ptrs(src, dst);
  if (rc) return rc;
  plgpu::Naive2DDesc g{src, dst, batch, rows, cols, p.search_radius, p.patch_radius,
                       weight_coef(p.h)};
  const int64_t work = (int64_t)batch * rows * cols;
  plgpu::nlm_2d_naive_kernel<<<(unsigned)((work + 127) / 128), 128, 0, as_stream(stream)>>>(g);
  return check_launch();
}

int pl_device_alloc(void** ptr, size_t bytes) {
  if (!ptr) return set_err(PL_ERR_ARG, "null pointer");
  PL_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
  return PL_OK;
}

int pl_device_free(void* ptr) {
  PL_CUDA(cudaFree(ptr));
  return PL_OK;
}

int pl_copy_to_device(void* dst, const void* src, size_t bytes) {
  PL_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  return PL_OK;
}

int pl_copy_to_host(void* dst, const void* src, size_t bytes) {
  PL_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  return PL_OK;
}

int pl_synchronize(void) {
  PL_CUDA(cudaDeviceSynchronize());
  return PL_OK;
}

int pl_host_alloc(void** ptr, size_t bytes) {
  if (!ptr) return set_err(PL_ERR_ARG, "null pointer");
  PL_CUDA(cudaMallocHost(ptr, bytes ? bytes : 1));
  return PL_OK;
}

int pl_host_free(void* ptr) {
  PL_CUDA(cudaFreeHost(ptr));
  return PL_OK;
}

int pl_stream_create(void** stream) {
  if (!stream) return set_err(PL_ERR_ARG, "null pointer");
  cudaStream_t s = nullptr;
  PL_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return PL_OK;
}

int pl_stream_destroy(void* stream) {
  PL_CUDA(cudaStreamDestroy(as_stream(stream)));
  return PL_OK;
}

int pl_stream_synchronize(void* stream) {
  PL_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return PL_OK;
}

int pl_copy_to_device_async(void* dst, const void* src, size_t bytes, void* stream) {
  PL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  return PL_OK;
}

int pl_copy_to_host_async(void* dst, const void* src, size_t bytes, void* stream) {
  PL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  return PL_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Fidelity metrics (metrics.cpp:98-158) on the device.
namespace {

plgpu::SsimWindow ssim_window() {  // metrics.cpp:25-37, same libm exp as the reference
  plgpu::SsimWindow w{};
  double total = 0.0;
  for (int t = 0; t < plgpu::kSsimWin; ++t) {
    const double x = t - (plgpu::kSsimWin - 1) / 2;
    w.k[t] = std::exp(-x * x / (2.0 * 1.5 * 1.5));
    total += w.k[t];
  }
  for (double& v : w.k) v /= total;
  return w;
}

template <typename T>
int image_metrics(const T* a, const T* b, int32_t batch, int32_t rows, int32_t cols, double* out,
                  void* stream) {
  int rc = validate_image(batch, rows, cols);
  if (!rc) rc = check_ptrs(a, b);
  if (rc) return rc;
  if (!out) return set_err(PL_ERR_ARG, "null output buffer");
  cudaStream_t st = as_stream(stream);
  // Images under 11x11 have no SSIM (the reference throws); mse/psnr still hold.
  const bool has_ssim = rows >= plgpu::kSsimWin && cols >= plgpu::kSsimWin;
  const int wo = has_ssim ? cols - plgpu::kSsimWin + 1 : 0;
  const int ho = has_ssim ? rows - plgpu::kSsimWin + 1 : 0;
  const dim3 tiles((wo + plgpu::kSsimTW - 1) / plgpu::kSsimTW, (ho + plgpu::kSsimTH - 1) / plgpu::kSsimTH,
                   batch);
  const int64_t ntiles = (int64_t)tiles.x * tiles.y;
  double* part = nullptr;  // stream-ordered scratch: MSE partials, then SSIM partials
  const size_t n_mse = (size_t)batch * plgpu::kMseBlocks;
  PL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part),
                          sizeof(double) * (n_mse + (size_t)batch * ntiles), st));
  const int64_t n = (int64_t)rows * cols;
  plgpu::mse_partial_kernel<T><<<dim3(plgpu::kMseBlocks, batch), plgpu::kMetricThreads, 0, st>>>(
      a, b, n, part);
  if (has_ssim)
    plgpu::ssim_partial_kernel<T><<<tiles, plgpu::kMetricThreads, 0, st>>>(a, b, rows, cols,
                                                                          ssim_window(), part + n_mse);
  plgpu::metrics_finish_kernel<<<batch, plgpu::kMetricThreads, 0, st>>>(
      part, part + n_mse, ntiles, n, (int64_t)wo * ho, out);
  rc = check_launch();
  PL_CUDA(cudaFreeAsync(part, st));
  return rc;
}

}  // namespace

int pl_image_metrics_f32(const float* a, const float* b, int32_t batch, int32_t rows, int32_t cols,
                         double* out, void* stream) {
  return image_metrics(a, b, batch, rows, cols, out, stream);
}

int pl_image_metrics_f64(const double* a, const double* b, int32_t batch, int32_t rows,
                         int32_t cols, double* out, void* stream) {
  return image_metrics(a, b, batch, rows, cols, out, stream);
}

// plgpu_launch.cuh -- launchers of the S-specialised kernels.  Each radius is
// explicitly instantiated in its own generated translation unit
// (build/gen/inst_S<ST>.cu, see paper_1407_2343_b200/build.py) so the large
// unrolled walkers compile in parallel; plgpu.cu only sees the declarations.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "plgpu_walk.cuh"
#include "plgpu_walk2.cuh"
#include "plgpu_walk3.cuh"
#include "plgpu_walk64.cuh"

namespace plgpu {

template <int ST>
void launch_pass(const PassDesc& g, cudaStream_t st);

// fp64 reference-precision walker (plgpu_walk64.cuh), defined inline there.

template <int ST, typename T>
void launch_band(const BandDesc& g, cudaStream_t st);

// Production pass kernel (plgpu_walk2.cuh): LINES = 2 (packed f32x2) for
// radii <= 16, 1 above (register budget); rows selects the transposing stage.
template <int ST>
void launch_pass2(const Pass2Desc& g, bool rows, cudaStream_t st);
constexpr int pass2_lines(int ST) { return ST <= 16 ? 2 : 1; }

// Hot-configuration kernel (plgpu_walk3.cuh) for the (K, S) pairs of the
// configs; returns false if (g.K, ST) has no instantiation.
// io: 0 column staging + column flush, 1 row + row, 2 row staging + column
// flush (plgpu_walk3.cuh).
template <int ST>
bool launch_pass3(const Pass3Desc& d, int io, cudaStream_t st);
// Folded 1D pass (plgpu_walk3.cuh, Pass3FoldDesc); lines = lines per lane.
template <int ST>
bool launch_pass3_fold(const Pass3FoldDesc& d, int lines, cudaStream_t st);
constexpr int pass3_k_for(int ST) { return ST == 10 ? 3 : ST == 15 ? 5 : ST == 25 ? 7 : -1; }
// warps per CTA the configs run with (PLGPU_WPC can override for io 0/1)
constexpr int pass3_default_wpc(int ST) { return ST >= 15 ? kLockWpc : 2; }

#ifdef PLGPU_DEFINE_LAUNCHERS
template <int ST>
void launch_pass(const PassDesc& g, cudaStream_t st) {
  const int64_t work = g.n_lines * g.nseg;
  const int threads = 128;
  const int64_t blocks = (work + threads - 1) / threads;
  nlm_pass_kernel<ST><<<(unsigned)blocks, threads, 0, st>>>(g);
}

template <int ST, typename T>
void launch_band(const BandDesc& g, cudaStream_t st) {
  const int64_t work = g.n_lines * g.nseg;
  distance_band_kernel<ST, T><<<(unsigned)((work + 127) / 128), 128, 0, st>>>(g);
}

template <int ST, int KT>
void launch_pass2_k(const Pass2Desc& g, bool rows, cudaStream_t st) {
  constexpr int L = pass2_lines(ST);
  const unsigned blocks = (unsigned)((g.total_warps + kWarpsPerCta - 1) / kWarpsPerCta);
  if (rows) {
    const size_t smem = sizeof(float) * kWarpsPerCta * pass2_smem_floats_per_warp<L, true>();
    nlm_pass2_kernel<ST, KT, L, true><<<blocks, 32 * kWarpsPerCta, smem, st>>>(g);
  } else {
    const size_t smem = sizeof(float) * kWarpsPerCta * pass2_smem_floats_per_warp<L, false>();
    nlm_pass2_kernel<ST, KT, L, false><<<blocks, 32 * kWarpsPerCta, smem, st>>>(g);
  }
}

template <int ST>
void launch_pass2(const Pass2Desc& g, bool rows, cudaStream_t st) {
  launch_pass2_k<ST, -1>(g, rows, st);  // runtime K (K <= 7)
}

template <int ST, int KT, int L, int IO, int WPC, bool AVG, bool EXP = false>
void launch3(const Pass3Desc& d, cudaStream_t st) {
  const size_t smem = sizeof(float) * WPC * pass3_smem_floats_per_warp<ST, L, IO>();
  unsigned grid;
  if constexpr (WPC == kLockWpc) {  // WPC line groups of one segment per CTA
    const int64_t groups = d.b.total_warps / d.b.nseg;
    const int64_t images = groups / d.b.groups_per_img;
    grid = (unsigned)(images * ((d.b.groups_per_img + WPC - 1) / WPC) * d.b.nseg);
  } else {
    grid = (unsigned)((d.b.total_warps + WPC - 1) / WPC);
  }
  auto k = nlm_pass3_kernel<ST, KT, L, IO, WPC, AVG, EXP>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, 32 * WPC, smem, st>>>(d);
}

template <int ST>
bool launch_pass3(const Pass3Desc& d, int io, cudaStream_t st) {
  constexpr int KT = pass3_k_for(ST);
  if constexpr (KT < 0) {
    return false;
  } else {
    if (d.b.K != KT || d.b.S != ST) return false;
    if (d.b.dexp && io != 1) return false;
    constexpr int DW = pass3_default_wpc(ST);
    // (register-capped variants, minb 6/8, measured slower on B200: profiles/README.md)
    auto go = [&](auto lines_tag) {
      constexpr int L = decltype(lines_tag)::value;
      if (d.b.dexp) {  // debug distance export (row pass only, checked below)
        launch3<ST, KT, L, 1, DW, false, true>(d, st);
        return;
      }
      if (io == 1) {
        if (d.wpc == kLockWpc) launch3<ST, KT, L, 1, kLockWpc, false>(d, st);
        else launch3<ST, KT, L, 1, 2, false>(d, st);
      } else if (io == 0 && !d.b.avg) {
        if (d.wpc == kLockWpc) launch3<ST, KT, L, 0, kLockWpc, false>(d, st);
        else launch3<ST, KT, L, 0, 2, false>(d, st);
      } else if (io == 0) {
        launch3<ST, KT, L, 0, DW, true>(d, st);
      } else if (d.b.avg) {
        launch3<ST, KT, L, 2, DW, true>(d, st);
      } else {
        launch3<ST, KT, L, 2, DW, false>(d, st);
      }
    };
    if constexpr (ST <= 16) {
      if (d.lines == 2) go(std::integral_constant<int, 2>{});
      else go(std::integral_constant<int, 1>{});
    } else {
      go(std::integral_constant<int, 1>{});
    }
    return true;
  }
}

template <int ST>
bool launch_pass3_fold(const Pass3FoldDesc& d, int lines, cudaStream_t st) {
  constexpr int KT = pass3_k_for(ST);
  if constexpr (KT < 0) {
    return false;
  } else {
    if (d.edge.K != KT || d.edge.S != ST) return false;
    auto go = [&](auto lines_tag) {
      constexpr int L = decltype(lines_tag)::value;
      const size_t smem = sizeof(float) * kWarpsPerCta * pass3_smem_floats_per_warp<ST, L, 1>();
      const unsigned grid =
          (unsigned)(d.fold_ctas + (d.edge_warps + kWarpsPerCta - 1) / kWarpsPerCta);
      auto k = nlm_pass3_fold_kernel<ST, KT, L>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<grid, 32 * kWarpsPerCta, smem, st>>>(d);
    };
    if constexpr (ST <= 16) {
      if (lines == 2) go(std::integral_constant<int, 2>{});
      else go(std::integral_constant<int, 1>{});
    } else {
      go(std::integral_constant<int, 1>{});
    }
    return true;
  }
}

#define PLGPU_INSTANTIATE(ST)                                              \
  template bool launch_pass3<ST>(const Pass3Desc&, int, cudaStream_t);     \
  template bool launch_pass3_fold<ST>(const Pass3FoldDesc&, int, cudaStream_t); \
  template void launch_pass<ST>(const PassDesc&, cudaStream_t);            \
  template void launch_pass2<ST>(const Pass2Desc&, bool, cudaStream_t);    \
  template void launch_pass64<ST>(const Pass64Desc&, cudaStream_t);        \
  template void launch_band<ST, float>(const BandDesc&, cudaStream_t);     \
  template void launch_band<ST, int32_t>(const BandDesc&, cudaStream_t);
#endif

// Instantiated template radii (keep in sync with build.py WALK_RADII).
#define PLGPU_FOR_EACH_RADIUS(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(15) X(16) X(20) X(25) X(32)

}  // namespace plgpu

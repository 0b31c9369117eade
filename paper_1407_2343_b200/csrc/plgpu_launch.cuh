// plgpu_launch.cuh -- launchers of the S-specialised kernels.  Each radius is
// explicitly instantiated in its own generated translation unit
// (build/gen/inst_S<ST>.cu, see paper_1407_2343_b200/build.py) so the large
// unrolled walkers compile in parallel; plgpu.cu only sees the declarations.
#pragma once

#include <cuda_runtime.h>

#include "plgpu_walk.cuh"

namespace plgpu {

template <int ST>
void launch_pass(const PassDesc& g, cudaStream_t st);

template <int ST, typename T>
void launch_band(const BandDesc& g, cudaStream_t st);

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

#define PLGPU_INSTANTIATE(ST)                                              \
  template void launch_pass<ST>(const PassDesc&, cudaStream_t);            \
  template void launch_band<ST, float>(const BandDesc&, cudaStream_t);     \
  template void launch_band<ST, int32_t>(const BandDesc&, cudaStream_t);
#endif

// Instantiated template radii (keep in sync with build.py WALK_RADII).
#define PLGPU_FOR_EACH_RADIUS(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(15) X(16) X(20) X(25) X(32)

}  // namespace plgpu

// ubench.cu -- pipe-throughput microbenchmarks for the roofline denominators
// MEASURED_PEAKS.json does not carry: MUFU.EX2 (the exp pipe the filter is
// bound by) and FP32 FFMA / packed FFMA2 issue.  Built as lib/libplubench.so,
// used by bench.py; not part of the product C ABI.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 8;

__global__ void ex2_kernel(float* out, int iters, float c) {
  float x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = -0.001f * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
      x[k] = -y;  // folded into the next MUFU operand modifier
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == c) out[threadIdx.x] = s;
}

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long x[kChains];
  unsigned long long av, bv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a), "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b), "f"(b));
#pragma unroll
  for (int k = 0; k < kChains; ++k) {
    float lo = threadIdx.x + k, hi = threadIdx.x - k;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[k]) : "f"(lo), "f"(hi));
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kChains; ++k) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[k]));
    s += lo + hi;
  }
  if (s == 1.2345f) out[threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Returns lane-operations per second (ex2: exps/s; ffma: FMAs/s; ffma2: FMAs/s
// counting 2 per packed instruction) and the measured milliseconds; -1 on error.
double plub_rate(int which, int blocks_per_sm, int threads, int iters, double* ms_out) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return -1;
  const int blocks = sms * blocks_per_sm;
  auto launch = [&]() {
    if (which == 0) ex2_kernel<<<blocks, threads>>>(out, iters, 3.0f);
    else if (which == 1) ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    else ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
  };
  launch();  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1;
  const double per_lane = (which == 2 ? 2.0 : 1.0) * kChains * (double)iters;
  const double ops = per_lane * (double)blocks * threads * reps;
  if (ms_out) *ms_out = ms / reps;
  return ops / (ms * 1e-3);
}

int plub_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
}

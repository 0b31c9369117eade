// ubench.cu -- pipe-throughput microbenchmarks for the roofline denominators
// MEASURED_PEAKS.json does not carry: MUFU.EX2 (the exp pipe the filter is
// bound by) and FP32 FFMA / packed FFMA2 issue.  Built as lib/libplubench.so,
// used by bench.py; not part of the product C ABI.
#include <cuda_runtime.h>

#include <cstdint>

#include "plgpu_walk2.cuh"

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

// The walker's per-pair update on register-resident data (no rings, no
// memory): LINES=2 packed form.  NK independent offsets per step; every
// accumulation pattern of the real kernel is kept (two num/den chains).
template <int NK, bool PRESCALE = false>
__global__ void pair2_kernel(float* out, int iters, float c) {
  using O = plgpu::VecOps<2>;
  using V = O::V;
  V p[NK + 1], q[NK + 1], f[NK + 1], d[NK + 1], an[NK + 1], ad[NK + 1];
#pragma unroll
  for (int k = 0; k <= NK; ++k) {
    p[k] = O::splat(threadIdx.x * 0.001f + k);
    q[k] = O::splat(threadIdx.x * 0.002f + k);
    f[k] = O::splat(k * 1.5f);
    d[k] = O::splat(0.f);
    an[k] = O::splat(0.f);
    ad[k] = O::splat(0.f);
  }
  const V cv = O::splat(c), one = O::splat(1.f);
  V num = O::splat(0.f), den = O::splat(0.f);
  V a = p[0], b = q[0];
  const V drift = O::splat(1e-7f);
  for (int it = 0; it < iters; ++it) {
    a = O::add(a, drift);
    b = O::add(b, drift);
    const V fi = f[0];
    num = O::add(num, fi);
    den = O::add(den, one);
#pragma unroll
    for (int k = 1; k <= NK; ++k) {
      const V dn = O::sub(a, p[k]);
      V dk = O::fma(dn, dn, d[k]);
      const V dq = O::sub(b, q[k]);
      dk = O::fms(dq, dq, dk);
      d[k] = dk;
      const V w = PRESCALE ? O::ex2(dk) : O::ex2(O::mul(dk, cv));
      num = O::fma(w, f[k], num);
      den = O::add(w, den);
      an[k] = O::fma(w, fi, an[k]);
      ad[k] = O::add(w, ad[k]);
    }
  }
  float s = O::lo(num) + O::hi(den);
#pragma unroll
  for (int k = 1; k <= NK; ++k) s += O::lo(an[k]) + O::hi(ad[k]) + O::lo(d[k]);
  if (s == c) out[threadIdx.x] = s;
}

// LINES=1 form with {num, den} packed in one f32x2 accumulator:
// {num, den} += w * {f, 1} is ONE FFMA2 (w broadcast).
template <int NK>
__global__ void pair1_kernel(float* out, int iters, float c) {
  using O2 = plgpu::VecOps<2>;
  using V2 = O2::V;
  float p[NK + 1], q[NK + 1], d[NK + 1];
  V2 f1[NK + 1], acc[NK + 1];
#pragma unroll
  for (int k = 0; k <= NK; ++k) {
    p[k] = threadIdx.x * 0.001f + k;
    q[k] = threadIdx.x * 0.002f + k;
    f1[k] = plgpu::f2_make(k * 1.5f, 1.f);
    d[k] = 0.f;
    acc[k] = O2::splat(0.f);
  }
  V2 nd = O2::splat(0.f);
  float a = p[0], b = q[0];
  for (int it = 0; it < iters; ++it) {
    a += 1e-7f;
    b += 1e-7f;
    const V2 fi = f1[0];
    nd = O2::add(nd, fi);
#pragma unroll
    for (int k = 1; k <= NK; ++k) {
      const float dn = a - p[k];
      float dk = fmaf(dn, dn, d[k]);
      const float dq = b - q[k];
      dk = fmaf(-dq, dq, dk);
      d[k] = dk;
      const float w = plgpu::ex2_approx(dk * c);
      const V2 wv = O2::splat(w);
      nd = O2::fma(wv, f1[k], nd);
      acc[k] = O2::fma(wv, fi, acc[k]);
    }
  }
  float s = O2::lo(nd) + O2::hi(nd);
#pragma unroll
  for (int k = 1; k <= NK; ++k) s += O2::lo(acc[k]) + O2::hi(acc[k]) + d[k];
  if (s == c) out[threadIdx.x] = s;
}

// Packed-op throughput with full register-pair operands (no broadcast):
// op 0: FFMA2 a*b+c (3 pairs), 1: FADD2 a+b (2 pairs), 2: FMUL2 a*b,
// 3: FFMA2 + FADD2 alternating, 4: scalar FFMA 3 regs, 5: scalar FADD.
template <int OP>
__global__ void pk_kernel(float* out, int iters) {
  using O = plgpu::VecOps<2>;
  using V = O::V;
  constexpr int NC = 8;
  V x[NC], y[NC];
  float xs[NC], ys[NC];
  int xi[NC], yi[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    x[k] = plgpu::f2_make(threadIdx.x * 1e-3f + k, k * 0.5f);
    y[k] = plgpu::f2_make(0.999f - k * 1e-4f, 1.0001f + k * 1e-5f);
    xs[k] = threadIdx.x * 1e-3f + k;
    ys[k] = 0.999f - k * 1e-4f;
    xi[k] = threadIdx.x * 7 + k;
    yi[k] = 3 + (int)threadIdx.x * k;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int j = (k + 3) % NC;
      if (OP == 0) x[k] = O::fma(x[k], y[k], x[j]);
      if (OP == 1) x[k] = O::add(x[k], y[j]);
      if (OP == 2) x[k] = O::mul(x[k], y[j]);
      if (OP == 3) { x[k] = (k & 1) ? O::add(x[k], y[j]) : O::fma(x[k], y[k], x[j]); }
      if (OP == 4) xs[k] = fmaf(xs[k], ys[k], xs[j]);
      if (OP == 5) xs[k] = xs[k] + ys[j];
      if (OP == 6) xi[k] = xi[k] * yi[k] + xi[j];
      if (OP == 7) xi[k] = xi[k] + yi[j] - xi[(k + 5) % NC];
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NC; ++k) s += (float)xi[k];
#pragma unroll
  for (int k = 0; k < NC; ++k) s += O::lo(x[k]) + O::hi(x[k]) + xs[k];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

// Mixed-pipe issue test: per iteration NF2 independent FFMA2, NF1 scalar
// FFMA, NMU MUFU.EX2 (8 rotating chains) and NAL integer ALU ops.  Comparing
// the mixes tells whether FFMA2 and MUFU share the dispatch port (times add)
// or overlap (time = max).
template <int NF2, int NF1, int NMU, int NAL>
__global__ void mix_kernel(float* out, int iters) {
  using O = plgpu::VecOps<2>;
  using V = O::V;
  V x[8], y[8];
  float xs[16], m[8];
  int xi[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    x[k] = plgpu::f2_make(threadIdx.x * 1e-3f + k, k * 0.5f);
    y[k] = plgpu::f2_make(0.999f - k * 1e-4f, 1.0001f + k * 1e-5f);
    m[k] = -0.5f - k * 0.01f;
    xi[k] = threadIdx.x * 7 + k;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) xs[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < (NF2 > 8 ? 8 : NF2); ++k) x[k] = O::fma(x[k], y[k], x[(k + 3) % 8]);
#pragma unroll
    for (int k = 8; k < NF2; ++k) x[k - 8] = O::fma(x[k - 8], y[k - 8], x[(k + 1) % 8]);
#pragma unroll
    for (int k = 0; k < NF1; ++k) xs[k % 16] = fmaf(xs[k % 16], 0.999f, xs[(k + 5) % 16]);
#pragma unroll
    for (int k = 0; k < NMU; ++k) {
      const int j = (it * NMU + k) & 7;
      m[j] = -plgpu::ex2_approx(m[j]);
    }
#pragma unroll
    for (int k = 0; k < NAL; ++k) xi[k & 7] = xi[k & 7] + xi[(k + 3) & 7];
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += O::lo(x[k]) + O::hi(x[k]) + m[k] + (float)xi[k];
#pragma unroll
  for (int k = 0; k < 16; ++k) s += xs[k];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Cycles per loop iteration per SM sub-partition (at the given clock in MHz)
// for mix_kernel preset `which`; -1 on error.
double plub_mix_cycles(int which, int blocks_per_sm, int threads, int iters, double mhz) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return -1;
  const int blocks = sms * blocks_per_sm;
  auto launch = [&]() {
    switch (which) {
      case 0: mix_kernel<8, 0, 0, 0><<<blocks, threads>>>(out, iters); break;
      case 1: mix_kernel<0, 0, 2, 0><<<blocks, threads>>>(out, iters); break;
      case 2: mix_kernel<8, 0, 2, 0><<<blocks, threads>>>(out, iters); break;
      case 3: mix_kernel<0, 16, 0, 0><<<blocks, threads>>>(out, iters); break;
      case 4: mix_kernel<0, 16, 2, 0><<<blocks, threads>>>(out, iters); break;
      case 5: mix_kernel<8, 0, 0, 8><<<blocks, threads>>>(out, iters); break;
      case 6: mix_kernel<0, 0, 0, 8><<<blocks, threads>>>(out, iters); break;
      case 7: mix_kernel<12, 0, 2, 0><<<blocks, threads>>>(out, iters); break;
      default: mix_kernel<6, 0, 2, 0><<<blocks, threads>>>(out, iters); break;
    }
  };
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1;
  // warps per SMSP = blocks_per_sm * threads / 32 / 4; each runs iters iterations
  const double warp_iters_per_smsp = 3.0 * iters * blocks_per_sm * (threads / 32) / 4.0;
  return (ms * 1e-3) * mhz * 1e6 / warp_iters_per_smsp;
}


// Warp-instructions per second per SM for pk_kernel<op>.
double plub_pk_rate(int op, int blocks_per_sm, int threads, int iters) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return -1;
  const int blocks = sms * blocks_per_sm;
  auto launch = [&]() {
    switch (op) {
      case 0: pk_kernel<0><<<blocks, threads>>>(out, iters); break;
      case 1: pk_kernel<1><<<blocks, threads>>>(out, iters); break;
      case 2: pk_kernel<2><<<blocks, threads>>>(out, iters); break;
      case 3: pk_kernel<3><<<blocks, threads>>>(out, iters); break;
      case 4: pk_kernel<4><<<blocks, threads>>>(out, iters); break;
      case 5: pk_kernel<5><<<blocks, threads>>>(out, iters); break;
      case 6: pk_kernel<6><<<blocks, threads>>>(out, iters); break;
      default: pk_kernel<7><<<blocks, threads>>>(out, iters); break;
    }
  };
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1;
  const double warp_instr = 8.0 * iters * (double)blocks * (threads / 32) * 3;
  return warp_instr / (ms * 1e-3) / sms;
}

// Pair-update throughput: unique pairs per second (each lane-line-offset is
// one pair).  form 0: LINES=2 packed; form 1: LINES=1 with {num,den} packed.
double plub_pair_rate(int form, int blocks_per_sm, int threads, int iters, double* ms_out) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return -1;
  const int blocks = sms * blocks_per_sm;
  constexpr int NK = 10;
  auto launch = [&]() {
    if (form == 0) pair2_kernel<NK><<<blocks, threads>>>(out, iters, -1e-4f);
    else if (form == 2) pair2_kernel<NK, true><<<blocks, threads>>>(out, iters, -1e-4f);
    else pair1_kernel<NK><<<blocks, threads>>>(out, iters, -1e-4f);
  };
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1;
  const double pairs = (form != 1 ? 2.0 : 1.0) * NK * (double)iters * blocks * threads * 3;
  if (ms_out) *ms_out = ms / 3;
  return pairs / (ms * 1e-3);
}

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

// FMA-pipe throughput probe.  MEASURED_PEAKS.json carries only bf16 and HBM,
// so the FP64 / FP32 roofline denominators of the covariance kernels are
// measured by bench.py on the same GPU, right before the timed region.
//
// The loop is the complex multiply-accumulate of the kernels (16 lags, all
// operands per-thread registers) with each x component repeated in one
// operand slot across consecutive FMAs, so the operand-reuse cache relieves
// the register file: measured on B200 this is the highest FMA rate reachable
// (FP64 ~33 TF/s, FP32 ~62 TF/s at 1965 MHz); three distinct 64-bit sources
// per DFMA reach only ~24.7 TF/s (register-bank bound, 42.5 DFMA/clk/SM).
#pragma once

#include "common.cuh"

namespace covgpu {

template <typename T>
__global__ void __launch_bounds__(256) k_fma_probe(T* out, int iters, T seed) {
  constexpr int E = 16;
  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    ar[e] = ai[e] = (T)0;
    yr[e] = seed + (T)(e + threadIdx.x) * (T)1e-7;
    yi[e] = seed - (T)(threadIdx.x & 7) * (T)1e-7;
  }
  T xr = seed * (T)0.5 + (T)threadIdx.x * (T)1e-8, xi = seed * (T)0.25 - (T)threadIdx.x * (T)1e-8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = fma(xr, yr[e], ar[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ai[e] = fma(xi, yr[e], ai[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = fma(xi, yi[e], ar[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ai[e] = fma(-xr, yi[e], ai[e]);
    xr = xr + (T)1e-9;
  }
  T s = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) s += ar[e] + ai[e];
  if (s == (T)-1.2345) out[0] = s;  // keep the chains live
}

// FP64 tensor-core (DMMA m8n8k4) throughput: 8 independent accumulator tiles
// per warp; the roofline denominator of the tensor-core bulk kernel
// (measured on B200: 37.2 TF/s at 1965 MHz = the nominal FP64 rate).
__global__ void __launch_bounds__(256) k_dmma_probe(double* out, int iters, double seed) {
  constexpr int CH = 8;
  const double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

}  // namespace covgpu

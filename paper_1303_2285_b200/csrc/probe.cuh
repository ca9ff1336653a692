// FMA-pipe throughput probe.  MEASURED_PEAKS.json carries only bf16 and HBM,
// so the FP64 / FP32 roofline denominators of the covariance kernels are
// measured by bench.py with this loop on the same GPU, right before the timed
// region: 16 independent FMA chains per thread, all operands in registers
// (the covariance kernels' operand form), a full-chip grid.
#pragma once

#include "common.cuh"

namespace covgpu {

template <typename T>
__global__ void __launch_bounds__(256) k_fma_probe(T* out, int iters, T seed) {
  constexpr int CH = 16;
  T acc[CH], x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    acc[c] = (T)(threadIdx.x + c) * (T)1e-3;
    x[c] = seed + (T)c * (T)1e-7 + (T)(threadIdx.x & 7) * (T)1e-9;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], x[c], x[(c + 5) % CH]);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == (T)-1.2345) out[0] = s;  // keep the chains live
}

}  // namespace covgpu

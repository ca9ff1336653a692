// Throughput probe for the FP64 / FP32 FMA pipes and shared-memory loads on the
// device the bench runs on.  MEASURED_PEAKS.json carries only bf16 and HBM, so
// the covariance roofline denominators (DFMA, FFMA) are measured here.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  // all three operands in registers, as in the covariance kernels
  T acc[CHAINS], x[CHAINS], y[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    acc[c] = (T)(threadIdx.x + c);
    x[c] = a + (T)(c * 1e-9) * (T)threadIdx.x;
    y[c] = b * (T)(c + 1 + (threadIdx.x & 3));
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(x[c], y[(c + 1) % CHAINS], acc[c]);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == (T)12345.678) out[0] = s;
}

template <typename T, int CHAINS>
double run(int blocks, int threads, int iters) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_loop<T, CHAINS><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_loop<T, CHAINS><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  double flops = 2.0 * CHAINS * (double)iters * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", prop.name, sms, clk);
  printf(", \"fp64_tflops\": %.3f", run<double, 8>(sms * 8, 256, 1 << 16));
  printf(", \"fp64_tflops_b4\": %.3f", run<double, 8>(sms * 4, 256, 1 << 16));
  printf(", \"fp32_tflops\": %.3f", run<float, 8>(sms * 8, 256, 1 << 17));
  printf(", \"fp32_tflops_b4\": %.3f", run<float, 8>(sms * 4, 256, 1 << 17));
  printf("}\n");
  return 0;
}

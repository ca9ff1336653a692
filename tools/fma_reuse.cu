// FMA throughput when one source operand repeats in the same slot across
// consecutive instructions (operand-reuse cache) vs three distinct sources.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void k_distinct(T* out, int iters, T seed) {
  T acc[CH], x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c] = (T)(threadIdx.x + c) * (T)1e-3; x[c] = seed + (T)c * (T)1e-7 + (T)(threadIdx.x & 7) * (T)1e-9; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(x[(c + 3) % CH], x[c], acc[c]);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == (T)-1.2345) out[0] = s;
}

// complex MAC pattern of the covariance kernels, grouped so x.x / x.y repeat
template <typename T, int E>
__global__ void k_cmac(T* out, int iters, T seed) {
  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) { ar[e] = ai[e] = (T)0; yr[e] = seed + (T)(e + threadIdx.x) * (T)1e-7; yi[e] = seed - (T)(threadIdx.x & 7) * (T)1e-7; }
  T xr = seed * (T)0.5 + (T)threadIdx.x * (T)1e-8, xi = seed * (T)0.25 - (T)threadIdx.x * (T)1e-8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = fma(xr, yr[e], ar[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = fma(xi, yi[e], ar[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ai[e] = fma(xi, yr[e], ai[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) ai[e] = fma(-xr, yi[e], ai[e]);
    xr = xr + (T)1e-9;   // keep x live / varying
  }
  T s = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) s += ar[e] + ai[e];
  if (s == (T)-1.2345) out[0] = s;
}


int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* od; float* of; cudaMalloc(&od, 16); cudaMalloc(&of, 16);
  float ms;
#define TIME(launch, fmas, label) \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
  cudaEventElapsedTime(&ms, e0, e1); printf("%-28s %.2f TFLOP/s\n", label, 2.0 * (fmas) / (ms * 1e-3) / 1e12);
  const int it = 1 << 15;
  TIME((k_distinct<double, 16><<<sms * 2, 256>>>(od, it, 0.999999)), 16.0 * it * sms * 2 * 256, "fp64 distinct 3-src");
  TIME((k_cmac<double, 16><<<sms * 1, 256>>>(od, it, 0.999999)), 64.0 * it * sms * 1 * 256, "fp64 cmac E=16 1blk");
  TIME((k_cmac<double, 16><<<sms * 2, 128>>>(od, it, 0.999999)), 64.0 * it * sms * 2 * 128, "fp64 cmac E=16 2x128");
  TIME((k_cmac<double, 8><<<sms * 2, 256>>>(od, it, 0.999999)), 32.0 * it * sms * 2 * 256, "fp64 cmac E=8");
  TIME((k_distinct<float, 16><<<sms * 2, 256>>>(of, it * 2, 0.999999f)), 16.0 * it * 2 * sms * 2 * 256, "fp32 distinct 3-src");
  TIME((k_cmac<float, 16><<<sms * 2, 256>>>(of, it * 2, 0.999999f)), 64.0 * it * 2 * sms * 2 * 256, "fp32 cmac E=16");
  TIME((k_cmac<float, 16><<<sms * 3, 256>>>(of, it * 2, 0.999999f)), 64.0 * it * 2 * sms * 3 * 256, "fp32 cmac E=16 3blk");
  return 0;
}

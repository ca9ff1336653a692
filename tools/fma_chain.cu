// Complex MAC orderings vs FMA-pipe rate (operand-reuse chains).
#include <cstdio>
#include <cuda_runtime.h>

// chain order with split accumulators: every FMA shares one operand (same
// slot) with its predecessor, and no accumulator is touched twice per step
template <typename T, int E>
__global__ void k_chain(T* out, int iters, T seed) {
  T a1[E], b1[E], a2[E], b2[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) { a1[e] = b1[e] = a2[e] = b2[e] = (T)0; yr[e] = seed + (T)(e + threadIdx.x) * (T)1e-7; yi[e] = seed - (T)(threadIdx.x & 7) * (T)1e-7 + (T)e * (T)1e-8; }
  T xr = seed * (T)0.5 + (T)threadIdx.x * (T)1e-8, xi = seed * (T)0.25 - (T)threadIdx.x * (T)1e-8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a1[e] = fma(xr, yr[e], a1[e]);
      b1[e] = fma(xi, yr[e], b1[e]);
      a2[e] = fma(xi, yi[e], a2[e]);
      b2[e] = fma(-xr, yi[e], b2[e]);
    }
    xr = xr + (T)1e-9;
    xi = xi - (T)1e-9;
  }
  T s = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) s += a1[e] + b1[e] + a2[e] + b2[e];
  if (s == (T)-1.2345) out[0] = s;
}

// same but single accumulators (dependency distance 2)
template <typename T, int E>
__global__ void k_chain1(T* out, int iters, T seed) {
  T a[E], b[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) { a[e] = b[e] = (T)0; yr[e] = seed + (T)(e + threadIdx.x) * (T)1e-7; yi[e] = seed - (T)(threadIdx.x & 7) * (T)1e-7 + (T)e * (T)1e-8; }
  T xr = seed * (T)0.5 + (T)threadIdx.x * (T)1e-8, xi = seed * (T)0.25 - (T)threadIdx.x * (T)1e-8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a[e] = fma(xr, yr[e], a[e]);
      b[e] = fma(xi, yr[e], b[e]);
      a[e] = fma(xi, yi[e], a[e]);
      b[e] = fma(-xr, yi[e], b[e]);
    }
    xr = xr + (T)1e-9;
    xi = xi - (T)1e-9;
  }
  T s = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) s += a[e] + b[e];
  if (s == (T)-1.2345) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* od; float* of; cudaMalloc(&od, 16); cudaMalloc(&of, 16);
  float ms;
#define TIME(launch, fmas, label) \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
  cudaEventElapsedTime(&ms, e0, e1); printf("%-34s %.2f TFLOP/s\n", label, 2.0 * (fmas) / (ms * 1e-3) / 1e12);
  const int it = 1 << 15;
  TIME((k_chain<double, 8><<<sms * 2, 256>>>(od, it, 0.999999)), 32.0 * it * sms * 2 * 256, "fp64 chain split E=8 2x256");
  TIME((k_chain<double, 8><<<sms * 4, 128>>>(od, it, 0.999999)), 32.0 * it * sms * 4 * 128, "fp64 chain split E=8 4x128");
  TIME((k_chain<double, 8><<<sms * 1, 256>>>(od, it, 0.999999)), 32.0 * it * sms * 1 * 256, "fp64 chain split E=8 1x256");
  TIME((k_chain1<double, 16><<<sms * 1, 256>>>(od, it, 0.999999)), 64.0 * it * sms * 1 * 256, "fp64 chain1 E=16 1x256");
  TIME((k_chain1<double, 8><<<sms * 2, 256>>>(od, it, 0.999999)), 32.0 * it * sms * 2 * 256, "fp64 chain1 E=8 2x256");
  TIME((k_chain<float, 8><<<sms * 2, 256>>>(of, it * 2, 0.999999f)), 32.0 * it * 2 * sms * 2 * 256, "fp32 chain split E=8 2x256");
  TIME((k_chain<float, 16><<<sms * 2, 256>>>(of, it * 2, 0.999999f)), 64.0 * it * 2 * sms * 2 * 256, "fp32 chain split E=16 2x256");
  TIME((k_chain1<float, 16><<<sms * 2, 256>>>(of, it * 2, 0.999999f)), 64.0 * it * 2 * sms * 2 * 256, "fp32 chain1 E=16 2x256");
  return 0;
}

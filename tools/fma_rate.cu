// Per-SM FMA issue rate: cycles measured with clock64 inside the kernel,
// SM clock from clock64 vs globaltimer.  Prints FMA/clk/SM for FP64 and FP32
// at several chain counts and occupancies.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void k(T* out, int iters, T seed, unsigned long long* cyc, unsigned long long* ns) {
  T acc[CH], x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c] = (T)(threadIdx.x + c) * (T)1e-3; x[c] = seed + (T)c * (T)1e-7 + (T)(threadIdx.x & 7) * (T)1e-9; }
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], x[c], x[(c + 5) % CH]);
  }
  unsigned long long c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == (T)-1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { *cyc = c1 - c0; *ns = t1 - t0; }
}

template <typename T, int CH>
void run(const char* name, int sms, int bps, int threads, int iters) {
  T* out; unsigned long long *cyc, *ns;
  cudaMalloc(&out, 16); cudaMallocManaged(&cyc, 8); cudaMallocManaged(&ns, 8);
  k<T, CH><<<sms * bps, threads>>>(out, iters, (T)0.999999, cyc, ns);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<T, CH><<<sms * bps, threads>>>(out, iters, (T)0.999999, cyc, ns);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)CH * iters * sms * bps * threads;
  double mhz = (double)*cyc / (double)*ns * 1e3;
  // per SM per clock, using the in-kernel cycle count of block 0 (all blocks co-resident)
  double per_clk = (double)CH * iters * bps * threads / (double)*cyc;
  printf("%s CH=%d blocks/SM=%d thr=%d: %.2f TFLOP/s, clk %.0f MHz, %.1f FMA/clk/SM (block0 view)\n",
         name, CH, bps, threads, 2 * fmas / (ms * 1e-3) / 1e12, mhz, per_clk);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<double, 8>("fp64", sms, 1, 256, 1 << 16);
  run<double, 16>("fp64", sms, 1, 256, 1 << 16);
  run<double, 16>("fp64", sms, 2, 256, 1 << 16);
  run<double, 16>("fp64", sms, 4, 256, 1 << 15);
  run<double, 32>("fp64", sms, 1, 512, 1 << 15);
  run<double, 8>("fp64", sms, 2, 1024, 1 << 15);
  run<float, 16>("fp32", sms, 1, 256, 1 << 17);
  run<float, 16>("fp32", sms, 2, 512, 1 << 16);
  run<float, 32>("fp32", sms, 2, 256, 1 << 16);
  run<double, 16>("fp64-long", sms, 2, 256, 1 << 20);
  return 0;
}

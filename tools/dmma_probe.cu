// FP64 tensor-core (DMMA, mma.sync f64) throughput on this GPU, for the
// shapes PTX offers: m8n8k4 (sm_80+) and m16n8k4 / m16n8k8 / m16n8k16 (sm_90+).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_m8n8k4(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

template <int CH, int K>
__global__ void k_m16n8(double* out, int iters, double seed) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = seed + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = seed - (threadIdx.x + i) * 1e-9;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if constexpr (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if constexpr (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* od; cudaMalloc(&od, 16);
  float ms;
#define TIME(launch, fmas, label) \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
  cudaEventElapsedTime(&ms, e0, e1); printf("%-32s %.2f TFLOP/s  (%s)\n", label, 2.0 * (fmas) / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  const int it = 1 << 14;
  for (int tpb : {128, 256, 512}) {
    char l[64];
    snprintf(l, 64, "m8n8k4 CH=8 tpb=%d", tpb);
    TIME((k_m8n8k4<8><<<sms * 2, tpb>>>(od, it, 0.999999)), 256.0 * 8 * it * sms * 2 * (tpb / 32), l);
    snprintf(l, 64, "m16n8k4 CH=4 tpb=%d", tpb);
    TIME((k_m16n8<4, 4><<<sms * 2, tpb>>>(od, it, 0.999999)), 512.0 * 4 * it * sms * 2 * (tpb / 32), l);
    snprintf(l, 64, "m16n8k8 CH=4 tpb=%d", tpb);
    TIME((k_m16n8<4, 8><<<sms * 2, tpb>>>(od, it, 0.999999)), 1024.0 * 4 * it * sms * 2 * (tpb / 32), l);
    snprintf(l, 64, "m16n8k16 CH=4 tpb=%d", tpb);
    TIME((k_m16n8<4, 16><<<sms * 2, tpb>>>(od, it / 2, 0.999999)), 2048.0 * 4 * (it / 2) * sms * 2 * (tpb / 32), l);
  }
  return 0;
}

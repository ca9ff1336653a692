// Warp-level (mma.sync) low-precision tensor-core throughput on this GPU:
// tf32 m16n8k8, bf16 m16n8k16, s8 m16n8k32 (f32 / s32 accumulate).  These
// are the legacy (pre-tcgen05) instructions: register fragments, so an
// operand can be any gather from SMEM (the Toeplitz operands of the bulk
// sums).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/mma_lowp_probe tools/mma_lowp_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_tf32(float* out, int iters, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = seed + threadIdx.x, b1 = b0 * 11u;
  float c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

template <int CH>
__global__ void k_bf16(float* out, int iters, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = seed + threadIdx.x, b1 = b0 * 11u;
  float c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

template <int CH>
__global__ void k_s8(int* out, int iters, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = seed + threadIdx.x, b1 = b0 * 11u;
  int c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -12345) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* of; cudaMalloc(&of, 16);
  int* oi; cudaMalloc(&oi, 16);
  float ms;
#define TIME(launch, macs, label) \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
  cudaEventElapsedTime(&ms, e0, e1); printf("%-28s %8.1f TFLOP/s  (%s)\n", label, 2.0 * (macs) / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  const int it = 1 << 13;
  for (int tpb : {128, 256, 512}) {
    char l[64];
    double warps = double(sms) * 2 * (tpb / 32);
    snprintf(l, 64, "tf32 m16n8k8 CH=8 tpb=%d", tpb);
    TIME((k_tf32<8><<<sms * 2, tpb>>>(of, it, 12345u)), 1024.0 * 8 * it * warps, l);
    snprintf(l, 64, "bf16 m16n8k16 CH=8 tpb=%d", tpb);
    TIME((k_bf16<8><<<sms * 2, tpb>>>(of, it, 12345u)), 2048.0 * 8 * it * warps, l);
    snprintf(l, 64, "s8 m16n8k32 CH=8 tpb=%d", tpb);
    TIME((k_s8<8><<<sms * 2, tpb>>>(oi, it, 12345u)), 4096.0 * 8 * it * warps, l);
  }
  return 0;
}

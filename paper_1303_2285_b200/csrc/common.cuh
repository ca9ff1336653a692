// Shared device-side types and helpers for the covgpu kernels.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "../../include/covgpu.h"

namespace covgpu {

template <typename T>
struct CT;
template <>
struct CT<double> {
  using c = double2;
};
template <>
struct CT<float> {
  using c = float2;
};

// One offset class (dr, dc) of UC (combinations.py:53-62) and where its
// intermediate sums live.
struct ClassDesc {
  int dr, dc;
  int pv, qu;  // slot grid: v in [0, pv) along the diagonal, u in [0, qu)
  int s1, s2;  // row shift of the first / second element: max(-dr,0), max(dr,0)
  int d;       // output diagonal dc*P + dr
  int uc;      // index in UC order
  long long rc_off;    // 2*(pv-1) edge-row sums (top rows, then bottom rows)
  long long ccol_off;  // 2*(qu-1) edge-column sums (left cols, then right cols)
  long long slot_off;  // offset of the class's pv*qu slots (compact layout / scratch)
};

struct Problem {
  int N, M, P, Q;
  int bh, bw;  // window-placement extents N-P+1, M-Q+1 (the box of every slot sum)
  int PQ;
};

__host__ __device__ inline int class_index(int dr, int dc, int P, int Q) {
  // position in UC order (combinations.py:53-62)
  return dr >= 0 ? dr * Q + dc : P * Q + (dr + P - 1) * (Q - 1) + (dc - 1);
}

__host__ __device__ inline bool in_uc(int dr, int dc, int P, int Q) {
  return (dr >= 0 && dr < P && dc >= 0 && dc < Q) || (dr < 0 && dr > -P && dc >= 1 && dc < Q);
}

__host__ __device__ inline long long packed_off(long long k1, long long k2, long long dim) {
  // core.py:60-72, 0-based: row k1 of the upper triangle starts after
  // k1*dim - k1(k1-1)/2 entries
  return k1 * dim - (k1 * (k1 - 1)) / 2 + (k2 - k1);
}

__device__ inline double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ inline double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// a * conj(b) as 4 FMAs in T, widened to double
template <typename T>
__device__ inline double2 cmulconj(typename CT<T>::c a, typename CT<T>::c b) {
  T re = a.x * b.x;
  re = fma(a.y, b.y, re);
  T im = a.y * b.x;
  im = fma(-a.x, b.y, im);
  return make_double2((double)re, (double)im);
}

__device__ inline double2 shfl_xor2(double2 v, int off) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, off);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, off);
  return v;
}

// fixed-order butterfly sum: every lane gets the same bits
__device__ inline double2 warp_sum(double2 v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = cadd(v, shfl_xor2(v, off));
  return v;
}

// exclusive prefix sum over the warp (lane 0 gets 0); `total` = inclusive sum
__device__ inline double2 warp_excl_scan(double2 v, double2* total) {
  const int lane = threadIdx.x & 31;
  double2 inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    double2 n;
    n.x = __shfl_up_sync(0xffffffffu, inc.x, off);
    n.y = __shfl_up_sync(0xffffffffu, inc.y, off);
    if (lane >= off) inc = cadd(inc, n);
  }
  total->x = __shfl_sync(0xffffffffu, inc.x, 31);
  total->y = __shfl_sync(0xffffffffu, inc.y, 31);
  return csub(inc, v);
}

// Output element write for slot (v, u) of class c (single writer per element).
template <typename T>
__device__ inline void write_slot(typename CT<T>::c* R, int layout, long long base, const ClassDesc& c,
                                  const Problem& pr, int v, int u, double re, double im) {
  using C2 = typename CT<T>::c;
  C2 val;
  val.x = (T)re;
  val.y = (T)im;
  if (layout == COVGPU_COMPACT) {
    R[base + c.slot_off + (long long)u * c.pv + v] = val;
    return;
  }
  const long long k1 = (long long)pr.P * u + c.s1 + v;
  const long long k2 = k1 + c.d;
  if (layout == COVGPU_DENSE) {
    const long long D = pr.PQ;
    R[base + k1 * D + k2] = val;
    if (c.d != 0) {
      C2 cv;
      cv.x = val.x;
      cv.y = -val.y;  // lower triangle = exact conjugate of the upper
      R[base + k2 * D + k1] = cv;
    }
  } else {
    R[base + packed_off(k1, k2, pr.PQ)] = val;
  }
}

// cp.async of one complex element with zero fill when !valid
template <int BYTES>
__device__ inline void cp_async_elem(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int src = valid ? BYTES : 0;
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  }
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier / TMA (sm_90+; used on sm_100a) ------------------------------
__device__ inline unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ inline void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ inline void fence_mbarrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ inline void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ inline void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ inline bool mbar_try(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ inline void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// waiting loop for a warp that is usually early (the TMA producer): back off
// so its polling does not take issue slots from the compute warps
__device__ inline void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  unsigned ns = 32;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 2048 ? ns * 2 : 2048;
  }
}
// Wait until the band counter written by the host path's copy stream
// (cuStreamWriteValue32 after each band's H2D copy) reaches `need`
// (wrap-safe), then order the TMA (async proxy) reads after it.
__device__ inline void wait_band(const unsigned* flag, unsigned need) {
  unsigned ns = 64;
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - need) >= 0) break;
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : 1024;
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 3-D tensor tile -> SMEM, completion counted on `bar` (bytes)
__device__ inline void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace covgpu

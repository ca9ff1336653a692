// K2 — edge-row sums RC'.
//
// The edge rows of class (dr, dc) are the pane rows whose window-row range is
// clipped: top rows, where both elements sit in A's first P-1 rows, and
// bottom rows, where both sit in the last P-1 rows.  Over all classes they
// are exactly the ordered row pairs (r1, r2) inside the top strip [0, P-1)
// and inside the bottom strip [N-P+1, N).  Each thread owns one pair and D
// consecutive column lags dc0..dc0+D-1 and walks c1 in [0, M-Q] — the
// columns of the slot u = 0 box, i.e. the left corner plus the core columns —
// the D second-element columns in flight rotating in a register window
// (2 loads per D products).  RC'_i = fullT_i(0) (resp. fullB_i(0)) is the
// starting value of the finalize's walk along u.  The column walk may be
// split into nseg segments; the finalize sums the segment partials in order.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace covgpu {

template <typename T, int D>
__global__ void __launch_bounds__(128)
    k_edge_rows(const typename CT<T>::c* __restrict__ A, Problem pr, int S, int ndg, int nseg,
                const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
                double2* __restrict__ rc, long long tot_rc, long long total) {
  using C2 = typename CT<T>::c;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const int N = pr.N, M = pr.M, P = pr.P, Q = pr.Q;
  const long long SS = (long long)S * S;
  long long t = tid;
  const int p = (int)(t % SS);
  t /= SS;
  const int seg = (int)(t % nseg);
  t /= nseg;
  const int g = (int)(t % ndg);
  t /= ndg;
  const int strip = (int)(t % 2);
  const int b = (int)(t / 2);

  const int base = strip ? pr.bh : 0;
  const int r1 = base + p % S, r2 = base + p / S;
  const int dr = r2 - r1;
  const int dc0 = g * D;
  unsigned valid = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int dc = dc0 + d;
    if (in_uc(dr, dc, P, Q) && cls_slot[class_index(dr, dc, P, Q)] >= 0) valid |= 1u << d;
  }
  if (!valid) return;

  const int cstart = 0;
  const int cend = M - Q;  // inclusive: the slot-0 box columns [0, bw)
  const int seglen = (cend - cstart + nseg) / nseg;  // ceil(len / nseg)
  const int cs = cstart + seg * seglen;
  const int ce = min(cend, cs + seglen - 1);
  const C2* __restrict__ x = A + ((long long)b * N + r1) * M;
  const C2* __restrict__ y = A + ((long long)b * N + r2) * M;

  T ar[D], ai[D], yr[D], yi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    ar[d] = ai[d] = yr[d] = yi[d] = (T)0;
  }
  if (cs <= ce) {
#pragma unroll
    for (int d = 0; d < D - 1; ++d) {
      const int col = min(cs + dc0 + d, M - 1);
      const C2 v = y[col];
      yr[d] = v.x;
      yi[d] = v.y;
    }
    for (int c0 = cs; c0 <= ce; c0 += D) {
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        const int c = c0 + cc;
        if (c <= ce) {
          const C2 yn = y[min(c + dc0 + D - 1, M - 1)];
          const C2 xv = x[c];
          yr[(cc + D - 1) % D] = yn.x;
          yi[(cc + D - 1) % D] = yn.y;
#pragma unroll
          for (int d = 0; d < D; ++d) ar[d] = fma(xv.x, yr[(cc + d) % D], ar[d]);
#pragma unroll
          for (int d = 0; d < D; ++d) ai[d] = fma(xv.y, yr[(cc + d) % D], ai[d]);
#pragma unroll
          for (int d = 0; d < D; ++d) ar[d] = fma(xv.y, yi[(cc + d) % D], ar[d]);
#pragma unroll
          for (int d = 0; d < D; ++d) ai[d] = fma(-xv.x, yi[(cc + d) % D], ai[d]);
        }
      }
    }
  }
  const int i = min(r1, r2);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (!(valid & (1u << d))) continue;
    const ClassDesc& cd = cls[cls_slot[class_index(dr, dc0 + d, P, Q)]];
    const int a_r = cd.pv - 1;
    const int k = strip ? a_r + (i - pr.bh) : i;
    rc[((long long)b * tot_rc + cd.rc_off + k) * nseg + seg] =
        make_double2((double)ar[d], (double)ai[d]);
  }
}

}  // namespace covgpu

namespace covgpu {

// ---- TMA variant -------------------------------------------------------------
// CTA = (snapshot, strip, column-lag group, r2 group of R2G rows, column
// segment).  Thread (r1, r2) as above, r1 = lanes (consecutive strip rows),
// r2 from the CTA's group.  The strip's rows for a 32-column chunk are staged
// by TMA into SMEM (X: all S strip rows x 32 columns, row pitch XW odd so the
// 32 lanes' rows fall in distinct banks; Y: the R2G second-element rows x
// (32+D-1) columns starting at column lag dc0) through a S-stage ring fed by
// a producer warp.
constexpr int EDGE_CW = 32;      // columns per stage (multiple of D)
constexpr int EDGE_STAGES = 4;
constexpr int EDGE_WARPS = 8;    // compute warps

template <typename T, int D>
struct EdgeCfg {
  using C2 = typename CT<T>::c;
  static constexpr int XW = sizeof(T) == 8 ? EDGE_CW + 1 : EDGE_CW + 2;  // X pitch (elements)
  static constexpr int YW = EDGE_CW + D - 1 + (sizeof(T) == 8 ? 0 : ((EDGE_CW + D - 1) & 1));
  __host__ __device__ static size_t xbytes(int S) { return sizeof(C2) * (size_t)S * XW; }
  __host__ __device__ static size_t ybytes(int R2G) { return sizeof(C2) * (size_t)R2G * YW; }
  // TMA destinations must be 128-byte aligned: Y starts at xoff
  __host__ __device__ static size_t xoff(int S) { return (xbytes(S) + 127) / 128 * 128; }
  __host__ __device__ static size_t stage(int S, int R2G) { return (xoff(S) + ybytes(R2G) + 127) / 128 * 128; }
  // ring depth that fits the SMEM budget (0: TMA variant unusable for this S)
  __host__ __device__ static int stages(int S, int R2G) {
    const size_t st = stage(S, R2G);
    const int n = (int)((200 * 1024 - 8 * EDGE_STAGES) / st);
    return n < 2 ? 0 : (n > EDGE_STAGES ? EDGE_STAGES : n);
  }
  __host__ __device__ static size_t smem(int S, int R2G) {
    return stages(S, R2G) * stage(S, R2G) + 8 * EDGE_STAGES;
  }
};

template <typename T, int D>
__global__ void __launch_bounds__((EDGE_WARPS + 1) * 32, 1)
    k_edge_tma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
               Problem pr, int S, int R2G, int n_r2g, int ndg, int nseg,
               const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
               double2* __restrict__ rc, long long tot_rc) {
  using C2 = typename CT<T>::c;
  using Cfg = EdgeCfg<T, D>;
  constexpr int XW = Cfg::XW, YW = Cfg::YW, CW = EDGE_CW;
  extern __shared__ __align__(128) unsigned char esm[];
  const size_t xb = Cfg::xbytes(S), yb = Cfg::ybytes(R2G), sb = Cfg::stage(S, R2G);
  const size_t xo = Cfg::xoff(S);
  const int NS = Cfg::stages(S, R2G);
  uint64_t* full = reinterpret_cast<uint64_t*>(esm + Cfg::stages(S, R2G) * sb);
  long long t = blockIdx.x;
  const int seg = (int)(t % nseg);
  t /= nseg;
  const int r2g = (int)(t % n_r2g);
  t /= n_r2g;
  const int g = (int)(t % ndg);
  t /= ndg;
  const int strip = (int)(t % 2);
  const int b = (int)(t / 2);
  const int M = pr.M, P = pr.P, Q = pr.Q;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int base = strip ? pr.bh : 0;
  const int dc0 = g * D;
  const int cend = M - Q;  // columns [0, bw)
  const int seglen = ((cend + 1 + nseg - 1) / nseg + CW - 1) / CW * CW;
  const int cs = seg * seglen;
  const int ce = min(cend, cs + seglen - 1);
  const int nchunks = ce >= cs ? (ce - cs + CW) / CW : 0;

  // this thread's pair
  const int tix = threadIdx.x;
  const int r1l = tix % S, r2l = tix / S;  // valid for compute warps with tix < R2G*S
  const int r2 = r2g * R2G + r2l;
  const bool pair_ok = w < EDGE_WARPS && r2l < R2G && r2 < S;
  const int dr = (base + r2) - (base + r1l);
  unsigned valid = 0;
  if (pair_ok) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int dc = dc0 + d;
      if (in_uc(dr, dc, P, Q) && cls_slot[class_index(dr, dc, P, Q)] >= 0) valid |= 1u << d;
    }
  }
  if (!__syncthreads_or(valid != 0) || nchunks == 0) {
    // still write zero partials for this segment so the finalize sums are defined
    if (valid && nchunks == 0) {
      const int i = min(r1l, r2);
      for (int d = 0; d < D; ++d) {
        if (!(valid & (1u << d))) continue;
        const ClassDesc& cd = cls[cls_slot[class_index(dr, dc0 + d, P, Q)]];
        const int a_r = cd.pv - 1;
        const int k = strip ? a_r + (base + i - pr.bh) : i;
        rc[((long long)b * tot_rc + cd.rc_off + k) * nseg + seg] = make_double2(0.0, 0.0);
      }
    }
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbarrier_init();
  }
  __syncthreads();
  __shared__ uint64_t emptyb[EDGE_STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&emptyb[s], EDGE_WARPS);
    fence_mbarrier_init();
  }
  __syncthreads();

  if (w == EDGE_WARPS) {  // producer
    if (lane == 0) {
      for (int k = 0; k < nchunks; ++k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait_sleep(&emptyb[s], ((k - NS) / NS) & 1);
        const int c0 = cs + k * CW;
        unsigned char* st = esm + s * sb;
        mbar_expect_tx(&full[s], (unsigned)(xb + yb));
        tma_load_3d(st, &tmx, 2 * c0, base, b, &full[s]);
        tma_load_3d(st + xo, &tmy, 2 * (c0 + dc0), base + r2g * R2G, b, &full[s]);
      }
    }
    return;
  }

  T ar[D], ai[D], yr[D], yi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) ar[d] = ai[d] = yr[d] = yi[d] = (T)0;
  for (int k = 0; k < nchunks; ++k) {
    const int s = k % NS;
    mbar_wait(&full[s], (k / NS) & 1);
    const C2* X = reinterpret_cast<const C2*>(esm + s * sb) + r1l * XW;
    const C2* Y = reinterpret_cast<const C2*>(esm + s * sb + xo) + r2l * YW;
    if (valid) {
      if (k == 0) {
#pragma unroll
        for (int d = 0; d < D - 1; ++d) {
          const C2 v = Y[d];
          yr[d] = v.x;
          yi[d] = v.y;
        }
      }
      const int c0 = cs + k * CW;
      const int ncol = min(CW, ce - c0 + 1);
      for (int t0 = 0; t0 < CW; t0 += D) {
        if (t0 >= ncol) break;
        if (t0 + D <= ncol) {
#pragma unroll
          for (int cc = 0; cc < D; ++cc) {
            const C2 yn = Y[t0 + cc + D - 1];
            const C2 xv = X[t0 + cc];
            yr[(cc + D - 1) % D] = yn.x;
            yi[(cc + D - 1) % D] = yn.y;
#pragma unroll
            for (int d = 0; d < D; ++d) ar[d] = fma(xv.x, yr[(cc + d) % D], ar[d]);
#pragma unroll
            for (int d = 0; d < D; ++d) ai[d] = fma(xv.y, yr[(cc + d) % D], ai[d]);
#pragma unroll
            for (int d = 0; d < D; ++d) ar[d] = fma(xv.y, yi[(cc + d) % D], ar[d]);
#pragma unroll
            for (int d = 0; d < D; ++d) ai[d] = fma(-xv.x, yi[(cc + d) % D], ai[d]);
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < D; ++cc) {
            if (t0 + cc < ncol) {
              const C2 yn = Y[t0 + cc + D - 1];
              const C2 xv = X[t0 + cc];
              yr[(cc + D - 1) % D] = yn.x;
              yi[(cc + D - 1) % D] = yn.y;
#pragma unroll
              for (int d = 0; d < D; ++d) ar[d] = fma(xv.x, yr[(cc + d) % D], ar[d]);
#pragma unroll
              for (int d = 0; d < D; ++d) ai[d] = fma(xv.y, yr[(cc + d) % D], ai[d]);
#pragma unroll
              for (int d = 0; d < D; ++d) ar[d] = fma(xv.y, yi[(cc + d) % D], ar[d]);
#pragma unroll
              for (int d = 0; d < D; ++d) ai[d] = fma(-xv.x, yi[(cc + d) % D], ai[d]);
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&emptyb[s]);
  }
  if (!valid) return;
  const int i = min(r1l, r2);  // pane row (strip-relative)
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (!(valid & (1u << d))) continue;
    const ClassDesc& cd = cls[cls_slot[class_index(dr, dc0 + d, P, Q)]];
    const int a_r = cd.pv - 1;
    const int k = strip ? a_r + (base + i - pr.bh) : i;
    rc[((long long)b * tot_rc + cd.rc_off + k) * nseg + seg] = make_double2((double)ar[d], (double)ai[d]);
  }
}

}  // namespace covgpu

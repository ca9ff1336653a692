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

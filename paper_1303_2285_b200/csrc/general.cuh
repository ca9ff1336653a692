// General path for "unclean" shapes (N < 2P-2, M < 2Q-2, or Q > kMaxCleanQ),
// where the edge-row and edge-column ranges of a class overlap and the
// T/C/B x L/C/R decomposition of the bulk path does not apply.
#pragma once

#include "common.cuh"

namespace covgpu {

// General path (shapes with N < 2P-2 or M < 2Q-2, or very wide windows):
// the reference's vectorised algorithm (_numpy_kernels.py:30-53) — one
// product pane per class, a 2-D prefix sum, four-corner box sums.  Products
// are still formed once; arithmetic in FP64 for both dtypes.
template <typename T>
__global__ void k_sat_rows(const typename CT<T>::c* __restrict__ A, Problem pr,
                           const ClassDesc* __restrict__ cls, int c0, int ncls, int batch,
                           double2* __restrict__ sat) {
  // one thread per (class, batch, pane row); writes row prefix sums
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int N = pr.N, M = pr.M;
  const long long per = (long long)batch * N;
  if (tid >= per * ncls) return;
  const int lc = (int)(tid / per);
  const int b = (int)((tid % per) / N);
  const int i = (int)(tid % N);
  const ClassDesc c = cls[c0 + lc];
  const int H = N - abs(c.dr), W = M - c.dc;
  double2* X = sat + ((long long)lc * batch + b) * (long long)(N + 1) * (M + 1);
  if (i == 0)
    for (int j = 0; j <= M; ++j) X[j] = make_double2(0.0, 0.0);
  if (i >= H) return;
  const auto* Ab = A + (long long)b * N * M;
  const auto* x = Ab + (long long)(i + c.s1) * M;
  const auto* y = Ab + (long long)(i + c.s2) * M + c.dc;
  double2* row = X + (long long)(i + 1) * (M + 1);
  row[0] = make_double2(0.0, 0.0);
  double sr = 0.0, si = 0.0;
  const bool self = (c.dr == 0 && c.dc == 0);
  for (int j = 0; j < W; ++j) {
    const double xr = (double)x[j].x, xi = (double)x[j].y;
    if (self) {
      sr += xr * xr + xi * xi;
    } else {
      const double yr = (double)y[j].x, yi = (double)y[j].y;
      sr += xr * yr + xi * yi;
      si += xi * yr - xr * yi;
    }
    row[j + 1] = make_double2(sr, si);
  }
}

__global__ void k_sat_cols(Problem pr, const ClassDesc* __restrict__ cls, int c0, int ncls,
                           int batch, double2* __restrict__ sat) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int N = pr.N, M = pr.M;
  const long long per = (long long)batch * (M + 1);
  if (tid >= per * ncls) return;
  const int lc = (int)(tid / per);
  const int b = (int)((tid % per) / (M + 1));
  const int j = (int)(tid % (M + 1));
  const ClassDesc c = cls[c0 + lc];
  const int H = N - abs(c.dr), W = M - c.dc;
  if (j > W) return;
  double2* X = sat + ((long long)lc * batch + b) * (long long)(N + 1) * (M + 1);
  double2 acc = make_double2(0.0, 0.0);
  for (int i = 1; i <= H; ++i) {
    acc = cadd(acc, X[(long long)i * (M + 1) + j]);
    X[(long long)i * (M + 1) + j] = acc;
  }
}

template <typename T>
__global__ void k_sat_gather(Problem pr, const ClassDesc* __restrict__ cls, int c0, int ncls,
                             int batch, const double2* __restrict__ sat, int max_slots,
                             typename CT<T>::c* __restrict__ R, int layout, long long r_bstride,
                             double scale) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)batch * max_slots;
  if (tid >= per * ncls) return;
  const int lc = (int)(tid / per);
  const int b = (int)((tid % per) / max_slots);
  const int s = (int)(tid % max_slots);
  const ClassDesc c = cls[c0 + lc];
  if (s >= c.pv * c.qu) return;
  const int u = s / c.pv, v = s % c.pv;
  const int N = pr.N, M = pr.M;
  const double2* X = sat + ((long long)lc * batch + b) * (long long)(N + 1) * (M + 1);
  const long long ld = M + 1;
  const int bh = pr.bh, bw = pr.bw;
  const double2 a = X[(long long)(v + bh) * ld + (u + bw)];
  const double2 bb = X[(long long)v * ld + (u + bw)];
  const double2 cc = X[(long long)(v + bh) * ld + u];
  const double2 dd = X[(long long)v * ld + u];
  const double re = ((a.x - bb.x) - cc.x + dd.x) * scale;
  const double im = (c.d == 0) ? 0.0 : ((a.y - bb.y) - cc.y + dd.y) * scale;
  write_slot<T>(R, layout, (long long)b * r_bstride, c, pr, v, u, re, im);
}


}  // namespace covgpu

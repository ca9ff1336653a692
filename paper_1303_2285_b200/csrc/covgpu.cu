// covgpu — B200-native windowed covariance estimation (arXiv 1303.2285).
//
// Hot path: for every offset class (dr, dc) of the
// reference's unique-combination set UC (combinations.py:53-62) compute the
// class's (P-|dr|) x (Q-dc) slot sums
//     S(v,u) = sum_{i=v}^{v+bh-1} sum_{j=u}^{u+bw-1} prod[i,j],
//     prod[i,j] = A[i+s1, j] * conj(A[i+s2, j+dc])         (_numba_kernels.py:62-107)
// with every product formed exactly once, and write them (scaled by 1/K) to
// the class's diagonal segments of R.
//
// Decomposition: the pane rows split into top edge T=[0,a_r),
// core C=[a_r,bh), bottom edge B=[bh,H); columns into L=[0,a_c), C=[a_c,bw),
// Rt=[bw,W), a_r = P-|dr|-1, a_c = Q-dc-1.  Then
//     S(v,u) = G(u) + sum_{i=v}^{a_r-1} fullT_i(u) + sum_{t<v} fullB_t(u)
//     G(u)   = CC + sum_{j>=u} CColL[j] + sum_{t<u} CColR[t]
// where CC is the core x core sum, CCol* are edge-column sums over core rows,
// fullT/B are edge-row sums over cols(u).  The v-walk is the paper's
// diagonal-segment recurrence: S(v+1,u) = S(v,u) - fullT_v(u) + fullB_v(u).
//
// Kernels
//   k_bulk      core rows x all columns: lanes = columns, walk rows, E row
//               lags (dr) in a rotating register window.  Emits CC partials
//               per column block and the edge-column sums CCol.      (FP pipe)
//   k_edge_rows edge rows x core columns: RC (edge-row sums).
//   k_finalize  per class: G(u), corner products, the v-walk, 1/K, writes R.
//   k_sat_*     general path for "unclean" shapes (N < 2P-2 or M < 2Q-2),
//               the reference's SAT algorithm (_numpy_kernels.py:30-53).
//
// Every R element has a single writer; no atomics anywhere; all reductions
// run in a fixed order, so results are bitwise reproducible and independent
// of how classes are sharded across launches or GPUs.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/covgpu.h"

namespace {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(COVGPU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// complex helpers
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// class table
// ---------------------------------------------------------------------------
struct ClassDesc {
  int dr, dc;
  int pv, qu;  // slot grid
  int s1, s2;  // first/second element row shift
  int d;       // output diagonal dc*P + dr
  int uc;      // index in UC order
  long long rc_off;    // 2*(pv-1) edge-row sums: top rows then bottom rows
  long long ccol_off;  // 2*(qu-1) edge-column sums: left cols then right cols
  long long slot_off;  // compact class-major offset (u-major, then v)
};

struct Problem {
  int N, M, P, Q;
  int bh, bw;  // box (window-placement) extents N-P+1, M-Q+1
  int PQ;
};

__host__ __device__ inline int class_index(int dr, int dc, int P, int Q) {
  // UC order, combinations.py:53-62
  return dr >= 0 ? dr * Q + dc : P * Q + (dr + P - 1) * (Q - 1) + (dc - 1);
}

__host__ __device__ inline long long packed_off(long long k1, long long k2, long long dim) {
  // core.py:60-72 (0-based): row k1 contributes dim - k1 entries
  return k1 * dim - (k1 * (k1 - 1)) / 2 + (k2 - k1);
}

// Output element write for slot (v,u) of class c. Single writer per element.
template <typename T>
__device__ inline void write_slot(typename CT<T>::c* R, int layout, long long bstride,
                                  const ClassDesc& c, const Problem& pr, int v, int u,
                                  double re, double im) {
  using C2 = typename CT<T>::c;
  const long long k1 = (long long)pr.P * u + c.s1 + v;
  const long long k2 = k1 + c.d;
  C2 val;
  val.x = (T)re;
  val.y = (T)im;
  if (layout == COVGPU_DENSE) {
    const long long D = pr.PQ;
    R[bstride + k1 * D + k2] = val;
    if (c.d != 0) {
      C2 cv;
      cv.x = val.x;
      cv.y = -val.y;
      R[bstride + k2 * D + k1] = cv;
    }
  } else if (layout == COVGPU_PACKED) {
    R[bstride + packed_off(k1, k2, pr.PQ)] = val;
  } else {
    R[bstride + c.slot_off + (long long)u * c.pv + v] = val;
  }
}

// ---------------------------------------------------------------------------
// K1: bulk kernel.  One warp = (snapshot b, work group g = (dc, dr0..dr0+E-1),
// column block cb).  Lane l owns first-element column c1 = 32*cb + l and walks
// the first-element rows r1 of the union of the group's core-row ranges;
// lag e (dr = dr0+e) accumulates A[r1,c1] * conj(A[r1+dr, c1+dc]) while r1 is
// a core row of that class.  The E second-element rows in flight live in a
// rotating register window, so each step loads 2 complex values for E
// products.
// ---------------------------------------------------------------------------
struct GroupDesc {
  int dc, dr0;
};

template <typename T, int E>
__global__ void __launch_bounds__(256) k_bulk(const typename CT<T>::c* __restrict__ A, Problem pr,
                                              const GroupDesc* __restrict__ groups, int ngroups,
                                              int ncb, int nclasses,
                                              const int* __restrict__ cls_slot,  // UC -> local or -1
                                              const ClassDesc* __restrict__ cls,
                                              double2* __restrict__ ccpart,
                                              double2* __restrict__ ccol, long long tot_ccol,
                                              long long total_warps) {
  using C2 = typename CT<T>::c;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= total_warps) return;
  const int lane = threadIdx.x & 31;
  long long t = wid;
  const int cb = (int)(t % ncb);
  t /= ncb;
  const int g = (int)(t % ngroups);
  const int b = (int)(t / ngroups);

  const int N = pr.N, M = pr.M, P = pr.P, Q = pr.Q;
  const GroupDesc gd = groups[g];
  const int dc = gd.dc, dr0 = gd.dr0;
  const C2* __restrict__ Ab = A + (long long)b * N * M;

  int lo[E], hi[E], cid[E];
  int rlo = INT_MAX, rhi = INT_MIN;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int dr = dr0 + e;
    const bool ok = dr > -P && dr < P && (dc > 0 || dr >= 0);
    const int uc = ok ? class_index(dr, dc, P, Q) : -1;
    const int loc = uc >= 0 ? cls_slot[uc] : -1;
    cid[e] = loc;
    if (loc >= 0) {
      lo[e] = P - 1 - max(dr, 0);
      hi[e] = N - P + max(-dr, 0);
      rlo = min(rlo, lo[e]);
      rhi = max(rhi, hi[e]);
    } else {
      lo[e] = INT_MAX;
      hi[e] = INT_MIN;
    }
  }
  if (rlo > rhi) return;  // no selected class in this group

  const int c1 = cb * 32 + lane;
  const int cx = min(c1, M - 1);
  const int cy = min(c1 + dc, M - 1);

  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    ar[e] = (T)0;
    ai[e] = (T)0;
  }
  auto yrow = [&](int r) { return min(max(r, 0), N - 1); };
#pragma unroll
  for (int e = 0; e < E - 1; ++e) {
    const C2 y = Ab[(long long)yrow(rlo + dr0 + e) * M + cy];
    yr[e] = y.x;
    yi[e] = y.y;
  }
  for (int base = rlo; base <= rhi; base += E) {
#pragma unroll
    for (int tt = 0; tt < E; ++tt) {
      const int r = base + tt;
      if (r <= rhi) {
        const C2 y = Ab[(long long)yrow(r + dr0 + E - 1) * M + cy];
        yr[(tt + E - 1) % E] = y.x;
        yi[(tt + E - 1) % E] = y.y;
        const C2 x = Ab[(long long)r * M + cx];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (r >= lo[e] && r <= hi[e]) {
            const int s = (tt + e) % E;
            ar[e] = fma(x.x, yr[s], ar[e]);
            ar[e] = fma(x.y, yi[s], ar[e]);
            ai[e] = fma(x.y, yr[s], ai[e]);
            ai[e] = fma(-x.x, yi[s], ai[e]);
          }
        }
      }
    }
  }

  // epilogue: per class, core-column lanes -> CC partial of this column
  // block (fixed-order shuffle tree), edge-column lanes -> CCol entries.
  const bool lane_ok = c1 < M - dc;
  const int left_end = Q - 1 - dc;  // c1 < left_end: left edge column
  const int right_beg = M - Q + 1;  // c1 >= right_beg: right edge column
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (cid[e] < 0) continue;
    const ClassDesc& c = cls[cid[e]];
    double vr = (double)ar[e], vi = (double)ai[e];
    const bool core = lane_ok && c1 >= left_end && c1 < right_beg;
    if (lane_ok && !core) {
      const long long base_off = (long long)b * tot_ccol + c.ccol_off;
      const int ac = c.qu - 1;
      const long long idx = c1 < left_end ? c1 : (long long)ac + (c1 - right_beg);
      ccol[base_off + idx] = make_double2(vr, vi);
    }
    if (!core) {
      vr = 0.0;
      vi = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      vr += __shfl_xor_sync(0xffffffffu, vr, off);
      vi += __shfl_xor_sync(0xffffffffu, vi, off);
    }
    if (lane == 0) ccpart[((long long)b * nclasses + cid[e]) * ncb + cb] = make_double2(vr, vi);
  }
}

// ---------------------------------------------------------------------------
// K2: edge-row sums.  Thread = (b, class, edge row k).  RC[k] = sum over the
// class's core columns of prod[i, j] for pane row i = k (top) or bh+k-a_r
// (bottom).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) k_edge_rows(const typename CT<T>::c* __restrict__ A, Problem pr,
                                                   const ClassDesc* __restrict__ cls,
                                                   double2* __restrict__ rc, long long tot_rc) {
  using C2 = typename CT<T>::c;
  const ClassDesc c = cls[blockIdx.x];
  const int b = blockIdx.y;
  const int ar = c.pv - 1;
  if (ar <= 0) return;
  const int N = pr.N, M = pr.M, Q = pr.Q;
  const C2* __restrict__ Ab = A + (long long)b * N * M;
  const int jlo = Q - 1 - c.dc, jhi = M - Q;  // core columns (inclusive)
  for (int k = threadIdx.x; k < 2 * ar; k += blockDim.x) {
    const int i = k < ar ? k : pr.bh + (k - ar);
    const C2* __restrict__ x = Ab + (long long)(i + c.s1) * M;
    const C2* __restrict__ y = Ab + (long long)(i + c.s2) * M + c.dc;
    T sr = 0, si = 0;
    for (int j = jlo; j <= jhi; ++j) {
      const C2 a = x[j], bb = y[j];
      sr = fma(a.x, bb.x, sr);
      sr = fma(a.y, bb.y, sr);
      si = fma(a.y, bb.x, si);
      si = fma(-a.x, bb.y, si);
    }
    rc[(long long)b * tot_rc + c.rc_off + k] = make_double2((double)sr, (double)si);
  }
}

// ---------------------------------------------------------------------------
// K3: finalize.  CTA = (class, b).  Builds G(u), then walks the diagonal
// segment v = a_r..0 adding top-edge rows (pass T, into the compact slot
// scratch), then v = 0..a_r adding bottom-edge rows (pass B, final values,
// scaled and written to R).  Corner products (edge row x edge column) are
// formed here, once each.
// ---------------------------------------------------------------------------
constexpr int FIN_VB = 16;  // edge rows per SMEM chunk

__device__ inline double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ inline double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

template <typename T>
__device__ inline double2 cprod(const typename CT<T>::c* Ab, int M, int r1, int c1, int r2, int c2) {
  const auto a = Ab[(long long)r1 * M + c1];
  const auto b = Ab[(long long)r2 * M + c2];
  T re = fma(a.x, b.x, (T)0);
  re = fma(a.y, b.y, re);
  T im = fma(a.y, b.x, (T)0);
  im = fma(-a.x, b.y, im);
  return make_double2((double)re, (double)im);
}

template <typename T>
__global__ void __launch_bounds__(256) k_finalize(const typename CT<T>::c* __restrict__ A, Problem pr,
                                                  const ClassDesc* __restrict__ cls, int nclasses,
                                                  int ncb, const double2* __restrict__ ccpart,
                                                  const double2* __restrict__ ccol, long long tot_ccol,
                                                  const double2* __restrict__ rc, long long tot_rc,
                                                  double2* __restrict__ slots, long long tot_slots,
                                                  typename CT<T>::c* __restrict__ R, int layout,
                                                  long long r_bstride, double scale) {
  extern __shared__ double2 sm[];
  const int ci = blockIdx.x;
  const int b = blockIdx.y;
  const ClassDesc c = cls[ci];
  const int N = pr.N, M = pr.M;
  const int qu = c.qu, pv = c.pv;
  const int ar = pv - 1, ac = qu - 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const auto* Ab = A + (long long)b * N * M;
  // SMEM: G[qu] | run[qu] | F[FIN_VB][qu] | Pt[FIN_VB][2*ac]
  double2* G = sm;
  double2* run = G + qu;
  double2* F = run + qu;
  double2* Pt = F + FIN_VB * qu;
  const double2* cc_p = ccpart + ((long long)b * nclasses + ci) * ncb;
  const double2* cl = ccol + (long long)b * tot_ccol + c.ccol_off;
  const double2* rcc = rc + (long long)b * tot_rc + c.rc_off;
  double2* sl = slots + (long long)b * tot_slots + c.slot_off;
  const bool zero_im = (c.d == 0);  // class (0,0): main diagonal, exactly real

  // CC: fixed-order sum of the column-block partials
  __shared__ double2 s_cc;
  if (tid < 32) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = tid; k < ncb; k += 32) acc = cadd(acc, cc_p[k]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (tid == 0) s_cc = acc;
  }
  __syncthreads();
  // G(u) = CC + sum_{j=u}^{ac-1} CColL[j] + sum_{t<u} CColR[t]
  for (int u = tid; u < qu; u += nt) {
    double2 g = s_cc;
    for (int j = u; j < ac; ++j) g = cadd(g, cl[j]);
    for (int t = 0; t < u; ++t) g = cadd(g, cl[ac + t]);
    G[u] = g;
    run[u] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  const int bw = pr.bw, bh = pr.bh;
  // slot v = ar (last on the segment) has no top-edge contribution
  for (int u = tid; u < qu; u += nt) sl[(long long)u * pv + ar] = G[u];

  // ---- pass T: rows i = ar-1 .. 0 (descending chunks) ----------------------
  for (int i_hi = ar; i_hi > 0; i_hi -= FIN_VB) {
    const int i_lo = max(0, i_hi - FIN_VB);
    const int nr = i_hi - i_lo;
    // corner products of rows [i_lo, i_hi): left cols j<ac, right cols bw+t
    for (int k = tid; k < nr * 2 * ac; k += nt) {
      const int ii = k / (2 * ac), jj = k % (2 * ac);
      const int i = i_lo + ii;
      const int j = jj < ac ? jj : bw + (jj - ac);
      Pt[ii * 2 * ac + jj] = cprod<T>(Ab, M, i + c.s1, j, i + c.s2, j + c.dc);
    }
    __syncthreads();
    // row scan: fullT_i(u) = RC_T[i] + sum_{j>=u} PL[j] + sum_{t<u} PR[t]
    for (int ii = tid; ii < nr; ii += nt) {
      const double2* pl = Pt + ii * 2 * ac;
      double2 val = rcc[i_lo + ii];
      for (int j = 0; j < ac; ++j) val = cadd(val, pl[j]);
      for (int u = 0; u < qu; ++u) {
        F[ii * qu + u] = val;
        if (u < ac) val = cadd(csub(val, pl[u]), pl[ac + u]);
      }
    }
    __syncthreads();
    for (int u = tid; u < qu; u += nt) {
      double2 acc = run[u];
      for (int ii = nr - 1; ii >= 0; --ii) {
        acc = cadd(acc, F[ii * qu + u]);
        sl[(long long)u * pv + (i_lo + ii)] = cadd(G[u], acc);
      }
      run[u] = acc;
    }
    __syncthreads();
  }

  // ---- pass B: rows t = 0 .. ar-1 (ascending chunks) -> final values ------
  for (int u = tid; u < qu; u += nt) run[u] = make_double2(0.0, 0.0);
  __syncthreads();
  using C2 = typename CT<T>::c;
  const long long rb = (long long)b * r_bstride;
  auto emit = [&](int v, int u, double2 s) {
    double re = s.x * scale, im = zero_im ? 0.0 : s.y * scale;
    if (layout == COVGPU_COMPACT) {
      C2 val;
      val.x = (T)re;
      val.y = (T)im;
      R[rb + c.slot_off + (long long)u * pv + v] = val;
    } else {
      write_slot<T>(R, layout, rb, c, pr, v, u, re, im);
    }
  };
  for (int u = tid; u < qu; u += nt) emit(0, u, sl[(long long)u * pv + 0]);
  for (int t_lo = 0; t_lo < ar; t_lo += FIN_VB) {
    const int t_hi = min(ar, t_lo + FIN_VB);
    const int nr = t_hi - t_lo;
    for (int k = tid; k < nr * 2 * ac; k += nt) {
      const int ii = k / (2 * ac), jj = k % (2 * ac);
      const int i = bh + t_lo + ii;
      const int j = jj < ac ? jj : bw + (jj - ac);
      Pt[ii * 2 * ac + jj] = cprod<T>(Ab, M, i + c.s1, j, i + c.s2, j + c.dc);
    }
    __syncthreads();
    for (int ii = tid; ii < nr; ii += nt) {
      const double2* pl = Pt + ii * 2 * ac;
      double2 val = rcc[ar + t_lo + ii];
      for (int j = 0; j < ac; ++j) val = cadd(val, pl[j]);
      for (int u = 0; u < qu; ++u) {
        F[ii * qu + u] = val;
        if (u < ac) val = cadd(csub(val, pl[u]), pl[ac + u]);
      }
    }
    __syncthreads();
    for (int u = tid; u < qu; u += nt) {
      double2 acc = run[u];
      for (int ii = 0; ii < nr; ++ii) {
        acc = cadd(acc, F[ii * qu + u]);
        const int v = t_lo + ii + 1;
        emit(v, u, cadd(sl[(long long)u * pv + v], acc));
      }
      run[u] = acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// General path (shapes with N < 2P-2 or M < 2Q-2, or very wide windows):
// the reference's vectorised algorithm (_numpy_kernels.py:30-53) — one
// product pane per class, a 2-D prefix sum, four-corner box sums.  Products
// are still formed once; arithmetic in FP64 for both dtypes.
// ---------------------------------------------------------------------------
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
  using C2 = typename CT<T>::c;
  if (layout == COVGPU_COMPACT) {
    C2 val;
    val.x = (T)re;
    val.y = (T)im;
    R[(long long)b * r_bstride + c.slot_off + (long long)u * c.pv + v] = val;
  } else {
    write_slot<T>(R, layout, (long long)b * r_bstride, c, pr, v, u, re, im);
  }
}

__global__ void k_warm(int* p) {
  if (threadIdx.x == 0 && p) *p = 1;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
constexpr int kMaxCleanQ = 4096;

}  // namespace

struct covgpu_plan {
  int device = 0;
  int dtype = COVGPU_C128;
  long long batch = 1;
  Problem pr{};
  bool clean = true;
  int E = 16;
  int ncb = 0;
  int nclasses = 0;                 // selected classes
  std::vector<ClassDesc> h_cls;     // selected classes
  std::vector<GroupDesc> h_groups;  // bulk groups containing >= 1 selected class
  long long tot_rc = 0, tot_ccol = 0, tot_slots = 0;
  long long compact_elems = 0;
  int max_slots = 0;
  // device
  ClassDesc* d_cls = nullptr;
  GroupDesc* d_groups = nullptr;
  int* d_cls_slot = nullptr;
  double2* d_ccpart = nullptr;
  double2* d_ccol = nullptr;
  double2* d_rc = nullptr;
  double2* d_slots = nullptr;
  double2* d_sat = nullptr;
  int sat_chunk = 0;
  long long ws_bytes = 0;
  size_t fin_smem = 0;
  int launches = 0;
};

namespace {

int validate(long long batch, long long n, long long m, int p, int q, int dtype) {
  if (batch < 1) return fail(COVGPU_EINVAL, "batch must contain at least one matrix");
  if (n < 1 || m < 1)
    return fail(COVGPU_EINVAL, "input matrix must be non-empty, got shape (" + std::to_string(n) +
                                   ", " + std::to_string(m) + ")");
  if (p < 1 || q < 1)
    return fail(COVGPU_EINVAL, "window dimensions must be positive, got " + std::to_string(p) +
                                   "x" + std::to_string(q));
  if (p > n || q > m)
    return fail(COVGPU_EINVAL, std::to_string(p) + "x" + std::to_string(q) +
                                   " window does not fit a " + std::to_string(n) + "x" +
                                   std::to_string(m) + " matrix");
  const long long pq = (long long)p * q;
  if (pq * (pq + 1) / 2 > 2147483647LL)
    return fail(COVGPU_ECAPACITY, "packed triangle of a " + std::to_string(pq) + "x" +
                                      std::to_string(pq) + " matrix exceeds 2^31-1 entries");
  if (n > INT_MAX / 2 || m > INT_MAX / 2) return fail(COVGPU_EINVAL, "matrix too large");
  if (dtype != COVGPU_C128 && dtype != COVGPU_C64) return fail(COVGPU_EINVAL, "unknown dtype");
  return COVGPU_OK;
}

template <typename X>
int dalloc(X** p, size_t count, long long* acc) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(X));
  if (e != cudaSuccess) return fail(COVGPU_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  *acc += (long long)(count * sizeof(X));
  return COVGPU_OK;
}

void plan_free(covgpu_plan* pl) {
  cudaFree(pl->d_cls);
  cudaFree(pl->d_groups);
  cudaFree(pl->d_cls_slot);
  cudaFree(pl->d_ccpart);
  cudaFree(pl->d_ccol);
  cudaFree(pl->d_rc);
  cudaFree(pl->d_slots);
  cudaFree(pl->d_sat);
}

int pick_E(int P) {
  const int span = 2 * P - 1;
  if (span <= 4) return 4;
  if (span <= 8) return 8;
  return 16;
}

template <typename T>
int launch_all(covgpu_plan* pl, const void* A_dev, void* R_dev, int layout, double scale,
               cudaStream_t st) {
  using C2 = typename CT<T>::c;
  const C2* A = (const C2*)A_dev;
  C2* R = (C2*)R_dev;
  const Problem& pr = pl->pr;
  const int B = (int)pl->batch;
  long long r_bstride;
  if (layout == COVGPU_DENSE)
    r_bstride = (long long)pr.PQ * pr.PQ;
  else if (layout == COVGPU_PACKED)
    r_bstride = (long long)pr.PQ * (pr.PQ + 1) / 2;
  else
    r_bstride = pl->compact_elems;
  int launches = 0;
  if (pl->nclasses == 0) return COVGPU_OK;

  if (!pl->clean) {
    // general path in class chunks bounded by the SAT scratch
    for (int c0 = 0; c0 < pl->nclasses; c0 += pl->sat_chunk) {
      const int nc = std::min(pl->sat_chunk, pl->nclasses - c0);
      const long long rows = (long long)nc * B * pr.N;
      k_sat_rows<T><<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(A, pr, pl->d_cls, c0, nc, B,
                                                                    pl->d_sat);
      const long long cols = (long long)nc * B * (pr.M + 1);
      k_sat_cols<<<(unsigned)((cols + 127) / 128), 128, 0, st>>>(pr, pl->d_cls, c0, nc, B,
                                                                 pl->d_sat);
      const long long sl = (long long)nc * B * pl->max_slots;
      k_sat_gather<T><<<(unsigned)((sl + 127) / 128), 128, 0, st>>>(
          pr, pl->d_cls, c0, nc, B, pl->d_sat, pl->max_slots, R, layout, r_bstride, scale);
      launches += 3;
    }
    CUDA_TRY(cudaGetLastError());
    pl->launches = launches;
    return COVGPU_OK;
  }

  const int ng = (int)pl->h_groups.size();
  const long long warps = (long long)B * ng * pl->ncb;
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  if (ng > 0) {
    switch (pl->E) {
      case 4:
        k_bulk<T, 4><<<blocks, 256, 0, st>>>(A, pr, pl->d_groups, ng, pl->ncb, pl->nclasses,
                                             pl->d_cls_slot, pl->d_cls, pl->d_ccpart, pl->d_ccol,
                                             pl->tot_ccol, warps);
        break;
      case 8:
        k_bulk<T, 8><<<blocks, 256, 0, st>>>(A, pr, pl->d_groups, ng, pl->ncb, pl->nclasses,
                                             pl->d_cls_slot, pl->d_cls, pl->d_ccpart, pl->d_ccol,
                                             pl->tot_ccol, warps);
        break;
      default:
        k_bulk<T, 16><<<blocks, 256, 0, st>>>(A, pr, pl->d_groups, ng, pl->ncb, pl->nclasses,
                                              pl->d_cls_slot, pl->d_cls, pl->d_ccpart, pl->d_ccol,
                                              pl->tot_ccol, warps);
    }
    ++launches;
  }
  dim3 gcls((unsigned)pl->nclasses, (unsigned)B);
  k_edge_rows<T><<<gcls, 128, 0, st>>>(A, pr, pl->d_cls, pl->d_rc, pl->tot_rc);
  ++launches;
  k_finalize<T><<<gcls, 256, pl->fin_smem, st>>>(A, pr, pl->d_cls, pl->nclasses, pl->ncb,
                                                 pl->d_ccpart, pl->d_ccol, pl->tot_ccol, pl->d_rc,
                                                 pl->tot_rc, pl->d_slots, pl->tot_slots, R, layout,
                                                 r_bstride, scale);
  ++launches;
  CUDA_TRY(cudaGetLastError());
  pl->launches = launches;
  return COVGPU_OK;
}

struct PlanKey {
  int device, dtype;
  long long batch, n, m;
  int p, q;
  std::vector<int32_t> ids;
  bool operator<(const PlanKey& o) const {
    return std::tie(device, dtype, batch, n, m, p, q, ids) <
           std::tie(o.device, o.dtype, o.batch, o.n, o.m, o.p, o.q, o.ids);
  }
};

std::mutex g_cache_mu;
std::map<PlanKey, covgpu_plan*> g_cache;

}  // namespace

extern "C" {

const char* covgpu_last_error(void) { return g_last_error.c_str(); }

const char* covgpu_version(void) { return "covgpu 0.1.0 (sm_100a)"; }

int64_t covgpu_num_classes(int32_t p, int32_t q) {
  if (p < 1 || q < 1) return 0;
  return (int64_t)p * q + (int64_t)(p - 1) * (q - 1);
}

int covgpu_init(int device) {
  CUDA_TRY(cudaSetDevice(device));
  k_warm<<<1, 32>>>(nullptr);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return COVGPU_OK;
}

int64_t covgpu_output_elems(int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q,
                            int32_t layout, const int32_t* class_ids, int32_t n_classes) {
  (void)n;
  (void)m;
  const long long pq = (long long)p * q;
  if (batch < 1 || p < 1 || q < 1) return -1;
  if (layout == COVGPU_DENSE) return batch * pq * pq;
  if (layout == COVGPU_PACKED) return batch * (pq * (pq + 1) / 2);
  if (layout == COVGPU_COMPACT) {
    if (!class_ids) return batch * (pq * (pq + 1) / 2);
    long long tot = 0;
    const int nuc = (int)covgpu_num_classes(p, q);
    for (int k = 0; k < n_classes; ++k) {
      const int uc = class_ids[k];
      if (uc < 0 || uc >= nuc) return -1;
      int dr, dc;
      if (uc < p * q) {
        dr = uc / q;
        dc = uc % q;
      } else {
        const int r = uc - p * q;
        dr = r / (q - 1) - (p - 1);
        dc = r % (q - 1) + 1;
      }
      tot += (long long)(p - std::abs(dr)) * (q - dc);
    }
    return batch * tot;
  }
  return -1;
}

int covgpu_plan_create(covgpu_plan_t* out, int device, int64_t batch, int64_t n, int64_t m,
                       int32_t p, int32_t q, int32_t dtype, const int32_t* class_ids,
                       int32_t n_classes) {
  if (!out) return fail(COVGPU_EINVAL, "plan pointer is NULL");
  *out = nullptr;
  int rc = validate(batch, n, m, p, q, dtype);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(device));
  auto pl = std::make_unique<covgpu_plan>();
  pl->device = device;
  pl->dtype = dtype;
  pl->batch = batch;
  Problem& pr = pl->pr;
  pr.N = (int)n;
  pr.M = (int)m;
  pr.P = p;
  pr.Q = q;
  pr.bh = (int)n - p + 1;
  pr.bw = (int)m - q + 1;
  pr.PQ = p * q;
  pl->clean = (n >= 2LL * p - 2) && (m >= 2LL * q - 2) && q <= kMaxCleanQ;
  pl->E = pick_E(p);
  pl->ncb = (int)((m + 31) / 32);

  const int nuc = (int)covgpu_num_classes(p, q);
  std::vector<char> sel(nuc, class_ids ? 0 : 1);
  if (class_ids) {
    for (int k = 0; k < n_classes; ++k) {
      const int uc = class_ids[k];
      if (uc < 0 || uc >= nuc) return fail(COVGPU_EINVAL, "class id out of range");
      sel[uc] = 1;
    }
  }
  std::vector<int> cls_slot(nuc, -1);
  long long rc_off = 0, ccol_off = 0, slot_off = 0;
  int max_slots = 0;
  for (int uc = 0; uc < nuc; ++uc) {
    if (!sel[uc]) continue;
    ClassDesc c{};
    if (uc < p * q) {
      c.dr = uc / q;
      c.dc = uc % q;
    } else {
      const int r = uc - p * q;
      c.dr = r / (q - 1) - (p - 1);
      c.dc = r % (q - 1) + 1;
    }
    c.pv = p - std::abs(c.dr);
    c.qu = q - c.dc;
    c.s1 = std::max(-c.dr, 0);
    c.s2 = std::max(c.dr, 0);
    c.d = c.dc * p + c.dr;
    c.uc = uc;
    c.rc_off = rc_off;
    c.ccol_off = ccol_off;
    c.slot_off = slot_off;
    rc_off += 2LL * (c.pv - 1);
    ccol_off += 2LL * (c.qu - 1);
    slot_off += (long long)c.pv * c.qu;
    max_slots = std::max(max_slots, c.pv * c.qu);
    cls_slot[uc] = (int)pl->h_cls.size();
    pl->h_cls.push_back(c);
  }
  pl->nclasses = (int)pl->h_cls.size();
  pl->tot_rc = rc_off;
  pl->tot_ccol = ccol_off;
  pl->tot_slots = slot_off;
  pl->compact_elems = slot_off;
  pl->max_slots = max_slots;

  // bulk groups: dc = 0 -> dr in [0, P); dc >= 1 -> dr in [-(P-1), P)
  const int E = pl->E;
  for (int dc = 0; dc < q; ++dc) {
    const int dr_first = dc == 0 ? 0 : -(p - 1);
    for (int dr0 = dr_first; dr0 < p; dr0 += E) {
      bool any = false;
      for (int e = 0; e < E && dr0 + e < p; ++e) {
        const int uc = class_index(dr0 + e, dc, p, q);
        if (sel[uc]) any = true;
      }
      if (any) pl->h_groups.push_back(GroupDesc{dc, dr0});
    }
  }

  long long ws = 0;
  const size_t nc = (size_t)std::max(pl->nclasses, 1);
  if ((rc = dalloc(&pl->d_cls, nc, &ws)) || (rc = dalloc(&pl->d_cls_slot, (size_t)nuc, &ws)) ||
      (rc = dalloc(&pl->d_groups, std::max<size_t>(pl->h_groups.size(), 1), &ws))) {
    plan_free(pl.get());
    return rc;
  }
  if (pl->clean) {
    if ((rc = dalloc(&pl->d_ccpart, (size_t)batch * nc * pl->ncb, &ws)) ||
        (rc = dalloc(&pl->d_ccol, (size_t)(batch * std::max(pl->tot_ccol, 1LL)), &ws)) ||
        (rc = dalloc(&pl->d_rc, (size_t)(batch * std::max(pl->tot_rc, 1LL)), &ws)) ||
        (rc = dalloc(&pl->d_slots, (size_t)(batch * std::max(pl->tot_slots, 1LL)), &ws))) {
      plan_free(pl.get());
      return rc;
    }
    const int qmax = q;
    const int acmax = std::max(q - 1, 1);
    pl->fin_smem = sizeof(double2) * ((size_t)2 * qmax + (size_t)FIN_VB * qmax + (size_t)FIN_VB * 2 * acmax);
    if (pl->fin_smem > 48 * 1024) {
      cudaError_t e;
      e = cudaFuncSetAttribute(k_finalize<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)pl->fin_smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_finalize<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pl->fin_smem);
      if (e != cudaSuccess) {
        plan_free(pl.get());
        return fail(COVGPU_ECUDA, std::string("finalize smem: ") + cudaGetErrorString(e));
      }
    }
  } else {
    // SAT scratch: bounded to ~512 MB per chunk of classes
    const long long per_class = batch * (n + 1) * (m + 1) * (long long)sizeof(double2);
    long long chunk = std::max(1LL, (512LL << 20) / std::max(per_class, 1LL));
    chunk = std::min<long long>(chunk, pl->nclasses);
    pl->sat_chunk = (int)std::max(1LL, chunk);
    if ((rc = dalloc(&pl->d_sat, (size_t)(pl->sat_chunk * batch * (n + 1) * (m + 1)), &ws))) {
      plan_free(pl.get());
      return rc;
    }
  }
  pl->ws_bytes = ws;
  cudaError_t e = cudaMemcpy(pl->d_cls, pl->h_cls.data(), sizeof(ClassDesc) * pl->h_cls.size(),
                             cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(pl->d_cls_slot, cls_slot.data(), sizeof(int) * cls_slot.size(),
                   cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !pl->h_groups.empty())
    e = cudaMemcpy(pl->d_groups, pl->h_groups.data(), sizeof(GroupDesc) * pl->h_groups.size(),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    plan_free(pl.get());
    return fail(COVGPU_ECUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  }
  *out = pl.release();
  return COVGPU_OK;
}

int covgpu_plan_execute(covgpu_plan_t pl, const void* A_dev, void* R_dev, int32_t layout,
                        double scale, void* stream) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  if (!A_dev || !R_dev) return fail(COVGPU_EINVAL, "A and R must be device pointers");
  if (layout < COVGPU_DENSE || layout > COVGPU_COMPACT) return fail(COVGPU_EINVAL, "unknown layout");
  CUDA_TRY(cudaSetDevice(pl->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (pl->dtype == COVGPU_C128) return launch_all<double>(pl, A_dev, R_dev, layout, scale, st);
  return launch_all<float>(pl, A_dev, R_dev, layout, scale, st);
}

int64_t covgpu_plan_workspace_bytes(covgpu_plan_t pl) { return pl ? pl->ws_bytes : -1; }
int32_t covgpu_plan_num_groups(covgpu_plan_t pl) { return pl ? (int32_t)pl->h_groups.size() : -1; }
int32_t covgpu_plan_launches(covgpu_plan_t pl) { return pl ? pl->launches : -1; }

int covgpu_plan_destroy(covgpu_plan_t pl) {
  if (!pl) return COVGPU_OK;
  cudaSetDevice(pl->device);
  plan_free(pl);
  delete pl;
  return COVGPU_OK;
}

static int cached_plan(covgpu_plan_t* out, int device, int64_t batch, int64_t n, int64_t m,
                       int32_t p, int32_t q, int32_t dtype, const int32_t* ids, int32_t nids) {
  PlanKey key{device, dtype, batch, n, m, p, q, {}};
  if (ids) key.ids.assign(ids, ids + nids);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *out = it->second;
    return COVGPU_OK;
  }
  if (g_cache.size() >= 16) {
    for (auto& kv : g_cache) covgpu_plan_destroy(kv.second);
    g_cache.clear();
  }
  int rc = covgpu_plan_create(out, device, batch, n, m, p, q, dtype, ids, nids);
  if (rc) return rc;
  g_cache[key] = *out;
  return COVGPU_OK;
}

int covgpu_estimate(const void* A_dev, int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q,
                    int32_t dtype, int32_t layout, const int32_t* class_ids, int32_t n_classes,
                    double scale, void* R_dev, void* stream) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  covgpu_plan_t pl = nullptr;
  int rc = cached_plan(&pl, dev, batch, n, m, p, q, dtype, class_ids, n_classes);
  if (rc) return rc;
  return covgpu_plan_execute(pl, A_dev, R_dev, layout, scale, stream);
}

int covgpu_estimate_host(const void* A_host, int64_t batch, int64_t n, int64_t m, int32_t p,
                         int32_t q, int32_t dtype, int32_t layout, double scale, void* R_host,
                         int device) {
  int rc = validate(batch, n, m, p, q, dtype);
  if (rc) return rc;
  if (!A_host || !R_host) return fail(COVGPU_EINVAL, "host buffers must be non-NULL");
  CUDA_TRY(cudaSetDevice(device));
  covgpu_plan_t pl = nullptr;
  rc = cached_plan(&pl, device, batch, n, m, p, q, dtype, nullptr, 0);
  if (rc) return rc;
  const size_t esz = dtype == COVGPU_C128 ? 16 : 8;
  const size_t a_bytes = (size_t)batch * n * m * esz;
  const int64_t r_elems = covgpu_output_elems(batch, n, m, p, q, layout, nullptr, 0);
  if (r_elems < 0) return fail(COVGPU_EINVAL, "unknown layout");
  const size_t r_bytes = (size_t)r_elems * esz;
  void *dA = nullptr, *dR = nullptr;
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t e = cudaMallocAsync(&dA, a_bytes, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dR, r_bytes, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A_host, a_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    return fail(COVGPU_ECUDA, std::string("estimate_host: ") + cudaGetErrorString(e));
  }
  rc = covgpu_plan_execute(pl, dA, dR, layout, scale, st);
  if (rc == COVGPU_OK) {
    e = cudaMemcpyAsync(R_host, dR, r_bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(COVGPU_ECUDA, std::string("estimate_host: ") + cudaGetErrorString(e));
  }
  cudaFreeAsync(dA, st);
  cudaFreeAsync(dR, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

int covgpu_combination(const void* A_dev, int64_t n, int64_t m, int32_t dr, int32_t dc, int32_t p,
                       int32_t q, void* out_dev, void* stream) {
  int rc = validate(1, n, m, p, q, COVGPU_C128);
  if (rc) return rc;
  const bool in_uc = (dr >= 0 && dr < p && dc >= 0 && dc < q) || (dr < 0 && dr > -p && dc >= 1 && dc < q);
  if (!in_uc)
    return fail(COVGPU_EINVAL, "offset (" + std::to_string(dr) + ", " + std::to_string(dc) +
                                   ") is not a unique combination for a " + std::to_string(p) +
                                   "x" + std::to_string(q) + " window");
  const int32_t uc = class_index(dr, dc, p, q);
  return covgpu_estimate(A_dev, 1, n, m, p, q, COVGPU_C128, COVGPU_PACKED, &uc, 1, 1.0, out_dev,
                         stream);
}

}  // extern "C"

// K1 — the bulk recurrence kernel (FP64 / FP32 CUDA cores).
//
// CTA = (snapshot b, row-lag group drg, column-lag block dcb, column block cb).
//   * lane l of warp w owns first-element column c1 = 32*cb + l and column
//     lag dc = NW*dcb + w;
//   * the CTA walks first-element rows r1; at each row, lag e of every warp
//     (dr = dr0 + e) adds A[r1, c1] * conj(A[r1+dr, c1+dc]) to its own
//     accumulator while r1 is a core row of class (dr, dc)
//     (core rows: P-1-max(dr,0) <= r1 <= N-P+max(-dr,0));
//   * the E second-element rows in flight sit in a rotating register window,
//     so each step reads 2 complex values from SMEM for E products;
//   * rows arrive in SMEM in chunks of BULK_RC through a 2-stage cp.async
//     pipeline: X tile RC x 32 (first elements), Y tile (RC+E-1) x (32+NW-1)
//     (second elements of every lag of every warp).  Rows / columns outside A
//     are zero-filled.
// Epilogue per (warp, lag): core-column lanes are summed (fixed butterfly)
// into the class's CC partial for this column block; edge-column lanes store
// their sums as the class's edge-column sums CCol (left: c1 < Q-1-dc;
// right: c1 > M-Q).
#pragma once

#include "common.cuh"

namespace covgpu {

constexpr int BULK_RC = 32;  // rows per SMEM stage (multiple of every E)

template <typename T, int E, int NW>
struct BulkCfg {
  using C2 = typename CT<T>::c;
  static constexpr int RC = BULK_RC;
  static constexpr int XW = 32;
  static constexpr int YW = 32 + NW - 1;
  static constexpr int YR = RC + E - 1;
  static constexpr size_t smem = sizeof(C2) * 2 * ((size_t)RC * XW + (size_t)YR * YW);
};

template <typename T, int E, int NW>
__global__ void __launch_bounds__(NW * 32, sizeof(T) == 8 ? 1 : 2)
    k_bulk(const typename CT<T>::c* __restrict__ A, Problem pr, int n_drg, int n_dcb, int ncb,
           int nclasses, const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
           double2* __restrict__ ccpart, double2* __restrict__ ccol, long long tot_ccol) {
  using Cfg = BulkCfg<T, E, NW>;
  using C2 = typename CT<T>::c;
  constexpr int RC = Cfg::RC, XW = Cfg::XW, YW = Cfg::YW, YR = Cfg::YR;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* Xs = reinterpret_cast<C2*>(smraw);  // [2][RC][XW]
  C2* Ys = Xs + 2 * RC * XW;              // [2][YR][YW]

  long long t = blockIdx.x;
  const int cb = (int)(t % ncb);
  t /= ncb;
  const int dcb = (int)(t % n_dcb);
  t /= n_dcb;
  const int drg = (int)(t % n_drg);
  const int b = (int)(t / n_drg);

  const int N = pr.N, M = pr.M, P = pr.P, Q = pr.Q;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dr0 = -(P - 1) + drg * E;
  const int dc_base = dcb * NW;
  const int dc = dc_base + w;
  const C2* __restrict__ Ab = A + (long long)b * N * M;

  // lags of this warp that are selected classes
  unsigned valid = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int dr = dr0 + e;
    if (dc < Q && in_uc(dr, dc, P, Q) && cls_slot[class_index(dr, dc, P, Q)] >= 0) valid |= 1u << e;
  }
  if (!__syncthreads_or(valid != 0)) return;  // CTA-uniform

  // CTA row range (union over lags), and the body where every lag is core
  const int dr_lo = dr0, dr_hi = min(dr0 + E - 1, P - 1);
  const int rlo = P - 1 - max(dr_hi, 0);
  const int rhi = N - P + max(-dr_lo, 0);
  const int body_lo = P - 1 - max(dr_lo, 0);
  const int body_hi = N - P + max(-dr_hi, 0);
  const int nrows = rhi - rlo + 1;
  const int nchunks = (nrows + RC - 1) / RC;
  const int col0 = cb * 32;
  const int ycol0 = col0 + dc_base;

  auto stage = [&](int c, int buf) {
    const int r0 = rlo + c * RC;
    C2* X = Xs + buf * RC * XW;
    C2* Y = Ys + buf * YR * YW;
    for (int idx = threadIdx.x; idx < RC * XW; idx += NW * 32) {
      const int rr = idx / XW, cc = idx % XW;
      const int row = r0 + rr, col = col0 + cc;
      const bool ok = row <= rhi && col < M;
      cp_async_elem<sizeof(C2)>(X + idx, ok ? Ab + (long long)row * M + col : Ab, ok);
    }
    for (int idx = threadIdx.x; idx < YR * YW; idx += NW * 32) {
      const int rr = idx / YW, cc = idx % YW;
      const int row = r0 + dr0 + rr, col = ycol0 + cc;
      const bool ok = row >= 0 && row < N && col < M;
      cp_async_elem<sizeof(C2)>(Y + idx, ok ? Ab + (long long)row * M + col : Ab, ok);
    }
  };

  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    ar[e] = (T)0;
    ai[e] = (T)0;
    yr[e] = (T)0;
    yi[e] = (T)0;
  }

  stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < nchunks) {
      stage(c + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const C2* X = Xs + buf * RC * XW + lane;
    const C2* Y = Ys + buf * YR * YW + lane + w;
    if (valid) {
      if (c == 0) {
#pragma unroll
        for (int e = 0; e < E - 1; ++e) {
          const C2 y = Y[e * YW];
          yr[e] = y.x;
          yi[e] = y.y;
        }
      }
      const int r0 = rlo + c * RC;
      if (r0 >= body_lo && r0 + RC - 1 <= body_hi) {
        // ---- body chunk: every lag is core, no predicates ----
        for (int t0 = 0; t0 < RC; t0 += E) {
#pragma unroll
          for (int tt = 0; tt < E; ++tt) {
            const C2 yn = Y[(t0 + tt + E - 1) * YW];
            const C2 x = X[(t0 + tt) * XW];
            yr[(tt + E - 1) % E] = yn.x;
            yi[(tt + E - 1) % E] = yn.y;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int s = (tt + e) % E;
              ar[e] = fma(x.x, yr[s], ar[e]);
              ar[e] = fma(x.y, yi[s], ar[e]);
              ai[e] = fma(x.y, yr[s], ai[e]);
              ai[e] = fma(-x.x, yi[s], ai[e]);
            }
          }
        }
      } else {
        // ---- head / tail chunk: lag e is active for e_min <= e <= e_max ----
        for (int t0 = 0; t0 < RC; t0 += E) {
#pragma unroll
          for (int tt = 0; tt < E; ++tt) {
            const int r = r0 + t0 + tt;
            if (r <= rhi) {
              const C2 yn = Y[(t0 + tt + E - 1) * YW];
              const C2 x = X[(t0 + tt) * XW];
              yr[(tt + E - 1) % E] = yn.x;
              yi[(tt + E - 1) % E] = yn.y;
              const int e_min = r >= P - 1 ? 0 : P - 1 - r - dr0;
              const int e_max = r <= N - P ? E - 1 : -dr0 - (r - N + P);
#pragma unroll
              for (int e = 0; e < E; ++e) {
                if (e >= e_min && e <= e_max) {
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
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's stage
  }
  if (!valid) return;

  // ---- epilogue ----
  const int c1 = col0 + lane;
  const bool lane_ok = c1 < M - dc;
  const int left_end = Q - 1 - dc;  // c1 < left_end: left edge column
  const int right_beg = M - Q + 1;  // c1 >= right_beg: right edge column
  const bool core = lane_ok && c1 >= left_end && c1 < right_beg;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (!(valid & (1u << e))) continue;  // warp-uniform
    const int cid = cls_slot[class_index(dr0 + e, dc, P, Q)];
    double2 v = make_double2((double)ar[e], (double)ai[e]);
    if (lane_ok && !core) {
      const ClassDesc& cd = cls[cid];
      const int ac = cd.qu - 1;
      const long long idx = c1 < left_end ? c1 : (long long)ac + (c1 - right_beg);
      ccol[(long long)b * tot_ccol + cd.ccol_off + idx] = v;
    }
    if (!core) v = make_double2(0.0, 0.0);
    v = warp_sum(v);
    if (lane == 0) ccpart[((long long)b * nclasses + cid) * ncb + cb] = v;
  }
}

}  // namespace covgpu

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
//   * rows arrive in SMEM in chunks of BULK_RC: X tile RC x 32 (first
//     elements) and Y tile (RC+E-1) x YW (second elements of every lag of
//     every warp).  Rows / columns outside A are zero-filled.
//     k_bulk_tma moves the tiles with TMA (cp.async.bulk.tensor) through an
//     S-stage full/empty mbarrier ring — one thread issues, no per-element
//     address arithmetic; k_bulk (cp.async, 2 stages) serves shapes whose
//     rows are not 16-byte aligned (complex64 with odd M).
// Epilogue per (warp, lag): core-column lanes are summed (fixed butterfly)
// into the class's CC partial for this column block; edge-column lanes store
// their sums as the class's edge-column sums CCol (left: c1 < Q-1-dc;
// right: c1 > M-Q).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace covgpu {

constexpr int BULK_RC = 32;      // rows per SMEM stage (multiple of every E)
constexpr int BULK_RC_BIG = 32;  // rows per stage for 1-CTA/SM variants
constexpr int BULK_MAX_STAGES = 4;
constexpr size_t BULK_SMEM_SM = 227 * 1024;  // usable SMEM per SM

template <typename T, int E, int NW, int MINB = 1>
struct BulkCfg {
  using C2 = typename CT<T>::c;
  static constexpr int RC = MINB == 1 ? BULK_RC_BIG : BULK_RC;
  static constexpr int XW = 32;
  static constexpr int YW = 32 + NW;  // 32+NW-1 needed; +1 keeps TMA rows 16B multiples
  static constexpr int YR = RC + E - 1;
  static constexpr size_t xbytes = sizeof(C2) * (size_t)RC * XW;
  static constexpr size_t ybytes = sizeof(C2) * (size_t)YR * YW;
  static constexpr size_t ybytes_al = (ybytes + 127) / 128 * 128;
  static constexpr size_t stage_bytes = xbytes + ybytes_al;
  static constexpr size_t smem = 2 * stage_bytes;  // cp.async: double buffer
  // TMA ring: as many stages (<= 4) as fit MINB CTAs per SM
  static constexpr int fit = (int)((BULK_SMEM_SM / MINB - 1024 - 64) / stage_bytes);
  static constexpr int stages = fit > BULK_MAX_STAGES ? BULK_MAX_STAGES : fit;
  static constexpr size_t smem_tma = stages * stage_bytes + 2 * 8 * BULK_MAX_STAGES;  // + mbarriers
};

// (A packed-FP32 variant with 2 FFMA2 (fma.rn.f32x2) per lag was measured
// slower on B200: cfg4 bulk 1.12 vs 0.88 ms; FFMA2 loops peak at 54-59 TF/s
// against 65.6 TF/s for FFMA — tools/ffma2.cu.)
// acc[e] += x * conj(y[(tt+e) % E]) for every lag, in four passes that each
// keep one x component in the same operand slot, so consecutive FMAs can read
// it from the operand-reuse cache (three distinct 64-bit sources per DFMA
// are register-bank bound at 2/3 of the DFMA rate on B200).
template <typename T, int E>
__device__ __forceinline__ void cmac_all(int tt, typename CT<T>::c x, const T* yr, const T* yi, T* ar,
                                         T* ai) {
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = fma(x.x, yr[(tt + e) % E], ar[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ai[e] = fma(x.y, yr[(tt + e) % E], ai[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = fma(x.y, yi[(tt + e) % E], ar[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ai[e] = fma(-x.x, yi[(tt + e) % E], ai[e]);
}

// Per-warp view of one CTA's geometry.
struct BulkGeom {
  int b, cb, rs, dr0, dc_base, dc;
  int rlo, rhi, body_lo, body_hi, nchunks;
  int col0, ycol0;
  unsigned valid;  // selected lags of this warp
};

// ncb_l + ncb_r > 0 (edge-only mode, next to the tensor-core core sums):
// the grid covers only the first ncb_l and last ncb_r column blocks, the
// blocks holding edge columns.
template <int E, int NW, int RC>
__device__ inline BulkGeom bulk_geom(const Problem& pr, int n_drg, int n_dcb, int ncb, int nrs,
                                     const int* __restrict__ cls_slot, int ncb_l = 0, int ncb_r = 0) {
  BulkGeom g;
  long long t = blockIdx.x;
  g.rs = (int)(t % nrs);  // row segment (small problems split the row walk)
  t /= nrs;
  g.cb = (int)(t % ncb);
  t /= ncb;
  const int dcb = (int)(t % n_dcb);
  t /= n_dcb;
  const int drg = (int)(t % n_drg);
  g.b = (int)(t / n_drg);
  const int P = pr.P, Q = pr.Q, N = pr.N;
  const int w = threadIdx.x >> 5;
  g.dr0 = -(P - 1) + drg * E;
  g.dc_base = dcb * NW;
  g.dc = g.dc_base + w;
  g.valid = 0;
  if (w < NW) {  // (warp NW of the TMA variant is the producer)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int dr = g.dr0 + e;
      if (g.dc < Q && in_uc(dr, g.dc, P, Q) && cls_slot[class_index(dr, g.dc, P, Q)] >= 0)
        g.valid |= 1u << e;
    }
  }
  // CTA row range (union over lags), and the body where every lag is core
  const int dr_lo = g.dr0, dr_hi = min(g.dr0 + E - 1, P - 1);
  g.rlo = P - 1 - max(dr_hi, 0);
  g.rhi = N - P + max(-dr_lo, 0);
  g.body_lo = P - 1 - max(dr_lo, 0);
  g.body_hi = N - P + max(-dr_hi, 0);
  if (nrs > 1) {
    const int nrows = g.rhi - g.rlo + 1;
    const int seglen = ((nrows + nrs - 1) / nrs + RC - 1) / RC * RC;
    const int lo = g.rlo + g.rs * seglen;
    g.rhi = min(g.rhi, lo + seglen - 1);
    g.rlo = lo;
  }
  g.nchunks = g.rhi >= g.rlo ? (g.rhi - g.rlo + RC) / RC : 0;
  if (ncb_l + ncb_r > 0) {
    if (g.cb >= ncb_l) g.cb = (pr.M + 31) / 32 - ncb_r + (g.cb - ncb_l);
    // skip CTAs without an edge column: left edge c1 < Q-1-dc, right edge
    // M-Q+1 <= c1 < M-dc (widest for the CTA's smallest lag dc_base)
    const int c0 = g.cb * 32, dcb0 = g.dc_base;
    const bool left = c0 < Q - 1 - dcb0;
    const bool right = c0 + 31 >= pr.M - Q + 1 && dcb0 < Q - 1;
    if (!left && !right) g.valid = 0;
  }
  g.col0 = g.cb * 32;
  g.ycol0 = g.col0 + g.dc_base;
  return g;
}

// One SMEM chunk of rows [r0, r0+RC) for one warp.
template <typename T, int E, int NW, int MINB>
__device__ __forceinline__ void bulk_chunk(const BulkGeom& g, const Problem& pr, int c,
                                           const typename CT<T>::c* __restrict__ X,
                                           const typename CT<T>::c* __restrict__ Y, T* yr, T* yi,
                                           T* ar, T* ai) {
  using C2 = typename CT<T>::c;
  using Cfg = BulkCfg<T, E, NW, MINB>;
  constexpr int RC = Cfg::RC, XW = Cfg::XW, YW = Cfg::YW;
  const int N = pr.N, P = pr.P;
  if (c == 0) {
#pragma unroll
    for (int e = 0; e < E - 1; ++e) {
      const C2 y = Y[e * YW];
      yr[e] = y.x;
      yi[e] = y.y;
    }
  }
  const int r0 = g.rlo + c * RC;
  if (r0 >= g.body_lo && r0 + RC - 1 <= g.body_hi) {
    // ---- whole chunk in the body: every lag is core, no predicates ----
#pragma unroll 1
    for (int t0 = 0; t0 < RC; t0 += E) {
#pragma unroll
      for (int tt = 0; tt < E; ++tt) {
        const C2 yn = Y[(t0 + tt + E - 1) * YW];
        const C2 x = X[(t0 + tt) * XW];
        yr[(tt + E - 1) % E] = yn.x;
        yi[(tt + E - 1) % E] = yn.y;
        cmac_all<T, E>(tt, x, yr, yi, ar, ai);
      }
    }
    return;
  }
  for (int t0 = 0; t0 < RC; t0 += E) {
    const int rb = r0 + t0;
    if (rb > g.rhi) break;
    if (rb >= g.body_lo && rb + E - 1 <= g.body_hi) {
      // ---- body block: every lag is core, no predicates ----
#pragma unroll
      for (int tt = 0; tt < E; ++tt) {
        const C2 yn = Y[(t0 + tt + E - 1) * YW];
        const C2 x = X[(t0 + tt) * XW];
        yr[(tt + E - 1) % E] = yn.x;
        yi[(tt + E - 1) % E] = yn.y;
        cmac_all<T, E>(tt, x, yr, yi, ar, ai);
      }
    } else {
      // ---- head / tail block: lag e is active for e_min <= e <= e_max ----
#pragma unroll
      for (int tt = 0; tt < E; ++tt) {
        const int r = rb + tt;
        if (r <= g.rhi) {
          const C2 yn = Y[(t0 + tt + E - 1) * YW];
          const C2 x = X[(t0 + tt) * XW];
          yr[(tt + E - 1) % E] = yn.x;
          yi[(tt + E - 1) % E] = yn.y;
          const int e_min = r >= P - 1 ? 0 : P - 1 - r - g.dr0;
          const int e_max = r <= N - P ? E - 1 : -g.dr0 - (r - N + P);
          // inactive lags see y = 0 (they add exact zeros)
          T mr[E], mi[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const bool on = e >= e_min && e <= e_max;
            mr[(tt + e) % E] = on ? yr[(tt + e) % E] : (T)0;
            mi[(tt + e) % E] = on ? yi[(tt + e) % E] : (T)0;
          }
          cmac_all<T, E>(tt, x, mr, mi, ar, ai);
        }
      }
    }
  }
}

template <typename T, int E>
__device__ inline void bulk_epilogue(const BulkGeom& g, const Problem& pr, int nclasses, int ncb, int nrs,
                                     const int* __restrict__ cls_slot,
                                     const ClassDesc* __restrict__ cls, double2* __restrict__ ccpart,
                                     double2* __restrict__ ccol, long long tot_ccol, const T* ar,
                                     const T* ai, bool edge_only = false) {
  const int lane = threadIdx.x & 31;
  const int M = pr.M, Q = pr.Q, P = pr.P;
  const int c1 = g.col0 + lane;
  const bool lane_ok = c1 < M - g.dc;
  const int left_end = Q - 1 - g.dc;  // c1 < left_end: left edge column
  const int right_beg = M - Q + 1;    // c1 >= right_beg: right edge column
  const bool core = lane_ok && c1 >= left_end && c1 < right_beg;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (!(g.valid & (1u << e))) continue;  // warp-uniform
    const int cid = cls_slot[class_index(g.dr0 + e, g.dc, P, Q)];
    double2 v = make_double2((double)ar[e], (double)ai[e]);
    if (edge_only) {  // core sums come from the tensor-core kernel
      if (lane_ok && !core) {
        const ClassDesc& cd = cls[cid];
        const int ac = cd.qu - 1;
        const long long idx = c1 < left_end ? c1 : (long long)ac + (c1 - right_beg);
        ccol[((long long)g.b * tot_ccol + cd.ccol_off + idx) * nrs + g.rs] = v;
      }
      continue;
    }
    if constexpr (sizeof(T) == 4) {
      // FP32: the 32-lane butterfly in FP32 (half the shuffles of FP64)
      float sr = (lane_ok && core) ? (float)ar[e] : 0.f, si = (lane_ok && core) ? (float)ai[e] : 0.f;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, off);
        si += __shfl_xor_sync(0xffffffffu, si, off);
      }
      if (lane_ok && !core) {
        const ClassDesc& cd = cls[cid];
        const int ac = cd.qu - 1;
        const long long idx = c1 < left_end ? c1 : (long long)ac + (c1 - right_beg);
        ccol[((long long)g.b * tot_ccol + cd.ccol_off + idx) * nrs + g.rs] = v;
      }
      if (lane == 0)
        ccpart[((long long)g.b * nclasses + cid) * ncb * nrs + g.cb * nrs + g.rs] =
            make_double2((double)sr, (double)si);
      continue;
    }
    if (lane_ok && !core) {
      const ClassDesc& cd = cls[cid];
      const int ac = cd.qu - 1;
      const long long idx = c1 < left_end ? c1 : (long long)ac + (c1 - right_beg);
      ccol[((long long)g.b * tot_ccol + cd.ccol_off + idx) * nrs + g.rs] = v;
    }
    if (!core) v = make_double2(0.0, 0.0);
    v = warp_sum(v);
    if (lane == 0) ccpart[((long long)g.b * nclasses + cid) * ncb * nrs + g.cb * nrs + g.rs] = v;
  }
}

// ---- cp.async variant (any alignment) --------------------------------------
template <typename T, int E, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_bulk(const typename CT<T>::c* __restrict__ A, Problem pr, int n_drg, int n_dcb, int ncb,
           int nrs, int nclasses, const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
           double2* __restrict__ ccpart, double2* __restrict__ ccol, long long tot_ccol) {
  using Cfg = BulkCfg<T, E, NW, MINB>;
  using C2 = typename CT<T>::c;
  constexpr int RC = Cfg::RC, XW = Cfg::XW, YW = Cfg::YW, YR = Cfg::YR;
  extern __shared__ __align__(128) unsigned char smraw[];
  const BulkGeom g = bulk_geom<E, NW, RC>(pr, n_drg, n_dcb, ncb, nrs, cls_slot);
  if (!__syncthreads_or(g.valid != 0)) return;  // CTA-uniform
  const int N = pr.N, M = pr.M;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const C2* __restrict__ Ab = A + (long long)g.b * N * M;

  auto stage = [&](int c, int buf) {
    const int r0 = g.rlo + c * RC;
    C2* X = reinterpret_cast<C2*>(smraw + buf * Cfg::stage_bytes);
    C2* Y = reinterpret_cast<C2*>(smraw + buf * Cfg::stage_bytes + Cfg::xbytes);
    for (int idx = threadIdx.x; idx < RC * XW; idx += NW * 32) {
      const int rr = idx / XW, cc = idx % XW;
      const int row = r0 + rr, col = g.col0 + cc;
      const bool ok = row < N && col < M;
      cp_async_elem<sizeof(C2)>(X + idx, ok ? Ab + (long long)row * M + col : Ab, ok);
    }
    for (int idx = threadIdx.x; idx < YR * YW; idx += NW * 32) {
      const int rr = idx / YW, cc = idx % YW;
      const int row = r0 + g.dr0 + rr, col = g.ycol0 + cc;
      const bool ok = row >= 0 && row < N && col < M;
      cp_async_elem<sizeof(C2)>(Y + idx, ok ? Ab + (long long)row * M + col : Ab, ok);
    }
  };

  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = ai[e] = yr[e] = yi[e] = (T)0;

  stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < g.nchunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < g.nchunks) {
      stage(c + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const C2* X = reinterpret_cast<const C2*>(smraw + buf * Cfg::stage_bytes) + lane;
    const C2* Y = reinterpret_cast<const C2*>(smraw + buf * Cfg::stage_bytes + Cfg::xbytes) + lane + w;
    if (g.valid) bulk_chunk<T, E, NW, MINB>(g, pr, c, X, Y, yr, yi, ar, ai);
    __syncthreads();  // buffer `buf` is refilled by the next iteration's stage
  }
  if (!g.valid) return;
  bulk_epilogue<T, E>(g, pr, nclasses, ncb, nrs, cls_slot, cls, ccpart, ccol, tot_ccol, ar, ai);
}

// ---- TMA variant ------------------------------------------------------------
// A is described to TMA as a 3-D tensor of reals {2M, N, B}; the X box is
// {64, RC, 1}, the Y box {2*YW, YR, 1}; negative / past-the-end coordinates
// are zero-filled by the hardware.
template <typename T, int E, int NW, int MINB>
__global__ void __launch_bounds__((NW + 1) * 32, MINB)
    k_bulk_tma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
               Problem pr, int n_drg, int n_dcb, int ncb, int nrs, int nclasses, int B, int nsnap,
               const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
               double2* __restrict__ ccpart, double2* __restrict__ ccol, long long tot_ccol,
               int ncb_l, int ncb_r) {
  // one CTA walks `nsnap` consecutive snapshots back to back: the TMA ring
  // keeps streaming across snapshot boundaries, accumulators and the lag
  // window restart, and the epilogue of one snapshot overlaps the next
  // snapshot's loads
  using Cfg = BulkCfg<T, E, NW, MINB>;
  using C2 = typename CT<T>::c;
  constexpr int S = Cfg::stages, RC = Cfg::RC;
  static_assert(S >= 2, "TMA ring needs two stages");
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + S * Cfg::stage_bytes);
  uint64_t* empty = full + S;
  BulkGeom g = bulk_geom<E, NW, RC>(pr, n_drg, n_dcb, ncb, nrs, cls_slot, ncb_l, ncb_r);  // g.b = snapshot group
  const int b0 = g.b * nsnap;
  const int nb = min(nsnap, B - b0);
  if (!__syncthreads_or(g.valid != 0) || nb <= 0) return;  // CTA-uniform
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int total = nb * g.nchunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbarrier_init();
  }
  __syncthreads();
  auto issue = [&](int k) {  // k = global chunk index over (snapshot, chunk)
    const int s = k % S;
    const int b = b0 + k / g.nchunks;
    const int r0 = g.rlo + (k % g.nchunks) * RC;
    unsigned char* base = smraw + s * Cfg::stage_bytes;
    mbar_expect_tx(&full[s], (unsigned)(Cfg::xbytes + Cfg::ybytes));
    tma_load_3d(base, &tmx, 2 * g.col0, r0, b, &full[s]);
    tma_load_3d(base + Cfg::xbytes, &tmy, 2 * g.ycol0, r0 + g.dr0, b, &full[s]);
  };
  if (w == NW) {  // producer warp: keep the ring full
    if (lane == 0) {
      for (int k = 0; k < total; ++k) {
        if (k >= S) mbar_wait_sleep(&empty[k % S], ((k - S) / S) & 1);
        issue(k);
      }
    }
    return;
  }

  T ar[E], ai[E], yr[E], yi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = ai[e] = yr[e] = yi[e] = (T)0;

  int k = 0;  // global chunk index (ring stage and phase)
  for (int bi = 0; bi < nb; ++bi) {
    for (int c = 0; c < g.nchunks; ++c, ++k) {
      const int s = k % S;
      mbar_wait(&full[s], (k / S) & 1);
      const C2* X = reinterpret_cast<const C2*>(smraw + s * Cfg::stage_bytes) + lane;
      const C2* Y =
          reinterpret_cast<const C2*>(smraw + s * Cfg::stage_bytes + Cfg::xbytes) + lane + w;
      if (g.valid) bulk_chunk<T, E, NW, MINB>(g, pr, c, X, Y, yr, yi, ar, ai);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (g.valid) {  // snapshot done
      g.b = b0 + bi;
      bulk_epilogue<T, E>(g, pr, nclasses, ncb, nrs, cls_slot, cls, ccpart, ccol, tot_ccol, ar, ai,
                          ncb_l + ncb_r > 0);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = ai[e] = (T)0;
  }
}

}  // namespace covgpu

// K1 on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64) — complex128 only.
//
// The core sums of every class are one GEMM.  For row lag dr and column lag
// dc, CC(dr, dc) = sum over core rows r1 and core columns c of
//     A[r1, c] * conj(A[r1 + dr, c + dc]).
// Index the K dimension by (r2, c), r2 = r1 + dr the second element's row:
//     CC[dr, dc] = sum_{r2, c} X[r2 - dr, c] * conj(Y[r2, c + dc])
// is a (lags x lags) = (K-long) x (K-long)^T product whose A operand
// (m = dr, k = c) is a row-Toeplitz gather of A's rows and whose B operand
// (k = c, n = dc) is a Toeplitz gather of one row — both read straight from
// the SMEM tiles, nothing is materialised.  The class's core restriction
// splits into position-only masks that TMA applies for free:
//   * core columns: c <= M-Q (X tensor map is M-Q+1 columns wide; the
//     out-of-bounds columns are zero-filled) and c + dc >= Q-1 (Y tensor map
//     starts at column Q-1; negative coordinates are zero-filled);
//   * core rows: max(r1, r2) >= P-1 and min(r1, r2) <= N-P, which holds for
//     every lag when r2 is in [P-1, N-P]; the few head / tail rows outside
//     zero the A fragment of the lags they do not belong to.
// Complex arithmetic = 4 real DMMAs per 8x8x4 tile: Re += xr*yr + xi*yi,
// Im += xi*yr - xr*yi.
//
// CTA = (snapshot, 32-lag tile, DC-lag tile, split p of G): 4 compute warps as
// 2 (16 lags) x 2 (DC/2 lags) warp tiles and one TMA producer warp.  The
// tile's (16-row x 32-column) chunks, row-major, are dealt round-robin to
// its G CTAs (chunks p, p+G, ...), so all CTAs sweep A top to bottom
// together — which lets the host path stream A in row bands while the kernel
// runs (band_flag: the producer waits for the band a chunk needs); each
// chunk is one TMA stage: X = the 47 first-element rows x 36 columns the 16
// rows' 32 lags touch, Y = the 16 second-element rows x (32+DC) columns.  The
// CTA writes its 32 x DC partial sums to the class's partial slot p; the
// finalize adds the G partials in order, so the result is deterministic.
// Edge-column sums CCol come from the CUDA-core kernel restricted to the
// column blocks holding edge columns (bulk.cuh, edge-only mode).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace covgpu {

constexpr int MMA_DR = 32;                   // row lags per CTA
constexpr int MMA_RC = 16;                   // second-element rows per chunk
constexpr int MMA_W = 32;                    // first-element columns per chunk
constexpr int MMA_XP = 36;                   // X row pitch (complex): 576 B = 64 mod 128
constexpr int MMA_XR = MMA_RC + MMA_DR - 1;  // X rows per chunk
constexpr int MMA_STAGES = 2;
constexpr int MMA_WARPS = 4;  // compute warps (+1 producer)

template <int DC>
struct MmaCfg {
  static constexpr int NT = DC / 16;     // 8-wide lag tiles per warp (2 warps across DC)
  static constexpr int YP = MMA_W + DC;  // Y row pitch (complex); W + DC - 1 used
  static constexpr size_t xbytes = 16 * (size_t)MMA_XR * MMA_XP;
  static constexpr size_t xoff = (xbytes + 127) / 128 * 128;
  static constexpr size_t ybytes = 16 * (size_t)MMA_RC * YP;
  static constexpr size_t stage = xoff + (ybytes + 127) / 128 * 128;
  static constexpr size_t smem = MMA_STAGES * stage + 64;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// One k-step (4 columns at one second-element row): fragments from SMEM,
// 4 passes of 2*NT independent DMMAs (dependent tiles 2*NT DMMAs apart).
template <int NT>
__device__ __forceinline__ void mma_kstep(const double2* __restrict__ xa0, const double2* __restrict__ xa1,
                                          const double2* __restrict__ yb, bool on0, bool on1,
                                          double (&cr)[2][NT][2], double (&ci)[2][NT][2]) {
  double2 a[2];
  a[0] = *xa0;
  a[1] = *xa1;
  if (!on0) a[0] = make_double2(0.0, 0.0);
  if (!on1) a[1] = make_double2(0.0, 0.0);
  double2 bv[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) bv[j] = yb[8 * j];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma(cr[i][j][0], cr[i][j][1], a[i].x, bv[j].x);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma(ci[i][j][0], ci[i][j][1], a[i].y, bv[j].x);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma(cr[i][j][0], cr[i][j][1], a[i].y, bv[j].y);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double nx = -a[i].x;
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma(ci[i][j][0], ci[i][j][1], nx, bv[j].y);
  }
}

// The MMA_RC rows of one chunk.  MASKED: head / tail rows, lags whose core
// rows exclude the row see a zero A fragment.  FULL: all MMA_W columns.
template <int NT, int YP, bool MASKED, bool FULL>
__device__ __forceinline__ void mma_rows(const double2* __restrict__ X, const double2* __restrict__ Y,
                                         int xrow0, int kq, int ycol0, int nks, int R, int dra,
                                         const Problem& pr, double (&cr)[2][NT][2],
                                         double (&ci)[2][NT][2]) {
  const int P = pr.P, N = pr.N;
#pragma unroll 1
  for (int tr = 0; tr < MMA_RC; ++tr) {
    const double2* xa0 = X + (tr + xrow0) * MMA_XP + kq;
    const double2* xa1 = xa0 - 8 * MMA_XP;  // lags + 8: rows - 8
    const double2* yb = Y + tr * YP + ycol0;
    bool on0 = true, on1 = true;
    if constexpr (MASKED) {
      const int r2 = R + tr, r1a = r2 - dra, r1b = r1a - 8;
      on0 = max(r1a, r2) >= P - 1 && min(r1a, r2) <= N - P;
      on1 = max(r1b, r2) >= P - 1 && min(r1b, r2) <= N - P;
    }
    if constexpr (FULL) {
#pragma unroll
      for (int ks = 0; ks < MMA_W / 4; ++ks)
        mma_kstep<NT>(xa0 + 4 * ks, xa1 + 4 * ks, yb + 4 * ks, on0, on1, cr, ci);
    } else {
#pragma unroll 1
      for (int ks = 0; ks < nks; ++ks)
        mma_kstep<NT>(xa0 + 4 * ks, xa1 + 4 * ks, yb + 4 * ks, on0, on1, cr, ci);
    }
  }
}

// The X tile of a chunk at rows [R, R+MMA_RC) starts MMA_DR-1 rows above R - dr0.
template <int DC>
__global__ void __launch_bounds__((MMA_WARPS + 1) * 32, 2)
    k_bulk_dmma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                Problem pr, int n_drt, int n_dct, int G, int nclasses,
                const int* __restrict__ cls_slot, double2* __restrict__ ccpart,
                const unsigned* __restrict__ band_flag, unsigned band_base, int band_rows) {
  using Cfg = MmaCfg<DC>;
  constexpr int NT = Cfg::NT, YP = Cfg::YP, S = MMA_STAGES;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + S * Cfg::stage);
  uint64_t* empty = full + S;
  long long t = blockIdx.x;
  const int p = (int)(t % G);
  t /= G;
  const int dct = (int)(t % n_dct);
  t /= n_dct;
  const int drt = (int)(t % n_drt);
  const int b = (int)(t / n_drt);
  const int P = pr.P, Q = pr.Q, N = pr.N, M = pr.M;
  const int dr0 = -(P - 1) + drt * MMA_DR;
  const int dc0 = dct * DC;
  const int drmax = min(dr0 + MMA_DR - 1, P - 1);
  // second-element rows where at least one lag of the tile has core rows
  const int rlo = max(0, P - 1 + min(dr0, 0));
  const int rhi = min(N - 1, N - P + max(drmax, 0));
  const int nrc = (rhi - rlo + MMA_RC) / MMA_RC;
  const int xcols = M - Q + 1;  // first-element columns of core products
  const int ncbk = (xcols + MMA_W - 1) / MMA_W;
  const long long nch = (long long)nrc * ncbk;
  const long long nmine = p < nch ? (nch - p + G - 1) / G : 0;  // chunks p, p+G, ...
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MMA_WARPS);
    }
    fence_mbarrier_init();
  }
  __syncthreads();

  if (w == MMA_WARPS) {  // producer
    if (lane == 0) {
      for (long long k = 0; k < nmine; ++k) {
        const int s = (int)(k % S);
        if (k >= S) mbar_wait_sleep(&empty[s], (int)(((k - S) / S) & 1));
        const long long q = p + k * G;
        const int R = rlo + (int)(q / ncbk) * MMA_RC;
        const int C0 = (int)(q % ncbk) * MMA_W;
        if (band_flag) {  // A still streaming in: wait for the last row this chunk reads
          const int rneed = min(N - 1, R + MMA_RC - 1 + max(-dr0, 0));
          wait_band(band_flag, band_base + (unsigned)(rneed / band_rows) + 1u);
        }
        unsigned char* st = smraw + s * Cfg::stage;
        mbar_expect_tx(&full[s], (unsigned)(Cfg::xbytes + Cfg::ybytes));
        tma_load_3d(st, &tmx, 2 * C0, R - dr0 - (MMA_DR - 1), b, &full[s]);
        tma_load_3d(st + Cfg::xoff, &tmy, 2 * (C0 + dc0 - (Q - 1)), R, b, &full[s]);
      }
    }
    return;
  }

  const int wm = w & 1, wn = w >> 1;
  const int m = lane >> 2, kq = lane & 3;
  double cr[2][NT][2], ci[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  // this lane's A rows: lag dr0 + 16 wm + 8 i + m -> X tile row tr + 31 - 16 wm - 8 i - m
  const int xrow0 = MMA_DR - 1 - 16 * wm - m;
  const int ycol0 = kq + wn * (DC / 2) + m;

  for (long long k = 0; k < nmine; ++k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (int)((k / S) & 1));
    const long long q = p + k * G;
    const int R = rlo + (int)(q / ncbk) * MMA_RC;
    const int C0 = (int)(q % ncbk) * MMA_W;
    const int nks = min(MMA_W, xcols - C0 + 3) / 4;
    const double2* X = reinterpret_cast<const double2*>(smraw + s * Cfg::stage);
    const double2* Y = reinterpret_cast<const double2*>(smraw + s * Cfg::stage + Cfg::xoff);
    const bool masked = R < P - 1 || R + MMA_RC - 1 > N - P;
    const int dra = dr0 + 16 * wm + m;
    if (nks == MMA_W / 4) {
      if (!masked)
        mma_rows<NT, YP, false, true>(X, Y, xrow0, kq, ycol0, nks, R, dra, pr, cr, ci);
      else
        mma_rows<NT, YP, true, true>(X, Y, xrow0, kq, ycol0, nks, R, dra, pr, cr, ci);
    } else {
      mma_rows<NT, YP, true, false>(X, Y, xrow0, kq, ycol0, nks, R, dra, pr, cr, ci);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: C fragment (m, 2 kq + e) of tile (i, j) = lag (dr, dc)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int dr = dr0 + 16 * wm + 8 * i + m;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int dc = dc0 + wn * (DC / 2) + 8 * j + 2 * kq + e;
        if (dr > P - 1 || dc >= Q || !in_uc(dr, dc, P, Q)) continue;
        const int cid = cls_slot[class_index(dr, dc, P, Q)];
        if (cid < 0) continue;
        ccpart[((long long)b * nclasses + cid) * G + p] = make_double2(cr[i][j][e], ci[i][j][e]);
      }
  }
}

// ---- edge-column sums on the tensor cores ------------------------------------
// For lag dr and one edge strip of Q-1 columns starting at o (left: o = 0;
// right: o = M-Q+1), the edge-column sums
//     CCol(dr, dc)[c1] = sum_{core rows} x[r2-dr, o+c1] * conj(y[r2, o+c1+dc]),
// c1 + dc <= Q-2, are the upper triangle (e = c1 + dc >= c1) of the strip's
// lag-dr cross Gram  G[c1, e] = sum_{r2} X[r2-dr, o+c1] conj(Y[r2, o+e]) — a
// GEMM with K = the class's core rows r2 in [P-1+min(dr,0), N-P+max(dr,0)].
// 8x8 tiles (ti, tj), tj >= ti, of the <= 64-column strip: warp w owns tile
// rows w and 7-w (9 tiles).  CTA = (snapshot, strip, dr, row split g of G);
// each chunk stages 16 rows of X (shifted by dr) and Y, 66-complex pitch
// (4 rows x 2 columns of a fragment phase hit distinct banks).  With G > 1
// the last CTA of an item (ticket counter, self-resetting) adds the G
// partial tiles in slot order — deterministic — and writes CCol.
constexpr int ECM_RC = 16;
constexpr int ECM_PITCH = 66;
constexpr int ECM_STAGES = 3;
constexpr size_t ECM_TILE = 16 * (size_t)ECM_RC * ECM_PITCH;
constexpr size_t ECM_STAGE = 2 * ECM_TILE;
constexpr size_t ECM_SMEM = ECM_STAGES * ECM_STAGE + 64;
constexpr int ECM_SLOTS = 9;
constexpr int ECM_PART = MMA_WARPS * ECM_SLOTS * 2 * 32;  // double2 per CTA partial

struct EcmItem {
  int b, side, dr, lo, hi, o;
};

__device__ __forceinline__ EcmItem ecm_item(long long item, const Problem& pr) {
  EcmItem it;
  const int span = 2 * pr.P - 1;
  it.dr = (int)(item % span) - (pr.P - 1);
  it.side = (int)((item / span) % 2);
  it.b = (int)(item / (2LL * span));
  it.lo = pr.P - 1 + min(it.dr, 0);
  it.hi = pr.N - pr.P + max(it.dr, 0);
  it.o = it.side ? pr.M - pr.Q + 1 : 0;
  return it;
}

template <int W>
__device__ __forceinline__ void ecm_consume(const unsigned char* smraw, uint64_t* full, uint64_t* empty,
                                            int nchunks, int R0, int hi, int nt, double (&p1)[ECM_SLOTS][2],
                                            double (&p2)[ECM_SLOTS][2], double (&p3)[ECM_SLOTS][2]) {
  const int lane = threadIdx.x & 31, m = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int sl = 0; sl < ECM_SLOTS; ++sl)
    p1[sl][0] = p1[sl][1] = p2[sl][0] = p2[sl][1] = p3[sl][0] = p3[sl][1] = 0.0;
  constexpr int NB = 8 - W;  // slots (W, W+sl) for sl < NB, then (7-W, 7-W + sl-NB)
  for (int k = 0; k < nchunks; ++k) {
    const int s = k % ECM_STAGES;
    mbar_wait(&full[s], (k / ECM_STAGES) & 1);
    const double2* X = reinterpret_cast<const double2*>(smraw + s * ECM_STAGE);
    const double2* Y = X + ECM_TILE / 16;
    const int R = R0 + k * ECM_RC;
#pragma unroll 1
    for (int kk = 0; kk < ECM_RC / 4; ++kk) {
      const int row = 4 * kk + kq;
      const bool on = R + row <= hi;
      double2 a0 = X[row * ECM_PITCH + 8 * W + m], a1 = X[row * ECM_PITCH + 8 * (7 - W) + m];
      if (!on) a0 = a1 = make_double2(0.0, 0.0);
      const double s0 = a0.x + a0.y, s1 = a1.x + a1.y;
      // Gauss form per slot: P1 += a.x b.x, P2 += a.y b.y, P3 += (a.x+a.y)(b.x-b.y);
      // B fragments loaded per slot (keeps registers for 2 CTAs/SM)
#pragma unroll
      for (int sl = 0; sl < ECM_SLOTS; ++sl) {
        const int tj = sl < NB ? W + sl : 7 - W + (sl - NB);
        if (tj < nt) {
          const double2 bv = Y[row * ECM_PITCH + 8 * tj + m];
          const double bd = bv.x - bv.y;
          const double2& av = sl < NB ? a0 : a1;
          const double as = sl < NB ? s0 : s1;
          dmma(p1[sl][0], p1[sl][1], av.x, bv.x);
          dmma(p2[sl][0], p2[sl][1], av.y, bv.y);
          dmma(p3[sl][0], p3[sl][1], as, bd);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

__global__ void __launch_bounds__((MMA_WARPS + 1) * 32, 2)
    k_edge_cols_dmma(const __grid_constant__ CUtensorMap tms, Problem pr, int G,
                     const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls,
                     double2* __restrict__ ccol, long long tot_ccol, double2* __restrict__ part,
                     unsigned* __restrict__ tickets, int kpart, int knparts) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + ECM_STAGES * ECM_STAGE);
  uint64_t* empty = full + ECM_STAGES;
  __shared__ int s_last;
  const long long item = blockIdx.x / G;
  const int g = (int)(blockIdx.x % G);
  const EcmItem it = ecm_item(item, pr);
  const int P = pr.P, Q = pr.Q;
  // multi-GPU row band kpart of knparts, then split g of G within it
  const int nrc_all = (it.hi - it.lo + ECM_RC) / ECM_RC;
  const int b_lo = nrc_all * kpart / knparts, nrc = nrc_all * (kpart + 1) / knparts - b_lo;
  const int c0 = b_lo + nrc * g / G, c1 = b_lo + nrc * (g + 1) / G;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ECM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MMA_WARPS);
    }
    fence_mbarrier_init();
  }
  __syncthreads();
  if (w == MMA_WARPS) {  // producer
    if (lane == 0) {
      for (int k = 0; k < c1 - c0; ++k) {
        const int s = k % ECM_STAGES;
        if (k >= ECM_STAGES) mbar_wait_sleep(&empty[s], ((k - ECM_STAGES) / ECM_STAGES) & 1);
        const int R = it.lo + (c0 + k) * ECM_RC;
        unsigned char* st = smraw + s * ECM_STAGE;
        mbar_expect_tx(&full[s], (unsigned)ECM_STAGE);
        tma_load_3d(st, &tms, 2 * it.o, R - it.dr, it.b, &full[s]);
        tma_load_3d(st + ECM_TILE, &tms, 2 * it.o, R, it.b, &full[s]);
      }
    }
    return;
  }
  const int nt = (Q - 1 + 7) / 8;
  const int R0 = it.lo + c0 * ECM_RC;
  double cr[ECM_SLOTS][2], ci[ECM_SLOTS][2];
  {
    double p1[ECM_SLOTS][2], p2[ECM_SLOTS][2], p3[ECM_SLOTS][2];
    switch (w) {
      case 0: ecm_consume<0>(smraw, full, empty, c1 - c0, R0, it.hi, nt, p1, p2, p3); break;
      case 1: ecm_consume<1>(smraw, full, empty, c1 - c0, R0, it.hi, nt, p1, p2, p3); break;
      case 2: ecm_consume<2>(smraw, full, empty, c1 - c0, R0, it.hi, nt, p1, p2, p3); break;
      default: ecm_consume<3>(smraw, full, empty, c1 - c0, R0, it.hi, nt, p1, p2, p3);
    }
#pragma unroll
    for (int sl = 0; sl < ECM_SLOTS; ++sl)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        cr[sl][e] = p1[sl][e] + p2[sl][e];
        ci[sl][e] = p3[sl][e] - p1[sl][e] + p2[sl][e];
      }
  }
  if (G > 1) {
    double2* mine = part + (item * G + g) * ECM_PART + (long long)w * ECM_SLOTS * 64;
#pragma unroll
    for (int sl = 0; sl < ECM_SLOTS; ++sl)
#pragma unroll
      for (int e = 0; e < 2; ++e) mine[(sl * 2 + e) * 32 + lane] = make_double2(cr[sl][e], ci[sl][e]);
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(MMA_WARPS * 32));
    if (threadIdx.x == 0) s_last = atomicAdd(&tickets[item], 1u) == (unsigned)(G - 1);
    asm volatile("bar.sync 1, %0;" ::"n"(MMA_WARPS * 32));
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int sl = 0; sl < ECM_SLOTS; ++sl)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double sr = 0.0, si = 0.0;
        for (int gg = 0; gg < G; ++gg) {
          const double2 v = __ldcg(part + (item * G + gg) * ECM_PART + (long long)w * ECM_SLOTS * 64 +
                                   (sl * 2 + e) * 32 + lane);
          sr += v.x;
          si += v.y;
        }
        cr[sl][e] = sr;
        ci[sl][e] = si;
      }
    if (threadIdx.x == 0) tickets[item] = 0u;  // ready for the next execute
  }
  // CCol entries: C fragment (m, 2 kq + e) of slot tile (ti, tj)
  const int m = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int sl = 0; sl < ECM_SLOTS; ++sl) {
    const int nb = 8 - w;
    const int ti = sl < nb ? w : 7 - w;
    const int tj = sl < nb ? w + sl : 7 - w + (sl - nb);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c1c = 8 * ti + m, ec = 8 * tj + 2 * kq + e;
      const int dc = ec - c1c;
      if (c1c >= Q - 1 || ec > Q - 2 || dc < 0 || !in_uc(it.dr, dc, P, Q)) continue;
      const int cid = cls_slot[class_index(it.dr, dc, P, Q)];
      if (cid < 0) continue;
      const ClassDesc& cd = cls[cid];
      const long long idx = it.side ? (long long)(cd.qu - 1) + c1c : c1c;
      ccol[(long long)it.b * tot_ccol + cd.ccol_off + idx] = make_double2(cr[sl][e], ci[sl][e]);
    }
  }
}

// ---- edge-row sums on the tensor cores ----------------------------------------
// K2's RC' (edge.cuh) for one strip (top: rows [0, P-1); bottom: [N-P+1, N))
// and one second-element row r2 of it: for every first-element row r1 of the
// strip and lag dc,
//     RC'(r1, r2, dc) = sum_{c=0}^{M-Q} x[r1, c] * conj(y[r2, c + dc])
// — a (strip rows x lags) GEMM with K = columns, A operand = the strip's
// rows (plain tile), B operand = the Toeplitz gather of row r2 (as in the
// core kernel).  The X tensor map is M-Q+1 columns wide (zero-filled beyond).
// CTA = (snapshot, strip, r2, DC-lag tile, column segment g of nseg): 4 warps
// as 2 (32 rows) x 2 (32 lags); the segment partials land in RC's nseg slots
// and the finalize adds them in order.
constexpr int ERM_XR = 64;  // strip rows per tile (P-1 <= 64)
constexpr int ERM_DC = 64;
constexpr int ERM_WM = 4, ERM_WN = 4;    // warp grid: rows x lags
constexpr int ERM_WARPS = ERM_WM * ERM_WN;
constexpr int ERM_MT = ERM_XR / 8 / ERM_WM;  // 8-row tiles per warp
constexpr int ERM_NT = ERM_DC / 8 / ERM_WN;  // 8-lag tiles per warp
constexpr int ERM_YP = MMA_W + ERM_DC;
constexpr size_t ERM_XBYTES = 16 * (size_t)ERM_XR * MMA_XP;
constexpr size_t ERM_YBYTES = 16 * (size_t)ERM_YP;
constexpr size_t ERM_STAGE = ERM_XBYTES + (ERM_YBYTES + 127) / 128 * 128;
constexpr int ERM_STAGES = 4;
constexpr size_t ERM_SMEM = ERM_STAGES * ERM_STAGE + 64;

__global__ void __launch_bounds__((ERM_WARPS + 1) * 32, 1)
    k_edge_rows_dmma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                     Problem pr, int n_dct, int nseg, const int* __restrict__ cls_slot,
                     const ClassDesc* __restrict__ cls, double2* __restrict__ rc, long long tot_rc,
                     int kpart, int knparts) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + ERM_STAGES * ERM_STAGE);
  uint64_t* empty = full + ERM_STAGES;
  const int P = pr.P, Q = pr.Q, S = P - 1;
  long long t = blockIdx.x;
  const int seg = (int)(t % nseg);
  t /= nseg;
  const int dct = (int)(t % n_dct);
  t /= n_dct;
  const int r2 = (int)(t % S);
  t /= S;
  const int strip = (int)(t % 2);
  const int b = (int)(t / 2);
  const int base = strip ? pr.bh : 0;
  const int dc0 = dct * ERM_DC;
  const int xcols = pr.M - Q + 1;
  const int ncbk = (xcols + MMA_W - 1) / MMA_W;
  // multi-GPU: segment seg belongs to part seg % knparts; the others write zeros
  const bool mine = seg % knparts == kpart;
  const int k0 = ncbk * seg / nseg, k1 = mine ? ncbk * (seg + 1) / nseg : k0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ERM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ERM_WARPS);
    }
    fence_mbarrier_init();
  }
  __syncthreads();
  if (w == ERM_WARPS) {  // producer
    if (lane == 0) {
      for (int k = 0; k < k1 - k0; ++k) {
        const int s = k % ERM_STAGES;
        if (k >= ERM_STAGES) mbar_wait_sleep(&empty[s], ((k - ERM_STAGES) / ERM_STAGES) & 1);
        const int C0 = (k0 + k) * MMA_W;
        unsigned char* st = smraw + s * ERM_STAGE;
        mbar_expect_tx(&full[s], (unsigned)(ERM_XBYTES + ERM_YBYTES));
        tma_load_3d(st, &tmx, 2 * C0, base, b, &full[s]);
        tma_load_3d(st + ERM_XBYTES, &tmy, 2 * (C0 + dc0), base + r2, b, &full[s]);
      }
    }
    return;
  }
  const int wm = w % ERM_WM, wn = w / ERM_WM, m = lane >> 2, kq = lane & 3;
  constexpr int MT = ERM_MT, NT = ERM_NT;
  double p1[MT][NT][2], p2[MT][NT][2], p3[MT][NT][2];  // Gauss form (see k_bulk_dmma3)
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
      p1[i][j][0] = p1[i][j][1] = p2[i][j][0] = p2[i][j][1] = p3[i][j][0] = p3[i][j][1] = 0.0;
  for (int k = 0; k < k1 - k0; ++k) {
    const int s = k % ERM_STAGES;
    mbar_wait(&full[s], (k / ERM_STAGES) & 1);
    const double2* X =
        reinterpret_cast<const double2*>(smraw + s * ERM_STAGE) + (8 * MT * wm + m) * MMA_XP + kq;
    const double2* Y =
        reinterpret_cast<const double2*>(smraw + s * ERM_STAGE + ERM_XBYTES) + kq + 8 * NT * wn + m;
    const int nks = min(MMA_W, xcols - (k0 + k) * MMA_W + 3) / 4;
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
      double2 a[MT], bv[NT];
      double as[MT], bd[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        a[i] = X[8 * i * MMA_XP + 4 * ks];
        as[i] = a[i].x + a[i].y;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        bv[j] = Y[8 * j + 4 * ks];
        bd[j] = bv[j].x - bv[j].y;
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(p1[i][j][0], p1[i][j][1], a[i].x, bv[j].x);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(p2[i][j][0], p2[i][j][1], a[i].y, bv[j].y);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(p3[i][j][0], p3[i][j][1], as[i], bd[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // RC' of pane row min(r1, r2) (strip-relative) of class (r2 - r1, dc)
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int r1 = 8 * MT * wm + 8 * i + m;
    if (r1 >= S) continue;
    const int dr = r2 - r1;
    const int row = min(r1, r2);
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int dc = dc0 + 8 * NT * wn + 8 * j + 2 * kq + e;
        if (dc >= Q || !in_uc(dr, dc, P, Q)) continue;
        const int cid = cls_slot[class_index(dr, dc, P, Q)];
        if (cid < 0) continue;
        const ClassDesc& cd = cls[cid];
        const int kk = strip ? cd.pv - 1 + row : row;
        rc[((long long)b * tot_rc + cd.rc_off + kk) * nseg + seg] =
            make_double2(p1[i][j][e] + p2[i][j][e], p3[i][j][e] - p1[i][j][e] + p2[i][j][e]);
      }
  }
}

// ---- K1 with 3 real GEMMs per complex GEMM (Gauss) ----------------------------
// x * conj(y) = (a + ib)(c - id) = (ac + bd) + i(bc - ad).  With
//   P1 = sum a c,  P2 = sum b d,  P3 = sum (a + b)(c - d):
//   Re = P1 + P2,  Im = P3 - P1 + P2
// — 3 DMMAs per complex 8x8x4 tile instead of 4.  The operand sums are one
// DADD per fragment — on B200 DMMA and DADD share the FP64 datapath, so with
// PREP the producer warp writes a+b / c-d for each landed stage into SMEM
// once (instead of every warp recomputing them per fragment) and the compute
// warps wait on a second per-stage barrier.  Rounding: every
// partial is a sum of products bounded by 2|x||y|, so the error stays at the
// level of the 4-multiplication form (relative Frobenius ~1e-16 at cfg5,
// tests/test_gpu_parity.py).  Same data flow as k_bulk_dmma; CTA tile DR =
// WM*MT*8 lags x DC = WN*NTW*8 lags, WM*WN compute warps of MT x NTW tiles.
template <int WM, int WN, int MT, int NTW, int MINB, bool PREP = false, int RC_ = MMA_RC>
struct Mma3Cfg {
  static constexpr int RC = RC_;  // second-element rows per chunk
  static constexpr int WARPS = WM * WN;
  static constexpr int DR = WM * MT * 8;
  static constexpr int DC = WN * NTW * 8;
  static constexpr int XR = RC + DR - 1;
  static constexpr int YP = MMA_W + DC;
  static constexpr size_t xbytes = 16 * (size_t)XR * MMA_XP;
  static constexpr size_t xoff = (xbytes + 127) / 128 * 128;
  static constexpr size_t ybytes = 16 * (size_t)RC * YP;
  static constexpr size_t yend = xoff + (ybytes + 127) / 128 * 128;
  // PREP: a+b of every X element, c-d of every Y element (doubles)
  static constexpr size_t xsoff = yend;
  static constexpr size_t ydoff = xsoff + (8 * (size_t)XR * MMA_XP + 127) / 128 * 128;
  static constexpr size_t stage = PREP ? ydoff + (8 * (size_t)RC * YP + 127) / 128 * 128 : yend;
  static constexpr int fit = (int)((227 * 1024 / MINB - 2048) / stage);
  static constexpr int S = fit > 4 ? 4 : fit;
  static constexpr size_t smem = S * stage + 128;  // + full / empty / prepped barriers
};

template <int MT, int NTW, bool MASKED, bool FULL, bool PREP, int RC>
__device__ __forceinline__ void mma3_rows(const double2* __restrict__ X, const double2* __restrict__ Y,
                                          const double* __restrict__ Xs, const double* __restrict__ Yd,
                                          int xrow0, int kq, int ycol0, int yp, int nks, int R,
                                          int dra, const Problem& pr, double (&p1)[MT][NTW][2],
                                          double (&p2)[MT][NTW][2], double (&p3)[MT][NTW][2]) {
  const int P = pr.P, N = pr.N;
#pragma unroll 1
  for (int tr = 0; tr < RC; ++tr) {
    const int xo = (tr + xrow0) * MMA_XP + kq;  // m-tile i: rows - 8 i
    const int yo = tr * yp + ycol0;
    const double2* xa = X + xo;
    const double2* yb = Y + yo;
    bool on[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      on[i] = true;
      if constexpr (MASKED) {
        const int r2 = R + tr, r1 = r2 - dra - 8 * i;
        on[i] = max(r1, r2) >= P - 1 && min(r1, r2) <= N - P;
      }
    }
    auto kstep = [&](int ks) {
      double2 a[MT], bv[NTW];
      double as[MT], bd[NTW];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        a[i] = xa[4 * ks - 8 * i * MMA_XP];
        if constexpr (PREP)
          as[i] = Xs[xo + 4 * ks - 8 * i * MMA_XP];
        else
          as[i] = a[i].x + a[i].y;
        if (MASKED && !on[i]) {
          a[i] = make_double2(0.0, 0.0);
          as[i] = 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        bv[j] = yb[4 * ks + 8 * j];
        if constexpr (PREP)
          bd[j] = Yd[yo + 4 * ks + 8 * j];
        else
          bd[j] = bv[j].x - bv[j].y;
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(p1[i][j][0], p1[i][j][1], a[i].x, bv[j].x);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(p2[i][j][0], p2[i][j][1], a[i].y, bv[j].y);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(p3[i][j][0], p3[i][j][1], as[i], bd[j]);
    };
    if constexpr (FULL) {
#pragma unroll
      for (int ks = 0; ks < MMA_W / 4; ++ks) kstep(ks);
    } else {
#pragma unroll 1
      for (int ks = 0; ks < nks; ++ks) kstep(ks);
    }
  }
}

template <int WM, int WN, int MT, int NTW, int MINB, bool PREP = false, int RC = MMA_RC>
__global__ void __launch_bounds__((WM * WN + 1) * 32, MINB)
    k_bulk_dmma3(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                 Problem pr, int n_drt, int n_dct, int G, int nclasses,
                 const int* __restrict__ cls_slot, double2* __restrict__ ccpart,
                 const unsigned* __restrict__ band_flag, unsigned band_base, int band_rows, int part,
                 int nparts) {
  // part / nparts: multi-GPU row bands — this launch covers row chunks
  // [nrc*part/nparts, nrc*(part+1)/nparts) of every tile (partial sums)
  using Cfg = Mma3Cfg<WM, WN, MT, NTW, MINB, PREP, RC>;
  constexpr int S = Cfg::S, DR = Cfg::DR, DC = Cfg::DC, NW = Cfg::WARPS;
  static_assert(S >= 2, "TMA ring needs two stages");
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + S * Cfg::stage);
  uint64_t* empty = full + S;
  uint64_t* prepped = empty + S;  // PREP: operand sums of the stage written
  long long t = blockIdx.x;
  const int p = (int)(t % G);
  t /= G;
  const int dct = (int)(t % n_dct);
  t /= n_dct;
  const int drt = (int)(t % n_drt);
  const int b = (int)(t / n_drt);
  const int P = pr.P, Q = pr.Q, N = pr.N, M = pr.M;
  const int dr0 = -(P - 1) + drt * DR;
  const int dc0 = dct * DC;
  const int drmax = min(dr0 + DR - 1, P - 1);
  const int rlo = max(0, P - 1 + min(dr0, 0));
  const int rhi = min(N - 1, N - P + max(drmax, 0));
  const int nrc_all = (rhi - rlo + RC) / RC;
  const int rc_lo = (int)((long long)nrc_all * part / nparts);
  const int nrc = (int)((long long)nrc_all * (part + 1) / nparts) - rc_lo;
  const int rbase = rlo + rc_lo * RC;  // first row of this band
  const int xcols = M - Q + 1;
  const int ncbk = (xcols + MMA_W - 1) / MMA_W;
  const long long nch = (long long)nrc * ncbk;
  const long long nmine = p < nch ? (nch - p + G - 1) / G : 0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
      mbar_init(&prepped[s], 1);
    }
    fence_mbarrier_init();
  }
  __syncthreads();

  if (w == NW && PREP) {  // producer: TMA issue + operand sums of landed stages
    auto issue = [&](long long k) {
      const int s = (int)(k % S);
      if (k >= S) mbar_wait_sleep(&empty[s], (int)(((k - S) / S) & 1));
      const long long q = p + k * G;
      const int R = rbase + (int)(q / ncbk) * RC;
      const int C0 = (int)(q % ncbk) * MMA_W;
      if (band_flag) {
        const int rneed = min(N - 1, R + RC - 1 + max(-dr0, 0));
        wait_band(band_flag, band_base + (unsigned)(rneed / band_rows) + 1u);
      }
      unsigned char* st = smraw + s * Cfg::stage;
      mbar_expect_tx(&full[s], (unsigned)(Cfg::xbytes + Cfg::ybytes));
      tma_load_3d(st, &tmx, 2 * C0, R - dr0 - (DR - 1), b, &full[s]);
      tma_load_3d(st + Cfg::xoff, &tmy, 2 * (C0 + dc0 - (Q - 1)), R, b, &full[s]);
    };
    long long issued = 0;
    if (lane == 0)
      for (; issued < nmine && issued < S - 1; ++issued) issue(issued);
    for (long long k = 0; k < nmine; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&full[s], (int)((k / S) & 1));
      const unsigned char* st = smraw + s * Cfg::stage;
      const double2* X = reinterpret_cast<const double2*>(st);
      const double2* Y = reinterpret_cast<const double2*>(st + Cfg::xoff);
      double* Xs = reinterpret_cast<double*>(smraw + s * Cfg::stage + Cfg::xsoff);
      double* Yd = reinterpret_cast<double*>(smraw + s * Cfg::stage + Cfg::ydoff);
#pragma unroll 4
      for (int i = lane; i < Cfg::XR * MMA_XP; i += 32) {
        const double2 v = X[i];
        Xs[i] = v.x + v.y;
      }
#pragma unroll 4
      for (int i = lane; i < RC * Cfg::YP; i += 32) {
        const double2 v = Y[i];
        Yd[i] = v.x - v.y;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&prepped[s]);
        if (issued < nmine) issue(issued++);  // refill (waits for the slot's consumers)
      }
      __syncwarp();
    }
    return;
  }
  if (w == NW) {  // producer
    if (lane == 0) {
      for (long long k = 0; k < nmine; ++k) {
        const int s = (int)(k % S);
        if (k >= S) mbar_wait_sleep(&empty[s], (int)(((k - S) / S) & 1));
        const long long q = p + k * G;
        const int R = rbase + (int)(q / ncbk) * RC;
        const int C0 = (int)(q % ncbk) * MMA_W;
        if (band_flag) {
          const int rneed = min(N - 1, R + RC - 1 + max(-dr0, 0));
          wait_band(band_flag, band_base + (unsigned)(rneed / band_rows) + 1u);
        }
        unsigned char* st = smraw + s * Cfg::stage;
        mbar_expect_tx(&full[s], (unsigned)(Cfg::xbytes + Cfg::ybytes));
        tma_load_3d(st, &tmx, 2 * C0, R - dr0 - (DR - 1), b, &full[s]);
        tma_load_3d(st + Cfg::xoff, &tmy, 2 * (C0 + dc0 - (Q - 1)), R, b, &full[s]);
      }
    }
    return;
  }

  const int wm = w % WM, wn = w / WM;
  const int m = lane >> 2, kq = lane & 3;
  double p1[MT][NTW][2], p2[MT][NTW][2], p3[MT][NTW][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j)
      p1[i][j][0] = p1[i][j][1] = p2[i][j][0] = p2[i][j][1] = p3[i][j][0] = p3[i][j][1] = 0.0;
  const int xrow0 = DR - 1 - MT * 8 * wm - m;
  const int ycol0 = kq + wn * NTW * 8 + m;
  const int dra = dr0 + MT * 8 * wm + m;

  for (long long k = 0; k < nmine; ++k) {
    const int s = (int)(k % S);
    if constexpr (PREP)
      mbar_wait(&prepped[s], (int)((k / S) & 1));
    else
      mbar_wait(&full[s], (int)((k / S) & 1));
    const long long q = p + k * G;
    const int R = rbase + (int)(q / ncbk) * RC;
    const int C0 = (int)(q % ncbk) * MMA_W;
    const int nks = min(MMA_W, xcols - C0 + 3) / 4;
    const double2* X = reinterpret_cast<const double2*>(smraw + s * Cfg::stage);
    const double2* Y = reinterpret_cast<const double2*>(smraw + s * Cfg::stage + Cfg::xoff);
    const double* Xs = reinterpret_cast<const double*>(smraw + s * Cfg::stage + Cfg::xsoff);
    const double* Yd = reinterpret_cast<const double*>(smraw + s * Cfg::stage + Cfg::ydoff);
    const bool masked = R < P - 1 || R + RC - 1 > N - P;
    if (nks == MMA_W / 4) {
      if (!masked)
        mma3_rows<MT, NTW, false, true, PREP, RC>(X, Y, Xs, Yd, xrow0, kq, ycol0, Cfg::YP, nks, R, dra, pr, p1,
                                              p2, p3);
      else
        mma3_rows<MT, NTW, true, true, PREP, RC>(X, Y, Xs, Yd, xrow0, kq, ycol0, Cfg::YP, nks, R, dra, pr, p1,
                                             p2, p3);
    } else {
      mma3_rows<MT, NTW, true, false, PREP, RC>(X, Y, Xs, Yd, xrow0, kq, ycol0, Cfg::YP, nks, R, dra, pr, p1,
                                            p2, p3);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int dr = dra + 8 * i;
#pragma unroll
    for (int j = 0; j < NTW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int dc = dc0 + wn * NTW * 8 + 8 * j + 2 * kq + e;
        if (dr > P - 1 || dc >= Q || !in_uc(dr, dc, P, Q)) continue;
        const int cid = cls_slot[class_index(dr, dc, P, Q)];
        if (cid < 0) continue;
        const double re = p1[i][j][e] + p2[i][j][e];
        const double im = p3[i][j][e] - p1[i][j][e] + p2[i][j][e];
        ccpart[((long long)b * nclasses + cid) * G + p] = make_double2(re, im);
      }
  }
}

}  // namespace covgpu

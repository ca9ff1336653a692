// Edge sums by blocked short-lag correlation (the default of the spectral
// engine; replaces one full-length FFT per line pair, spectral.cuh
// k_spec_ccol / k_spec_rc).
//
// Both edge families are short-lag correlations of pairs of LINES of A:
//   CCol(dr, dc)[c1] = sum_r x_c1[r] conj(y_e[r + dr])    (e = c1 + dc; lines =
//       the Q-1 columns of the left / right strip, samples along the N rows,
//       |dr| < P; x, y = the column under the two core-row masks), and
//   RC'(dr, dc) of pane row min(i1, i2) = sum_c x_i1[c] conj(a_i2[c + dc])
//       (lines = the P-1 rows of the top / bottom strip, samples along the M
//       columns, 0 <= dc < Q; x = the row masked to the slot-0 box columns
//       [0, M-Q], a = the row itself)
// (the reference forms these products one by one inside its class kernel,
// _numba_kernels.py:62-107; DESIGN.md §3 for the split into CC / CCol / RC').
//
// Only nlag << len lags are kept, so the line is cut into blocks of
// bk = Lb - nlag + 1 samples (Lb = FFT length, ~4 nlag) and each line gets two
// block spectra:
//   S_l[k] = FFT_Lb(samples [k bk, k bk + bk) under the "first element" mask, zero-padded)
//   G_l[k] = FFT_Lb(samples [k bk, k bk + Lb) under the "second element" mask)
// For lags 0 <= t < nlag no index wraps (bk - 1 + nlag - 1 < Lb), hence
//   sum_n s_i[n] conj(g_j[n + t]) = (1/Lb) FFT_Lb( sum_k S_i[k] conj(G_j[k]) )[t].
// The negative row lags of CCol come from the same two spectra with the roles
// swapped: x- / y- (spectral.cuh k_spec_colfft versions 2, 3) carry the masks
// of G / S, and sum_r x_c1[r] conj(y_e[r - t]) = conj( corr(S_e, G_c1)[t] ).
// So every ordered pair (i, j) of one strip's lines is one accumulation over
// the blocks plus one FFT of length Lb: cfg5 7938 pairs x (11 blocks x 256
// frequencies) = 2.2e7 complex MACs and 7938 FFT-256 per edge family, against
// 7938 FFT-2048 of 2 x 2048 operand loads each before.
//
// k_eb_spec: one FFT per (snapshot, strip, type, line, block).
// k_eb_pairs: CTA = (snapshot, strip, TI x TJ tile of ordered line pairs),
// thread = frequency: the tile's TI S-values and TJ G-values of a block feed
// TI TJ accumulators (each operand is read once per tile, coalesced); the
// tile's cross spectra go through SMEM to NP / 8 rounds of 8 concurrent FFTs,
// whose first nlag outputs are stored straight into CCol / RC'.
// Every sum runs in a fixed order (blocks ascending): bitwise reproducible;
// a pair's value does not depend on the tiling, the batch or the part split.
#pragma once

#include "spectral.cuh"

namespace covgpu {

struct EbGeom {
  int logLb, bk, nblk;  // FFT length 2^logLb, samples per short block, blocks per line
  int nlines;           // lines per strip (Q-1 columns / P-1 rows)
  int len;              // samples per line (N / M)
  int s_hi;             // short type: samples n <= s_hi are kept
  int g_lo;             // long type: samples n >= g_lo are kept
  int nlag;             // lags kept (P / Q)
};

// FFT length for nlag lags: ~4 nlag (3/4 of every transform is new samples), 64 .. 512
inline int eb_logLb(int nlag) {
  int lg = 6;
  while ((1 << lg) < 4 * nlag && lg < 9) ++lg;
  return lg;
}
inline EbGeom eb_geom(int nlag, int nlines, int len, int s_hi, int g_lo) {
  EbGeom g;
  g.logLb = eb_logLb(nlag);
  g.bk = (1 << g.logLb) - nlag + 1;
  g.nblk = (len + g.bk - 1) / g.bk;
  g.nlines = nlines;
  g.len = len;
  g.s_hi = s_hi;
  g.g_lo = g_lo;
  g.nlag = nlag;
  return g;
}
// block spectra of one snapshot: [strip 0/1][type S/G][line][block][Lb]
inline size_t eb_spec_elems(const EbGeom& g) { return (size_t)4 * g.nlines * g.nblk << g.logLb; }

template <typename T, int LOGLB>
__global__ void __launch_bounds__(spec_threads<LOGLB>())
    k_eb_spec(long long nitems, const typename CT<T>::c* __restrict__ A, Problem pr, EbGeom g, int cols,
              const double2* __restrict__ tw, double2* __restrict__ SP) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGLB;
  double2* sb;
  const SpecItem si = spec_item<LOGLB>(nitems, sb, sbuf);
  // the line varies fastest: the transforms of one CTA read neighbouring
  // columns of the same rows (column strips)
  long long t = si.item;
  const int line = (int)(t % g.nlines);
  t /= g.nlines;
  const int blk = (int)(t % g.nblk);
  t /= g.nblk;
  const int type = (int)(t % 2);
  t /= 2;
  const int strip = (int)(t % 2);
  const long long b = t / 2;
  const int n0 = blk * g.bk;
  const int cnt = type ? L : g.bk;
  const int lo = type ? g.g_lo : 0, hi = type ? g.len - 1 : g.s_hi;
  const typename CT<T>::c* base;
  long long stride;
  if (cols) {
    base = A + b * pr.N * (long long)pr.M + (strip ? pr.M - pr.Q + 1 + line : line);
    stride = pr.M;
  } else {
    base = A + (b * pr.N + (strip ? pr.N - (pr.P - 1) + line : line)) * (long long)pr.M;
    stride = 1;
  }
  double2* out = SP + (((((b * 2 + strip) * 2 + type) * g.nlines + line) * g.nblk + blk) << LOGLB);
  const bool ok = si.valid;
  spec_fft_block<LOGLB>(
      sb, si.tl, tw,
      [&](int idx) {
        const int n = n0 + idx;
        return (ok && idx < cnt && n >= lo && n <= hi) ? widen2(base[n * stride]) : make_double2(0.0, 0.0);
      },
      [&](int idx, double2 v) {
        if (ok) out[idx] = v;
      });
}

template <int LOGLB>
struct EbTile {  // 16 pairs per CTA (8 for the 512-thread length: registers)
  static constexpr int TI = 4, TJ = LOGLB >= 9 ? 2 : 4;
};
template <int LOGLB>
__host__ __device__ constexpr size_t eb_pairs_smem() {
  return sizeof(double2) * ((size_t)EbTile<LOGLB>::TI * EbTile<LOGLB>::TJ * (1 << LOGLB) + 8 * spec_sb_elems<LOGLB>());
}

// cols = 1: CCol of the column strips; cols = 0: RC' of the row strips.
// Multi-GPU row bands: tile t belongs to part t mod nparts and only the
// part's tiles are launched (the caller zeroes dst first; the parts are summed).
template <int LOGLB>
__global__ void __launch_bounds__(1 << LOGLB)
    k_eb_pairs(const double2* __restrict__ SP, Problem pr, EbGeom g, int cols, const double2* __restrict__ tw,
               const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls, double2* __restrict__ dst,
               long long tot, int part, int nparts, long long ntiles) {
  constexpr int L = 1 << LOGLB, TI = EbTile<LOGLB>::TI, TJ = EbTile<LOGLB>::TJ, NP = TI * TJ, NT = L / 8;
  static_assert(NP % 8 == 0, "whole rounds of 8 transforms");
  extern __shared__ double2 sbuf[];
  double2* const Z = sbuf;
  long long tile = (long long)blockIdx.x * nparts + part;
  if (tile >= ntiles) return;
  const int nti = (g.nlines + TI - 1) / TI, ntj = (g.nlines + TJ - 1) / TJ;
  const int tj = (int)(tile % ntj);
  tile /= ntj;
  const int ti = (int)(tile % nti);
  tile /= nti;
  const int strip = (int)(tile % 2);
  const long long b = tile / 2;
  const int f = threadIdx.x;
  const long long lstride = (long long)g.nblk << LOGLB;  // next line
  const double2* sS = SP + ((b * 2 + strip) * 2 + 0) * g.nlines * lstride + f;
  const double2* sG = SP + ((b * 2 + strip) * 2 + 1) * g.nlines * lstride + f;
  const int i0 = ti * TI, j0 = tj * TJ;
  double2 acc[TI][TJ];
#pragma unroll
  for (int a = 0; a < TI; ++a)
#pragma unroll
    for (int c = 0; c < TJ; ++c) acc[a][c] = make_double2(0.0, 0.0);
#pragma unroll 2
  for (int k = 0; k < g.nblk; ++k) {
    double2 s[TI], y[TJ];
#pragma unroll
    for (int a = 0; a < TI; ++a)
      s[a] = i0 + a < g.nlines ? sS[(i0 + a) * lstride + ((long long)k << LOGLB)] : make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < TJ; ++c)
      y[c] = j0 + c < g.nlines ? sG[(j0 + c) * lstride + ((long long)k << LOGLB)] : make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < TI; ++a)
#pragma unroll
      for (int c = 0; c < TJ; ++c) {  // += s conj(y)
        acc[a][c].x = fma(s[a].x, y[c].x, acc[a][c].x);
        acc[a][c].x = fma(s[a].y, y[c].y, acc[a][c].x);
        acc[a][c].y = fma(s[a].y, y[c].x, acc[a][c].y);
        acc[a][c].y = fma(-s[a].x, y[c].y, acc[a][c].y);
      }
  }
#pragma unroll
  for (int a = 0; a < TI; ++a)
#pragma unroll
    for (int c = 0; c < TJ; ++c) Z[(a * TJ + c) * L + f] = acc[a][c];
  __syncthreads();
  const int grp = threadIdx.x / NT, tl = threadIdx.x % NT;
  double2* const sb = sbuf + NP * L + grp * spec_sb_elems<LOGLB>();
  const int P = pr.P, Q = pr.Q;
  const double inv = 1.0 / (double)L;
  for (int round = 0; round < NP / 8; ++round) {
    const int pi = round * 8 + grp;
    const int i = i0 + pi / TJ, j = j0 + pi % TJ;  // S line i, G line j
    const bool valid = i < g.nlines && j < g.nlines;
    const double2* z = Z + pi * L;
    spec_fft_block<LOGLB>(
        sb, tl, tw, [&](int idx) { return z[idx]; },
        [&](int idx, double2 v) {
          if (!valid || idx >= g.nlag) return;
          int dr, dc, pos;
          double2 val = make_double2(v.x * inv, v.y * inv);
          if (cols) {
            if (i <= j) {  // (c1, e) = (i, j), row lag +idx
              dr = idx;
              dc = j - i;
              pos = i;
            } else {  // (c1, e) = (j, i), row lag -idx: the conjugate of corr(S_e, G_c1)
              if (idx == 0) return;
              dr = -idx;
              dc = i - j;
              pos = j;
              val.y = -val.y;
            }
          } else {  // strip rows (i1, i2) = (i, j), column lag idx
            dr = j - i;
            dc = idx;
            pos = min(i, j);
          }
          if (!in_uc(dr, dc, P, Q)) return;
          const int cid = cls_slot[class_index(dr, dc, P, Q)];
          if (cid < 0) return;
          const ClassDesc& cd = cls[cid];
          const long long o = cols ? cd.ccol_off + (strip ? (cd.qu - 1) + pos : pos)
                                   : cd.rc_off + (strip ? (cd.pv - 1) + pos : pos);
          dst[b * tot + o] = val;
        });
  }
}

}  // namespace covgpu

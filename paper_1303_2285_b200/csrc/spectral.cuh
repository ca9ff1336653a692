// K1 in the frequency domain — the core sums CC(dr, dc) of every class at
// once through FFTs along A's rows (FP64 arithmetic; complex128 or complex64
// inputs).
//
// With x_r = row r of A restricted to the core first-element columns
// c <= M-Q and y_r = row r restricted to the core second-element columns
// c' >= Q-1 (the two position-only core-column masks of DESIGN.md §3),
//     CC(dr, dc) = sum_{r2 in rows(dr)} sum_c x_{r2-dr}[c] conj(y_{r2}[c+dc]),
// rows(dr) = [P-1, N-P+dr] for dr >= 0 and [P-1+dr, N-P] for dr < 0 (the core
// rows).  For an FFT length L >= M (power of two) no circular wrap occurs
// (c + dc <= M-1 < L), so with X_r = FFT_L(x_r), Y_r = FFT_L(y_r),
// w = exp(-2 pi i / L):
//     sum_c x_a[c] conj(y_b[c+dc]) = (1/L) sum_f X_a[f] conj(Y_b[f]) w^(f dc)
// and therefore
//     G(dr, f)   = sum_{r2 in rows(dr)} X_{r2-dr}[f] conj(Y_{r2}[f])     (k_spec_corr)
//     CC(dr, dc) = (1/L) sum_f G(dr, f) w^(f dc)                         (k_spec_dft)
// — the row-lag correlation is done per frequency, the column lags by one
// short DFT per row lag.  Cost: 2N row FFTs (k_spec_fft) + (2P-1) L N complex
// MACs + (2P-1) Q L for the DFT: cfg5 5.3e8 MACs against 3.1e10 core products
// for the direct sums (mma.cuh).
//
// Accuracy: the FFT rounds at ~eps log2(L) of the row energy.  For dr != 0
// the sum over r2 is incoherent and CC keeps ~1e-14 relative accuracy on
// white noise; for dr = 0 the terms X_r conj(Y_r) are coherent (|X_r|^2 for
// the shared columns), so the dr = 0 classes are transformed row by row and
// summed over rows in the space domain (k_spec_rowac).
// Every sum runs in a fixed order: results are bitwise reproducible.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace covgpu {

constexpr int SPEC_E = 16;        // row lags per k_spec_corr thread
constexpr int SPEC_CW = 4;        // warps (32-frequency columns) per k_spec_corr CTA
constexpr int SPEC_MAX_Q = 512;   // edge-column pairs grow as Q^2
#ifndef SPEC_CTA_THREADS
#define SPEC_CTA_THREADS 256        // FFT kernels: transforms per CTA up to this many threads
#endif

template <typename C2>
__device__ __forceinline__ double2 widen2(C2 v) {
  return make_double2((double)v.x, (double)v.y);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// In-register R-point forward DFTs (w = exp(-2 pi i / R)).
__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // a * (-i)

template <int R>
__device__ __forceinline__ void dft_small(double2* u);
template <>
__device__ __forceinline__ void dft_small<2>(double2* u) {
  const double2 a = u[0], b = u[1];
  u[0] = cadd2(a, b);
  u[1] = csub2(a, b);
}
template <>
__device__ __forceinline__ void dft_small<4>(double2* u) {
  const double2 t0 = cadd2(u[0], u[2]), t1 = csub2(u[0], u[2]);
  const double2 t2 = cadd2(u[1], u[3]), t3 = mul_mi(csub2(u[1], u[3]));
  u[0] = cadd2(t0, t2);
  u[2] = csub2(t0, t2);
  u[1] = cadd2(t1, t3);
  u[3] = csub2(t1, t3);
}
template <>
__device__ __forceinline__ void dft_small<8>(double2* u) {
  constexpr double c = 0.70710678118654752440;  // sqrt(1/2)
  double2 e[4] = {u[0], u[2], u[4], u[6]}, o[4] = {u[1], u[3], u[5], u[7]};
  dft_small<4>(e);
  dft_small<4>(o);
  // o[k] *= w8^k: w8 = (c, -c), w8^2 = -i, w8^3 = (-c, -c)
  const double2 o1 = make_double2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
  const double2 o2 = mul_mi(o[2]);
  const double2 o3 = make_double2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
  u[0] = cadd2(e[0], o[0]);
  u[4] = csub2(e[0], o[0]);
  u[1] = cadd2(e[1], o1);
  u[5] = csub2(e[1], o1);
  u[2] = cadd2(e[2], o2);
  u[6] = csub2(e[2], o2);
  u[3] = cadd2(e[3], o3);
  u[7] = csub2(e[3], o3);
}

// SMEM index with one pad element per 8: the strided Stockham stores hit
// distinct 16-byte bank groups
__device__ __forceinline__ int fpad(int i) { return i + (i >> 3); }

// Twiddle table, pass-major: for each pass after the first (p = product of
// the earlier radices, radix R) the entries w_{pR}^(r k), r in [1, R),
// k in [0, p), at [(r-1) p + k] — consecutive lanes (consecutive k) read
// consecutive entries.  spec_tw_off(logL, p) = offset of the pass; the same
// walk builds the table on the host (spec_twiddles).
__host__ __device__ constexpr int spec_tw_off(int logL, int P0) {
  int off = 0, p = 1, rem = logL;
  while (p < P0) {
    const int lr = rem >= 3 ? 3 : rem;
    if (p > 1) off += ((1 << lr) - 1) * p;
    p <<= lr;
    rem -= lr;
  }
  return off;
}

// One radix-R Stockham pass (autosort, no bit reversal): item i of L/R,
// k = i mod p (p = product of the radices already applied):
//     u_r = in[i + r L/R] * w_L^(r k L/(pR)),  DFT_R(u),  out[(i - k) R + k + r p] = u_r.
// One transform per group of L/8 threads (tl = thread in the group, sb = the
// group's SMEM), so a thread holds at most 8 values; in place in SMEM with a
// CTA barrier between the reads and the writes (every group of the CTA runs
// the same pass sequence).  The first pass reads its input through `ld(idx)`
// (global memory, coalesced), the last pass hands the natural-order spectrum
// to `st(idx, v)`.
template <int LOGL>
__host__ __device__ constexpr int spec_nt() {  // threads per transform
  return (1 << LOGL) / 8;
}
template <int LOGL>
__host__ __device__ constexpr int spec_g() {  // transforms per CTA: >= 256 threads for short lengths
  return spec_nt<LOGL>() >= SPEC_CTA_THREADS ? 1 : SPEC_CTA_THREADS / spec_nt<LOGL>();
}
template <int LOGL>
__host__ __device__ constexpr int spec_threads() {
  return spec_nt<LOGL>() * spec_g<LOGL>();
}
template <int LOGL>
__host__ __device__ constexpr int spec_sb_elems() {  // SMEM complex values per transform (one pad per 8)
  return (1 << LOGL) + (1 << LOGL) / 8;
}

template <int LOGL, int R, int P0, class Load, class Store>
__device__ __forceinline__ void spec_pass(double2* sb, int tl, const double2* __restrict__ tw, const Load& ld,
                                          const Store& st) {
  constexpr int L = 1 << LOGL, T = L / R, NTHR = spec_nt<LOGL>();
  constexpr int IPT = (T + NTHR - 1) / NTHR;
  constexpr bool first = P0 == 1, last = P0 * R == L;
  double2 u[IPT][R];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int i = tl + it * NTHR;
    if (i < T) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int idx = i + r * T;
        if constexpr (first)
          u[it][r] = ld(idx);
        else
          u[it][r] = sb[fpad(idx)];
      }
    }
  }
  if constexpr (!first) __syncthreads();
  const double2* __restrict__ twp = tw + spec_tw_off(LOGL, P0);
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int i = tl + it * NTHR;
    if (i < T) {
      const int k = i & (P0 - 1);
      if (k) {
        // w^(rk) for r = 1..R-1 from at most two table reads (w^k, w^4k) and
        // products of depth <= 2: fewer L1 wavefronts (the FFT kernels are
        // LSU-bound), twiddle error <= ~3 ulp
        double2 w[R];
        w[1] = twp[k];
        if constexpr (R >= 4) {
          w[2] = cmul(w[1], w[1]);
          w[3] = cmul(w[2], w[1]);
        }
        if constexpr (R == 8) {
          w[4] = twp[3 * P0 + k];
          w[5] = cmul(w[4], w[1]);
          w[6] = cmul(w[4], w[2]);
          w[7] = cmul(w[4], w[3]);
        }
#pragma unroll
        for (int r = 1; r < R; ++r) u[it][r] = cmul(u[it][r], w[r]);
      }
      dft_small<R>(u[it]);
      const int j = i * R - k * (R - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int idx = j + r * P0;
        if constexpr (last)
          st(idx, u[it][r]);
        else
          sb[fpad(idx)] = u[it][r];
      }
    }
  }
  if constexpr (!last) __syncthreads();
}

// The whole forward FFT of length 2^LOGL: radix-8 passes, then one radix-4 /
// radix-2 pass.  tw = the pass-major twiddle table (spec_tw_off).
template <int LOGL, int P0 = 1, class Load, class Store>
__device__ __forceinline__ void spec_fft_block(double2* sb, int tl, const double2* __restrict__ tw, const Load& ld,
                                               const Store& st) {
  constexpr int done = P0 == 1 ? 0 : __builtin_ctz(P0);
  constexpr int rem = LOGL - done;
  if constexpr (rem > 0) {
    constexpr int lr = rem >= 3 ? 3 : rem;
    spec_pass<LOGL, (1 << lr), P0>(sb, tl, tw, ld, st);
    spec_fft_block<LOGL, (P0 << lr)>(sb, tl, tw, ld, st);
  }
}

// Output-pruned transform for the kernels that keep only the first NOUT = 64
// outputs (edge sums, dr = 0 rows, output FFT: Q, P <= 64).  With
// n = m + (L/64) n', the two radix-8 passes leave V_m[k] = sum_n' u[m + (L/64) n']
// w_64^(n' k) at SMEM position 64 m + k (Stockham layout), and
//     out[k] = sum_{m < L/64} w_L^(m k) V_m[k],   k < 64,
// replaces the remaining passes (L = 2048: 2 of 4 SMEM round trips, 30 % of
// the butterflies).  Thread (k, q) sums a contiguous quarter of the m in order
// (twiddles from the full table, then a depth <= L/256 recurrence), the
// quarters are added in a fixed order.  twf[j] = w_L^j (host-made).
constexpr int SPEC_LOGOUT = 6;

template <int LOGL, int P0, int LOGSTOP, class Load, class Store>
__device__ __forceinline__ void spec_passes_upto(double2* sb, int tl, const double2* __restrict__ tw,
                                                 const Load& ld, const Store& st) {
  constexpr int done = P0 == 1 ? 0 : __builtin_ctz(P0);
  if constexpr (done < LOGSTOP) {
    constexpr int lr = (LOGL - done) >= 3 ? 3 : (LOGL - done);
    static_assert(done + lr <= LOGSTOP, "pruned FFT: the radix-8 passes must land on 2^LOGSTOP");
    spec_pass<LOGL, (1 << lr), P0>(sb, tl, tw, ld, st);
    spec_passes_upto<LOGL, (P0 << lr), LOGSTOP>(sb, tl, tw, ld, st);
  }
}

template <int LOGL, class Load, class Store>
__device__ __forceinline__ void spec_fft_pruned(double2* sb, int tl, const double2* __restrict__ tw,
                                                const double2* __restrict__ twf, const Load& ld, const Store& st) {
  constexpr int L = 1 << LOGL, NOUT = 1 << SPEC_LOGOUT, M1 = L / NOUT;
  constexpr int NT = spec_nt<LOGL>(), NQ = NT / NOUT;
  static_assert(LOGL >= SPEC_LOGOUT + 3 && NQ >= 1, "pruned FFT needs L >= 8 NOUT");
  spec_passes_upto<LOGL, 1, SPEC_LOGOUT>(sb, tl, tw, ld, [](int, double2) {});
  const int k = tl % NOUT, q = tl / NOUT;
  constexpr int MQ = M1 / NQ;
  double2 acc = make_double2(0.0, 0.0);
  {
    const int m0 = q * MQ;
    double2 w = twf[(m0 * k) & (L - 1)];
    const double2 step = twf[k];
#pragma unroll 4
    for (int m = m0; m < m0 + MQ; ++m) {
      acc = cadd(acc, cmul(sb[fpad(m * NOUT + k)], w));
      w = cmul(w, step);
    }
  }
  if constexpr (NQ > 1) {
    __syncthreads();  // every V read
    sb[tl] = acc;
    __syncthreads();
    if (q == 0) {
      double2 s = sb[k];
#pragma unroll
      for (int qq = 1; qq < NQ; ++qq) s = cadd(s, sb[k + qq * NOUT]);
      st(k, s);
    }
  } else {
    st(k, acc);
  }
}

// This thread's transform: item = CTA * G + group (valid < nitems), tl, SMEM
struct SpecItem {
  long long item;
  int tl;
  bool valid;
};
template <int LOGL>
__device__ __forceinline__ SpecItem spec_item(long long nitems, double2*& sb, double2* sbuf) {
  SpecItem it;
  const int grp = threadIdx.x / spec_nt<LOGL>();
  it.tl = threadIdx.x % spec_nt<LOGL>();
  it.item = (long long)blockIdx.x * spec_g<LOGL>() + grp;
  it.valid = it.item < nitems;
  if (!it.valid) it.item = nitems - 1;  // keep the index math in range; loads / stores are skipped
  sb = sbuf + grp * spec_sb_elems<LOGL>();
  return it;
}

// Row spectra X_r, Y_r live f-block-major: [b][f / 32][PADR + r][f % 32],
// with PADR zero rows above and below every block (never written), so that
// a run of rows of one 32-frequency block is one contiguous bulk copy.
struct SpecLayout {
  int nfb;   // 32-frequency blocks (L / 32)
  int padr;  // zero rows above and below
  int np;    // rows per block: N + 2 padr
  __host__ __device__ long long at(long long b, int r, int f) const {
    return ((b * nfb + (f >> 5)) * np + padr + r) * 32LL + (f & 31);
  }
};

// Row FFTs.  mode 0: CTA = (snapshot b, row r, which): which 0 -> X_r
// (columns c <= M-Q), 1 -> Y_r (columns c >= Q-1).  mode 1 (edge rows):
// CTA = (b, strip row s of 2(P-1)) -> Y0_s, the unmasked row of the top
// strip [0, P-1) / bottom strip [N-P+1, N).  Zero-padded to L = 2^LOGL.
// mode 2 (symmetric core sums): CTA = (b, row r) -> X_r only, the row under
// ONE mask for both elements, the core columns [Q-1, M-Q].  mode 3 (the
// strips' correction of the symmetric sums): "snapshot" 2 b + s = strip s of
// snapshot b, the first (s = 0) / last (s = 1) 2Q-2 columns of the row at
// positions [0, 2Q-2); which 0 -> the strip's first-element columns
// [0, Q-1), which 1 -> its second-element columns [Q-1, 2Q-2).
template <typename T, int LOGL>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_fft(long long nitems, const typename CT<T>::c* __restrict__ A, Problem pr, int mode, SpecLayout lay,
               const double2* __restrict__ tw, double2* __restrict__ FX, double2* __restrict__ FY, int row0,
               int nrows) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  long long t = si.item;
  const int N = pr.N, M = pr.M, Q = pr.Q, S = pr.P - 1;
  int r, clo, chi;
  long long orow;
  double2* out;
  int which = 0, strip = 0;
  if (mode == 0 || mode == 3) {  // rows [row0, row0 + nrows)
    which = (int)(t & 1);
    t >>= 1;
    r = row0 + (int)(t % nrows);
    const long long b = t / nrows;  // (mode 3: 2 snapshot + strip)
    clo = which ? Q - 1 : 0;
    chi = which ? M - 1 : M - Q;
    strip = (int)(b & 1);
    orow = (mode == 3 ? b >> 1 : b) * N + r;
    out = (which ? FY : FX) + lay.at(b, r, 0);
  } else if (mode == 2) {
    r = row0 + (int)(t % nrows);
    const long long b = t / nrows;
    clo = Q - 1;
    chi = M - Q;
    orow = b * N + r;
    out = FX + lay.at(b, r, 0);
  } else {
    const int sr = (int)(t % (2 * S));
    const long long b = t / (2 * S);
    r = sr < S ? sr : N - S + (sr - S);
    clo = 0;
    chi = M - 1;
    orow = b * N + r;
    out = FY + (b * 2 * S + sr) * (long long)L;  // row-major (mode 1 stride: 32 per block)
  }
  const typename CT<T>::c* row = A + orow * (long long)M;
  const long long fstride = mode != 1 ? (long long)lay.np * 32 : 32;  // next 32-frequency block
  const bool ok = si.valid;
  const int W2 = 2 * Q - 2;
  spec_fft_block<LOGL>(
      sb, si.tl, tw,
      [&](int idx) {
        if (mode == 3) {
          const bool in = ok && idx < W2 && (which ? idx >= Q - 1 : idx < Q - 1);
          return in ? widen2(row[strip ? M - W2 + idx : idx]) : make_double2(0.0, 0.0);
        }
        return (ok && idx >= clo && idx <= chi) ? widen2(row[idx]) : make_double2(0.0, 0.0);
      },
      [&](int idx, double2 v) {
        if (ok) out[(idx >> 5) * fstride + (idx & 31)] = v;
      });
}

// Column FFTs of the edge-column strips (left: columns [0, Q-1), right:
// [M-Q+1, M)), four row-masked versions each: v0 x+ = rows [0, N-P],
// v1 y+ = rows [P-1, N-1] (row lags dr >= 0), v2 x- = rows [P-1, N-1],
// v3 y- = rows [0, N-P] (dr < 0).  CTA = (b, side, version, strip column j);
// FC[((b*2 + side)*4 + v)*(Q-1) + j][0 .. Lr).
template <typename T, int LOGL>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_colfft(long long nitems, const typename CT<T>::c* __restrict__ A, Problem pr,
                  const double2* __restrict__ tw, double2* __restrict__ FC) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  const int N = pr.N, M = pr.M, P = pr.P, Q = pr.Q;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  long long t = si.item;
  const int j = (int)(t % (Q - 1));
  t /= Q - 1;
  const int v = (int)(t % 4);
  t /= 4;
  const int side = (int)(t % 2);
  const long long b = t / 2;
  const int col = side ? M - Q + 1 + j : j;
  const int rlo = (v == 1 || v == 2) ? P - 1 : 0;
  const int rhi = (v == 1 || v == 2) ? N - 1 : N - P;
  const typename CT<T>::c* base = A + b * N * (long long)M + col;
  double2* out = FC + (((b * 2 + side) * 4 + v) * (Q - 1) + j) * (long long)L;
  const bool ok = si.valid;
  spec_fft_block<LOGL>(
      sb, si.tl, tw,
      [&](int idx) {
        return (ok && idx >= rlo && idx <= rhi) ? widen2(base[(long long)idx * M]) : make_double2(0.0, 0.0);
      },
      [&](int idx, double2 v2) {
        if (ok) out[idx] = v2;
      });
}

// Edge-column sums CCol from the column spectra: for strip side, sign and
// column pair (c1, e = c1 + dc), e <= Q-2,
//     CCol(dr, dc)[c1] = (1/Lr) sum_f Xc1[f] conj(Ye[f]) w^(f dr),
// dr in [0, P) from the + versions (index dr), dr in (-P, 0) from the -
// versions (index Lr + dr).  CTA = (b, side, sign, c1, e); pairs with e < c1
// (and e == c1 for sign -) exit; in multi-GPU row-band mode item g belongs
// to part g mod nparts, and only the part's items are launched (the caller
// zeroes CCol first: the parts are summed).
template <int LOGL, bool PRUNE = false>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_ccol(long long nitems, const double2* __restrict__ FC, Problem pr, const double2* __restrict__ tw,
                const double2* __restrict__ twf,
                const int* __restrict__ cls_slot, const ClassDesc* __restrict__ cls, double2* __restrict__ ccol,
                long long tot_ccol, int part, int nparts, long long total) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  const int P = pr.P, Q = pr.Q, S1 = Q - 1;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  long long g = si.item * nparts + part;  // this part's items: g = part (mod nparts)
  const bool own = si.valid && g < total;
  if (!own) g = total - 1;                 // (index math in range; loads / stores skipped)
  // item = (b, side, pair q): sign 0 pairs e >= c1 first, then sign 1 pairs e > c1
  const long long np0 = (long long)S1 * (S1 + 1) / 2, np1 = (long long)S1 * (S1 - 1) / 2;
  long long q = g % (np0 + np1);
  const long long bs = g / (np0 + np1);
  const int side = (int)(bs % 2);
  const long long b = bs / 2;
  const int sign = q < np0 ? 0 : 1;
  if (sign) q -= np0;
  int c1 = 0;
  for (;;) {
    const int cnt = S1 - c1 - sign;
    if (q < cnt) break;
    q -= cnt;
    ++c1;
  }
  const int e = c1 + sign + (int)q;
  const int dc = e - c1;
  const bool mine = own;
  const double2* fx = FC + (((b * 2 + side) * 4 + 2 * sign) * S1 + c1) * (long long)L;
  const double2* fy = FC + (((b * 2 + side) * 4 + 2 * sign + 1) * S1 + e) * (long long)L;
  const double inv = 1.0 / (double)L;
  // CCol of class (dr, dc) at strip column c1 (zero where this part does not own the pair)
  auto emit = [&](int dr, double2 v) {
    if (!in_uc(dr, dc, P, Q)) return;
    const int cid = cls_slot[class_index(dr, dc, P, Q)];
    if (cid < 0) return;
    const ClassDesc& cd = cls[cid];
    const long long o = side ? (long long)(cd.qu - 1) + c1 : c1;
    ccol[b * tot_ccol + cd.ccol_off + o] = v;
  };
  // the last pass hands over the natural-order outputs: only the P row lags
  // of this sign are kept, stored straight to CCol (no SMEM round trip)
  if constexpr (PRUNE) {
    // lags dr < 0 sit at the top of the spectrum (L + dr): transform the
    // conjugate product and conjugate the first outputs instead
    spec_fft_pruned<LOGL>(
        sb, si.tl, tw, twf,
        [&](int idx) {
          if (!mine) return make_double2(0.0, 0.0);
          const double2 x = fx[idx], y = fy[idx];
          const double re = fma(x.x, y.x, x.y * y.y), im = fma(x.y, y.x, -x.x * y.y);  // x conj(y)
          return make_double2(re, sign ? -im : im);
        },
        [&](int idx, double2 v) {
          if (!mine || idx >= P) return;
          if (sign == 0)
            emit(idx, make_double2(v.x * inv, v.y * inv));
          else if (idx > 0)
            emit(-idx, make_double2(v.x * inv, -v.y * inv));
        });
  } else {
    spec_fft_block<LOGL>(
        sb, si.tl, tw,
        [&](int idx) {
          if (!mine) return make_double2(0.0, 0.0);
          const double2 x = fx[idx], y = fy[idx];
          return make_double2(fma(x.x, y.x, x.y * y.y), fma(x.y, y.x, -x.x * y.y));  // x conj(y)
        },
        [&](int idx, double2 v) {
          const int dr = sign ? idx - L : idx;
          if (mine && ((sign == 0 && idx < P) || (sign == 1 && dr > -P)))
            emit(dr, make_double2(v.x * inv, v.y * inv));
        });
  }
}

// Edge-row sums RC' from the row spectra: for strip rows (i1, i2) (first
// element row base + i1, second base + i2, dr = i2 - i1),
//     RC'(dr, dc) of pane row min(i1, i2) = (1/L) sum_f X_{base+i1}[f] conj(Y0_{i2}[f]) w^(f dc)
// (X masked to the slot-0 box columns [0, M-Q], Y0 unmasked).  CTA = (b,
// strip, i1, i2); multi-GPU: item g belongs to part g mod nparts, only the
// part's items are launched (the caller zeroes RC' first).  RC' has one
// segment here (nseg = 1).
template <int LOGL, bool PRUNE = false>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_rc(long long nitems, const double2* __restrict__ FX, const double2* __restrict__ FY0, Problem pr,
              SpecLayout lay, const double2* __restrict__ tw, const double2* __restrict__ twf, const int* __restrict__ cls_slot,
              const ClassDesc* __restrict__ cls, double2* __restrict__ rc, long long tot_rc, int part, int nparts,
              long long total) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  const int N = pr.N, P = pr.P, Q = pr.Q, S = P - 1;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  long long g = si.item * nparts + part;
  const bool own = si.valid && g < total;
  if (!own) g = total - 1;
  long long t = g;
  const int i2 = (int)(t % S);
  t /= S;
  const int i1 = (int)(t % S);
  t /= S;
  const int strip = (int)(t % 2);
  const long long b = t / 2;
  const int dr = i2 - i1;
  const int base = strip ? N - S : 0;
  const bool mine = own;
  const double2* fx = FX + lay.at(b, base + i1, 0);
  const long long fxs = (long long)lay.np * 32;
  const double2* fy = FY0 + (b * 2 * S + strip * S + i2) * (long long)L;
  const double inv = 1.0 / (double)L;
  const int i = min(i1, i2);
  auto emit = [&](int dc, double2 v) {
    if (!in_uc(dr, dc, P, Q)) return;
    const int cid = cls_slot[class_index(dr, dc, P, Q)];
    if (cid < 0) return;
    const ClassDesc& cd = cls[cid];
    const int k = strip ? (cd.pv - 1) + i : i;
    rc[b * tot_rc + cd.rc_off + k] = v;
  };
  auto ld = [&](int idx) {
    if (!mine) return make_double2(0.0, 0.0);
    const double2 x = fx[(idx >> 5) * fxs + (idx & 31)], y = fy[idx];
    return make_double2(fma(x.x, y.x, x.y * y.y), fma(x.y, y.x, -x.x * y.y));
  };
  auto stf = [&](int idx, double2 v) {
    if (mine && idx < Q) emit(idx, make_double2(v.x * inv, v.y * inv));  // outputs dc < Q only
  };
  if constexpr (PRUNE)
    spec_fft_pruned<LOGL>(sb, si.tl, tw, twf, ld, stf);
  else
    spec_fft_block<LOGL>(sb, si.tl, tw, ld, stf);
}

__device__ __forceinline__ int spec_lo(int dr, int P) { return P - 1 + min(dr, 0); }
__device__ __forceinline__ int spec_hi(int dr, int P, int N) { return N - P + max(dr, 0); }

// acc[e] += X_{r2 - dr0 - e} conj(y) for the E lags: the X rows sit in a
// rotating register window (slot (tt + E - 1 - e) % E holds row r2 - dr0 - e
// at step tt).  Grouped by the y component so consecutive FMAs share it.
template <int E>
__device__ __forceinline__ void spec_mac(int tt, double2 y, const double* wr, const double* wi, double* ar,
                                         double* ai) {
  const double ny = -y.y;
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = fma(wr[(tt + E - 1 - e) % E], y.x, ar[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ai[e] = fma(wi[(tt + E - 1 - e) % E], y.x, ai[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = fma(wi[(tt + E - 1 - e) % E], y.y, ar[e]);
#pragma unroll
  for (int e = 0; e < E; ++e) ai[e] = fma(wr[(tt + E - 1 - e) % E], ny, ai[e]);
}

// Per-frequency row-lag correlation G(dr, f), partial over row segments.
// CTA = (snapshot b, row segment, 128-frequency block, lag group of E row
// lags; the lag group varies fastest so the CTAs reading the same X / Y rows
// run together and share them in L2); lane = frequency.  The row range of
// the group (union of its lags' core rows) is cut into nparts bands (multi-GPU
// row bands) x nseg segments; rows where every lag is active run without
// predicates.
template <int E>
__global__ void __launch_bounds__(SPEC_CW * 32, 2)
    k_spec_corr(const double2* __restrict__ FX, const double2* __restrict__ FY, Problem pr, SpecLayout lay, int L,
                int nfb,
                int ngrp, int nseg, int part, int nparts, double2* __restrict__ Gp) {
  long long t = blockIdx.x;
  const int g = (int)(t % ngrp);
  t /= ngrp;
  const int fb = (int)(t % nfb);
  t /= nfb;
  const int seg = (int)(t % nseg);
  const long long b = t / nseg;
  const int f = (fb * SPEC_CW + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31);
  if (f >= L) return;
  const int P = pr.P, N = pr.N;
  const int nlag = 2 * P - 1;
  const int dr0 = -(P - 1) + g * E;
  const int drl = min(dr0 + E - 1, P - 1);
  const int rlo = spec_lo(dr0, P), rhi = spec_hi(drl, P, N);
  const int nr = rhi - rlo + 1;
  const int pieces = nparts * nseg, idx = part * nseg + seg;
  const int a = rlo + (int)((long long)nr * idx / pieces);
  const int z = rlo + (int)((long long)nr * (idx + 1) / pieces) - 1;  // last row (inclusive)
  const int blo = spec_lo(drl, P), bhi = min(spec_hi(dr0, P, N), z);  // every lag active
  // rows of one 32-frequency block are 32 apart (SpecLayout)
  const double2* fx = FX + lay.at(b, 0, f);
  const double2* fy = FY + lay.at(b, 0, f);

  double ar[E], ai[E], wr[E], wi[E];
#pragma unroll
  for (int e = 0; e < E; ++e) ar[e] = ai[e] = wr[e] = wi[e] = 0.0;
  // window: slot k holds X row (a - dr0) - (E - 1) + k for k < E - 1
  {
    const int t0 = a - dr0;
#pragma unroll
    for (int k = 0; k < E - 1; ++k) {
      const int row = t0 - (E - 1) + k;
      if (row >= 0 && row < N) {
        const double2 v = fx[(long long)row * 32];
        wr[k] = v.x;
        wi[k] = v.y;
      }
    }
  }
  for (int rb = a; rb <= z; rb += E) {
    const int t0 = rb - dr0;
    if (rb >= blo && rb + E - 1 <= bhi) {
      const double2* px = fx + (long long)t0 * 32;
      const double2* py = fy + (long long)rb * 32;
#pragma unroll
      for (int tt = 0; tt < E; ++tt) {
        const double2 xn = px[(long long)tt * 32];
        const double2 y = py[(long long)tt * 32];
        wr[(tt + E - 1) % E] = xn.x;
        wi[(tt + E - 1) % E] = xn.y;
        spec_mac<E>(tt, y, wr, wi, ar, ai);
      }
    } else {
#pragma unroll
      for (int tt = 0; tt < E; ++tt) {
        const int r2 = rb + tt, row = t0 + tt;
        double2 xn = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (row >= 0 && row < N) xn = fx[(long long)row * 32];
        if (r2 <= z) y = fy[(long long)r2 * 32];
        wr[(tt + E - 1) % E] = xn.x;
        wi[(tt + E - 1) % E] = xn.y;
        const double ny = -y.y;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int dr = dr0 + e;
          const bool on = r2 >= spec_lo(dr, P) && r2 <= spec_hi(dr, P, N);
          const double yx = on ? y.x : 0.0, yy = on ? y.y : 0.0, nyy = on ? ny : 0.0;
          const int s = (tt + E - 1 - e) % E;
          ar[e] = fma(wr[s], yx, ar[e]);
          ai[e] = fma(wi[s], yx, ai[e]);
          ar[e] = fma(wi[s], yy, ar[e]);
          ai[e] = fma(wr[s], nyy, ai[e]);
        }
      }
    }
  }
  double2* out = Gp + (b * nseg + seg) * (long long)nlag * L + f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int dr = dr0 + e;
    if (dr <= P - 1) out[(long long)(dr + P - 1) * L] = make_double2(ar[e], ai[e]);
  }
}

// The same correlation with the rows staged in SMEM (P <= 64): CTA = (b,
// 32-frequency block, row segment), NG compute warps = the 16-lag groups of
// all 2P-1 lags (so the X / Y rows are read from L2 once per CTA instead of
// once per lag group) + one producer warp.  Per chunk of SC_RC second-element
// rows R.., the producer bulk-copies (cp.async.bulk, mbarrier ring) the
// contiguous runs Y rows [R, R+SC_RC) and X rows [R-(P-1), R+SC_RC+P-2) of the
// f-block (zero pad rows cover the ends); warp g walks the chunk with its 16
// X rows in a rotating register window (2 LDS.128 per 16 complex MACs).
constexpr int SC_RC = 32;
constexpr size_t SC_SMEM_BUDGET = 220 * 1024;

// (posonly: the symmetric sums keep the lags dr >= 0 only — the second
// element's rows [R, R+SC_RC) are the tail of the first element's rows
// [R-(P-1), R+SC_RC) of the same spectrum: one copy)
__host__ __device__ inline size_t spec_corr_stage_bytes(int P, bool posonly = false) {
  return sizeof(double2) * 32 * (size_t)(posonly ? SC_RC + P - 1 : 2 * SC_RC + 2 * P - 2);
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// E row lags per warp, NG = blockDim / 32 warps (<= MAXW): E = 16 with 8
// warps (255 registers) or E = 8 with 16 warps (128 registers)
template <int E, int MAXW>
__global__ void __launch_bounds__(MAXW * 32, 1)
    k_spec_corr_smem(const double2* __restrict__ FX, const double2* __restrict__ FY, Problem pr, SpecLayout lay,
                     int nseg, int part, int nparts, int stages, double2* __restrict__ Gp, int slot0, int nslots,
                     int posonly) {
  const int NG = blockDim.x >> 5;
  extern __shared__ __align__(128) unsigned char scraw[];
  const int P = pr.P, N = pr.N;
  const int nlag = 2 * P - 1, XR = posonly ? SC_RC + P - 1 : SC_RC + 2 * P - 2;
  const size_t stage_bytes = spec_corr_stage_bytes(P, posonly != 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(scraw + stages * stage_bytes);
  uint64_t* empty = full + stages;
  long long t = blockIdx.x;
  const int seg = (int)(t % nseg);
  t /= nseg;
  const int fb = (int)(t % lay.nfb);
  const long long b = t / lay.nfb;
  const int nch = (N + SC_RC - 1) / SC_RC;
  const int pieces = nparts * nseg, idx = part * nseg + seg;
  const int ca = (int)((long long)nch * idx / pieces), cz = (int)((long long)nch * (idx + 1) / pieces);
  const int nk = cz - ca;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* fxb = FX + ((b * lay.nfb + fb) * lay.np + lay.padr) * 32LL;  // row 0 of the block
  const double2* fyb = FY + ((b * lay.nfb + fb) * lay.np + lay.padr) * 32LL;
  // thread 0 is also the producer (keeps 2 warps per SM sub-partition: the
  // register budget of 8 warps is 255 per thread, 9 warps would cap it at 168)
  auto issue = [&](int k) {
    const int s = k % stages;
    if (k >= stages) mbar_wait(&empty[s], ((k - stages) / stages) & 1);
    const int R = (ca + k) * SC_RC;
    unsigned char* st = scraw + s * stage_bytes;
    mbar_expect_tx(&full[s], (unsigned)stage_bytes);
    if (posonly) {
      bulk_g2s(st, fxb + (long long)(R - (P - 1)) * 32, (unsigned)(sizeof(double2) * 32 * XR), &full[s]);
    } else {
      bulk_g2s(st, fyb + (long long)R * 32, (unsigned)(sizeof(double2) * 32 * SC_RC), &full[s]);
      bulk_g2s(st + sizeof(double2) * 32 * SC_RC, fxb + (long long)(R - (P - 1)) * 32,
               (unsigned)(sizeof(double2) * 32 * XR), &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NG);
    }
    fence_mbarrier_init();
    for (int k = 0; k < stages - 1 && k < nk; ++k) issue(k);
  }
  __syncthreads();
  // warps 0 .. ngn-1 take the negative lags [-(P-1), -1], the others [0, P-1]
  // (E per warp, never both signs): the core-row condition then becomes two
  // per-ROW masks — dr >= 0: y rows r2 >= P-1, x rows r1 <= N-P; dr < 0:
  // y rows r2 <= N-P, x rows r1 >= P-1 — applied once per row as it enters
  // the registers, with no per-lag predicates
  const int ngn = posonly ? 0 : (P - 1 + E - 1) / E;
  const bool neg = w < ngn;
  const int dr0 = neg ? -(P - 1) + w * E : (w - ngn) * E;
  const int drmax = neg ? -1 : P - 1;
  // Gauss form: s1 += xr yr, s2 += xi yi, s3 += (xr + xi)(yr - yi), then
  // Re = s1 + s2, Im = s3 - s1 + s2 — 3 DFMAs per complex MAC instead of 4
  // (the operand sums: one DADD per X row entering the window, one per y)
  double s1[E], s2[E], s3[E], wr[E], wi[E], ws[E];
#pragma unroll
  for (int e = 0; e < E; ++e) s1[e] = s2[e] = s3[e] = wr[e] = wi[e] = ws[e] = 0.0;
  const int xoff = (P - 1) - dr0;  // stage X row of (r2 = R + j, lag e) = j + xoff - e
  const int ylo = neg ? 0 : P - 1, yhi = neg ? N - P : N - 1;  // valid second-element rows
  const int xlo = neg ? P - 1 : 0, xhi = neg ? N - 1 : N - P;  // valid first-element rows
  for (int k = 0; k < nk; ++k) {
    if (threadIdx.x == 0 && k + stages - 1 < nk) issue(k + stages - 1);
    const int s = k % stages;
    mbar_wait(&full[s], (k / stages) & 1);
    const int R = (ca + k) * SC_RC;
    const double2* const S0 = reinterpret_cast<const double2*>(scraw + s * stage_bytes) + lane;
    const double2* X = posonly ? S0 : S0 + 32 * SC_RC;
    const double2* Y = posonly ? S0 + 32 * (P - 1) : S0;
    // window: slot kk holds X row t = R - dr0 - (E-1) + kk (stage row xoff - (E-1) + kk; clamped
    // stage rows only feed lags past the warp's range).  Filled at the
    // segment's first chunk only: SC_RC is a multiple of E, so at a chunk
    // boundary the slots already hold exactly these rows (entered, masked,
    // during the previous chunk)
    static_assert(SC_RC % E == 0, "chunk rows must be a multiple of the lag window");
    if (k == 0) {
#pragma unroll
      for (int kk = 0; kk < E - 1; ++kk) {
        const int trow = R - dr0 - (E - 1) + kk;
        double2 v = X[max(xoff - (E - 1) + kk, 0) * 32];
        if (trow < xlo || trow > xhi) v = make_double2(0.0, 0.0);
        wr[kk] = v.x;
        wi[kk] = v.y;
        ws[kk] = v.x + v.y;
      }
    }
    // the row masks only bite in the first / last chunks: interior chunks
    // (every entering X row and every Y row valid) run without them
    const bool interior = R - dr0 >= xlo && R + SC_RC - 1 - dr0 <= xhi && R >= ylo && R + SC_RC - 1 <= yhi;
    auto walk = [&](auto masked) {
#pragma unroll 2
      for (int j0 = 0; j0 < SC_RC; j0 += E) {
#pragma unroll
        for (int tt = 0; tt < E; ++tt) {
          const int r2 = R + j0 + tt, trow = r2 - dr0;
          double2 xn = X[(j0 + tt + xoff) * 32];
          double2 y = Y[(j0 + tt) * 32];
          if constexpr (decltype(masked)::value) {
            if (trow < xlo || trow > xhi) xn = make_double2(0.0, 0.0);
            if (r2 < ylo || r2 > yhi) y = make_double2(0.0, 0.0);
          }
          const int nw = (tt + E - 1) % E;
          wr[nw] = xn.x;
          wi[nw] = xn.y;
          ws[nw] = xn.x + xn.y;
          const double yd = y.x - y.y;
#pragma unroll
          for (int e = 0; e < E; ++e) s1[e] = fma(wr[(tt + E - 1 - e) % E], y.x, s1[e]);
#pragma unroll
          for (int e = 0; e < E; ++e) s2[e] = fma(wi[(tt + E - 1 - e) % E], y.y, s2[e]);
#pragma unroll
          for (int e = 0; e < E; ++e) s3[e] = fma(ws[(tt + E - 1 - e) % E], yd, s3[e]);
        }
      }
    };
    if (interior)
      walk(std::false_type{});
    else
      walk(std::true_type{});
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  const int f = fb * 32 + lane;
  double2* out = Gp + (b * nslots + slot0 + seg) * (long long)nlag * (lay.nfb * 32) + f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int dr = dr0 + e;
    if (dr <= drmax)
      out[(long long)(dr + P - 1) * (lay.nfb * 32)] = make_double2(s1[e] + s2[e], s3[e] - s1[e] + s2[e]);
  }
}

// dr = 0 core sums, one row at a time: for each core row r (both elements
// on row r),
//     CC_r(0, dc) = (1/L) sum_f X_r[f] conj(Y_r[f]) w^(f dc),   dc < Q,
// one FFT per row; the rows are then added in the space domain (k_spec_dft,
// in order).  Summing X_r conj(Y_r) over the rows first (as G does for
// dr != 0) would add the rows' |X_r|^2 coherently and leave ~1e-12 relative
// error at dc > 0 (numpy, cfg5); per row the error is ~eps log L of the row
// energy and adds incoherently over rows (~1e-15 relative, numpy, cfg5).
// CTA = (b, row r of the band [row_a, row_a + nrows)).
template <int LOGL, bool PRUNE = false>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_rowac(long long nitems, const double2* __restrict__ FX, const double2* __restrict__ FY, Problem pr,
                 SpecLayout lay, const double2* __restrict__ tw, const double2* __restrict__ twf, int row_a, int nrows, int nd0, int kbase,
                 double2* __restrict__ D0p) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  const int Q = pr.Q;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  const bool ok = si.valid;
  const int k = (int)(si.item % nrows);
  const long long b = si.item / nrows;
  const int r = row_a + k;
  const double2* fx = FX + lay.at(b, r, 0);
  const double2* fy = FY + lay.at(b, r, 0);
  const long long fs = (long long)lay.np * 32;
  const double inv = 1.0 / (double)L;
  double2* out = D0p + (b * nd0 + kbase + k) * (long long)Q;
  auto ld = [&](int idx) {
    if (!ok) return make_double2(0.0, 0.0);
    const long long o = (idx >> 5) * fs + (idx & 31);
    const double2 x = fx[o], y = fy[o];
    return make_double2(fma(x.x, y.x, x.y * y.y), fma(x.y, y.x, -x.x * y.y));  // x conj(y)
  };
  auto stf = [&](int idx, double2 v) {
    if (ok && idx < Q) out[idx] = make_double2(v.x * inv, v.y * inv);
  };
  if constexpr (PRUNE)
    spec_fft_pruned<LOGL>(sb, si.tl, tw, twf, ld, stf);
  else
    spec_fft_block<LOGL>(sb, si.tl, tw, ld, stf);
}

// k_spec_fft mode 2 with the dr = 0 row transform of k_spec_rowac fused (the
// symmetric core sums on the device path: one spectrum per row, X_r = Y_r):
// the CTA writes its row's spectrum, then transforms X_r conj(X_r) read back
// from the row it just wrote (L2 / L1, not HBM) — the same values in the
// same order as k_spec_rowac on that spectrum, so D0p is bitwise the same;
// the separate kernel's re-read of every spectrum and its launch are gone.
// Rows outside the core rows [row_a, row_a + nd0) run the second transform
// without storing (the FFT's barriers are CTA-wide).
template <typename T, int LOGL, bool PRUNE = false>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_fft_ac(long long nitems, const typename CT<T>::c* __restrict__ A, Problem pr, SpecLayout lay,
                  const double2* __restrict__ tw, const double2* __restrict__ twf, double2* FX, int row0, int nrows,
                  int row_a, int nd0, double2* __restrict__ D0p) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  const int M = pr.M, Q = pr.Q;
  const int r = row0 + (int)(si.item % nrows);
  const long long b = si.item / nrows;
  const int clo = Q - 1, chi = M - Q;
  double2* out = FX + lay.at(b, r, 0);
  const typename CT<T>::c* row = A + (b * pr.N + r) * (long long)M;
  const long long fs = (long long)lay.np * 32;  // next 32-frequency block
  const bool ok = si.valid;
  spec_fft_block<LOGL>(
      sb, si.tl, tw,
      [&](int idx) { return (ok && idx >= clo && idx <= chi) ? widen2(row[idx]) : make_double2(0.0, 0.0); },
      [&](int idx, double2 v) {
        if (ok) out[(idx >> 5) * fs + (idx & 31)] = v;
      });
  __syncthreads();  // the row's spectrum is visible to the CTA; sb is free
  const bool core = ok && r >= row_a && r < row_a + nd0;
  const double inv = 1.0 / (double)L;
  double2* d0 = D0p + (b * nd0 + (r - row_a)) * (long long)Q;
  auto ld = [&](int idx) {
    if (!core) return make_double2(0.0, 0.0);
    const double2 x = out[(idx >> 5) * fs + (idx & 31)];
    return make_double2(fma(x.x, x.x, x.y * x.y), fma(x.y, x.x, -x.x * x.y));  // x conj(x), as k_spec_rowac forms it
  };
  auto stf = [&](int idx, double2 v) {
    if (core && idx < Q) d0[idx] = make_double2(v.x * inv, v.y * inv);
  };
  if constexpr (PRUNE)
    spec_fft_pruned<LOGL>(sb, si.tl, tw, twf, ld, stf);
  else
    spec_fft_block<LOGL>(sb, si.tl, tw, ld, stf);
}

// CC(0, dc) = sum over the band's core rows of the per-row transforms
// (k_spec_rowac): CTA = (b, dc), thread = a contiguous run of rows summed in
// order, then a fixed-shape tree over the threads — deterministic.
__global__ void __launch_bounds__(256)
    k_spec_d0sum(const double2* __restrict__ D0p, int nd0, Problem pr, int nclasses,
                 const int* __restrict__ cls_slot, double2* __restrict__ ccpart, int cc_stride) {
  __shared__ double2 red[256];
  const int Q = pr.Q;
  const int dc = (int)(blockIdx.x % Q);
  const long long b = blockIdx.x / Q;
  const int t = threadIdx.x, nt = blockDim.x;
  const int k0 = (int)((long long)nd0 * t / nt), k1 = (int)((long long)nd0 * (t + 1) / nt);
  const double2* p = D0p + b * (long long)nd0 * Q + dc;
  double2 s = make_double2(0.0, 0.0);
  for (int k = k0; k < k1; ++k) s = cadd(s, p[(long long)k * Q]);
  red[t] = s;
  __syncthreads();
  for (int h = nt / 2; h > 0; h >>= 1) {
    if (t < h) red[t] = cadd(red[t], red[t + h]);
    __syncthreads();
  }
  if (t == 0) {
    const int cid = cls_slot[class_index(0, dc, pr.P, Q)];
    if (cid >= 0) ccpart[(b * nclasses + cid) * cc_stride] = red[0];
  }
}

// G partials of the row segments summed in order into segment 0 (one thread
// per (b, dr, f): the output FFT below then reads one value per frequency)
__global__ void __launch_bounds__(256)
    k_spec_gsum(double2* __restrict__ Gp, int nseg, long long per_seg, long long e_lo, long long e_cnt,
                long long total) {
  // elements [e_lo, e_lo + e_cnt) of every snapshot's [lag][f] block (the
  // symmetric sums fill the lags dr >= 0 only)
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const long long b = t / e_cnt, e = e_lo + t % e_cnt;
  double2* g = Gp + b * nseg * per_seg + e;
  double2 v[8];
  double2 s = g[0];
  int sg = 1;
  for (; sg + 8 <= nseg; sg += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = g[(sg + j) * per_seg];
#pragma unroll
    for (int j = 0; j < 8; ++j) s = cadd(s, v[j]);
  }
  for (; sg < nseg; ++sg) s = cadd(s, g[sg * per_seg]);
  g[0] = s;
}

// CC(dr, dc) = (1/L) sum_f G(dr, f) w^(f dc) for dr != 0: one forward FFT of
// G(dr, .) (segment 0 after k_spec_gsum) per row lag, outputs
// dc in [0, Q); for dr = 0 the ordered sum of the space-domain partials.
// CTA = (snapshot b, row lag dr).  Writes the classes' CC slot (one partial:
// npart = 1 for the finalize).
template <int LOGL, bool PRUNE = false>
__global__ void __launch_bounds__(spec_threads<LOGL>())
    k_spec_dft(long long nitems, const double2* __restrict__ Gp, const double2* __restrict__ tw,
               const double2* __restrict__ twf, Problem pr,
               int nseg, int nclasses, const int* __restrict__ cls_slot, double2* __restrict__ ccpart, int cc_stride,
               int cc_part, int sym, int with_d0, int strips) {
  extern __shared__ double2 sbuf[];
  constexpr int L = 1 << LOGL;
  const int P = pr.P, Q = pr.Q;
  const int nlag = 2 * P - 1;
  double2* sb;
  const SpecItem si = spec_item<LOGL>(nitems, sb, sbuf);
  const int li = (int)(si.item % nlag);
  const long long bg = si.item / nlag;  // G's snapshot index (strips: 2 snapshot + strip, one CC partial per strip)
  const long long b = strips ? bg >> 1 : bg;
  if (strips) cc_part += (int)(bg & 1);
  const int dr = li - (P - 1);
  const bool ok = si.valid && (dr != 0 || with_d0);  // dr = 0: k_spec_d0sum (unless with_d0)
  // sym: only G(dr >= 0, .) exists and G(-d, f) = conj(G(d, f)), so the lag
  // -d transforms the conjugate of lag d's row
  const bool cj = sym && dr < 0;
  const double2* g = Gp + (bg * nseg * nlag + (cj ? (P - 1) - dr : li)) * (long long)L;
  const double inv = 1.0 / (double)L;
  auto ld = [&](int idx) {  // segment 0: the ordered sum
    if (!ok) return make_double2(0.0, 0.0);
    const double2 v = g[idx];
    return cj ? make_double2(v.x, -v.y) : v;
  };
  auto stf = [&](int idx, double2 v) {
    if (ok && idx < Q && (dr >= 0 || idx > 0)) {
      const int cid = cls_slot[class_index(dr, idx, P, Q)];
      if (cid >= 0) ccpart[(b * nclasses + cid) * cc_stride + cc_part] = make_double2(v.x * inv, v.y * inv);
    }
  };
  if constexpr (PRUNE)
    spec_fft_pruned<LOGL>(sb, si.tl, tw, twf, ld, stf);
  else
    spec_fft_block<LOGL>(sb, si.tl, tw, ld, stf);
}

}  // namespace covgpu

// K2 — the class sums of one small complex64 snapshot inside one CTA, in FP32
// (the batched per-snapshot kernel; the reference's batch
// driver engine.py:219-255 runs its class kernel _numba_kernels.py:62-107 per
// snapshot).
//
// The same frequency-domain identity as spectral.cuh, with everything a
// snapshot needs held in the CTA's shared memory, so no spectrum ever goes
// to HBM: with x_r / y_r = row r under the two core-column masks and
// X_r = FFT_128(x_r), Y_r = FFT_128(y_r),
//     G(dr, f)   = sum_{r2 in rows(dr)} X_{r2-dr}[f] conj(Y_{r2}[f])
//     CC(dr, dc) = (1/L) FFT_128(G(dr, .))[dc]
// for all 2P-1 <= 15 row lags at once (P <= 8, M <= 128, Q <= 16).
//
// CTA = one snapshot, 256 threads.  Rows go through in chunks of 16:
//   transform phase: 16 groups of 16 threads, group g -> row 16 j + g, read
//     from global memory once (coalesced; the next chunk's row is prefetched
//     under the correlation) and transformed twice — X and Y, the two masked
//     versions, pass by pass together: radix-8 x radix-8 x radix-2 Stockham
//     passes in place in the destination rows of the X ring (3 chunks) / Y
//     ring (2 chunks);
//   correlation phase for the Y rows of chunk j-1 (their X rows r2 - dr lie in
//     chunks j-2 .. j): thread = (frequency f, lag sign), 8 lags in registers.
// After the last chunk the G rows are transformed in place (one group per
// lag) and the first Q outputs go to the plan's CC array (one partial per
// class); finally the edge-column sums CCol (core rows x the Q-1 edge columns
// of each side: correlations of pairs of strip columns along the rows, one
// pair per thread, the 15 lags in a rotating register window) and the
// edge-row sums RC' (ordered strip-row pairs x column lags) come from the
// strips, staged in the rings' shared memory once the core sums are done.
// FP32 arithmetic throughout (complex64 bar: 1e-5 relative Frobenius; measured
// ~1e-6); every sum has a fixed order, nothing depends on the batch size.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace covgpu {

constexpr int K2_L = 128;          // FFT length (M <= 128)
constexpr int K2_RS = 144;         // SMEM row stride: 128 + one pad per 8
constexpr int K2_CH = 16;          // rows per chunk (one row per 16-thread group: its X and its Y transform)
constexpr int K2_XR = 3 * K2_CH;   // X ring rows (chunks j-2 .. j)
constexpr int K2_E = 8;            // lags per correlation thread
constexpr int K2_W = 2 * K2_E - 1; // lag window of the edge-column pairs
constexpr int K2_MAXQ = 16;
constexpr int K2_THREADS = 256;

constexpr int K2_ERS = 129;        // strip-row stride (odd: the strip's rows fall in distinct banks)
// twiddles + max(the rings of the core sums, the strips of the edge sums staged
// in the same memory afterwards)
__host__ __device__ inline size_t k2_smem_bytes(int N, int P, int Q) {
  const size_t rings = (size_t)(K2_XR + 2 * K2_CH) * K2_RS;
  const size_t strips = (size_t)2 * N * (Q - 1) + (size_t)2 * (P - 1) * K2_ERS;
  return sizeof(float2) * (128 + (rings > strips ? rings : strips));
}

__device__ __forceinline__ int k2_pad(int i) { return i + (i >> 3); }
__device__ __forceinline__ float2 k2_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 k2_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 k2_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 k2_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)

__device__ __forceinline__ void k2_dft4(float2& a, float2& b, float2& c, float2& d) {
  const float2 t0 = k2_add(a, c), t1 = k2_sub(a, c), t2 = k2_add(b, d), t3 = k2_mi(k2_sub(b, d));
  a = k2_add(t0, t2);
  c = k2_sub(t0, t2);
  b = k2_add(t1, t3);
  d = k2_sub(t1, t3);
}
// forward 8-point DFT in registers (natural order in, natural order out)
__device__ __forceinline__ void k2_dft8(float2* u) {
  constexpr float c = 0.70710678118654752440f;
  float2 e0 = u[0], e1 = u[2], e2 = u[4], e3 = u[6], o0 = u[1], o1 = u[3], o2 = u[5], o3 = u[7];
  k2_dft4(e0, e1, e2, e3);
  k2_dft4(o0, o1, o2, o3);
  const float2 p1 = make_float2(c * (o1.x + o1.y), c * (o1.y - o1.x));
  const float2 p2 = k2_mi(o2);
  const float2 p3 = make_float2(c * (o3.y - o3.x), -c * (o3.x + o3.y));
  u[0] = k2_add(e0, o0);
  u[4] = k2_sub(e0, o0);
  u[1] = k2_add(e1, p1);
  u[5] = k2_sub(e1, p1);
  u[2] = k2_add(e2, p2);
  u[6] = k2_sub(e2, p2);
  u[3] = k2_add(e3, p3);
  u[7] = k2_sub(e3, p3);
}

// Forward FFT-128 by 16 threads (tl = thread in the group), the 8 inputs
// u[r] = in[tl + 16 r] already in registers; row = the destination (stride-
// padded, k2_pad), used in place for the two exchanges.  All groups of a warp
// run this together (__syncwarp).  tw64[k] = w_64^k (k < 64), tw128[k] = w_128^k.
__device__ __forceinline__ void k2_fft128(float2* u, float2* row, int tl, const float2* tw64,
                                          const float2* tw128) {
  // pass 1: radix 8, p = 1 (no twiddles): out[8 tl + r]
  k2_dft8(u);
#pragma unroll
  for (int r = 0; r < 8; ++r) row[k2_pad(8 * tl + r)] = u[r];
  __syncwarp();
  // pass 2: radix 8, p = 8: k = tl & 7, u_r = in[tl + 16 r] w_64^(r k), out[(tl - k) 8 + k + 8 r]
#pragma unroll
  for (int r = 0; r < 8; ++r) u[r] = row[k2_pad(tl + 16 * r)];
  __syncwarp();
  const int k = tl & 7;
#pragma unroll
  for (int r = 1; r < 8; ++r) u[r] = k2_mul(u[r], tw64[r * k]);
  k2_dft8(u);
#pragma unroll
  for (int r = 0; r < 8; ++r) row[k2_pad((tl - k) * 8 + k + 8 * r)] = u[r];
  __syncwarp();
  // pass 3: radix 2, p = 64: items i = tl + 16 it (i < 64): out[i] = in[i] + w in[i+64], out[i+64] = in[i] - w in[i+64]
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int i = tl + 16 * it;
    u[2 * it] = row[k2_pad(i)];
    u[2 * it + 1] = k2_mul(row[k2_pad(i + 64)], tw128[i]);
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int i = tl + 16 * it;
    row[k2_pad(i)] = k2_add(u[2 * it], u[2 * it + 1]);
    row[k2_pad(i + 64)] = k2_sub(u[2 * it], u[2 * it + 1]);
  }
  __syncwarp();
}

// Two transforms by the same 16 threads, pass by pass (twice the independent
// work between the warp barriers)
__device__ __forceinline__ void k2_fft128x2(float2* u, float2* v, float2* rowu, float2* rowv, int tl,
                                            const float2* tw64, const float2* tw128) {
  k2_dft8(u);
  k2_dft8(v);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    rowu[k2_pad(8 * tl + r)] = u[r];
    rowv[k2_pad(8 * tl + r)] = v[r];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    u[r] = rowu[k2_pad(tl + 16 * r)];
    v[r] = rowv[k2_pad(tl + 16 * r)];
  }
  __syncwarp();
  const int k = tl & 7;
#pragma unroll
  for (int r = 1; r < 8; ++r) {
    const float2 w = tw64[r * k];
    u[r] = k2_mul(u[r], w);
    v[r] = k2_mul(v[r], w);
  }
  k2_dft8(u);
  k2_dft8(v);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    rowu[k2_pad((tl - k) * 8 + k + 8 * r)] = u[r];
    rowv[k2_pad((tl - k) * 8 + k + 8 * r)] = v[r];
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int i = tl + 16 * it;
    const float2 w = tw128[i];
    u[2 * it] = rowu[k2_pad(i)];
    u[2 * it + 1] = k2_mul(rowu[k2_pad(i + 64)], w);
    v[2 * it] = rowv[k2_pad(i)];
    v[2 * it + 1] = k2_mul(rowv[k2_pad(i + 64)], w);
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int i = tl + 16 * it;
    rowu[k2_pad(i)] = k2_add(u[2 * it], u[2 * it + 1]);
    rowu[k2_pad(i + 64)] = k2_sub(u[2 * it], u[2 * it + 1]);
    rowv[k2_pad(i)] = k2_add(v[2 * it], v[2 * it + 1]);
    rowv[k2_pad(i + 64)] = k2_sub(v[2 * it], v[2 * it + 1]);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(K2_THREADS, 2)
    k_snap_spec(const float2* __restrict__ A, Problem pr, int B, int nclasses, const int* __restrict__ cls_slot,
                const ClassDesc* __restrict__ cls, double2* __restrict__ ccpart, double2* __restrict__ ccol,
                long long tot_ccol, double2* __restrict__ rc, long long tot_rc) {
  extern __shared__ __align__(16) unsigned char k2raw[];
  const int N = pr.N, M = pr.M, P = pr.P, Q = pr.Q, S1 = Q - 1;
  float2* const tw64 = reinterpret_cast<float2*>(k2raw);         // w_64^k
  float2* const tw128 = tw64 + 64;                               // w_128^k, k < 64
  float2* const xr = tw128 + 64;                                 // X ring [K2_XR][K2_RS]
  float2* const yr = xr + K2_XR * K2_RS;                         // Y ring [2][K2_CH][K2_RS]
  // (after the core sums, in the rings' memory:)
  float2* const sl = xr;                                         // left strip [N][Q-1]
  float2* const sr = sl + (size_t)N * S1;                        // right strip [N][Q-1]
  float2* const er = sr + (size_t)N * S1;                        // strip rows [2][P-1][K2_ERS] (edge-row sums)
  const int S = P - 1;
  const int t = threadIdx.x, b = blockIdx.x;
  const float2* Ab = A + (long long)b * N * M;

  if (t < 64) {
    float s, c;
    sincospif(-(float)t / 32.f, &s, &c);
    tw64[t] = make_float2(c, s);
    sincospif(-(float)t / 64.f, &s, &c);
    tw128[t] = make_float2(c, s);
  }
  __syncthreads();

  // ---- core sums -----------------------------------------------------------
  const int f = t & 127, half = t >> 7;  // half 1: lags dr = e >= 0; half 0: dr = -(e + 1)
  float ar[K2_E], ai[K2_E];
#pragma unroll
  for (int e = 0; e < K2_E; ++e) ar[e] = ai[e] = 0.f;
  const int grp = t >> 4, tl = t & 15;
  const int nchunks = (N + K2_CH - 1) / K2_CH;
  // the X rows of a thread's 8 lags sit in a rotating register window (slot =
  // row mod 8): half 1 (dr = e) holds rows r2-7 .. r2, half 0 (dr = -(e+1))
  // rows r2+1 .. r2+8; one row enters per second-element row r2.  The core-row
  // condition is two per-ROW masks, applied as a row enters the registers:
  // dr >= 0: y rows r2 >= P-1, x rows r1 <= N-P; dr < 0: y rows r2 <= N-P,
  // x rows r1 >= P-1
  float wr[K2_E], wi[K2_E];
#pragma unroll
  for (int e = 0; e < K2_E; ++e) wr[e] = wi[e] = 0.f;
  const float2* const xb = xr + k2_pad(f);
  // this group's row of chunk j: 8 inputs per thread (both transforms mask them)
  auto load_row = [&](int j, float2* u) {
    const int row = j * K2_CH + grp;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int c = tl + 16 * r;
      u[r] = (j < nchunks && row < N && c < M) ? Ab[(long long)row * M + c] : make_float2(0.f, 0.f);
    }
  };
  auto corr = [&](auto hs, int jc) {
    constexpr int H = decltype(hs)::value;
    const float2* yb = yr + (jc & 1) * K2_CH * K2_RS + k2_pad(f);
    int rslot = (jc * K2_CH + (H ? 0 : K2_E)) % K2_XR;  // ring slot of the entering row
#pragma unroll
    for (int t2 = 0; t2 < K2_CH; ++t2) {
      const int tt = t2 % K2_E;
      const int r2 = jc * K2_CH + t2;
      const int rin = H ? r2 : r2 + K2_E;  // the row entering the window (slot tt either way)
      float2 x = xb[rslot * K2_RS];
      rslot = rslot + 1 == K2_XR ? 0 : rslot + 1;
      float2 y = yb[t2 * K2_RS];
      if (H ? rin > N - P : (rin < P - 1 || rin >= N)) x = make_float2(0.f, 0.f);
      if (H ? (r2 < P - 1 || r2 >= N) : r2 > N - P) y = make_float2(0.f, 0.f);
      wr[tt] = x.x;
      wi[tt] = x.y;
      const float ny = -y.y;
#pragma unroll
      for (int e = 0; e < K2_E; ++e) {
        const int s = H ? (tt - e + K2_E) % K2_E : (tt + 1 + e) % K2_E;  // row r2 - e / r2 + 1 + e
        ar[e] = fmaf(wr[s], y.x, ar[e]);
        ai[e] = fmaf(wi[s], y.x, ai[e]);
        ar[e] = fmaf(wi[s], y.y, ar[e]);
        ai[e] = fmaf(wr[s], ny, ai[e]);
      }
    }
  };
  float2 u[8];
  load_row(0, u);
  for (int j = 0; j <= nchunks; ++j) {
    if (j < nchunks) {
      const int row = j * K2_CH + grp;
      // x: first-element columns c <= M-Q; y: second-element columns c >= Q-1
      float2 v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int c = tl + 16 * r;
        v[r] = c >= Q - 1 ? u[r] : make_float2(0.f, 0.f);
        if (c > M - Q) u[r] = make_float2(0.f, 0.f);
      }
      k2_fft128x2(u, v, xr + (row % K2_XR) * K2_RS, yr + ((j & 1) * K2_CH + grp) * K2_RS, tl, tw64, tw128);
    }
    load_row(j + 1, u);  // the next chunk's row: its latency hides under the correlation
    __syncthreads();
    if (j == 1 && !half) {
      // half 0's window before r2 = 0: rows 1 .. 7 (row 8 enters at r2 = 0)
#pragma unroll
      for (int x = 1; x < K2_E; ++x) {
        float2 w = xb[x * K2_RS];
        if (x < P - 1 || x >= N) w = make_float2(0.f, 0.f);
        wr[x] = w.x;
        wi[x] = w.y;
      }
    }
    if (j >= 1) {
      if (half)
        corr(std::integral_constant<int, 1>{}, j - 1);
      else
        corr(std::integral_constant<int, 0>{}, j - 1);
    }
    __syncthreads();
  }
  // G rows -> the X ring (row = lag index dr + P - 1), then one forward FFT per lag
#pragma unroll
  for (int e = 0; e < K2_E; ++e) {
    const int dr = half ? e : -(e + 1);
    if (dr > -P && dr < P) xr[(dr + P - 1) * K2_RS + k2_pad(f)] = make_float2(ar[e], ai[e]);
  }
  __syncthreads();
  {
    // every group transforms a ring row (warp-level barriers inside); rows
    // past the 2P-1 lags hold stale spectra and store nothing
    float2* row = xr + grp * K2_RS;
    float2 u[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = row[k2_pad(tl + 16 * r)];
    __syncwarp();
    k2_fft128(u, row, tl, tw64, tw128);
    const int dr = grp - (P - 1);
    if (grp < 2 * P - 1) {
      for (int dc = tl; dc < Q; dc += 16) {
        if (!in_uc(dr, dc, P, Q)) continue;
        const int slot = cls_slot[class_index(dr, dc, P, Q)];
        if (slot < 0) continue;
        const float2 v = row[k2_pad(dc)];
        ccpart[(long long)b * nclasses + slot] = make_double2((double)v.x / K2_L, (double)v.y / K2_L);
      }
    }
  }

  // ---- the strips of the edge sums, staged in the rings' memory -------------
  __syncthreads();  // (the G rows are read)
  // columns [0, Q-1) and [M-Q+1, M) of every row: thread = (row mod 16, column)
  if (tl < S1)
    for (int r = grp; r < N; r += 16) {
      sl[r * S1 + tl] = Ab[(long long)r * M + tl];
      sr[r * S1 + tl] = Ab[(long long)r * M + (M - S1) + tl];
    }
  // the top / bottom P-1 strip rows, zero beyond column M
  for (int row = t >> 7; row < 2 * S; row += 2) {
    const int c = t & 127, ra = row < S ? row : N - S + (row - S);
    er[row * K2_ERS + c] = c < M ? Ab[(long long)ra * M + c] : make_float2(0.f, 0.f);
  }
  __syncthreads();

  // ---- edge-column sums: pairs (j1 <= j2) of one strip's columns ------------
  const int npairs = S1 * (S1 + 1) / 2;
  for (int item = t; item < 2 * npairs; item += K2_THREADS) {
    const int side = item >= npairs;
    int q = item - side * npairs, j1 = 0;
    while (q >= S1 - j1) {  // pairs of column j1: j2 = j1 .. S1-1
      q -= S1 - j1;
      ++j1;
    }
    const int j2 = j1 + q, dc = q;
    const float2* st = side ? sr : sl;
    // lag slot e <-> dr = e - (K2_E - 1).  The window holds the first-element
    // column for rows r2 - 7 .. r2 + 7, row x in slot x mod K2_W: rows ahead of
    // r2 serve the negative lags (valid first-element rows >= P-1), row r2 and
    // the rows behind it the lags >= 0 (valid rows <= N-P) — a row is masked for
    // the negative lags as it enters and re-masked when r2 reaches it
    float wr[K2_W], wi[K2_W], cr[K2_W], ci[K2_W];
#pragma unroll
    for (int e = 0; e < K2_W; ++e) wr[e] = wi[e] = cr[e] = ci[e] = 0.f;
#pragma unroll
    for (int x = 0; x < K2_E - 1; ++x) {  // rows 0 .. 6 are ahead of r2 = 0
      if (x < N && x >= P - 1) {
        const float2 v = st[x * S1 + j1];
        wr[x] = v.x;
        wi[x] = v.y;
      }
    }
    // one block of K2_W rows; interior blocks (every row and every entering
    // row valid for both lag signs, the window already holding actual values)
    // run without masks and without the re-mask load
    auto block = [&](auto masked, int r2base) {
      constexpr bool MASK = decltype(masked)::value;
      const float2* px = st + (r2base + K2_E - 1) * S1 + j1;
      const float2* py = st + r2base * S1 + j2;
#pragma unroll
      for (int tt = 0; tt < K2_W; ++tt) {
        float ypx, ypy, ynx, yny;
        if constexpr (MASK) {
          const int r2 = r2base + tt, rin = r2 + K2_E - 1;
          float2 xin = make_float2(0.f, 0.f), xc = xin, y = xin;
          if (rin < N && rin >= P - 1) xin = px[tt * S1];
          if (r2 <= N - P) xc = st[r2 * S1 + j1];
          if (r2 < N) y = py[tt * S1];
          wr[(tt + K2_E - 1) % K2_W] = xin.x;
          wi[(tt + K2_E - 1) % K2_W] = xin.y;
          wr[tt] = xc.x;
          wi[tt] = xc.y;
          // second-element row masks: lags >= 0 need r2 >= P-1, lags < 0 need r2 <= N-P
          ypx = r2 >= P - 1 ? y.x : 0.f, ypy = r2 >= P - 1 ? y.y : 0.f;
          ynx = r2 <= N - P ? y.x : 0.f, yny = r2 <= N - P ? y.y : 0.f;
        } else {
          const float2 xin = px[tt * S1], y = py[tt * S1];
          wr[(tt + K2_E - 1) % K2_W] = xin.x;
          wi[(tt + K2_E - 1) % K2_W] = xin.y;
          ypx = ynx = y.x;
          ypy = yny = y.y;
        }
#pragma unroll
        for (int e = 0; e < K2_W; ++e) {
          const int dr = e - (K2_E - 1);
          const int s = (tt - dr + K2_W) % K2_W;  // slot of row r2 - dr
          const float yx = dr >= 0 ? ypx : ynx, yy = dr >= 0 ? ypy : yny;
          cr[e] = fmaf(wr[s], yx, cr[e]);
          cr[e] = fmaf(wi[s], yy, cr[e]);
          ci[e] = fmaf(wi[s], yx, ci[e]);
          ci[e] = fmaf(-wr[s], yy, ci[e]);
        }
      }
    };
    for (int r2base = 0; r2base < N; r2base += K2_W) {
      // interior: rows r2 in [P-1, N-P] and entering rows r2 + 7 < N throughout
      // (entering rows >= P-1 follows; rows behind r2 were re-masked in range)
      if (r2base >= P - 1 + K2_E - 1 && r2base + K2_W - 1 + K2_E - 1 <= N - P)
        block(std::false_type{}, r2base);
      else
        block(std::true_type{}, r2base);
    }
#pragma unroll
    for (int e = 0; e < K2_W; ++e) {
      const int dr = e - (K2_E - 1);
      if (dr <= -P || dr >= P || !in_uc(dr, dc, P, Q)) continue;
      const int slot = cls_slot[class_index(dr, dc, P, Q)];
      if (slot < 0) continue;
      const ClassDesc& cd = cls[slot];
      const int ac = cd.qu - 1;  // = Q - 1 - dc > j1
      ccol[(long long)b * tot_ccol + cd.ccol_off + (side ? ac : 0) + j1] = make_double2((double)cr[e], (double)ci[e]);
    }
  }
  // ---- edge-row sums RC' (edge.cuh k_edge_rows): ordered row pairs (r1, r2)
  // of one strip x column lags dc < Q, summed over the slot-0 box columns
  // c in [0, M-Q]; thread = (strip, pair, group of K2_E column lags), the
  // second-element columns in a rotating register window
  const int ndg = (Q + K2_E - 1) / K2_E;
  for (int item = t; item < 2 * S * S * ndg; item += K2_THREADS) {
    const int g = item % ndg;
    const int pq = item / ndg % (S * S), strip = item / (ndg * S * S);
    const int i1 = pq % S, i2 = pq / S, dr = i2 - i1, dc0 = g * K2_E;
    const float2* x = er + (strip * S + i1) * K2_ERS;
    const float2* y = er + (strip * S + i2) * K2_ERS;
    float cr[K2_E], ci[K2_E], vr[K2_E], vi[K2_E];
#pragma unroll
    for (int d = 0; d < K2_E; ++d) cr[d] = ci[d] = vr[d] = vi[d] = 0.f;
#pragma unroll
    for (int d = 0; d < K2_E - 1; ++d) {  // y columns dc0 .. dc0 + 6 (column c = 0's lags but the last)
      const float2 v = y[min(dc0 + d, K2_L - 1)];
      vr[d] = v.x;
      vi[d] = v.y;
    }
    auto cols = [&](auto masked, int c0) {
      constexpr bool MASK = decltype(masked)::value;
#pragma unroll
      for (int cc = 0; cc < K2_E; ++cc) {
        const int c = c0 + cc;
        float2 xv, yn;
        if constexpr (MASK) {
          xv = x[min(c, K2_L - 1)];
          if (c > M - Q) xv = make_float2(0.f, 0.f);
          yn = y[min(c + dc0 + K2_E - 1, K2_L - 1)];  // (columns past M are zero)
        } else {
          xv = x[c];
          yn = y[c + dc0 + K2_E - 1];
        }
        vr[(cc + K2_E - 1) % K2_E] = yn.x;
        vi[(cc + K2_E - 1) % K2_E] = yn.y;
#pragma unroll
        for (int d = 0; d < K2_E; ++d) {
          const int sl_ = (cc + d) % K2_E;  // column c + dc0 + d
          cr[d] = fmaf(xv.x, vr[sl_], cr[d]);
          ci[d] = fmaf(xv.y, vr[sl_], ci[d]);
          cr[d] = fmaf(xv.y, vi[sl_], cr[d]);
          ci[d] = fmaf(-xv.x, vi[sl_], ci[d]);
        }
      }
    };
    for (int c0 = 0; c0 <= M - Q; c0 += K2_E) {
      if (c0 + K2_E - 1 <= M - Q && c0 + dc0 + 2 * K2_E - 2 < K2_L)
        cols(std::false_type{}, c0);
      else
        cols(std::true_type{}, c0);
    }
    const int i = min(i1, i2);
#pragma unroll
    for (int d = 0; d < K2_E; ++d) {
      const int dc = dc0 + d;
      if (dc >= Q || !in_uc(dr, dc, P, Q)) continue;
      const int slot = cls_slot[class_index(dr, dc, P, Q)];
      if (slot < 0) continue;
      const ClassDesc& cd = cls[slot];
      const int k = strip ? (cd.pv - 1) + i : i;
      rc[(long long)b * tot_rc + cd.rc_off + k] = make_double2((double)cr[d], (double)ci[d]);
    }
  }
}

}  // namespace covgpu

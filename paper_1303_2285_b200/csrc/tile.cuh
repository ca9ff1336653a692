// K3 — tile finalize (k_fin_tile): the diagonal-segment walk written as
// coalesced row segments of R's P x P blocks.
//
// Block (u, u+dc) of R (rows P u + r1, columns P (u+dc) + r2, r1, r2 in
// [0, P)) holds, on its diagonal dr = r2 - r1, slot u of class (dr, dc):
// entry (r1, r1+dr) is slot (v = r1 - s1, u) (_numba_kernels.py:100-106).
// With the class's top / bottom edge-row state indexed by the pair of A rows
// it multiplies — F_T[r1][r2] = fullT_i(u), F_B[r1][r2] = fullB_i(u) with
// i = min(r1, r2) — the walk along the diagonal reads
//   O(r1)   = G(u) + sum_{k >= r1} F_T[k][k+dr] + sum_{k < r1} F_B[k][k+dr]
//   O(r1+1) = O(r1) - F_T[r1][r1+dr] + F_B[r1][r1+dr]
// (drop the leaving edge row, add the entering one), and the step u -> u+1
// of every class of one column offset dc is ONE rank-2 update of the state
// by four strip columns of A (the corner products, each formed once):
//   F_T += TR[u] (x) conj(TR[u+dc]) - TL[u] (x) conj(TL[u+dc])    (top strip)
//   F_B += BR[u] (x) conj(BR[u+dc]) - BL[u] (x) conj(BL[u+dc])    (bottom strip)
//   G   += CColR[u] - CColL[u].
//
// Circular diagonals: diagonal dr = c (rows [0, P-c)) and dr = c-P (rows
// [P-c, P)) have complementary rows, so lane c of a warp walks the block's
// entries (r1, (r1 + c) mod P) for all rows — two classes, one segment each,
// and no idle slot (dc > 0).  Unit = (snapshot, dc, band of 32 circular
// diagonals, steps [u_lo, u_hi)); warp w owns rows 8w .. 8w+7 and carries
// F_T / F_B of its 8 entries in registers.  Per step u: the row-group totals
// of both segments meet in SMEM (one unit barrier per step) to give each
// warp its carries; a warp's store of row r1 covers 32 consecutive columns
// (mod P) of R's row P u + r1 (straight-line stores under a predicate);
// dense R's mirrored block (u+dc, u) is written from an SMEM stage, again as
// row segments (units of 2 - 4 warps: double-buffered, one step later; 8
// warps: one buffer and a second barrier, so two units fit an SM); the strip
// columns of the next step are prefetched with cp.async.
//
// Walks are cut at u = ck j (ck = 4, 8 or 16 by window size, ft_ckstep): the
// same kernel in DELTA mode adds up each ck-step chunk's updates (from zero;
// it reads only the corner blocks of A, so it runs first, off the critical
// path), k_ck_scan sums them in chunk order, and a unit starting at
// u_lo = ck j takes F(u_lo) = F(0) + (delta_1 + ... + delta_j).  Every unit
// walks <= ck steps and the launch fills the SMs.  The cut grid is a fixed
// function of the window and of u, and every value depends only on its
// class's sums and the fixed 8-row grouping: class subsets (shards), layouts,
// batches and u-chunked launches give the same bits; packed R equals dense
// R's upper triangle bitwise.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace covgpu {

#ifndef FT_CTA_WARPS
#define FT_CTA_WARPS 8
#endif
constexpr int FT_RPT = 8;  // rows per thread
constexpr int FT_CK = 16;  // largest checkpoint spacing (steps); a plan picks 4, 8 or 16 (ft_ckstep)

template <int NWARP>
struct FtCfg {
  static constexpr int UPC = NWARP >= FT_CTA_WARPS ? 1 : FT_CTA_WARPS / NWARP;  // units per CTA
  static constexpr int THREADS = 32 * NWARP * UPC;
};

// walk state saved between u-chunked launches: F_T[8], F_B[8], G1, G2
constexpr int FT_STATE = 2 * FT_RPT + 2;

inline int ft_nwarp(int P) {
  int w = 1;
  while (w * FT_RPT < P) w <<= 1;
  return w;
}
// lanes per snapshot: small windows pack 32 / lanes snapshots into a warp
inline int ft_lanes(int P) { return P > 16 ? 32 : P > 8 ? 16 : 8; }
__host__ __device__ inline int ft_nck(int Q, int ck) { return (Q - 1) / ck; }  // checkpoints per (snapshot, dc)
// Checkpoint spacing of a plan: a function of the window only (never of the
// batch or the class subset, so a snapshot's bits do not depend on them).
// Large windows have enough (dc, band, chunk) units to fill the SMs with
// 16-step walks; small ones are latency-bound chains, so they are cut finer.
inline int ft_ckstep(int P, int Q) {
  // (P <= 8: several snapshots share a warp and a step is cheap — the
  // checkpoint traffic of a batch costs more than the longer chains)
  const int bands = (P + 31) / 32;
  return Q * bands >= 128 || P <= 8 ? 16 : Q * bands >= 48 ? 8 : 4;
}

// Corner blocks per (snapshot, column j of the (Q-1)-column strips), widened
// to double, in the layout one step's SMEM copy takes as is: first operands
// TL, TR, BL, BR ([PP] each: rows [0, P-1) of A's top / bottom strip, zero
// beyond), then second operands TL, TR, BL, BR ([2 PP] each: the P-1 strip
// rows and a zero, twice — index (r1 + c) mod P then needs no wrap — zero
// beyond 2P; the block strides depend on the instantiation only, so every
// SMEM offset of the walk is a compile-time constant).
__host__ __device__ inline int ft_colw(int P, int PP) {
  (void)P;
  return 12 * PP;
}

// SMEM per unit: strip vectors [2 bufs][subs][colw + 8] double2 (8 zeros of
// slack: rows past P read in range), row-group totals [2 bufs][T1, B1, T2,
// B2][nwarp][32] double2, edge-column sums of the step [2 bufs][class 1,
// 2][L, R][32] double2, stage [bufs][PP][32] (output precision)
__host__ __device__ inline size_t ft_vec_elems(int P, int PP) { return (size_t)ft_colw(P, PP) + 8; }
__host__ __device__ inline size_t ft_tot_bytes(int nwarp) { return (size_t)2 * 4 * nwarp * 32 * 16; }
__host__ __device__ inline size_t ft_gcol_bytes() { return (size_t)2 * 4 * 32 * 16; }
// (P > 64, or a one-warp unit: one stage buffer, the mirror follows its step
// after a second barrier — for one warp a __syncwarp)
#ifndef FT_STAGE2_MAXW
#define FT_STAGE2_MAXW 4
#endif
__host__ __device__ inline int ft_stage_bufs(int nwarp) { return nwarp >= 2 && nwarp <= FT_STAGE2_MAXW ? 2 : 1; }
__host__ __device__ inline size_t ft_vec_bytes(int P, int nwarp, int subs) {
  return (size_t)2 * subs * ft_vec_elems(P, nwarp * FT_RPT) * 16;
}
__host__ __device__ inline size_t ft_unit_smem(int P, int nwarp, int subs, size_t esz) {
  return ft_vec_bytes(P, nwarp, subs) + ft_tot_bytes(nwarp) + ft_gcol_bytes() +
         (size_t)ft_stage_bufs(nwarp) * nwarp * FT_RPT * 32 * esz;
}

__device__ __forceinline__ void ft_unit_sync(int id, int nthreads) {
  if (nthreads == 32)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One complex store under a predicate (no branch: the walk's stores sit in
// straight-line code); CS: evict-first (packed R is written once, never re-read)
template <bool CS>
__device__ __forceinline__ void ft_store(double2* p, double2 v, unsigned on) {
  if constexpr (CS)
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cs.v2.f64 [%1], {%2, %3}; }" ::"r"(on), "l"(p),
                 "d"(v.x), "d"(v.y)
                 : "memory");
  else
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.v2.f64 [%1], {%2, %3}; }" ::"r"(on), "l"(p),
                 "d"(v.x), "d"(v.y)
                 : "memory");
}
template <bool CS>
__device__ __forceinline__ void ft_store(float2* p, float2 v, unsigned on) {
  if constexpr (CS)
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cs.v2.f32 [%1], {%2, %3}; }" ::"r"(on), "l"(p),
                 "f"(v.x), "f"(v.y)
                 : "memory");
  else
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.v2.f32 [%1], {%2, %3}; }" ::"r"(on), "l"(p),
                 "f"(v.x), "f"(v.y)
                 : "memory");
}

// f += a (x) conj(b) - c (x) conj(d), accumulated with FMAs in double
__device__ __forceinline__ void ft_rank2(double2& f, double2 a, double2 b, double2 c, double2 d) {
  f.x = fma(a.x, b.x, f.x);
  f.x = fma(a.y, b.y, f.x);
  f.x = fma(-c.x, d.x, f.x);
  f.x = fma(-c.y, d.y, f.x);
  f.y = fma(a.y, b.x, f.y);
  f.y = fma(-a.x, b.y, f.y);
  f.y = fma(-c.y, d.x, f.y);
  f.y = fma(c.x, d.y, f.y);
}

// k_corners_d: the corner layout above, thread per element
template <typename T>
__global__ void k_corners_d(const typename CT<T>::c* __restrict__ A, Problem pr, int B, int PP,
                            double2* __restrict__ C) {
  const int P = pr.P, S = P - 1, Wc = pr.Q - 1, cw = ft_colw(P, PP);
  const long long per = (long long)Wc * cw;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= per * B) return;
  const int b = (int)(tid / per);
  const int j = (int)(tid % per / cw), x = (int)(tid % cw);
  int blk, i;
  if (x < 4 * PP) {
    blk = x / PP;
    i = x % PP;
  } else {
    blk = (x - 4 * PP) / (2 * PP);
    i = (x - 4 * PP) % (2 * PP);
    i = i < 2 * P ? i % P : S;  // (beyond the doubled strip: zero)
  }
  double2 v = make_double2(0.0, 0.0);
  if (i < S) {
    const int row = (blk < 2 ? 0 : pr.N - S) + i;
    const int col = ((blk & 1) ? pr.M - Wc : 0) + j;
    const auto a = A[((long long)b * pr.N + row) * pr.M + col];
    v = make_double2((double)a.x, (double)a.y);
  }
  C[tid] = v;
}

// The two classes on circular diagonal c of column offset dc: (c, dc) on
// rows [0, P-c) and (c-P, dc) on rows [P-c, P) (dc > 0, c > 0 only)
struct FtLane {
  int slot1, slot2;  // plan slots (-1: absent)
  long long rc1, rc2, cl1, cl2, so1, so2;
};
__device__ inline FtLane ft_lane(int c, int dc, int P, int Q, const ClassDesc* __restrict__ cls,
                                 const int* __restrict__ cls_slot, int lo, int hi) {
  FtLane L{-1, -1, 0, 0, 0, 0, 0, 0};
  if (c < P) {
    int s = cls_slot[class_index(c, dc, P, Q)];
    if (s >= lo && s < hi) {
      L.slot1 = s;
      L.rc1 = cls[s].rc_off;
      L.cl1 = cls[s].ccol_off;
      L.so1 = cls[s].slot_off;
    }
    if (dc > 0 && c > 0) {
      s = cls_slot[class_index(c - P, dc, P, Q)];
      if (s >= lo && s < hi) {
        L.slot2 = s;
        L.rc2 = cls[s].rc_off;
        L.cl2 = cls[s].ccol_off;
        L.so2 = cls[s].slot_off;
      }
    }
  }
  return L;
}

// F(0) of entry (r1, (r1 + c) mod P): full_i(0) = RC'_i (top), RC'_{ar+i}
// (bottom) of the entry's class, i = v = the entry's slot row
__device__ inline void ft_init_entry(int r1, int c, int P, const FtLane& L, const double2* __restrict__ rcb,
                                     int nseg, double2& fT, double2& fB) {
  fT = fB = make_double2(0.0, 0.0);
  const int bnd = P - c;
  const bool seg1 = r1 < bnd;
  const int v = seg1 ? r1 : r1 - bnd, ar = seg1 ? P - c - 1 : c - 1;
  if (r1 >= P || (seg1 ? L.slot1 : L.slot2) < 0 || v >= ar) return;
  const double2* rcp = rcb + (seg1 ? L.rc1 : L.rc2) * nseg;
  if (nseg == 1) {  // one column segment: two plain loads (the 8 rows' loads of a thread go out together)
    fT = rcp[v];
    fB = rcp[ar + v];
    return;
  }
  for (int g = 0; g < nseg; ++g) {
    fT = cadd(fT, rcp[(long long)v * nseg + g]);
    fB = cadd(fB, rcp[(long long)(ar + v) * nseg + g]);
  }
}

#ifndef FT_MINB
#define FT_MINB 2
#endif
#ifndef FT_DENSE_CS
#define FT_DENSE_CS true  // dense R's stores evict-first as well
#endif
// DELTA: unit = (snapshots, dc, band, chunk [16 (j-1), 16 j)); the chunk's
// state updates from zero go to ck[b][dc][j-1][T, B][row][c] (no output).
// LANES < 32: a warp holds 32 / LANES snapshots (lane = (snapshot, c)).
template <typename T, int NWARP, int LAYOUT, bool DELTA, int LANES>
__global__ void __launch_bounds__(FtCfg<NWARP>::THREADS, NWARP == 8 ? FT_MINB : 1)
    k_fin_tile(const double2* __restrict__ corners, Problem pr, int B, const ClassDesc* __restrict__ cls,
               const int* __restrict__ cls_slot, const int4* __restrict__ units, int nunits, int nclasses,
               int npart, const double2* __restrict__ ccpart, const double2* __restrict__ ccol,
               long long tot_ccol, const double2* __restrict__ rc, long long tot_rc, int nseg,
               double2* __restrict__ ck, typename CT<T>::c* __restrict__ R, long long r_bstride,
               double scale, int u_begin, int u_end, double2* __restrict__ wstate, int slot_lo, int slot_hi,
               int ckstep) {
  using C2 = typename CT<T>::c;
  constexpr int UPC = FtCfg<NWARP>::UPC, UT = 32 * NWARP, PP = NWARP * FT_RPT, SUBS = 32 / LANES;
  constexpr bool DENSE = LAYOUT == COVGPU_DENSE, PACKED = LAYOUT == COVGPU_PACKED;
  constexpr bool STAGE2 = NWARP >= 2 && NWARP <= FT_STAGE2_MAXW;  // double-buffered stage: the mirror runs one step later
  extern __shared__ __align__(16) unsigned char ft_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int us = warp / NWARP, w = warp - us * NWARP, ut = (int)threadIdx.x - us * UT;
  const int unit = blockIdx.x * UPC + us;
  if (unit >= nunits) return;  // unit-uniform: the barriers below involve only this unit
  const int4 un = units[unit];
  const int b0 = un.x, dc = un.y, d0 = un.z, u_lo = un.w & 0xffff, u_hi = un.w >> 16;
  const int P = pr.P, Q = pr.Q, ac = Q - dc - 1, Wc = Q - 1;
  // emitted steps of this launch; a unit resumed by a later u-chunk restores
  // the state the previous chunk saved, a fresh one starts from F(u_lo)
  const int e0 = max(u_lo, u_begin), e1 = min(u_hi, u_end);
  if (e0 >= e1) return;
  const bool resume = e0 > u_lo;
  constexpr int cw = 12 * PP, vstride = cw + 8;  // ft_colw, ft_vec_elems
  unsigned char* sb = ft_smem + (size_t)us * ft_unit_smem(P, NWARP, SUBS, sizeof(C2));
  double2* const vec = (double2*)sb;
  double2* const tot0 = (double2*)(sb + ft_vec_bytes(P, NWARP, SUBS));
  double2* const gcol0 = (double2*)(sb + ft_vec_bytes(P, NWARP, SUBS) + ft_tot_bytes(NWARP));
  C2* const stage0 = (C2*)(sb + ft_vec_bytes(P, NWARP, SUBS) + ft_tot_bytes(NWARP) + ft_gcol_bytes());
  const int bar = 1 + us;

  const int cl = lane & (LANES - 1), sub = lane / LANES;
  const int b = b0 + sub;  // this lane's snapshot
  const int c = d0 + cl;   // this lane's circular diagonal
  const FtLane L = b < B ? ft_lane(c, dc, P, Q, cls, cls_slot, slot_lo, slot_hi) : FtLane{-1, -1, 0, 0, 0, 0, 0, 0};
  const int bnd = P - c;  // first row of segment 2
  const int r0 = w * FT_RPT;
  const int pv1 = P - c, pv2 = c;
  const int bs = b < B ? b : B - 1;  // (index math of idle lanes in range)
  unsigned omask = 0;
#pragma unroll
  for (int k = 0; k < FT_RPT; ++k) {
    const int r1 = r0 + k;
    if (r1 < P && ((r1 < bnd) ? L.slot1 : L.slot2) >= 0) omask |= 1u << k;
  }
  const int r2_0 = (r0 + c) % P;  // second A row of row r0 (rows r0 + k: r2_0 + k in the doubled strip)
  // mirror writer: lane l handles the lane m of its snapshot with c(m) = d0 + LANES-1 - cl
  const int m = sub * LANES + (LANES - 1 - cl), cm = d0 + LANES - 1 - cl;
  const bool m1 = __shfl_sync(0xffffffffu, L.slot1, m) >= 0 && (dc > 0 || cm > 0);
  const bool m2 = __shfl_sync(0xffffffffu, L.slot2, m) >= 0;
  unsigned mmask = 0;
  const int msrc0 = cm < P ? ((r0 - cm) % P + P) % P : 0;  // mirror row r0 + k: source row (msrc0 + k) mod P
#pragma unroll
  for (int k = 0; k < FT_RPT; ++k) {
    const int r2 = r0 + k, src = (msrc0 + k) % P;
    if (cm < P && r2 < P && (src < P - cm ? m1 : m2)) mmask |= 1u << k;
  }
  const bool wout = __any_sync(0xffffffffu, omask != 0);
  const bool wmir = DENSE && __any_sync(0xffffffffu, mmask != 0);
  const double2* clb = ccol + (long long)bs * tot_ccol;
  double* const wsp = wstate ? (double*)(wstate + ((long long)unit * UT + ut) * FT_STATE) : nullptr;

  double2 fT[FT_RPT], fB[FT_RPT], G1 = make_double2(0.0, 0.0), G2 = G1;
  const long long per = (long long)P * P;
  const double2* ckb = ck + ((long long)bs * Q + dc) * ft_nck(Q, ckstep) * 2 * per + c;
  if (DELTA) {
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) fT[k] = fB[k] = make_double2(0.0, 0.0);
  } else if (resume) {
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) {
      fT[k] = make_double2(wsp[4 * k], wsp[4 * k + 1]);
      fB[k] = make_double2(wsp[4 * k + 2], wsp[4 * k + 3]);
    }
    G1 = make_double2(wsp[4 * FT_RPT], wsp[4 * FT_RPT + 1]);
    G2 = make_double2(wsp[4 * FT_RPT + 2], wsp[4 * FT_RPT + 3]);
  } else {
    // F(u_lo) = F(0) + (delta_1 + ... + delta_j), j = u_lo / ckstep: the
    // chunk updates are already summed in chunk order (k_ck_scan)
    const double2* rcb = rc + (long long)bs * tot_rc * nseg;
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) ft_init_entry(r0 + k, c, P, L, rcb, nseg, fT[k], fB[k]);
    if (u_lo > 0) {
      const double2* cj = ckb + (long long)(u_lo / ckstep - 1) * 2 * per;
#pragma unroll
      for (int k = 0; k < FT_RPT; ++k) {
        const int r1 = r0 + k;
        if (r1 < P && c < P) {
          fT[k] = cadd(fT[k], cj[(long long)r1 * P]);
          fB[k] = cadd(fB[k], cj[per + (long long)r1 * P]);
        }
      }
    }
    // G(u_lo) = CC + sum_{j < u_lo} CColR[j] + sum_{u_lo <= j < ac} CColL[j]
    // per class (the walk's G(0) plus its first u_lo updates): warp w adds
    // columns j = w (mod NWARP), the partials meet in SMEM (fixed order)
    double2 g1 = make_double2(0.0, 0.0), g2 = g1;
    if (w == 0) {
      for (int k = 0; k < npart; ++k) {
        if (L.slot1 >= 0) g1 = cadd(g1, ccpart[((long long)bs * nclasses + L.slot1) * npart + k]);
        if (L.slot2 >= 0) g2 = cadd(g2, ccpart[((long long)bs * nclasses + L.slot2) * npart + k]);
      }
    }
#pragma unroll 8
    for (int j = w; j < ac; j += NWARP) {
      const int o = j < u_lo ? ac + j : j;
      if (L.slot1 >= 0) g1 = cadd(g1, clb[L.cl1 + o]);
      if (L.slot2 >= 0) g2 = cadd(g2, clb[L.cl2 + o]);
    }
    tot0[w * 32 + lane] = g1;
    tot0[(NWARP + w) * 32 + lane] = g2;
    ft_unit_sync(bar, UT);
    for (int x = 0; x < NWARP; ++x) {
      G1 = cadd(G1, tot0[x * 32 + lane]);
      G2 = cadd(G2, tot0[(NWARP + x) * 32 + lane]);
    }
  }
  ft_unit_sync(bar, UT);  // tot0 is reused by the steps
  for (int e = ut; e < 2 * 4 * 32; e += UT) gcol0[e] = make_double2(0.0, 0.0);            // absent classes stay 0
  for (int e = ut; e < 2 * SUBS * vstride; e += UT) vec[e] = make_double2(0.0, 0.0);  // slack zeros
  ft_unit_sync(bar, UT);

  // one step's strip columns: the column-u and column-(u+dc) runs of the
  // corner layout (ft_colw), one contiguous copy per snapshot; copied by the
  // snapshot's own lanes (id = w * LANES + cl), plus each lane's CColL /
  // CColR of its two classes (gcol [class][L, R][lane], warp x % NWARP)
  const double2* cb = corners + (long long)bs * Wc * cw;
  const int cid = w * LANES + cl;
  auto prefetch = [&](int uu, int buf) {
    if (uu < ac && uu < e1) {
      double2* dst = vec + (buf * SUBS + sub) * vstride;
      if (b < B) {
        const double2* srcA = cb + (long long)uu * cw;
        const double2* srcB = cb + (long long)(uu + dc) * cw;
        for (int j = cid; j < cw; j += NWARP * LANES)
          cp_async_elem<16>(dst + j, (j < 4 * PP ? srcA : srcB) + j, true);
      }
      if (!DELTA) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const long long co = x < 2 ? L.cl1 : L.cl2;
          if (w == x % NWARP && (x < 2 ? L.slot1 : L.slot2) >= 0)
            cp_async_elem<16>(gcol0 + buf * 128 + x * 32 + lane, clb + co + ((x & 1) ? ac : 0) + uu, true);
        }
      }
    }
    cp_async_commit();
  };
  int u = e0;
  prefetch(u, u & 1);
  const double2* const vbase = vec + sub * vstride + r0;  // this thread's rows of buffer 0

  const long long D = pr.PQ;
  C2* const Rb = R + (long long)bs * r_bstride;
  const bool zero_im = dc == 0 && c == 0;  // class (0,0): R's real main diagonal (rows < bnd = P)
  const long long ostep = (long long)P * (D + 1);  // block (u, u+dc) -> (u+1, u+1+dc)
  constexpr int P2 = 2 * PP;  // stride of the second-operand blocks
  // rows k >= kb of this thread belong to segment 2 (the second class; the
  // block column wraps from P-1 to 0 there).  wstr: some lane of the warp
  // holds rows of both segments (a function of the geometry only)
  const int kb = bnd - r0;
  const bool wstr = __any_sync(0xffffffffu, kb > 0 && kb < FT_RPT);
  const int col0 = (r0 + c) % P;  // block column of row r0
  const int kbw = kb > 0 ? kb : FT_RPT;  // rows k >= kbw wrap to column col0 + k - P (kb <= 0: col0 is already wrapped)
  const int mwrap = P - msrc0;           // mirror rows k >= mwrap read source row msrc0 + k - P
  // warp-uniform row pointers, stepped by ostep per step: the emitted row
  // P u + r0 of block (u, u+dc) and the mirrored row P (u+dc) + r0 of block (u+dc, u)
  C2* rowp = Rb + ((long long)P * e0 + r0) * D + (long long)P * (e0 + dc);
  C2* mrowp = Rb + ((long long)P * (e0 + dc) + r0) * D + (long long)P * e0;
  // mirror of the step whose rows start at mrow: lower-block row r0 + k takes
  // the conjugate of source row (msrc0 + k) mod P of diagonal cm (the lower
  // triangle = exact conjugate of the upper)
  auto mirror = [&](C2* mrow, int buf) {
    const C2* stg = stage0 + (STAGE2 ? buf : 0) * PP * 32 + m;
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) {
      const int src = msrc0 + k - (k >= mwrap ? P : 0);
      C2 val = stg[src * 32];
      val.y = -val.y;
      ft_store<FT_DENSE_CS>(mrow + src, val, (mmask >> k) & 1u);
      mrow += D;
    }
  };
  // the walk over the thread's rows from O at its first row.  STR: the segment
  // switch is compiled in (warps without straddling lanes skip it); ZI: the
  // dc = 0 units hold class (0,0), whose imaginary part is written as exactly 0
  auto emit = [&](auto str, auto zi, double2 o1, double2 o2, int buf) {
    constexpr bool STR = decltype(str)::value, ZI = decltype(zi)::value;
    C2* const stg = stage0 + (STAGE2 ? buf : 0) * PP * 32 + r0 * 32 + lane;
    const long long k1 = (long long)P * u + r0;
    C2* rk;  // dense / packed: warp-uniform pointer of the row (the lane adds its column); compact: the lane's slot
    if constexpr (DENSE)
      rk = rowp;
    else if constexpr (PACKED)
      rk = Rb + (k1 * D - (k1 * (k1 - 1)) / 2 - k1 + (long long)P * (u + dc));
    else
      rk = Rb + (kb > 0 ? L.so1 + (long long)u * pv1 + r0 : L.so2 + (long long)u * pv2 + (r0 - bnd));
    double2 o = kb > 0 ? o1 : o2;
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) {
      int colk = col0 + k;
      if constexpr (STR) {
        if (k > 0 && k == kb) {
          o = o2;  // segment 2 starts: the second class's walk
          if constexpr (!DENSE && !PACKED) rk = Rb + L.so2 + (long long)u * pv2;
        }
        if (k > 0 && k >= kbw) colk -= P;
      }
      C2 val;
      val.x = (T)(o.x * scale);
      val.y = (T)(o.y * scale);
      if constexpr (ZI) {
        if (zero_im) val.y = (T)0;
      }
      const unsigned on = (omask >> k) & 1u;
      if constexpr (PACKED)
        ft_store<true>(rk + colk, val, on);
      else if constexpr (DENSE)
        ft_store<FT_DENSE_CS>(rk + colk, val, on);
      else
        ft_store<false>(rk, val, on);
      if constexpr (DENSE) stg[k * 32] = val;
      if (k + 1 < FT_RPT) {
        o = cadd(o, csub(fB[k], fT[k]));
        if constexpr (DENSE)
          rk += D;
        else if constexpr (PACKED)
          rk += D - 1 - (k1 + k);
        else
          rk += 1;
      }
    }
  };
  bool prev = false;  // the previous step emitted (its mirror is pending)
  for (; u < e1; ++u) {
    const int buf = u & 1;
    double2* const tot = tot0 + buf * 4 * NWARP * 32;
    if constexpr (!DELTA) {
      // row-group totals of the two segments (t: top states, b: bottom states)
      double2 t1 = make_double2(0.0, 0.0), b1 = t1, t2 = t1, b2 = t1;
      if (wstr) {
#pragma unroll
        for (int k = 0; k < FT_RPT; ++k) {
          if (k < kb) {
            t1 = cadd(t1, fT[k]);
            b1 = cadd(b1, fB[k]);
          } else {
            t2 = cadd(t2, fT[k]);
            b2 = cadd(b2, fB[k]);
          }
        }
        tot[w * 32 + lane] = t1;
        tot[(NWARP + w) * 32 + lane] = b1;
        tot[(2 * NWARP + w) * 32 + lane] = t2;
        tot[(3 * NWARP + w) * 32 + lane] = b2;
      } else {
        // one segment per lane: sum all rows, store under the lane's segment
#pragma unroll
        for (int k = 0; k < FT_RPT; ++k) {
          t1 = cadd(t1, fT[k]);
          b1 = cadd(b1, fB[k]);
        }
        const int sg = kb > 0 ? 0 : 2 * NWARP;
        tot[(sg + w) * 32 + lane] = t1;
        tot[(sg + NWARP + w) * 32 + lane] = b1;
        tot[(2 * NWARP - sg + w) * 32 + lane] = t2;  // (zeros: the lane has no rows of the other segment)
        tot[(3 * NWARP - sg + w) * 32 + lane] = b2;
      }
    }
    cp_async_wait<0>();  // this step's strip columns and edge-column sums
    ft_unit_sync(bar, UT);
    prefetch(u + 1, buf ^ 1);
    if (!DELTA && STAGE2 && DENSE && prev && wmir) mirror(mrowp - ostep, buf ^ 1);
    if (!DELTA && wout) {
      // O at the warp's first row of each segment: G + top rows from there
      // down + bottom rows above it (x < w: bottoms, x >= w: tops)
      double2 o1 = G1, o2 = G2;
#pragma unroll
      for (int x = 0; x < NWARP; ++x) {
        o1 = cadd(o1, tot[((x < w ? NWARP : 0) + x) * 32 + lane]);
        o2 = cadd(o2, tot[((x < w ? 3 * NWARP : 2 * NWARP) + x) * 32 + lane]);
      }
      if (dc == 0) {
        if (wstr)
          emit(std::true_type{}, std::true_type{}, o1, o2, buf);
        else
          emit(std::false_type{}, std::true_type{}, o1, o2, buf);
      } else {
        if (wstr)
          emit(std::true_type{}, std::false_type{}, o1, o2, buf);
        else
          emit(std::false_type{}, std::false_type{}, o1, o2, buf);
      }
    }
    prev = !DELTA;
    if constexpr (!DELTA && !STAGE2 && DENSE) {
      ft_unit_sync(bar, UT);
      if (wmir) mirror(mrowp, 0);
      prev = false;
    }
    rowp += ostep;
    mrowp += ostep;
    if (u < ac) {
      // every row (no guards): rows and entries outside the strip read zeros
      const double2* va = vbase + buf * (SUBS * vstride);
      const double2* vq = va + (4 * PP - r0) + r2_0;
#pragma unroll
      for (int k = 0; k < FT_RPT; ++k) {
        ft_rank2(fT[k], va[PP + k], vq[P2 + k], va[k], vq[k]);
        ft_rank2(fB[k], va[3 * PP + k], vq[3 * P2 + k], va[2 * PP + k], vq[2 * P2 + k]);
      }
      const double2* gc = gcol0 + buf * 128 + lane;
      G1 = cadd(G1, csub(gc[32], gc[0]));  // + CColR[u] - CColL[u]
      G2 = cadd(G2, csub(gc[96], gc[64]));
    }
  }
  cp_async_wait<0>();
  if constexpr (DELTA) {
    if (b < B) {
      double2* o = (double2*)ckb + (long long)(u_lo / ckstep) * 2 * per;
#pragma unroll
      for (int k = 0; k < FT_RPT; ++k) {
        const int r1 = r0 + k;
        if (r1 < P && c < P) {
          o[(long long)r1 * P] = fT[k];
          o[per + (long long)r1 * P] = fB[k];
        }
      }
    }
    return;
  }
  if (STAGE2 && DENSE && prev) {
    ft_unit_sync(bar, UT);
    if (wmir) mirror(mrowp - ostep, (e1 - 1) & 1);
  }
  if (wsp && e1 < u_hi) {
#pragma unroll
    for (int k = 0; k < FT_RPT; ++k) {
      wsp[4 * k] = fT[k].x;
      wsp[4 * k + 1] = fT[k].y;
      wsp[4 * k + 2] = fB[k].x;
      wsp[4 * k + 3] = fB[k].y;
    }
    wsp[4 * FT_RPT] = G1.x;
    wsp[4 * FT_RPT + 1] = G1.y;
    wsp[4 * FT_RPT + 2] = G2.x;
    wsp[4 * FT_RPT + 3] = G2.y;
  }
}

// k_ck_delta: the chunk updates of windows with P >= 32 as a register-tiled
// rank-2 update in R-block coordinates (the DELTA mode of k_fin_tile holds one
// circular diagonal per lane and re-reads the second operand per row: LSU
// bound).  Unit = (snapshot, dc, chunk, top / bottom strip); CTA = one 32 x 32
// sub-block of the P x P state, thread = 4 x 4 entries (r1, r2): per step 8
// first-operand and 8 second-operand loads feed 16 rank-2 updates.  Every
// entry takes the same FMA sequence as the walk (ft_rank2, steps ascending
// from zero): the values equal the DELTA mode's bitwise.  Output layout as
// there: ck[b][dc][j][T, B][r1][c], c = (r2 - r1) mod P.
constexpr int CKD_T = 4;     // tile side per thread
constexpr int CKD_SUB = 32;  // sub-block side per CTA (cfg5: 768 CTAs of 64 threads)
// SMEM: the chunk's strip columns [step][l1, h1, l2, h2][CKD_SUB] (l / h: left /
// right strip column, 1 / 2: rows r1 of column u / rows r2 of column u + dc);
// the second operands are stored tile-interleaved (entry e at (e % 4) (CKD_SUB / 4) +
// e / 4), so the threads of a tile row read consecutive values
__host__ __device__ inline size_t ckd_smem(int ckstep) { return (size_t)ckstep * 4 * CKD_SUB * sizeof(double2); }
__global__ void __launch_bounds__(256, 2)
    k_ck_delta(const double2* __restrict__ corners, int P, int Q, int PP, const int4* __restrict__ units, int nsub,
               int tw, double2* __restrict__ ck, int ckstep) {
  extern __shared__ __align__(16) unsigned char ckd_sm[];
  double2* const sm = (double2*)ckd_sm;
  const int ns2 = nsub * nsub;
  const int4 un = units[blockIdx.x / ns2];
  const int sb = blockIdx.x % ns2;
  const int rb1 = CKD_SUB * (sb / nsub), rb2 = CKD_SUB * (sb % nsub);  // (rb + 31 < PP: PP is a multiple of 32 >= P)
  const int b = un.x, dc = un.y, which = un.z, u0 = un.w & 0xffff, u1 = un.w >> 16;
  const int cw = 12 * PP;
  // first-operand blocks of the corner layout: [TL, TR, BL, BR][PP]; the
  // second operands of column u + dc are that column's first-operand blocks
  const double2* cb = corners + (long long)b * (Q - 1) * cw + (which ? 2 * PP : 0);
  for (int x = threadIdx.x; x < (u1 - u0) * 4 * CKD_SUB; x += blockDim.x) {
    const int e = x % CKD_SUB, blk = x / CKD_SUB % 4, st = x / (4 * CKD_SUB);
    const double2 v = __ldg(cb + (long long)(u0 + st + (blk >= 2 ? dc : 0)) * cw + ((blk & 1) ? PP : 0) +
                            (blk >= 2 ? rb2 : rb1) + e);
    sm[(st * 4 + blk) * CKD_SUB + (blk >= 2 ? (e % CKD_T) * (CKD_SUB / CKD_T) + e / CKD_T : e)] = v;
  }
  __syncthreads();
  const int ty = threadIdx.x / tw, tx = threadIdx.x % tw;
  const int r1 = rb1 + CKD_T * ty, r2 = rb2 + CKD_T * tx;
  if (ty >= tw || r1 >= P || r2 >= P) return;
  double2 f[CKD_T][CKD_T];
#pragma unroll
  for (int i = 0; i < CKD_T; ++i)
#pragma unroll
    for (int j = 0; j < CKD_T; ++j) f[i][j] = make_double2(0.0, 0.0);
  const double2* s1 = sm + CKD_T * ty;
  const double2* s2 = sm + 2 * CKD_SUB + tx;
#pragma unroll 2
  for (int u = u0; u < u1; ++u) {
    double2 l1[CKD_T], h1[CKD_T], l2[CKD_T], h2[CKD_T];
#pragma unroll
    for (int i = 0; i < CKD_T; ++i) {
      l1[i] = s1[i];
      h1[i] = s1[CKD_SUB + i];
      l2[i] = s2[i * (CKD_SUB / CKD_T)];
      h2[i] = s2[CKD_SUB + i * (CKD_SUB / CKD_T)];
    }
#pragma unroll
    for (int i = 0; i < CKD_T; ++i)
#pragma unroll
      for (int j = 0; j < CKD_T; ++j) ft_rank2(f[i][j], h1[i], h2[j], l1[i], l2[j]);
    s1 += 4 * CKD_SUB;
    s2 += 4 * CKD_SUB;
  }
  const long long per = (long long)P * P;
  double2* o = ck + ((((long long)b * Q + dc) * ft_nck(Q, ckstep) + u0 / ckstep) * 2 + which) * per;
#pragma unroll
  for (int i = 0; i < CKD_T; ++i)
#pragma unroll
    for (int j = 0; j < CKD_T; ++j) {
      const int a = r1 + i, e = r2 + j;
      if (a < P && e < P) o[(long long)a * P + (e >= a ? e - a : e - a + P)] = f[i][j];
    }
}

// The per-chunk state updates of one (snapshot, dc) summed in chunk order,
// in place: ck[j] <- delta_1 + ... + delta_{j+1}.  Thread per element of the
// [T, B][row][c] block; chunk j of column offset dc exists while
// (j + 1) ckstep < Q - dc.
__global__ void k_ck_scan(double2* __restrict__ ck, int B, int P, int Q, int ckstep) {
  const long long per2 = 2LL * P * P;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)B * Q * per2) return;
  const int dc = (int)(tid / per2 % Q);
  const int n = (Q - dc - 1) / ckstep;  // chunks with a cut after them
  double2* e = ck + (tid / per2) * ft_nck(Q, ckstep) * per2 + tid % per2;
  double2 acc = make_double2(0.0, 0.0);
  for (int j = 0; j < n; ++j) {
    acc = cadd(acc, e[(long long)j * per2]);
    e[(long long)j * per2] = acc;
  }
}

}  // namespace covgpu

// K3 — finalize.
//
// k_finalize_v (default, P <= 128): lanes own diagonal positions v; the warp
// walks u = 0 .. qu-1 carrying every edge row's full_i(u) in registers
// (full_i(u+1) = full_i(u) - pL_i[u] + pR_i[u]) and G(u) (G(u+1) = G(u) -
// CColL[u] + CColR[u]); at each u the whole column of slots follows the
// diagonal-segment recurrence S(0,u) = G(u) + sum_i fullT_i(u),
// S(v+1,u) = S(v,u) - fullT_v(u) + fullB_v(u): one segmented warp scan plus
// one reduction per column.  Classes with pv <= 16 pack 32/W snapshots per
// warp (W = pow2ceil(pv)-lane segments).  Corner reads come from the
// transposed corner blocks (k_corners), so lanes read consecutive addresses.
//
// k_finalize (P > 128): one warp per (snapshot, class), lanes own u.
//
// With a_r = pv-1 top/bottom edge rows and a_c = qu-1 left/right edge
// columns, slot (v, u) of the class is
//   S(v,u) = G(u) + sum_{i=v}^{a_r-1} fullT_i(u) + sum_{t<v} fullB_t(u)
//   G(u)   = CC + sum_{j>=u} CColL[j] + sum_{t<u} CColR[t]
//          = CC + sum_j CColL[j] + excl_prefix(CColR - CColL)(u)
//   full*_i(u) = RC_i + sum_{j>=u} pL_i[j] + sum_{t<u} pR_i[t]
//              = RC'_i + excl_prefix(pR_i - pL_i)(u),   RC'_i = full_i(0) (edge.cuh)
// where pL/pR are the row's corner products with the left/right edge columns
// (formed here, once each).  Lanes own u (32 per chunk).  Pass T walks the
// diagonal segment upward (v = a_r .. 0) accumulating top rows into an L2
// scratch; pass B walks downward (v = 0 .. a_r) adding bottom rows — the
// paper's "add the entering edge products, drop the leaving ones" — and
// writes the scaled result.
#pragma once

#include "common.cuh"

namespace covgpu {

constexpr int FIN_WARPS = 4;
constexpr int FINV_MAX_P = 128;
// complex64 walks with one row per lane (cfg4: short walks, latency-bound on
// the per-class sum reads): 6 CTAs per SM (80 registers) 0.249-0.253 ->
// 0.245-0.249 ms (within noise); 8 CTAs spill
#ifndef FIN_MINB_F1
#define FIN_MINB_F1 6
#endif
// CTAs per SM asked of ptxas (an explicit 1 would let it spend up to 255
// registers): the occupancy each instantiation reached without a hint
// (double KR = 2: 96 registers, 5 CTAs), except complex64 KR = 1 (above)
constexpr int fin_min_blocks(size_t tsize, int kr) {
  return (kr == 1 && tsize == 4) ? FIN_MINB_F1 : kr == 2 ? 5 : 4;
}

// Transposed corner blocks of A: C[b][k][j][ph], k = TL, TR, BL, BR, each
// (P-1) rows x (Q-1) columns of A (the only elements corner products read).
// Rows are stored permuted for k_finalize_v's rows-per-lane walk: row i sits
// at ph = (i % kr) * Wp + i / kr (Wp = ceil((P-1)/kr), column stride kr*Wp),
// so the lanes' reads of rows li*kr + k + s (fixed k, any shift s) are
// consecutive addresses while each lane still owns contiguous rows.
__host__ __device__ inline int corner_rows(int P, int kr) {
  const int S = P > 1 ? P - 1 : 0;
  return kr * ((S + kr - 1) / kr);
}
__host__ __device__ inline int corner_phys(int i, int P, int kr) {
  const int wp = corner_rows(P, kr) / kr;
  return (i % kr) * wp + i / kr;
}
template <typename T>
__global__ void k_corners(const typename CT<T>::c* __restrict__ A, Problem pr, int B, int kr,
                          typename CT<T>::c* __restrict__ C) {
  using C2 = typename CT<T>::c;
  const int S = pr.P - 1, Sp = corner_rows(pr.P, kr), Wc = pr.Q - 1, wp = Sp / kr;
  const long long per = 4LL * Sp * Wc;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= per * B) return;
  const int b = (int)(tid / per);
  long long r = tid % per;
  const int k = (int)(r / ((long long)Sp * Wc));
  r %= (long long)Sp * Wc;
  const int j = (int)(r / Sp), ph = (int)(r % Sp);
  const int i = (ph % wp) * kr + ph / wp;
  if (i >= S) {
    C2 z;
    z.x = z.y = (T)0;
    C[tid] = z;
    return;
  }
  const int row = (k < 2 ? 0 : pr.N - S) + i;
  const int col = ((k & 1) ? pr.M - Wc : 0) + j;
  C[tid] = A[((long long)b * pr.N + row) * pr.M + col];
}

__device__ inline double2 seg_sum(double2 v, int W) {
  for (int off = W >> 1; off > 0; off >>= 1) v = cadd(v, shfl_xor2(v, off));
  return v;
}

// inclusive suffix (toward higher lanes) and exclusive prefix scans inside
// aligned segments of W lanes; `total` = segment sum
__device__ inline double2 seg_suffix_incl(double2 v, int li, int W, double2* total) {
  double2 inc = v;
  for (int off = 1; off < W; off <<= 1) {
    double2 n;
    n.x = __shfl_down_sync(0xffffffffu, inc.x, off, W);
    n.y = __shfl_down_sync(0xffffffffu, inc.y, off, W);
    if (li + off < W) inc = cadd(inc, n);
  }
  total->x = __shfl_sync(0xffffffffu, inc.x, 0, W);
  total->y = __shfl_sync(0xffffffffu, inc.y, 0, W);
  return inc;
}
// inc += the value `off` lanes below, when that lane is in the segment: the
// shfl's own in-range predicate guards the adds (no selects of a zero)
__device__ inline void shfl_up_acc(double2& inc, int off, int segc) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 a0, a1, b0, b1;\n\t.reg .f64 t0, t1;\n\t"
      "mov.b64 {a0, a1}, %0;\n\t"
      "mov.b64 {b0, b1}, %1;\n\t"
      "shfl.sync.up.b32 a0|p, a0, %2, %3, -1;\n\t"
      "shfl.sync.up.b32 a1, a1, %2, %3, -1;\n\t"
      "shfl.sync.up.b32 b0, b0, %2, %3, -1;\n\t"
      "shfl.sync.up.b32 b1, b1, %2, %3, -1;\n\t"
      "mov.b64 t0, {a0, a1};\n\t"
      "mov.b64 t1, {b0, b1};\n\t"
      "@p add.f64 %0, %0, t0;\n\t"
      "@p add.f64 %1, %1, t1;\n\t}"
      : "+d"(inc.x), "+d"(inc.y)
      : "r"(off), "r"(segc));
}
__device__ inline double2 seg_prefix_excl(double2 v, int li, int W, double2* total) {
  (void)li;
  double2 inc = v;
  const int segc = (32 - W) << 8;
  for (int off = 1; off < W; off <<= 1) shfl_up_acc(inc, off, segc);
  total->x = __shfl_sync(0xffffffffu, inc.x, W - 1, W);
  total->y = __shfl_sync(0xffffffffu, inc.y, W - 1, W);
  return csub(inc, v);
}

// packed R (the host path's layout) is written once and not re-read on the
// device: evict-first stores (st.global.cs) — cfg5 packed finalize 0.171 ->
// 0.167-0.168 ms over two alternating runs; dense R keeps plain stores (its
// mirrored halves of a sector arrive from different walks and merge in L2:
// 0.210-0.214 plain vs 0.214-0.220 ms evict-first)
template <typename C2>
__device__ __forceinline__ void fin_store(C2* p, C2 v, bool stream) {
  if (stream) __stcs(p, v);
  else *p = v;
}

// task = (class, snapshot group); W = min(32, pow2ceil(pv)) lanes per snapshot
template <typename T, int KR, bool DIRECT, bool CONTIG>
__global__ void __launch_bounds__(FIN_WARPS * 32, fin_min_blocks(sizeof(T), KR))
    k_finalize_v(const typename CT<T>::c* __restrict__ corners, Problem pr,
                 const ClassDesc* __restrict__ cls, const int2* __restrict__ tasks, long long ntasks,
                 int nclasses, int ncb, int nrs, int B, const double2* __restrict__ ccpart,
                 const double2* __restrict__ ccol, long long tot_ccol, const double2* __restrict__ rc,
                 long long tot_rc, int nseg, typename CT<T>::c* __restrict__ R,
                 long long r_bstride, double scale, int dlayout, int u_begin, int u_end,
                 double2* __restrict__ wstate) {
  // R: compact (class-major) output, r_bstride elements per snapshot.
  // Columns [u_begin, u_end) of every walk: with wstate the walk state (fT,
  // fB, G per lane) is saved at u_end and restored at u_begin, so the walk can
  // run in u-chunks — R rows [P u_begin, P u_end) are complete after a chunk
  // (the host path copies them out while the next chunk runs)
  using C2 = typename CT<T>::c;
  const int lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * FIN_WARPS + (threadIdx.x >> 5);
  if (task >= ntasks) return;  // warp-uniform; no block barriers below
  const int2 tk = tasks[task];
  const ClassDesc c = cls[tk.x];
  const int pv = c.pv, qu = c.qu, ar = pv - 1, ac = qu - 1;
  if (u_begin >= qu) return;
  double2* ws = wstate ? wstate + (task * 32 + lane) * (2 * KR + 1) : nullptr;
  int W = 1;
  while (W < pv && W < 32) W <<= 1;
  const int li = lane & (W - 1);
  const int b_raw = tk.y * (32 / W) + lane / W;
  const bool active = b_raw < B;
  const int b = active ? b_raw : B - 1;
  constexpr int CKR = CONTIG ? KR : 1;  // corner row permutation (k_corners kr)
  const int Sx = corner_rows(pr.P, CKR), Wc = pr.Q - 1;
  const long long cstride = (long long)Sx * Wc;
  const C2* Cb = corners + (long long)b * 4 * cstride;
  (void)nrs;  // bulk row segments are off (nrs == 1): ccol holds whole-column sums
  const double2* cl = ccol + (long long)b * tot_ccol + c.ccol_off;
  const double2* rcc = rc + ((long long)b * tot_rc + c.rc_off) * nseg;

  // row ownership, kre = ceil(pv / W) <= KR rounds (classes with pv <= 32
  // run one).  CONTIG: lane li owns the contiguous rows v = li*kre + k (one
  // in-lane prefix + one segmented scan per column; the permuted corner
  // layout keeps each round's corner reads consecutive).  Otherwise rows are
  // strided, v = li + W k (one scan per round) — kept for dense R, whose
  // mirrored stores run markedly slower from the contiguous mapping (cfg5
  // 0.245 vs 0.214 ms, while compact / packed gain: 0.185 -> 0.163 ms)
  const int kre = min(KR, (pv + W - 1) / W);
  auto rowv = [&](int k) { return CONTIG ? li * kre + k : li + W * k; };
  double2 G, fT[KR], fB[KR];
  if (u_begin > 0) {
    // resume: the state saved by the previous chunk
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      fT[k] = ws[k];
      fB[k] = ws[KR + k];
    }
    G = ws[2 * KR];
  } else {
    // CC and G(0) = CC + sum_j CColL[j]
    const double2* cc_p = ccpart + ((long long)b * nclasses + tk.x) * ncb;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = li; k < ncb; k += W) acc = cadd(acc, cc_p[k]);
    for (int j = li; j < ac; j += W) acc = cadd(acc, cl[j]);
    G = seg_sum(acc, W);
    // edge-row state of the lane's rows
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int v = rowv(k);
      fT[k] = fB[k] = make_double2(0.0, 0.0);
      if (v < ar) {
        for (int g = 0; g < nseg; ++g) {
          fT[k] = cadd(fT[k], rcc[(long long)v * nseg + g]);
          fB[k] = cadd(fB[k], rcc[(long long)(ar + v) * nseg + g]);
        }
      }
    }
  }
  const bool zero_im = (c.d == 0);
  const int u_stop = min(qu, u_end);
  // incremental addressing (the per-slot 64-bit index products were a third
  // of the kernel's instructions): per row k, the corner pointers of column u
  // (o1) and u + dc (o2) step by Sx, the output offsets by one window column
  const long long cs = cstride;
  const C2* p1[KR];
  const C2* p2[KR];
  long long ro[KR], ro2[KR];
  int rk1[KR];
  const long long D = pr.PQ;
  const long long rb = (long long)b * r_bstride;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int v = rowv(k);
    p1[k] = Cb + (long long)u_begin * Sx + corner_phys(min(v, Sx - 1) + c.s1, pr.P, CKR);
    p2[k] = Cb + (long long)(u_begin + c.dc) * Sx + corner_phys(min(v, Sx - 1) + c.s2, pr.P, CKR);
    const long long k1 = (long long)pr.P * u_begin + c.s1 + v;
    rk1[k] = (int)k1;
    if constexpr (DIRECT) {
      if (dlayout == COVGPU_DENSE) {
        ro[k] = rb + k1 * (D + 1) + c.d;
        ro2[k] = rb + k1 * (D + 1) + (long long)c.d * D;
      } else {
        ro[k] = rb + packed_off(k1, k1 + c.d, D);
        ro2[k] = 0;
      }
    } else {
      ro[k] = rb + c.slot_off + (long long)u_begin * pv + v;
      ro2[k] = 0;
    }
  }
  const long long dstep = (long long)pr.P * (D + 1);
  const long long pstep0 = (long long)pr.P * D - (long long)pr.P * (pr.P - 1) / 2;
  for (int u = u_begin; u < u_stop; ++u) {
    // KR == 1: this column's corner / edge-column reads go out first, so
    // their latency overlaps the scan and the slot stores below (cfg3
    // finalize 0.058 -> 0.050 ms); with KR >= 2 the extra live registers cost
    // more occupancy than the overlap gains (cfg5 0.242 -> 0.277 ms), so the
    // reads stay next to their use
    const bool upd = u < ac;
    C2 q[8];
    double2 clr = make_double2(0.0, 0.0), cll = make_double2(0.0, 0.0);
    if constexpr (KR == 1) {
      if (upd) {
        if (li < ar) {
          const C2* a1 = p1[0];
          const C2* a2 = p2[0];
          q[0] = a1[cs];
          q[1] = a2[cs];
          q[2] = a1[0];
          q[3] = a2[0];
          q[4] = a1[3 * cs];
          q[5] = a2[3 * cs];
          q[6] = a1[2 * cs];
          q[7] = a2[2 * cs];
        }
        clr = cl[ac + u];
        cll = cl[u];
      }
    }
    // the diagonal-segment walk along v:  S(0) = G + sum_i fullT_i,
    // S(v+1) = S(v) - fullT_v + fullB_v  (drop the leaving edge row, add the
    // entering one) — one exclusive scan of (fB - fT) plus one reduction of fT
    double2 d[KR], tsum = make_double2(0.0, 0.0), run = make_double2(0.0, 0.0);
    double2 base = make_double2(0.0, 0.0);
    if constexpr (CONTIG) {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        d[k] = run;  // in-lane exclusive prefix
        if (k < kre) {
          run = cadd(run, csub(fB[k], fT[k]));
          tsum = cadd(tsum, fT[k]);
        }
      }
      double2 tot;
      base = seg_prefix_excl(run, li, W, &tot);
    } else {
      // rows li + W k: prefix over v = the earlier rounds' totals (all lanes)
      // + this round's exclusive lane prefix
#pragma unroll
      for (int k = 0; k < KR; ++k) tsum = cadd(tsum, fT[k]);
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        d[k] = run;
        if (k < kre) {
          double2 totk;
          d[k] = cadd(run, seg_prefix_excl(csub(fB[k], fT[k]), li, W, &totk));
          run = cadd(run, totk);
        }
      }
    }
    const double2 s0 = cadd(G, seg_sum(tsum, W));
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int v = rowv(k);
      if (k < kre && active && v < pv) {
        const double2 sv = cadd(s0, cadd(base, d[k]));
        C2 val;
        val.x = (T)(sv.x * scale);
        val.y = (T)(zero_im ? 0.0 : sv.y * scale);
        // DIRECT: dense / packed R straight from the walk (the scattered
        // diagonal stores merge in L2 well enough to beat a separate expand);
        // otherwise the compact slot (u-major, then v) for k_expand
        fin_store(R + ro[k], val, DIRECT && dlayout != COVGPU_DENSE);
        if constexpr (DIRECT) {
          if (dlayout == COVGPU_DENSE && !zero_im) {
            C2 cv;
            cv.x = val.x;
            cv.y = -val.y;  // lower triangle = exact conjugate of the upper
            fin_store(R + ro2[k], cv, false);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if constexpr (DIRECT) {
        if (dlayout == COVGPU_DENSE) {
          ro[k] += dstep;
          ro2[k] += dstep;
        } else {
          ro[k] += pstep0 - (long long)pr.P * rk1[k];
          rk1[k] += pr.P;
        }
      } else {
        ro[k] += pv;
      }
    }
    if (upd) {
      // corner products of column u (left) and u + dc (right), each formed once
      if constexpr (KR == 1) {
        if (li < ar) {
          fT[0] = cadd(fT[0], csub(cmulconj<T>(q[0], q[1]), cmulconj<T>(q[2], q[3])));
          fB[0] = cadd(fB[0], csub(cmulconj<T>(q[4], q[5]), cmulconj<T>(q[6], q[7])));
        }
        G = cadd(G, csub(clr, cll));
      } else {
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int v = rowv(k);
          if (k < kre && v < ar) {
            const C2* a1 = p1[k];
            const C2* a2 = p2[k];
            fT[k] = cadd(fT[k], csub(cmulconj<T>(a1[cs], a2[cs]), cmulconj<T>(a1[0], a2[0])));
            fB[k] = cadd(fB[k], csub(cmulconj<T>(a1[3 * cs], a2[3 * cs]), cmulconj<T>(a1[2 * cs], a2[2 * cs])));
          }
        }
        G = cadd(G, csub(cl[ac + u], cl[u]));
      }
    }
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      p1[k] += Sx;
      p2[k] += Sx;
    }
  }
  if (ws && u_stop < qu) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      ws[k] = fT[k];
      ws[KR + k] = fB[k];
    }
    ws[2 * KR] = G;
  }
}

template <typename T>
__global__ void __launch_bounds__(FIN_WARPS * 32)
    k_finalize(const typename CT<T>::c* __restrict__ A, Problem pr, const ClassDesc* __restrict__ cls,
               int nclasses, int ncb, int nrs, const double2* __restrict__ ccpart,
               const double2* __restrict__ ccol, long long tot_ccol, const double2* __restrict__ rc,
               long long tot_rc, int nseg, double2* __restrict__ scratch, long long tot_slots,
               typename CT<T>::c* __restrict__ R, int layout, long long r_bstride, double scale,
               long long ntasks, int qmax) {
  using C2 = typename CT<T>::c;
  extern __shared__ double2 fsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * FIN_WARPS + w;
  if (task >= ntasks) return;  // no block-level barriers below
  const int ci = (int)(task % nclasses);
  const int b = (int)(task / nclasses);
  const ClassDesc c = cls[ci];
  const int N = pr.N, M = pr.M;
  const int qu = c.qu, pv = c.pv, ar = pv - 1, ac = qu - 1;
  double2* G = fsm + (size_t)w * 4 * qmax;  // per-warp region
  double2* run = G + qmax;
  double2* pl = run + qmax;
  double2* prr = pl + qmax;
  const C2* Ab = A + (long long)b * N * M;
  const double2* cc_p = ccpart + ((long long)b * nclasses + ci) * ncb;
  const double2* clb = ccol + ((long long)b * tot_ccol + c.ccol_off) * nrs;
  auto cl = [&](int j) {
    if (nrs == 1) return clb[j];
    double2 v = clb[(long long)j * nrs];
    for (int r = 1; r < nrs; ++r) v = cadd(v, clb[(long long)j * nrs + r]);
    return v;
  };
  const double2* rcc = rc + ((long long)b * tot_rc + c.rc_off) * nseg;
  double2* sl = scratch + (long long)b * tot_slots + c.slot_off;  // [v][u]
  const bool zero_im = (c.d == 0);  // class (0,0) feeds the real main diagonal

  // CC = fixed-order sum of the column-block partials
  double2 cc = make_double2(0.0, 0.0);
  for (int k = lane; k < ncb; k += 32) cc = cadd(cc, cc_p[k]);
  cc = warp_sum(cc);
  // G(u)
  double2 totl = make_double2(0.0, 0.0);
  for (int j = lane; j < ac; j += 32) totl = cadd(totl, cl(j));
  totl = warp_sum(totl);
  {
    double2 carry = cadd(cc, totl);
    for (int u0 = 0; u0 < qu; u0 += 32) {
      const int u = u0 + lane;
      const double2 q = u < ac ? csub(cl(ac + u), cl(u)) : make_double2(0.0, 0.0);
      double2 tot;
      const double2 ex = warp_excl_scan(q, &tot);
      if (u < qu) {
        G[u] = cadd(carry, ex);
        run[u] = make_double2(0.0, 0.0);
        sl[(long long)ar * qu + u] = G[u];  // slot v = a_r: no top-edge row
      }
      carry = cadd(carry, tot);
    }
  }

  // one edge row's contribution full_i(u), u = u0 + lane, for all u-chunks:
  // products into pl/prr, then scan; returns via callback per chunk
  auto edge_row = [&](int i, double2 rcv, auto&& consume) {
    for (int j = lane; j < ac; j += 32) {
      const double2 a = cmulconj<T>(Ab[(long long)(i + c.s1) * M + j], Ab[(long long)(i + c.s2) * M + j + c.dc]);
      const int jr = pr.bw + j;
      const double2 bb =
          cmulconj<T>(Ab[(long long)(i + c.s1) * M + jr], Ab[(long long)(i + c.s2) * M + jr + c.dc]);
      pl[j] = a;
      prr[j] = bb;
    }
    __syncwarp();
    double2 carry = rcv;  // RC' = full_i(0) (edge.cuh)
    for (int u0 = 0; u0 < qu; u0 += 32) {
      const int u = u0 + lane;
      const double2 q = u < ac ? csub(prr[u], pl[u]) : make_double2(0.0, 0.0);
      double2 tot;
      const double2 ex = warp_excl_scan(q, &tot);
      if (u < qu) consume(u, cadd(carry, ex));
      carry = cadd(carry, tot);
    }
    __syncwarp();
  };
  auto rc_sum = [&](int k) {
    double2 s = make_double2(0.0, 0.0);
    for (int g = 0; g < nseg; ++g) s = cadd(s, rcc[(long long)k * nseg + g]);
    return s;
  };

  // pass T: v = a_r-1 .. 0
  for (int i = ar - 1; i >= 0; --i) {
    edge_row(i, rc_sum(i), [&](int u, double2 f) {
      const double2 acc = cadd(run[u], f);
      run[u] = acc;
      sl[(long long)i * qu + u] = cadd(G[u], acc);
    });
  }
  // pass B: v = 1 .. a_r, final values
  const long long rb = (long long)b * r_bstride;
  auto emit = [&](int v, int u, double2 s) {
    write_slot<T>(R, layout, rb, c, pr, v, u, s.x * scale, zero_im ? 0.0 : s.y * scale);
  };
  for (int u = lane; u < qu; u += 32) {
    run[u] = make_double2(0.0, 0.0);
    emit(0, u, sl[u]);
  }
  for (int t = 0; t < ar; ++t) {
    edge_row(pr.bh + t, rc_sum(ar + t), [&](int u, double2 f) {
      const double2 acc = cadd(run[u], f);
      run[u] = acc;
      emit(t + 1, u, cadd(sl[(long long)(t + 1) * qu + u], acc));
    });
  }
}

// K4 — scatter a class-major compact shard into the dense Hermitian R
// (the root's side of the multi-GPU gather; CovarianceMatrix.dense(),
// core.py:170-176, for a shard).  Thread per compact slot.
template <typename T>
__global__ void k_scatter_compact(const typename CT<T>::c* __restrict__ compact, Problem pr,
                                  const ClassDesc* __restrict__ cls, int nclasses, long long per_b,
                                  int B, typename CT<T>::c* __restrict__ R) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= per_b * B) return;
  const int b = (int)(tid / per_b);
  const long long s = tid % per_b;
  int lo = 0, hi = nclasses - 1;  // class whose slot range holds s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cls[mid].slot_off <= s) lo = mid; else hi = mid - 1;
  }
  const ClassDesc c = cls[lo];
  const long long r = s - c.slot_off;
  const int u = (int)(r / c.pv), v = (int)(r % c.pv);
  const auto val = compact[tid];
  write_slot<T>(R, COVGPU_DENSE, (long long)b * pr.PQ * pr.PQ, c, pr, v, u, (double)val.x,
                (double)val.y);
}

// K5 — expand the compact (class-major) result into the dense Hermitian R or
// the packed upper triangle with coalesced stores: thread per output element
// (k1, k2) reads its slot — class (dr, dc) = (k2%P - k1%P, k2/P - k1/P),
// u = k1/P, v = k1%P - s1 — from the L2-resident compact buffer.
// uc_off[uc] is the class's compact offset (-1: class not in this plan's
// shard -> element untouched).  (A P x P-block SMEM-transpose variant was
// measured no faster on B200: cfg5 0.155 vs 0.146 ms, cfg4 0.29 vs 0.12 ms.)
template <typename T>
__global__ void k_expand(const typename CT<T>::c* __restrict__ compact, long long cstride,
                         const long long* __restrict__ uc_off, Problem pr, int B, int layout,
                         typename CT<T>::c* __restrict__ R) {
  using C2 = typename CT<T>::c;
  const long long D = pr.PQ;
  const long long per = layout == COVGPU_DENSE ? D * D : D * (D + 1) / 2;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= per * B) return;
  const int b = (int)(tid / per);
  const long long e = tid % per;
  long long k1, k2;
  if (layout == COVGPU_DENSE) {
    k1 = e / D;
    k2 = e % D;
  } else {
    // packed row k1 starts at k1*D - k1(k1-1)/2: invert with a float guess + fix-up
    const double disc = (2.0 * D + 1.0) * (2.0 * D + 1.0) - 8.0 * (double)e;
    long long r = (long long)(((2.0 * D + 1.0) - sqrt(disc)) / 2.0);
    if (r < 0) r = 0;
    while (r > 0 && r * D - (r * (r - 1)) / 2 > e) --r;
    while ((r + 1) * D - ((r + 1) * r) / 2 <= e) ++r;
    k1 = r;
    k2 = k1 + (e - (k1 * D - (k1 * (k1 - 1)) / 2));
  }
  const bool lower = k2 < k1;
  const long long a = lower ? k2 : k1, c2 = lower ? k1 : k2;  // a <= c2
  const int P = pr.P, Q = pr.Q;
  const int ra = (int)(a % P), ca = (int)(a / P), rc = (int)(c2 % P), cc = (int)(c2 / P);
  const int dr = rc - ra, dc = cc - ca;
  const long long off = uc_off[class_index(dr, dc, P, Q)];
  if (off < 0) return;
  const int pv = P - abs(dr), s1 = dr < 0 ? -dr : 0;
  C2 val = compact[(long long)b * cstride + off + (long long)ca * pv + (ra - s1)];
  if (lower) val.y = -val.y;
  R[tid] = val;
}

// Reduce the partials of one execute into [CC | CCol | RC'] (one value per
// class / edge column / edge row): CC over the bulk kernel's npart partials,
// RC' over the edge-row kernel's nseg column segments, fixed order.
__global__ void k_reduce_sums(const double2* __restrict__ ccpart, int npart, long long ncc,
                              const double2* __restrict__ ccol, long long ncl,
                              const double2* __restrict__ rc, int nseg, long long nrc,
                              double2* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ncc) {
    double2 a = make_double2(0.0, 0.0);
    for (int g = 0; g < npart; ++g) a = cadd(a, ccpart[t * npart + g]);
    out[t] = a;
  } else if (t < ncc + ncl) {
    out[t] = ccol[t - ncc];
  } else if (t < ncc + ncl + nrc) {
    const long long r = t - ncc - ncl;
    double2 a = make_double2(0.0, 0.0);
    for (int g = 0; g < nseg; ++g) a = cadd(a, rc[r * nseg + g]);
    out[t] = a;
  }
}

}  // namespace covgpu

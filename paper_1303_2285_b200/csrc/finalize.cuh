// K3 — finalize: one warp per (snapshot, class).
//
// With a_r = pv-1 top/bottom edge rows and a_c = qu-1 left/right edge
// columns, slot (v, u) of the class is
//   S(v,u) = G(u) + sum_{i=v}^{a_r-1} fullT_i(u) + sum_{t<v} fullB_t(u)
//   G(u)   = CC + sum_{j>=u} CColL[j] + sum_{t<u} CColR[t]
//          = CC + sum_j CColL[j] + excl_prefix(CColR - CColL)(u)
//   full*_i(u) = RC_i + sum_{j>=u} pL_i[j] + sum_{t<u} pR_i[t]
//              = RC_i + sum_j pL_i[j] + excl_prefix(pR_i - pL_i)(u)
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

template <typename T>
__global__ void __launch_bounds__(FIN_WARPS * 32)
    k_finalize(const typename CT<T>::c* __restrict__ A, Problem pr, const ClassDesc* __restrict__ cls,
               int nclasses, int ncb, const double2* __restrict__ ccpart,
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
  const double2* cl = ccol + (long long)b * tot_ccol + c.ccol_off;
  const double2* rcc = rc + ((long long)b * tot_rc + c.rc_off) * nseg;
  double2* sl = scratch + (long long)b * tot_slots + c.slot_off;  // [v][u]
  const bool zero_im = (c.d == 0);  // class (0,0) feeds the real main diagonal

  // CC = fixed-order sum of the column-block partials
  double2 cc = make_double2(0.0, 0.0);
  for (int k = lane; k < ncb; k += 32) cc = cadd(cc, cc_p[k]);
  cc = warp_sum(cc);
  // G(u)
  double2 totl = make_double2(0.0, 0.0);
  for (int j = lane; j < ac; j += 32) totl = cadd(totl, cl[j]);
  totl = warp_sum(totl);
  {
    double2 carry = cadd(cc, totl);
    for (int u0 = 0; u0 < qu; u0 += 32) {
      const int u = u0 + lane;
      const double2 q = u < ac ? csub(cl[ac + u], cl[u]) : make_double2(0.0, 0.0);
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
    double2 tl = make_double2(0.0, 0.0);
    for (int j = lane; j < ac; j += 32) {
      const double2 a = cmulconj<T>(Ab[(long long)(i + c.s1) * M + j], Ab[(long long)(i + c.s2) * M + j + c.dc]);
      const int jr = pr.bw + j;
      const double2 bb =
          cmulconj<T>(Ab[(long long)(i + c.s1) * M + jr], Ab[(long long)(i + c.s2) * M + jr + c.dc]);
      pl[j] = a;
      prr[j] = bb;
      tl = cadd(tl, a);
    }
    tl = warp_sum(tl);
    __syncwarp();
    double2 carry = cadd(rcv, tl);
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

}  // namespace covgpu

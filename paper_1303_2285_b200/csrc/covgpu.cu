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
// CC (core x core) and CCol (edge columns x core rows) come from K1 (bulk.cuh),
// RC (edge rows x core columns) from K2 (edge.cuh); K3 (finalize.cuh) forms
// the corner products and walks each diagonal segment.  Shapes where the
// edge ranges overlap go to the SAT path (general.cuh).
//
// Every R element has a single writer; no atomics anywhere; all reductions
// run in a fixed order, so results are bitwise reproducible and independent
// of how classes are sharded across launches or GPUs.
// The C ABI (include/covgpu.h) is at the end of this file.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "bulk.cuh"
#include "common.cuh"
#include "edge.cuh"
#include "finalize.cuh"
#include "general.cuh"
#include "mma.cuh"
#include "probe.cuh"
#include "spectral.cuh"
#include "edgeblk.cuh"
#include "tile.cuh"
#include "snap.cuh"

using namespace covgpu;

namespace {

thread_local std::string g_last_error;

// The COVGPU_* environment switches (engine forcing, kernel variants) are
// test hooks: honoured only when COVGPU_TEST_HOOKS=1 is set (tests/conftest.py,
// bench.py's side runs, tools/); the product path reads no switch.
const char* hook_env(const char* name) {
  static const bool on = [] {
    const char* v = getenv("COVGPU_TEST_HOOKS");
    return v && atoi(v) != 0;
  }();
  return on ? getenv(name) : nullptr;
}

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

__global__ void k_warm(int* p) {
  if (threadIdx.x == 0 && p) *p = 1;
}

constexpr int kMaxCleanQ = 4096;
// direct core-sum work (batch (2P-1) Q N M) from which the spectral path is
// the default (below it the direct kernels' fewer launches win; measured on
// B200)
constexpr double kSpecMinWork = 1e8;  // per snapshot; cfg2 (3.3e7): direct 0.065 vs spectral 0.098 ms,
                                      // cfg4 (3.9e6 x 1024): 1.21 vs 2.04 ms; cfg3 (5.3e8): 0.225 vs 0.124 ms

}  // namespace

struct covgpu_plan {
  int device = 0;
  int dtype = COVGPU_C128;
  long long batch = 1;
  Problem pr{};
  bool clean = true;
  int E = 16;         // row lags per bulk warp
  int NW = 8;         // column lags (warps) per bulk CTA
  int bulk_variant = 0;
  bool use_tma = true;          // COVGPU_NO_TMA=1 forces the cp.async bulk kernel
  bool no_direct = false;       // COVGPU_NO_DIRECT=1: always finalize via compact + expand
  bool used_tma = false;
  const void* tmap_ptr = nullptr;  // A the cached tensor maps describe
  const void* tmap_kernel = nullptr;  // ... for this bulk kernel instance (box sizes)
  CUtensorMap tmx{}, tmy{};
  // FP64 tensor-core core sums (mma.cuh); CUDA-core bulk then covers only
  // the ncb_l + ncb_r column blocks that hold edge columns
  bool use_mma = false;
  int mma_dc = 64, n_drt = 0, n_dct = 0, mma_g = 0;
  int mma_kind = 1;  // 0: 4-DMMA complex tiles (k_bulk_dmma); 1-3: Gauss 3-DMMA (k_bulk_dmma3)
  int mtmap_kind = -1;
  int ncb_l = 0, ncb_r = 0;
  int edge_variant = 0;
  const void* mtmap_ptr = nullptr;
  CUtensorMap mtmx{}, mtmy{};
  // edge-column sums on the tensor cores too (Q <= 65): items x ecm_g CTAs
  bool use_ecm = false;
  int ecm_g = 1;
  long long ecm_items = 0;
  double2* d_ecm_part = nullptr;
  unsigned* d_ecm_tickets = nullptr;
  const void* ecm_ptr = nullptr;
  CUtensorMap ecm_tm{};
  // spectral core sums (spectral.cuh): row FFTs of length L = 2^spec_logL,
  // per-frequency row-lag correlation, output DFT; dr = 0 in the space domain
  bool use_snap = false;  // per-snapshot FP32 spectral sums (snap.cuh k_snap_spec)
  bool use_spec = false;
  int spec_logL = 0, spec_L = 0, spec_nseg = 1, spec_nfb = 1, spec_ngrp = 1;
  int spec_nd0 = 0;  // dr = 0 per-row partials (core rows)
  double2 *d_tw = nullptr, *d_fx = nullptr, *d_fy = nullptr, *d_gp = nullptr, *d_d0p = nullptr;
  SpecLayout spec_lay{};
  bool spec_smem = false;  // k_spec_corr_smem (P <= 64) instead of the L2-fed k_spec_corr
  int spec_e = 16;         // row lags per k_spec_corr_smem warp (16: up to 8 warps, 8: up to 16 warps)
  int spec_stages = 2;
  // symmetric core sums (spectral.cuh k_spec_fft modes 2 / 3): one spectrum per
  // row under one core-column mask, only the row lags dr >= 0 correlated; the
  // difference to CC is a correlation of the two 2Q-2 column strips (second,
  // small spectral problem: spec2_*), added as a second CC partial
  bool spec_sym = false;
  int spec2_logL = 0, spec2_nseg = 1;
  SpecLayout spec2_lay{};
  double2 *d_tw2 = nullptr, *d_twf2 = nullptr, *d_fx2 = nullptr, *d_fy2 = nullptr, *d_gp2 = nullptr;
  // spectral edge sums: column FFTs of length Lr = 2^spec_logLr (CCol), the
  // unmasked strip-row spectra (RC')
  bool spec_edges = false;
  int spec_logLr = 0;
  double2 *d_twr = nullptr, *d_fc = nullptr, *d_fy0 = nullptr;
  // full twiddle tables w_L^j / w_Lr^j for the output-pruned transforms
  double2 *d_twf = nullptr, *d_twrf = nullptr;
  bool spec_prune_q = false, spec_prune_p = false;  // Q <= 64 (row-spectrum pairs) / P <= 64 (column pairs)
  // edge sums by blocked short-lag correlation (edgeblk.cuh; the default):
  // block spectra of the strip columns / strip rows, twiddles of the block length
  bool spec_blk = false;
  EbGeom ebc{}, ebr{};
  double2 *d_ebc = nullptr, *d_ebr = nullptr, *d_twbc = nullptr, *d_twbr = nullptr;
  // edge-row sums on the tensor cores (P <= 65)
  // host path streaming A in row bands (batch 1, tensor-core path): the
  // copy stream bumps *d_band_flag after each band; k_bulk_dmma waits on it,
  // the side-stream kernels wait for ev_h2d (the whole of A)
  bool band_wait = false;
  // multi-GPU row bands (covgpu_plan_execute_sums): this execute computes
  // part ks_part of ks_nparts of every sum and reduces them into ks_out
  int ks_part = 0, ks_nparts = 1;
  bool ks_failed = false;
  double2* ks_out = nullptr;
  // finalize from reduced sums for a class range: cached task list
  int2* d_rtasks = nullptr;
  long long n_rtasks = 0;
  int rtask_lo = -1, rtask_hi = -1;
  unsigned* d_band_flag = nullptr;
  unsigned band_base = 0;
  int band_rows = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_h2d = nullptr;
  cudaEvent_t ev_strips = nullptr;  // spectral host path: edge columns + strip rows copied
  // spectral host path: one event per row band of A (recorded between the band
  // copies — unlike a stream memory operation it leaves no gap between two
  // DMA transfers: 16 bands x ~7 us at cfg5)
  std::vector<cudaEvent_t> ev_band;
  bool use_erm = false;
  int erm_dct = 1;
  const void* erm_ptr = nullptr;
  CUtensorMap erm_tmx{}, erm_tmy{};
  // edge-row kernel TMA variant (strips of >= 16 rows)
  bool edge_tma = false;
  int r2g = 1, n_r2g = 1;
  const void* etmap_ptr = nullptr;
  CUtensorMap etmx{}, etmy{};
  int D = 16;         // column lags per edge-row thread
  int ncb = 0;        // 32-column blocks
  int nrs = 1;        // bulk row segments (small problems: more CTAs)
  int n_drg = 0;      // bulk row-lag groups
  int n_dcb = 0;      // bulk column-lag blocks (NW lags each)
  int S = 0;          // edge strip height P-1
  int ndg = 0;        // edge-row column-lag groups
  int nseg = 1;       // edge-row column segments
  int nclasses = 0;   // selected classes
  std::vector<ClassDesc> h_cls;
  long long tot_rc = 0, tot_ccol = 0, tot_slots = 0;
  long long compact_elems = 0;
  int max_slots = 0;
  // device
  ClassDesc* d_cls = nullptr;
  int* d_cls_slot = nullptr;
  double2* d_ccpart = nullptr;
  double2* d_ccol = nullptr;
  double2* d_rc = nullptr;
  double2* d_slots = nullptr;
  double2* d_sat = nullptr;
  void* d_corners = nullptr;  // transposed corner blocks (k_corners)
  int2* d_tasks = nullptr;    // k_finalize_v tasks (class, snapshot group)
  std::vector<int2> h_tasks;
  long long* d_uc_off = nullptr;  // compact offset per UC index (-1: not in shard)
  long long ntasks = 0;
  int fin_kr = 0;             // k_finalize_v rows per lane (0: wide finalize)
  // tile finalize (tile.cuh): units (snapshot, dc, 32-diagonal band), longest walks first
  bool use_tile = false;
  int ft_nwarp = 1;
  int4* d_units = nullptr;
  long long n_units = 0;
  std::vector<int4> h_units;
  int4* d_runits = nullptr;   // class-range finalize: units holding a class of the range
  long long n_runits = 0;
  double2* d_ck = nullptr;    // per-chunk state updates delta_j (the tile kernel's DELTA mode), summed in chunk order
  int ft_ck = FT_CK;          // checkpoint spacing of the tile walk (ft_ckstep)
  int4* d_dunits = nullptr;   // DELTA-mode units (all classes) and for the class range
  long long n_dunits = 0;
  bool ck_tiled = false;      // chunk updates by k_ck_delta (P >= 32); d_dunits then holds its units
  int4* d_rdunits = nullptr;
  long long n_rdunits = 0;
  // chunked walk for the synchronous host path (covgpu_plan_execute_host):
  // u-chunk bounds, saved walk state, an event per chunk
  static constexpr int kMaxFinChunks = 4;
  int fin_nchunks = 1;
  int fin_ubound[kMaxFinChunks + 1] = {};
  double2* d_fin_state = nullptr;
  cudaEvent_t ev_fin_chunk[kMaxFinChunks] = {};
  cudaStream_t out_stream = nullptr;
  int sat_chunk = 0;
  long long ws_bytes = 0;
  size_t fin_smem = 0;
  int launches = 0;
  int spec_launches = 0;  // kernels launch_spectral enqueued (counted at the launch sites)
  // optional per-kernel timing of the last execute (events on its stream)
  bool timing = false;
  static constexpr int kMaxEv = 12;
  cudaEvent_t ev[kMaxEv] = {};
  const char* ev_name[kMaxEv] = {};  // kernel timed by the interval ending at ev[i]
  int nev = 0;
  // side stream for the edge-row / corner kernels (overlap with the bulk)
  cudaStream_t side_stream = nullptr;
  cudaStream_t delta_stream = nullptr;  // the walk's corner blocks / chunk updates (beside the edge sums)
  cudaStream_t cur_ds = nullptr;        // this execute's third stream (nullptr: none)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_djoin = nullptr;
  cudaEvent_t ev_d0 = nullptr;  // spectral: dr = 0 sums (side stream) done
  // end-to-end host path: cached stream and device buffers
  cudaStream_t host_stream = nullptr;
  void* hA = nullptr;
  void* hR = nullptr;
  size_t hA_bytes = 0, hR_bytes = 0;
  std::mutex host_mu;
  // streaming host path (covgpu_plan_execute_host_async): two slots of device
  // buffers, copy-in / compute (host_stream) / copy-out streams
  cudaStream_t as_in = nullptr, as_out = nullptr;
  void* asA[2] = {};
  void* asR[2] = {};
  size_t asA_bytes = 0, asR_bytes = 0;
  cudaEvent_t as_ev_in[2] = {}, as_ev_comp[2] = {}, as_ev_out[2] = {};
  long long as_n = 0;
  int as_err = 0;
  std::mutex exec_mu;  // executes mutate plan state (tensor-map cache, timing events)
  // the workspace is shared by every execute of the plan: an execute on a
  // stream other than the previous one's waits for it (event ev_done)
  cudaEvent_t ev_done = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // CUDA-graph replay of covgpu_plan_execute: the second call with the same
  // (A, R, layout, scale) captures the launch sequence (side-stream fork /
  // join included) on cap_stream; later identical calls launch the graph
  bool use_graph = true;  // COVGPU_NO_GRAPH=1: off
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const void* g_A = nullptr;
  void* g_R = nullptr;
  int g_layout = -1;
  double g_scale = 0.0;
  int g_hits = 0;
  // pipelined host path for batches: sub-batch plans, streams and buffers
  static constexpr int kPipeSlots = 3;
  covgpu_plan* pipe[kPipeSlots] = {};
  covgpu_plan* pipe_tail = nullptr;
  long long pipe_sub = 0, pipe_tail_b = 0;
  cudaStream_t pipe_stream[kPipeSlots] = {};
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  cudaEvent_t pipe_ev_in[kPipeSlots] = {}, pipe_ev_comp[kPipeSlots] = {}, pipe_ev_out[kPipeSlots] = {};
  void* pipe_A[kPipeSlots] = {};
  void* pipe_R[kPipeSlots] = {};
  size_t pipe_Ab = 0, pipe_Rb = 0;
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

void plan_free(covgpu_plan* pl);
void plan_free_pipe(covgpu_plan* pl) {
  for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
    if (pl->pipe[k]) {
      plan_free(pl->pipe[k]);
      delete pl->pipe[k];
      pl->pipe[k] = nullptr;
    }
    if (pl->pipe_stream[k]) cudaStreamDestroy(pl->pipe_stream[k]);
    pl->pipe_stream[k] = nullptr;
    cudaFree(pl->pipe_A[k]);
    cudaFree(pl->pipe_R[k]);
    pl->pipe_A[k] = pl->pipe_R[k] = nullptr;
  }
  if (pl->pipe_tail) {
    plan_free(pl->pipe_tail);
    delete pl->pipe_tail;
    pl->pipe_tail = nullptr;
  }
  pl->pipe_sub = pl->pipe_tail_b = 0;
  pl->pipe_Ab = pl->pipe_Rb = 0;
  if (pl->pipe_in) cudaStreamDestroy(pl->pipe_in);
  if (pl->pipe_out) cudaStreamDestroy(pl->pipe_out);
  pl->pipe_in = pl->pipe_out = nullptr;
  for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
    if (pl->pipe_ev_in[k]) cudaEventDestroy(pl->pipe_ev_in[k]);
    if (pl->pipe_ev_comp[k]) cudaEventDestroy(pl->pipe_ev_comp[k]);
    if (pl->pipe_ev_out[k]) cudaEventDestroy(pl->pipe_ev_out[k]);
    pl->pipe_ev_in[k] = pl->pipe_ev_comp[k] = pl->pipe_ev_out[k] = nullptr;
  }
}

void plan_free(covgpu_plan* pl) {
  plan_free_pipe(pl);
  for (auto& e : pl->ev)
    if (e) cudaEventDestroy(e);
  if (pl->host_stream) cudaStreamDestroy(pl->host_stream);
  if (pl->side_stream) cudaStreamDestroy(pl->side_stream);
  if (pl->delta_stream) cudaStreamDestroy(pl->delta_stream);
  if (pl->ev_djoin) cudaEventDestroy(pl->ev_djoin);
  if (pl->ev_fork) cudaEventDestroy(pl->ev_fork);
  if (pl->ev_join) cudaEventDestroy(pl->ev_join);
  if (pl->ev_d0) cudaEventDestroy(pl->ev_d0);
  cudaFree(pl->hA);
  cudaFree(pl->hR);
  cudaFree(pl->d_cls);
  cudaFree(pl->d_cls_slot);
  cudaFree(pl->d_ccpart);
  cudaFree(pl->d_ccol);
  cudaFree(pl->d_rc);
  cudaFree(pl->d_slots);
  cudaFree(pl->d_sat);
  cudaFree(pl->d_corners);
  cudaFree(pl->d_tasks);
  cudaFree(pl->d_units);
  cudaFree(pl->d_runits);
  cudaFree(pl->d_ck);
  cudaFree(pl->d_dunits);
  cudaFree(pl->d_rdunits);
  cudaFree(pl->d_uc_off);
  cudaFree(pl->d_ecm_part);
  cudaFree(pl->d_band_flag);
  cudaFree(pl->d_rtasks);
  if (pl->copy_stream) cudaStreamDestroy(pl->copy_stream);
  if (pl->ev_h2d) cudaEventDestroy(pl->ev_h2d);
  if (pl->ev_strips) cudaEventDestroy(pl->ev_strips);
  for (cudaEvent_t e : pl->ev_band)
    if (e) cudaEventDestroy(e);
  pl->ev_band.clear();
  cudaFree(pl->d_ecm_tickets);
  if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
  if (pl->ev_done) cudaEventDestroy(pl->ev_done);
  if (pl->cap_stream) cudaStreamDestroy(pl->cap_stream);
  if (pl->as_in) cudaStreamDestroy(pl->as_in);
  if (pl->as_out) cudaStreamDestroy(pl->as_out);
  for (int k = 0; k < 2; ++k) {
    cudaFree(pl->asA[k]);
    cudaFree(pl->asR[k]);
    if (pl->as_ev_in[k]) cudaEventDestroy(pl->as_ev_in[k]);
    if (pl->as_ev_comp[k]) cudaEventDestroy(pl->as_ev_comp[k]);
    if (pl->as_ev_out[k]) cudaEventDestroy(pl->as_ev_out[k]);
  }
  cudaFree(pl->d_fin_state);
  if (pl->out_stream) cudaStreamDestroy(pl->out_stream);
  for (auto& e : pl->ev_fin_chunk)
    if (e) cudaEventDestroy(e);
  cudaFree(pl->d_tw2);
  cudaFree(pl->d_twf2);
  cudaFree(pl->d_fx2);
  cudaFree(pl->d_fy2);
  cudaFree(pl->d_gp2);
  cudaFree(pl->d_tw);
  cudaFree(pl->d_fx);
  cudaFree(pl->d_fy);
  cudaFree(pl->d_gp);
  cudaFree(pl->d_d0p);
  cudaFree(pl->d_twr);
  cudaFree(pl->d_twf);
  cudaFree(pl->d_twrf);
  cudaFree(pl->d_fc);
  cudaFree(pl->d_fy0);
  cudaFree(pl->d_ebc);
  cudaFree(pl->d_ebr);
  cudaFree(pl->d_twbc);
  cudaFree(pl->d_twbr);
}

int pick_lags(int span) {
  if (span <= 4) return 4;
  if (span <= 8) return 8;
  return 16;
}

// Bulk kernel variants (row lags E, warps NW, min CTAs/SM): register
// budget vs occupancy.  FP64 E=8 x 2 CTAs keeps <= 128 registers so 16 warps
// hide the DFMA dependency latency; FP32 runs E=16.
struct BulkVariant {
  int E, NW, MINB;
};
constexpr BulkVariant kBulkVariants[] = {
    {4, 8, 2}, {8, 8, 2}, {16, 8, 1}, {8, 16, 1}, {16, 8, 2}, {16, 16, 1}, {16, 4, 2}, {8, 4, 2},
    {16, 4, 3}, {8, 4, 4},
};
constexpr int kNumBulkVariants = sizeof(kBulkVariants) / sizeof(kBulkVariants[0]);

// Bulk variant per shape, measured on B200 (tools/kt.py): 4 compute warps
// (column lags) per CTA and 2 CTAs/SM beat 8-warp CTAs for FP64; 16 row lags
// when the grid still has >= 6 waves (cfg5: bulk 9.09 -> 8.81 ms), else 8
// lags for more CTAs (cfg3 0.196 -> 0.174 ms, cfg2 0.036 -> 0.027 ms).  FP32
// keeps 8 warps x 8 lags on large grids (cfg4).  COVGPU_BULK_VARIANT
// overrides (tuning experiments).
int pick_bulk_variant(long long n, long long m, int p, int q, long long batch, int dtype) {
  (void)n;
  const int span = 2 * p - 1;
  auto waves = [&](int E, int NW, int MINB) {
    const long long ctas = batch * ((span + E - 1) / E) * (long long)((q + NW - 1) / NW) * ((m + 31) / 32);
    return (double)ctas / (148.0 * MINB);
  };
  int v;
  if (span <= 4)
    v = 0;  // E=4
  else if (dtype == COVGPU_C128)
    v = (span > 8 && waves(16, 4, 2) >= 6.0) ? 6 : 7;
  else
    v = waves(8, 8, 2) >= 6.0 ? 1 : 7;
  if (const char* env = hook_env("COVGPU_BULK_VARIANT")) {
    const int ev = atoi(env);
    if (ev >= 0 && ev < kNumBulkVariants) v = ev;
  }
  return v;
}

template <typename T, int E, int NW, int MINB>
cudaError_t bulk_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_bulk<T, E, NW, MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)BulkCfg<T, E, NW, MINB>::smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_bulk_tma<T, E, NW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)BulkCfg<T, E, NW, MINB>::smem_tma);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// A as a {2M, N, B} tensor of reals with a {bw, bh, 1} box.  width > 0: only
// `width` complex columns are in bounds (the rest read as zeros); col0 shifts
// the origin to complex column col0.
bool make_tmap(CUtensorMap* map, const void* A, bool fp64, long long B, long long N, long long M,
               int box_w, int box_h, long long width = -1, long long col0 = 0) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t esz = fp64 ? 8 : 4;
  if (width <= 0) width = M;
  A = (const char*)A + 2 * col0 * esz;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * width), (cuuint64_t)N, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)(2 * M) * esz, (cuuint64_t)(2 * M * N) * esz};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, fp64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
             const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T>
cudaError_t bulk_attrs() {
  cudaError_t e = cudaSuccess, r;
  if ((r = bulk_attr<T, 4, 8, 2>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 8, 8, 2>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 16, 8, 1>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 8, 16, 1>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 16, 8, 2>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 16, 16, 1>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 16, 4, 2>()) != cudaSuccess) e = r;
  if ((r = bulk_attr<T, 8, 4, 2>()) != cudaSuccess) e = r;
  if constexpr (sizeof(T) == 4) {  // FP32-only variants (FP64 tiles do not fit 3-4 CTAs/SM)
    if ((r = bulk_attr<T, 16, 4, 3>()) != cudaSuccess) e = r;
    if ((r = bulk_attr<T, 8, 4, 4>()) != cudaSuccess) e = r;
  }
  return e;
}

std::string g_attr_fail;  // the kernel whose attribute could not be set (error text)

template <typename T, int NW, int LANES>
cudaError_t fin_tile_attr() {
  // the largest window of this instantiation (P = 8 NW) needs the most SMEM
  const int smem = (int)(ft_unit_smem(8 * NW, NW, 32 / LANES, sizeof(typename CT<T>::c)) * FtCfg<NW>::UPC);
  g_attr_fail = "k_fin_tile<" + std::to_string(sizeof(T)) + "," + std::to_string(NW) + "> smem " + std::to_string(smem);
  cudaError_t e = cudaFuncSetAttribute(k_fin_tile<T, NW, COVGPU_DENSE, false, LANES>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaError_t r = cudaFuncSetAttribute(k_fin_tile<T, NW, COVGPU_PACKED, false, LANES>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (r != cudaSuccess) e = r;
  r = cudaFuncSetAttribute(k_fin_tile<T, NW, COVGPU_COMPACT, false, LANES>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (r != cudaSuccess) e = r;
  r = cudaFuncSetAttribute(k_fin_tile<T, NW, COVGPU_DENSE, true, LANES>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (r != cudaSuccess) e = r;
  if (e == cudaSuccess) g_attr_fail.clear();
  return e;
}
template <typename T>
cudaError_t fin_tile_attrs() {
  cudaError_t e = cudaSuccess, r;
  if ((r = fin_tile_attr<T, 1, 8>()) != cudaSuccess) return r;
  if ((r = fin_tile_attr<T, 2, 16>()) != cudaSuccess) return r;
  if ((r = fin_tile_attr<T, 4, 32>()) != cudaSuccess) return r;
  if ((r = fin_tile_attr<T, 8, 32>()) != cudaSuccess) return r;
  if ((r = fin_tile_attr<T, 16, 32>()) != cudaSuccess) return r;
  return e;
}

cudaError_t set_attrs() {
  static cudaError_t once = [] {
    cudaError_t e = bulk_attrs<double>();
    cudaError_t r = bulk_attrs<float>();
    if (r != cudaSuccess) e = r;
    if ((r = cudaFuncSetAttribute(k_finalize<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)MmaCfg<32>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)MmaCfg<64>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma3<2, 4, 2, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Mma3Cfg<2, 4, 2, 2, 2>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma3<4, 4, 2, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Mma3Cfg<4, 4, 2, 2, 1>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma3<2, 2, 2, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Mma3Cfg<2, 2, 2, 2, 2>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma3<4, 4, 2, 2, 1, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Mma3Cfg<4, 4, 2, 2, 1, true>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_bulk_dmma3<2, 4, 2, 2, 2, true, 8>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Mma3Cfg<2, 4, 2, 2, 2, true, 8>::smem)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_edge_cols_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ECM_SMEM)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_edge_rows_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ERM_SMEM)) != cudaSuccess)
      e = r;
    if ((r = cudaFuncSetAttribute(k_finalize<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024)) != cudaSuccess)
      e = r;
    if ((r = fin_tile_attrs<double>()) != cudaSuccess) e = r;
    if ((r = fin_tile_attrs<float>()) != cudaSuccess) e = r;

    return e;
  }();
  return once;
}

// ncb_l + ncb_r > 0: edge-only mode (TMA kernel only; the caller checked
// that the tensor maps can be made)
template <typename T, int E, int NW, int MINB>
void launch_bulk(covgpu_plan* pl, const typename CT<T>::c* A, cudaStream_t st, int ncb_l = 0,
                 int ncb_r = 0) {
  using Cfg = BulkCfg<T, E, NW, MINB>;
  const int n_drg = (2 * pl->pr.P - 1 + E - 1) / E, n_dcb = (pl->pr.Q + NW - 1) / NW;
  const int ncb = ncb_l + ncb_r > 0 ? ncb_l + ncb_r : pl->ncb;
  const long long units = (long long)n_drg * n_dcb * ncb * pl->nrs;  // CTAs per snapshot
  const long long blocks = pl->batch * units;
  const Problem& pr = pl->pr;
  // TMA needs 16-byte aligned rows: always for complex128, even M for complex64
  const bool tma_ok = pl->use_tma &&
                      ((uintptr_t)A % 16 == 0) && ((2LL * pr.M * sizeof(T)) % 16 == 0);
  if (tma_ok) {
    const void* kfn = (const void*)k_bulk_tma<T, E, NW, MINB>;
    if (pl->tmap_ptr != (const void*)A || pl->tmap_kernel != kfn) {
      CUtensorMap mx, my;
      if (make_tmap(&mx, A, sizeof(T) == 8, pl->batch, pr.N, pr.M, 2 * Cfg::XW, Cfg::RC) &&
          make_tmap(&my, A, sizeof(T) == 8, pl->batch, pr.N, pr.M, 2 * Cfg::YW, Cfg::YR)) {
        pl->tmx = mx;
        pl->tmy = my;
        pl->tmap_ptr = A;
        pl->tmap_kernel = kfn;
      } else {
        pl->tmap_ptr = nullptr;
      }
    }
    if (pl->tmap_ptr == (const void*)A) {
      // snapshots per CTA: keep ~2 waves of CTAs, stream the rest through the ring
      const long long slots = 148LL * MINB * 2;
      long long nsnap = std::max(1LL, (blocks + slots - 1) / slots);
      nsnap = std::min<long long>(nsnap, pl->batch);
      const long long groups = (pl->batch + nsnap - 1) / nsnap;
      k_bulk_tma<T, E, NW, MINB><<<(unsigned)(groups * units), (NW + 1) * 32, Cfg::smem_tma, st>>>(
          pl->tmx, pl->tmy, pr, n_drg, n_dcb, ncb, pl->nrs, pl->nclasses, (int)pl->batch,
          (int)nsnap, pl->d_cls_slot, pl->d_cls, pl->d_ccpart, pl->d_ccol, pl->tot_ccol, ncb_l, ncb_r);
      pl->used_tma = true;
      return;
    }
  }
  pl->used_tma = false;
  k_bulk<T, E, NW, MINB><<<(unsigned)blocks, NW * 32, Cfg::smem, st>>>(
      A, pr, n_drg, n_dcb, ncb, pl->nrs, pl->nclasses, pl->d_cls_slot, pl->d_cls, pl->d_ccpart,
      pl->d_ccol, pl->tot_ccol);
}

template <typename T>
void launch_bulk_variant(covgpu_plan* pl, const typename CT<T>::c* A, cudaStream_t st, int variant,
                         int ncb_l = 0, int ncb_r = 0) {
  switch (variant) {
    case 0: launch_bulk<T, 4, 8, 2>(pl, A, st, ncb_l, ncb_r); break;
    case 1: launch_bulk<T, 8, 8, 2>(pl, A, st, ncb_l, ncb_r); break;
    case 2: launch_bulk<T, 16, 8, 1>(pl, A, st, ncb_l, ncb_r); break;
    case 3: launch_bulk<T, 8, 16, 1>(pl, A, st, ncb_l, ncb_r); break;
    case 4: launch_bulk<T, 16, 8, 2>(pl, A, st, ncb_l, ncb_r); break;
    case 6: launch_bulk<T, 16, 4, 2>(pl, A, st, ncb_l, ncb_r); break;
    case 7: launch_bulk<T, 8, 4, 2>(pl, A, st, ncb_l, ncb_r); break;
    case 8:
      if constexpr (sizeof(T) == 4) {
        launch_bulk<T, 16, 4, 3>(pl, A, st, ncb_l, ncb_r);
        break;
      }
      launch_bulk<T, 16, 4, 2>(pl, A, st, ncb_l, ncb_r);
      break;
    case 9:
      if constexpr (sizeof(T) == 4) {
        launch_bulk<T, 8, 4, 4>(pl, A, st, ncb_l, ncb_r);
        break;
      }
      launch_bulk<T, 8, 4, 2>(pl, A, st, ncb_l, ncb_r);
      break;
    default: launch_bulk<T, 16, 16, 1>(pl, A, st, ncb_l, ncb_r);
  }
}

// FP64 tensor-core core sums; false when the tensor maps cannot describe A
// (the caller then runs the CUDA-core bulk over every column block)
template <int DC>
bool launch_dmma(covgpu_plan* pl, const double2* A, cudaStream_t st) {
  using Cfg = MmaCfg<DC>;
  const Problem& pr = pl->pr;
  if ((uintptr_t)A % 16 != 0) return false;
  if (pl->mtmap_ptr != (const void*)A || pl->mtmap_kind != 0) {
    CUtensorMap mx, my;
    const long long w = pr.M - pr.Q + 1;
    if (make_tmap(&mx, A, true, pl->batch, pr.N, pr.M, 2 * MMA_XP, MMA_XR, w, 0) &&
        make_tmap(&my, A, true, pl->batch, pr.N, pr.M, 2 * Cfg::YP, MMA_RC, w, pr.Q - 1)) {
      pl->mtmx = mx;
      pl->mtmy = my;
      pl->mtmap_ptr = A;
      pl->mtmap_kind = 0;
    } else {
      pl->mtmap_ptr = nullptr;
      return false;
    }
  }
  const long long blocks = pl->batch * (long long)pl->n_drt * pl->n_dct * pl->mma_g;
  k_bulk_dmma<DC><<<(unsigned)blocks, (MMA_WARPS + 1) * 32, Cfg::smem, st>>>(
      pl->mtmx, pl->mtmy, pr, pl->n_drt, pl->n_dct, pl->mma_g, pl->nclasses, pl->d_cls_slot,
      pl->d_ccpart, pl->band_wait ? pl->d_band_flag : nullptr, pl->band_base, pl->band_rows);
  return true;
}

// Gauss 3-DMMA core sums (k_bulk_dmma3); false when the tensor maps fail
template <int WM, int WN, int MT, int NTW, int MINB, bool PREP = false, int RC = MMA_RC>
bool launch_dmma3(covgpu_plan* pl, const double2* A, cudaStream_t st) {
  using Cfg = Mma3Cfg<WM, WN, MT, NTW, MINB, PREP, RC>;
  const Problem& pr = pl->pr;
  if ((uintptr_t)A % 16 != 0) return false;
  if (pl->mtmap_ptr != (const void*)A || pl->mtmap_kind != pl->mma_kind) {
    CUtensorMap mx, my;
    const long long w = pr.M - pr.Q + 1;
    if (make_tmap(&mx, A, true, pl->batch, pr.N, pr.M, 2 * MMA_XP, Cfg::XR, w, 0) &&
        make_tmap(&my, A, true, pl->batch, pr.N, pr.M, 2 * Cfg::YP, Cfg::RC, w, pr.Q - 1)) {
      pl->mtmx = mx;
      pl->mtmy = my;
      pl->mtmap_ptr = A;
      pl->mtmap_kind = pl->mma_kind;
    } else {
      pl->mtmap_ptr = nullptr;
      return false;
    }
  }
  const long long blocks = pl->batch * (long long)pl->n_drt * pl->n_dct * pl->mma_g;
  k_bulk_dmma3<WM, WN, MT, NTW, MINB, PREP, RC><<<(unsigned)blocks, (Cfg::WARPS + 1) * 32, Cfg::smem, st>>>(
      pl->mtmx, pl->mtmy, pr, pl->n_drt, pl->n_dct, pl->mma_g, pl->nclasses, pl->d_cls_slot,
      pl->d_ccpart, pl->band_wait ? pl->d_band_flag : nullptr, pl->band_base, pl->band_rows,
      pl->ks_part, pl->ks_nparts);
  return true;
}

// Pass-major twiddle table of an FFT of length 2^logL (spectral.cuh,
// spec_tw_off): w_{pR}^(r k) in long double, rounded once.
std::vector<double2> spec_twiddles(int logL) {
  std::vector<double2> t((size_t)1 << logL, make_double2(0.0, 0.0));
  const long double pi2 = 6.283185307179586476925286766559L;
  int p = 1, rem = logL;
  while (rem > 0) {
    const int lr = rem >= 3 ? 3 : rem, R = 1 << lr;
    if (p > 1) {
      const int off = spec_tw_off(logL, p);
      for (int r = 1; r < R; ++r)
        for (int k = 0; k < p; ++k) {
          const long double a = -pi2 * (long double)(r * k) / (long double)(p * R);
          t[(size_t)off + (size_t)(r - 1) * p + k] = make_double2((double)cosl(a), (double)sinl(a));
        }
    }
    p <<= lr;
    rem -= lr;
  }
  return t;
}

// G partial slots reserved for the banded correlation of the host path
constexpr int kMaxBandSlots = 32;
// rows per H2D band of the single-snapshot host path: ~9 bands, >= 64 rows (the band
// count is also the correlation's row-segment count: 64 f-blocks x 9 = 576 CTAs
// = 3.9 waves of 148, and fewer, longer segments than 16 — less per-CTA
// prologue / epilogue and G partial traffic: cfg5 step 0.463 -> 0.452 ms)
int host_band_rows(long long n) { return (int)std::max(64LL, (n + 8) / 9); }

// Spectral kernels are instantiated for FFT lengths 2^6 .. 2^12; SPEC_LOGL
// dispatches a launch on the runtime log2 length (SMEM attribute set once per
// instantiation: up to (L + L/8) complex values).
#define CUDA_TRY_V(expr) (void)(expr)

// cuStreamWaitValue32 through the runtime's driver entry point (no -lcuda)
PFN_cuStreamWaitValue32_v11070 stream_wait_value() {
  static PFN_cuStreamWaitValue32_v11070 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
  }();
  return fn;
}

template <typename K>
void spec_attr(K* fn, int logL) {
  // once per kernel instantiation (keyed on the function, not its type: the
  // LOGL instantiations of one kernel share a signature)
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  const void* f = (const void*)fn;
  if (std::find(done.begin(), done.end(), f) != done.end()) return;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 144 * 1024);
  done.push_back(f);
  (void)logL;
}
#define SPEC_LOGL(lg, KERNEL, GRID, ...)                                                        \
  do {                                                                                          \
    switch (lg) {                                                                               \
      case 6: SPEC_LAUNCH(6, KERNEL, GRID, __VA_ARGS__); break;                                 \
      case 7: SPEC_LAUNCH(7, KERNEL, GRID, __VA_ARGS__); break;                                 \
      case 8: SPEC_LAUNCH(8, KERNEL, GRID, __VA_ARGS__); break;                                 \
      case 9: SPEC_LAUNCH(9, KERNEL, GRID, __VA_ARGS__); break;                                 \
      case 10: SPEC_LAUNCH(10, KERNEL, GRID, __VA_ARGS__); break;                               \
      case 11: SPEC_LAUNCH(11, KERNEL, GRID, __VA_ARGS__); break;                               \
      default: SPEC_LAUNCH(12, KERNEL, GRID, __VA_ARGS__);                                      \
    }                                                                                           \
  } while (0)
#define SPEC_LAUNCH(LG, KERNEL, GRID, ...)                                                     \
  do {                                                                                          \
    auto fn_ = KERNEL<LG>();                                                                    \
    spec_attr(fn_, LG);                                                                         \
    const long long items_ = (long long)(GRID);                                                 \
    fn_<<<(unsigned)((items_ + spec_g<LG>() - 1) / spec_g<LG>()), spec_threads<LG>(),           \
          sizeof(double2) * spec_g<LG>() * spec_sb_elems<LG>(), st>>>(items_, __VA_ARGS__);     \
    ++pl->spec_launches;                                                                        \
  } while (0)

template <typename T>
struct SpecK {
  template <int LG>
  static auto fft() { return &k_spec_fft<T, LG>; }
  template <int LG>
  static auto colfft() { return &k_spec_colfft<T, LG>; }
  template <int LG>
  static auto dft() { return &k_spec_dft<LG>; }
  template <int LG>
  static auto ccol() { return &k_spec_ccol<LG>; }
  template <int LG>
  static auto rc() { return &k_spec_rc<LG>; }
  template <int LG>
  static auto rowac() { return &k_spec_rowac<LG>; }
  // output-pruned variants (first 64 outputs; L >= 512, else the full FFT)
  template <int LG>
  static auto rcp() {
    if constexpr (LG >= SPEC_LOGOUT + 3) return &k_spec_rc<LG, true>; else return &k_spec_rc<LG, false>;
  }
  template <int LG>
  static auto rowacp() {
    if constexpr (LG >= SPEC_LOGOUT + 3) return &k_spec_rowac<LG, true>; else return &k_spec_rowac<LG, false>;
  }
  template <int LG>
  static auto fftac() { return &k_spec_fft_ac<T, LG, false>; }
  template <int LG>
  static auto fftacp() {
    if constexpr (LG >= SPEC_LOGOUT + 3) return &k_spec_fft_ac<T, LG, true>; else return &k_spec_fft_ac<T, LG, false>;
  }
  template <int LG>
  static auto dftp() {
    if constexpr (LG >= SPEC_LOGOUT + 3) return &k_spec_dft<LG, true>; else return &k_spec_dft<LG, false>;
  }
  template <int LG>
  static auto ccolp() {
    if constexpr (LG >= SPEC_LOGOUT + 3) return &k_spec_ccol<LG, true>; else return &k_spec_ccol<LG, false>;
  }
};

// edge sums by blocked short-lag correlation (edgeblk.cuh): block spectra of
// one strip family (cols: the edge columns -> CCol; else the edge rows -> RC'),
// then the line-pair tiles of this part
template <typename T>
void launch_edges_blocked(covgpu_plan* pl, const typename CT<T>::c* A, cudaStream_t st, bool cols, int part,
                          int nparts) {
  const Problem& pr = pl->pr;
  const long long B = pl->batch;
  const EbGeom& g = cols ? pl->ebc : pl->ebr;
  if (g.nlines <= 0) return;
  double2* SP = cols ? pl->d_ebc : pl->d_ebr;
  const double2* tw = cols ? pl->d_twbc : pl->d_twbr;
  double2* dst = cols ? pl->d_ccol : pl->d_rc;
  const long long tot = cols ? pl->tot_ccol : pl->tot_rc;
  const long long nspec = B * 4 * g.nlines * g.nblk;
#define EB_LAUNCH(LG)                                                                                       \
  do {                                                                                                      \
    auto fs = &k_eb_spec<T, LG>;                                                                            \
    auto fp = &k_eb_pairs<LG>;                                                                              \
    spec_attr(fs, LG);                                                                                      \
    spec_attr(fp, LG);                                                                                      \
    fs<<<(unsigned)((nspec + spec_g<LG>() - 1) / spec_g<LG>()), spec_threads<LG>(),                         \
         sizeof(double2) * spec_g<LG>() * spec_sb_elems<LG>(), st>>>(nspec, A, pr, g, cols ? 1 : 0, tw, SP); \
    const long long nti = (g.nlines + EbTile<LG>::TI - 1) / EbTile<LG>::TI,                                 \
                    ntj = (g.nlines + EbTile<LG>::TJ - 1) / EbTile<LG>::TJ, ntiles = B * 2 * nti * ntj;     \
    fp<<<(unsigned)((ntiles + nparts - 1) / nparts), 1 << LG, eb_pairs_smem<LG>(), st>>>(                   \
        SP, pr, g, cols ? 1 : 0, tw, pl->d_cls_slot, pl->d_cls, dst, tot, part, nparts, ntiles);            \
    pl->spec_launches += 2;                                                                                 \
  } while (0)
  switch (g.logLb) {
    case 6: EB_LAUNCH(6); break;
    case 7: EB_LAUNCH(7); break;
    case 8: EB_LAUNCH(8); break;
    default: EB_LAUNCH(9);
  }
#undef EB_LAUNCH
}

// spectral core sums (spectral.cuh) for band ks_part of ks_nparts: writes
// the one CC partial per class (npart = 1); with spec_edges also the
// edge-column sums CCol and edge-row sums RC' (one segment)
template <typename T>
void launch_spectral(covgpu_plan* pl, const typename CT<T>::c* A, cudaStream_t st, cudaStream_t es,
                     const std::function<void(const char*)>& mark) {
  const Problem& pr = pl->pr;
  const long long B = pl->batch;
  const int L = pl->spec_L, part = pl->ks_part, nparts = pl->ks_nparts;
  const int rows_lo = pr.P - 1, nrows = pr.N - 2 * pr.P + 2;
  const int ra = rows_lo + (int)((long long)nrows * part / nparts);
  const int rz = rows_lo + (int)((long long)nrows * (part + 1) / nparts) - 1;
  const int S = pr.P - 1, S1 = pr.Q - 1;
  // side stream (es): the edge-column sums depend only on A; main stream:
  // row spectra -> dr = 0 per-row transforms, correlation -> output FFT ->
  // edge rows
  // correlation launch for chunk range `part_` of `nparts_` into G slots [slot0, slot0 + nseg_)
  const bool sym = pl->spec_sym && nparts == 1;  // (row parts keep the two-mask sums)
  auto corr_launch = [&](cudaStream_t cs, long long nb_, const double2* fx, const double2* fy, const SpecLayout& lay_,
                         double2* gp, bool posonly, int nseg_, int part_, int nparts_, int slot0, int nslots) {
    const int e = pl->spec_e;
    const int ngrp = posonly ? (pr.P + e - 1) / e : pl->spec_ngrp;
    const int stages = posonly ? 2 : pl->spec_stages;
    const size_t sm = stages * spec_corr_stage_bytes(pr.P, posonly) + 16 * stages;
    const unsigned blocks = (unsigned)(nb_ * lay_.nfb * nseg_);
    auto kern = pl->spec_e == 8 ? &k_spec_corr_smem<8, 16> : &k_spec_corr_smem<16, 8>;
    {
      static std::mutex mu;
      static std::vector<const void*> done;
      std::lock_guard<std::mutex> lk(mu);
      if (std::find(done.begin(), done.end(), (const void*)kern) == done.end()) {
        cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        done.push_back((const void*)kern);
      }
    }
    kern<<<blocks, ngrp * 32, sm, cs>>>(fx, fy, pr, lay_, nseg_, part_, nparts_, stages, gp, slot0, nslots,
                                        posonly ? 1 : 0);
    ++pl->spec_launches;
  };
  auto corr_smem = [&](int nseg_, int part_, int nparts_, int slot0, int nslots) {
    corr_launch(st, B, pl->d_fx, sym ? pl->d_fx : pl->d_fy, pl->spec_lay, pl->d_gp, sym, nseg_, part_, nparts_,
                slot0, nslots);
  };
  // row spectra of rows [r0, r0 + nr): X and Y (two column masks), or the one
  // symmetric spectrum
  auto fft_rows = [&](int r0, int nr) {
    if (nr <= 0) return;
    if (sym)
      SPEC_LOGL(pl->spec_logL, SpecK<T>::template fft, B * nr, A, pr, 2, pl->spec_lay, pl->d_tw, pl->d_fx, pl->d_fy,
                r0, nr);
    else
      SPEC_LOGL(pl->spec_logL, SpecK<T>::template fft, B * nr * 2, A, pr, 0, pl->spec_lay, pl->d_tw, pl->d_fx,
                pl->d_fy, r0, nr);
  };
  const double2* const fy_rows = sym ? pl->d_fx : pl->d_fy;  // second-element spectrum of the dr = 0 rows
  if (nparts > 1) {
    // only this part's edge pairs are computed: the others' CCol / RC' stay zero
    if (pl->spec_edges) {
      CUDA_TRY_V(cudaMemsetAsync(pl->d_ccol, 0, sizeof(double2) * (size_t)(B * pl->tot_ccol), es));
      CUDA_TRY_V(cudaMemsetAsync(pl->d_rc, 0, sizeof(double2) * (size_t)(B * pl->tot_rc), es));
      if (es != st) {
        cudaEventRecord(pl->ev_d0, es);
        cudaStreamWaitEvent(st, pl->ev_d0, 0);
      }
    }
  }
  int gslots = pl->spec_nseg;  // G partial slots the output FFT sums
  bool corr_done = false;
  const bool band_mode = pl->band_wait && B == 1 && stream_wait_value();
  // The blocked edge sums read only A: with a side stream they go first, under
  // the row FFTs and the correlation (queued behind the dr = 0 row transforms
  // they started after the correlation and ended ~50 us after the main chain
  // at cfg5).  Timing mode keeps them after the output FFT (one stream).
  const bool edges_first = pl->spec_edges && pl->spec_blk && !band_mode && es != st && !hook_env("COVGPU_EDGES_LAST");
  // symmetric sums on the device path: the dr = 0 row transforms run inside
  // the row-FFT kernel (k_spec_fft_ac)
  const bool fuse_d0 = sym && !band_mode && rz >= ra && !hook_env("COVGPU_NO_FUSE_D0");
  if (edges_first) {
    launch_edges_blocked<T>(pl, A, es, true, part, nparts);
    launch_edges_blocked<T>(pl, A, es, false, part, nparts);
  }
  if (band_mode) {
    // host path streaming A: the copy stream sends the edge columns and the
    // top / bottom strip rows first (ev_strips), then the remaining rows in
    // bands (band counter).  Strip-row spectra right after ev_strips (the
    // side stream's edge sums start from them); each band's row FFTs and
    // dr = 0 row transforms as soon as the band is signalled; each band's
    // rows of the correlation once its +P-1 halo is transformed — all under
    // the rest of the H2D.
    const int N = pr.N;
    CUDA_TRY_V(cudaStreamWaitEvent(st, pl->ev_strips, 0));
    fft_rows(0, S);
    fft_rows(N - S, S);
    if (pl->spec_edges && !pl->spec_blk)
      SPEC_LOGL(pl->spec_logL, SpecK<T>::template fft, B * 2 * S, A, pr, 1, pl->spec_lay, pl->d_tw, pl->d_fx,
                pl->d_fy0, 0, N);
    if (es != st) {  // the side stream: edge-row pair FFTs from the strip spectra
      cudaEventRecord(pl->ev_d0, st);
      cudaStreamWaitEvent(es, pl->ev_d0, 0);
    }
    const int br = pl->band_rows, nb = (N + br - 1) / br;
    const int nch = (N + SC_RC - 1) / SC_RC;
    const bool band_corr = pl->spec_smem && nb <= kMaxBandSlots;
    int fft_done = 0;  // bands transformed
    auto fft_upto = [&](int m) {  // rows of bands [fft_done, m] outside the strips
      for (; fft_done <= m && fft_done < nb; ++fft_done) {
        const int k = fft_done, r0 = std::max(S, k * br), r1 = std::min(N - S, (k + 1) * br);
        if (k < (int)pl->ev_band.size() && pl->ev_band[k])
          cudaStreamWaitEvent(st, pl->ev_band[k], 0);
        else
          stream_wait_value()(st, (CUdeviceptr)pl->d_band_flag, pl->band_base + (unsigned)k + 1u,
                              CU_STREAM_WAIT_VALUE_GEQ);
        if (r1 <= r0) continue;
        fft_rows(r0, r1 - r0);
        // dr = 0 rows: the core rows [P-1, N-P] = the non-strip rows
        if (pl->spec_prune_q)
          SPEC_LOGL(pl->spec_logL, SpecK<T>::template rowacp, B * (r1 - r0), pl->d_fx, fy_rows, pr,
                    pl->spec_lay, pl->d_tw, pl->d_twf, r0, r1 - r0, rz - ra + 1, r0 - ra, pl->d_d0p);
        else
          SPEC_LOGL(pl->spec_logL, SpecK<T>::template rowac, B * (r1 - r0), pl->d_fx, fy_rows, pr,
                    pl->spec_lay, pl->d_tw, pl->d_twf, r0, r1 - r0, rz - ra + 1, r0 - ra, pl->d_d0p);
      }
    };
    for (int j = 0; j < nb; ++j) {
      if (!band_corr) {
        fft_upto(j);
        continue;
      }
      // part j of nb chunk ranges reads X rows up to its last row + P-1
      const int cz = (int)((long long)nch * (j + 1) / nb);
      const int hi = std::min(N - 1, cz * SC_RC - 1 + pr.P - 1);
      fft_upto(hi / br);
      corr_smem(1, j, nb, j, nb);
    }
    fft_upto(nb - 1);
    if (band_corr) {
      gslots = nb;
      corr_done = true;
    }
    mark("spec_fft");
    k_spec_d0sum<<<(unsigned)(B * pr.Q), 256, 0, st>>>(pl->d_d0p, std::max(0, rz - ra + 1), pr, pl->nclasses,
                                                       pl->d_cls_slot, pl->d_ccpart, sym ? 3 : 1);
    ++pl->spec_launches;
    if (pl->spec_edges && !pl->spec_blk && es != st) {
      const cudaStream_t st_main = st;
      st = es;
      if (pl->spec_prune_q)
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rcp, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
      else
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rc, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
      st = st_main;
    }
    mark("spec_rowac");
  } else {
    if (nparts > 1 && pl->spec_smem) {
      // multi-GPU row band: transform only the rows this part reads — its
      // correlation rows +- P-1, its dr = 0 rows and the two strips (edge-row
      // pairs); overlapping ranges write the same values
      const int nch = (pr.N + SC_RC - 1) / SC_RC;
      const int pieces = nparts * pl->spec_nseg;
      const int c0 = (int)((long long)nch * part * pl->spec_nseg / pieces);
      const int c1 = (int)((long long)nch * (part + 1) * pl->spec_nseg / pieces);
      int ranges[4][2] = {{std::max(0, c0 * SC_RC - (pr.P - 1)), std::min(pr.N, c1 * SC_RC + pr.P - 1)},
                          {ra, rz + 1},
                          {0, S},
                          {pr.N - S, pr.N}};
      for (auto& rg : ranges) {
        const int r0 = std::max(0, rg[0]), r1 = std::min(pr.N, rg[1]);
        if (r1 > r0) fft_rows(r0, r1 - r0);
      }
    } else if (fuse_d0) {
      if (pl->spec_prune_q)
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template fftacp, B * pr.N, A, pr, pl->spec_lay, pl->d_tw, pl->d_twf,
                  pl->d_fx, 0, pr.N, ra, rz - ra + 1, pl->d_d0p);
      else
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template fftac, B * pr.N, A, pr, pl->spec_lay, pl->d_tw, pl->d_twf,
                  pl->d_fx, 0, pr.N, ra, rz - ra + 1, pl->d_d0p);
    } else {
      fft_rows(0, pr.N);
    }
    if (pl->spec_edges && !pl->spec_blk)
      SPEC_LOGL(pl->spec_logL, SpecK<T>::template fft, B * 2 * S, A, pr, 1, pl->spec_lay, pl->d_tw, pl->d_fx,
                pl->d_fy0, 0, pr.N);
    mark("spec_fft");
    // the dr = 0 row transforms and the edge-row pair FFTs need only the row
    // spectra: side stream after the FFTs (they fill the SMs around the
    // correlation kernel)
    const cudaStream_t st_main = st;
    if (es != st) {
      cudaEventRecord(pl->ev_d0, st);
      cudaStreamWaitEvent(es, pl->ev_d0, 0);
      st = es;
    }
    if (rz >= ra && !fuse_d0)
      if (pl->spec_prune_q)
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rowacp, B * (rz - ra + 1), pl->d_fx, fy_rows, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, ra, rz - ra + 1, rz - ra + 1, 0, pl->d_d0p);
      else
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rowac, B * (rz - ra + 1), pl->d_fx, fy_rows, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, ra, rz - ra + 1, rz - ra + 1, 0, pl->d_d0p);
    // (fused dr = 0 rows: only this small sum is left — on the main stream, the
    // side stream is busy with the edge sums until the end)
    k_spec_d0sum<<<(unsigned)(B * pr.Q), 256, 0, fuse_d0 && edges_first && !hook_env("COVGPU_D0_SIDE") ? st_main : st>>>(
        pl->d_d0p, std::max(0, rz - ra + 1), pr, pl->nclasses, pl->d_cls_slot, pl->d_ccpart, sym ? 3 : 1);
    ++pl->spec_launches;
    if (pl->spec_edges && !pl->spec_blk && es != st_main)
      if (pl->spec_prune_q)
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rcp, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
      else
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rc, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
    st = st_main;
    mark("spec_rowac");
  }
  if (corr_done) {
  } else if (pl->spec_smem) {
    corr_smem(pl->spec_nseg, part, nparts, 0, pl->spec_nseg);
  } else {
    k_spec_corr<SPEC_E><<<(unsigned)(B * pl->spec_nseg * pl->spec_nfb * pl->spec_ngrp), SPEC_CW * 32, 0, st>>>(
        pl->d_fx, pl->d_fy, pr, pl->spec_lay, L, pl->spec_nfb, pl->spec_ngrp, pl->spec_nseg, part, nparts,
        pl->d_gp);
    ++pl->spec_launches;
  }
  mark("spec_corr");
  if (gslots > 1) {  // row-segment partials -> slot 0, in order
    const long long per_seg = (long long)(2 * pr.P - 1) * L;
    const long long e_lo = sym ? (long long)(pr.P - 1) * L : 0, e_cnt = per_seg - e_lo, tot = B * e_cnt;
    k_spec_gsum<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->d_gp, gslots, per_seg, e_lo, e_cnt, tot);
    ++pl->spec_launches;
  }
  if (pl->spec_prune_q)
    SPEC_LOGL(pl->spec_logL, SpecK<T>::template dftp, B * (2 * pr.P - 1), pl->d_gp, pl->d_tw, pl->d_twf, pr, gslots,
              pl->nclasses, pl->d_cls_slot, pl->d_ccpart, sym ? 3 : 1, 0, sym ? 1 : 0, 0, 0);
  else
    SPEC_LOGL(pl->spec_logL, SpecK<T>::template dft, B * (2 * pr.P - 1), pl->d_gp, pl->d_tw, pl->d_twf, pr, gslots,
              pl->nclasses, pl->d_cls_slot, pl->d_ccpart, sym ? 3 : 1, 0, sym ? 1 : 0, 0, 0);
  if (pl->spec_edges && pl->spec_blk) {
    // blocked short-lag correlation (edgeblk.cuh) on the side stream: reads
    // only A's strips.  Timing names: spec_ccol = column strips, spec_rc = row strips
    mark("spec_dft");
    if (band_mode) {
      // host path: the strip rows arrived first, the edge columns are complete
      // only with the last band of A
      launch_edges_blocked<T>(pl, A, es, false, part, nparts);
      CUDA_TRY_V(cudaStreamWaitEvent(es, pl->ev_h2d, 0));
      launch_edges_blocked<T>(pl, A, es, true, part, nparts);
      mark("spec_ccol");
    } else if (!edges_first) {
      launch_edges_blocked<T>(pl, A, es, true, part, nparts);
      mark("spec_ccol");
      launch_edges_blocked<T>(pl, A, es, false, part, nparts);
    }
  } else if (pl->spec_edges) {
    mark("spec_dft");
    if (band_mode) CUDA_TRY_V(cudaStreamWaitEvent(es, pl->ev_h2d, 0));  // (edge columns of every row)
    {
      cudaStream_t st_main = st;
      st = es;  // SPEC_LOGL launches on `st`
      SPEC_LOGL(pl->spec_logLr, SpecK<T>::template colfft, B * 2 * 4 * S1, A, pr, pl->d_twr, pl->d_fc);
      if (pl->spec_prune_p)
        SPEC_LOGL(pl->spec_logLr, SpecK<T>::template ccolp, (B * 2 * (long long)S1 * S1 + nparts - 1) / nparts, pl->d_fc, pr,
                  pl->d_twr, pl->d_twrf, pl->d_cls_slot, pl->d_cls, pl->d_ccol, pl->tot_ccol, part, nparts,
                  B * 2 * (long long)S1 * S1);
      else
        SPEC_LOGL(pl->spec_logLr, SpecK<T>::template ccol, (B * 2 * (long long)S1 * S1 + nparts - 1) / nparts, pl->d_fc, pr,
                  pl->d_twr, pl->d_twrf, pl->d_cls_slot, pl->d_cls, pl->d_ccol, pl->tot_ccol, part, nparts,
                  B * 2 * (long long)S1 * S1);
      st = st_main;
    }
    mark("spec_ccol");
    if (es == st)  // (timing mode: everything in order on one stream)
      if (pl->spec_prune_q)
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rcp, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
      else
        SPEC_LOGL(pl->spec_logL, SpecK<T>::template rc, (B * 2 * (long long)S * S + nparts - 1) / nparts, pl->d_fx, pl->d_fy0, pr,
                  pl->spec_lay, pl->d_tw, pl->d_twf, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, part, nparts,
                  B * 2 * (long long)S * S);
  }
  if (sym) {
    mark("spec_rc");
    // the strips' correction E(dr, dc) (all lags, dr = 0 included) as the second
    // CC partial: a small spectral problem on the two 2Q-2 column strips, on the
    // side stream (host path: the edge columns are complete with the last band)
    const cudaStream_t st_main = st;
    if (es != st) st = pl->cur_ds ? pl->cur_ds : es;  // (the third stream, after the walk's chunk updates)
    if (band_mode) CUDA_TRY_V(cudaStreamWaitEvent(st, pl->ev_h2d, 0));
    SPEC_LOGL(pl->spec2_logL, SpecK<T>::template fft, B * 2 * pr.N * 2, A, pr, 3, pl->spec2_lay, pl->d_tw2, pl->d_fx2,
              pl->d_fy2, 0, pr.N);
    const int ns2 = pl->spec2_nseg;
    corr_launch(st, 2 * B, pl->d_fx2, pl->d_fy2, pl->spec2_lay, pl->d_gp2, false, ns2, 0, 1, 0, ns2);
    const int L2 = 1 << pl->spec2_logL;
    if (ns2 > 1) {
      const long long per_seg = (long long)(2 * pr.P - 1) * L2, tot = 2 * B * per_seg;
      k_spec_gsum<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->d_gp2, ns2, per_seg, 0, per_seg, tot);
      ++pl->spec_launches;
    }
    SPEC_LOGL(pl->spec2_logL, SpecK<T>::template dft, 2 * B * (2 * pr.P - 1), pl->d_gp2, pl->d_tw2, pl->d_twf2, pr,
              ns2, pl->nclasses, pl->d_cls_slot, pl->d_ccpart, 3, 1, 0, 1, 1);
    st = st_main;
  }
}

// edge-column sums on the tensor cores; false when the tensor map fails
bool launch_edge_cols_dmma(covgpu_plan* pl, const double2* A, cudaStream_t st) {
  const Problem& pr = pl->pr;
  if (pl->ecm_ptr != (const void*)A) {
    CUtensorMap tm;
    if (!make_tmap(&tm, A, true, pl->batch, pr.N, pr.M, 2 * ECM_PITCH, ECM_RC)) {
      pl->ecm_ptr = nullptr;
      return false;
    }
    pl->ecm_tm = tm;
    pl->ecm_ptr = A;
  }
  const long long blocks = pl->ecm_items * pl->ecm_g;
  k_edge_cols_dmma<<<(unsigned)blocks, (MMA_WARPS + 1) * 32, ECM_SMEM, st>>>(
      pl->ecm_tm, pr, pl->ecm_g, pl->d_cls_slot, pl->d_cls, pl->d_ccol, pl->tot_ccol, pl->d_ecm_part,
      pl->d_ecm_tickets, pl->ks_part, pl->ks_nparts);
  return true;
}

// edge-row sums on the tensor cores; false when the tensor maps fail
bool launch_edge_rows_dmma(covgpu_plan* pl, const double2* A, cudaStream_t st) {
  const Problem& pr = pl->pr;
  if ((uintptr_t)A % 16 != 0) return false;
  if (pl->erm_ptr != (const void*)A) {
    CUtensorMap mx, my;
    if (!make_tmap(&mx, A, true, pl->batch, pr.N, pr.M, 2 * MMA_XP, ERM_XR, pr.M - pr.Q + 1, 0) ||
        !make_tmap(&my, A, true, pl->batch, pr.N, pr.M, 2 * ERM_YP, 1)) {
      pl->erm_ptr = nullptr;
      return false;
    }
    pl->erm_tmx = mx;
    pl->erm_tmy = my;
    pl->erm_ptr = A;
  }
  const long long blocks = pl->batch * 2LL * pl->S * pl->erm_dct * pl->nseg;
  k_edge_rows_dmma<<<(unsigned)blocks, (ERM_WARPS + 1) * 32, ERM_SMEM, st>>>(
      pl->erm_tmx, pl->erm_tmy, pr, pl->erm_dct, pl->nseg, pl->d_cls_slot, pl->d_cls, pl->d_rc,
      pl->tot_rc, pl->ks_part, pl->ks_nparts);
  return true;
}

template <typename T, int D>
void launch_edge(covgpu_plan* pl, const typename CT<T>::c* A, cudaStream_t st) {
  const Problem& pr = pl->pr;
  if constexpr (sizeof(T) == 8) {
    if (pl->use_erm && launch_edge_rows_dmma(pl, (const double2*)A, st)) return;
  }
  if (pl->ks_nparts > 1) {  // the CUDA-core edge-row kernels have no row bands
    fail(COVGPU_ECUDA, "row-band sums: edge-row kernel unavailable");
    pl->ks_failed = true;
    return;
  }
  if (pl->edge_tma && ((uintptr_t)A % 16 == 0) && ((2LL * pr.M * sizeof(T)) % 16 == 0) &&
      EdgeCfg<T, D>::stages(pl->S, pl->r2g) >= 2) {
    using Cfg = EdgeCfg<T, D>;
    if (pl->etmap_ptr != (const void*)A) {
      CUtensorMap mx, my;
      if (make_tmap(&mx, A, sizeof(T) == 8, pl->batch, pr.N, pr.M, 2 * Cfg::XW, pl->S) &&
          make_tmap(&my, A, sizeof(T) == 8, pl->batch, pr.N, pr.M, 2 * Cfg::YW, pl->r2g)) {
        pl->etmx = mx;
        pl->etmy = my;
        pl->etmap_ptr = A;
      } else {
        pl->etmap_ptr = nullptr;
      }
    }
    if (pl->etmap_ptr == (const void*)A) {
      const size_t smem = Cfg::smem(pl->S, pl->r2g);
      static bool attr_done[2] = {false, false};  // per dtype, set once per process
      if (!attr_done[sizeof(T) == 8]) {
        cudaFuncSetAttribute(k_edge_tma<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr_done[sizeof(T) == 8] = true;
      }
      const long long blocks = pl->batch * 2LL * pl->ndg * pl->n_r2g * pl->nseg;
      k_edge_tma<T, D><<<(unsigned)blocks, (EDGE_WARPS + 1) * 32, smem, st>>>(
          pl->etmx, pl->etmy, pr, pl->S, pl->r2g, pl->n_r2g, pl->ndg, pl->nseg, pl->d_cls_slot,
          pl->d_cls, pl->d_rc, pl->tot_rc);
      return;
    }
  }
  const long long total = pl->batch * 2LL * pl->ndg * pl->nseg * (long long)pl->S * pl->S;
  if (total == 0) return;
  k_edge_rows<T, D><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
      A, pl->pr, pl->S, pl->ndg, pl->nseg, pl->d_cls_slot, pl->d_cls, pl->d_rc, pl->tot_rc, total);
}

// k_finalize_v row mapping: contiguous rows per lane (corners stored with the
// row permutation of kr = fin_kr) except for dense R written straight from
// the walk (strided rows, plain corner layout) — finalize.cuh
static inline bool fin_contig(const covgpu_plan* pl, int layout, bool direct) {
  (void)pl;
  return !(direct && layout == COVGPU_DENSE);
}
static inline int fin_corner_kr(const covgpu_plan* pl, int layout, bool direct) {
  return fin_contig(pl, layout, direct) ? std::max(pl->fin_kr, 1) : 1;
}

// Tile-finalize units (tile.cuh): (snapshot, dc, band of 32 circular
// diagonals, steps [u_lo, u_hi)) holding at least one class of plan slots
// [lo, hi).  Walks are cut at u = 16 j (the state there comes from
// k_fin_ckpt); pieces are ordered longest first, the bands of one
// (snapshot, dc, piece) adjacent (their row segments share sectors).
// delta: the chunk units [16 (j-1), 16 j) of every cut step 16 j < Q - dc
std::vector<int4> fin_tile_units(const covgpu_plan* pl, int lo, int hi, bool delta = false) {
  const int P = pl->pr.P, Q = pl->pr.Q;
  std::vector<char> has((size_t)(2 * P - 1) * Q, 0);
  for (int sl = lo; sl < hi; ++sl) {
    const ClassDesc& c = pl->h_cls[sl];
    has[(size_t)(c.dr + P - 1) * Q + c.dc] = 1;
  }
  struct Piece {
    int4 u;
    int len;
  };
  std::vector<Piece> pieces;
  const int lanes = ft_lanes(P), subs = 32 / lanes;  // snapshots per warp
  if (delta && pl->ck_tiled) {
    // k_ck_delta units: (snapshot, dc, top / bottom, chunk) of every column
    // offset that holds a class of the range
    std::vector<int4> units;
    for (int dc = 0; dc < Q; ++dc) {
      bool any = false;
      for (int dr = 0; dr < 2 * P - 1 && !any; ++dr) any = has[(size_t)dr * Q + dc];
      if (!any) continue;
      const int qu = Q - dc;
      for (int u0 = 0; u0 + pl->ft_ck < qu; u0 += pl->ft_ck)
        for (long long b = 0; b < pl->batch; ++b)
          for (int which = 0; which < 2; ++which)
            units.push_back(make_int4((int)b, dc, which, u0 | ((u0 + pl->ft_ck) << 16)));
    }
    return units;
  }
  for (int dc = 0; dc < Q; ++dc) {
    const int qu = Q - dc;
    for (int u0 = 0; u0 < qu; u0 += pl->ft_ck) {
      const int u1 = std::min(qu, u0 + pl->ft_ck);
      if (delta && u1 >= qu) break;  // no cut after this chunk
      for (long long b = 0; b < pl->batch; b += subs)
        for (int d0 = 0; d0 < P; d0 += lanes) {
          bool any = false;  // circular diagonal c holds classes (c, dc) and (c - P, dc)
          for (int c = d0; c < std::min(P, d0 + lanes); ++c)
            any = any || has[(size_t)(c + P - 1) * Q + dc] || (dc > 0 && c > 0 && has[(size_t)(c - 1) * Q + dc]);
          if (any) pieces.push_back({make_int4((int)b, dc, d0, u0 | (u1 << 16)), u1 - u0});
        }
    }
  }
  std::stable_sort(pieces.begin(), pieces.end(), [](const Piece& x, const Piece& y) { return x.len > y.len; });
  std::vector<int4> units;
  units.reserve(pieces.size());
  for (const Piece& pc : pieces) units.push_back(pc.u);
  return units;
}

template <typename T>
void launch_fin_tile(covgpu_plan* pl, const int4* units, long long nunits, const double2* ccpart, int npart,
                     const double2* ccol, const double2* rc, int nseg, typename CT<T>::c* R, long long rstride,
                     double scale, int layout, int u0, int u1, double2* wst, int slot_lo, int slot_hi,
                     cudaStream_t st, bool delta = false) {
  using C2 = typename CT<T>::c;
  if (nunits <= 0) return;
#define FT_LAUNCH(NW, LN, LAY, DEL)                                                                         \
  do {                                                                                                      \
    constexpr int upc = FtCfg<NW>::UPC;                                                                     \
    const unsigned grid = (unsigned)((nunits + upc - 1) / upc);                                             \
    const size_t smem = ft_unit_smem(pl->pr.P, NW, 32 / LN, sizeof(C2)) * upc;                              \
    k_fin_tile<T, NW, LAY, DEL, LN><<<grid, FtCfg<NW>::THREADS, smem, st>>>(                                \
        (const double2*)pl->d_corners, pl->pr, (int)pl->batch, pl->d_cls, pl->d_cls_slot, units,            \
        (int)nunits, pl->nclasses, npart, ccpart, ccol, pl->tot_ccol, rc, pl->tot_rc, nseg, pl->d_ck, R,    \
        rstride, scale, u0, u1, wst, slot_lo, slot_hi, pl->ft_ck);                                          \
  } while (0)
#define FT_LAY(NW, LN)                                                       \
  do {                                                                       \
    if (delta) FT_LAUNCH(NW, LN, COVGPU_DENSE, true);                        \
    else if (layout == COVGPU_DENSE) FT_LAUNCH(NW, LN, COVGPU_DENSE, false); \
    else if (layout == COVGPU_PACKED) FT_LAUNCH(NW, LN, COVGPU_PACKED, false); \
    else FT_LAUNCH(NW, LN, COVGPU_COMPACT, false);                           \
  } while (0)
  switch (pl->ft_nwarp) {
    case 1: FT_LAY(1, 8); break;
    case 2: FT_LAY(2, 16); break;
    case 4: FT_LAY(4, 32); break;
    case 8: FT_LAY(8, 32); break;
    default: FT_LAY(16, 32);
  }
#undef FT_LAY
#undef FT_LAUNCH
}

// the chunk updates delta_j of the units' (snapshot, dc, chunk)s: k_ck_delta
// for P >= 32, else the tile kernel's DELTA mode (same values)
template <typename T>
void launch_ck_delta(covgpu_plan* pl, const int4* dunits, long long ndunits, cudaStream_t st) {
  if (ndunits <= 0) return;
  if (pl->ck_tiled) {
    const int P = pl->pr.P, nsub = (P + CKD_SUB - 1) / CKD_SUB;
    const int tw = (std::min(P, CKD_SUB) + CKD_T - 1) / CKD_T;
    const int threads = (tw * tw + 31) / 32 * 32;
    static const cudaError_t attr =
        cudaFuncSetAttribute(k_ck_delta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ckd_smem(FT_CK));
    (void)attr;
    k_ck_delta<<<(unsigned)(ndunits * nsub * nsub), threads, ckd_smem(pl->ft_ck), st>>>(
        (const double2*)pl->d_corners, P, pl->pr.Q, 8 * pl->ft_nwarp, dunits, nsub, tw, pl->d_ck, pl->ft_ck);
    return;
  }
  launch_fin_tile<T>(pl, dunits, ndunits, nullptr, 1, nullptr, nullptr, 1, nullptr, 0, 1.0, COVGPU_DENSE, 0,
                     1 << 30, nullptr, 0, INT_MAX, st, true);
}

// chunk updates -> running sums over the chunks (tile.cuh k_ck_scan)
void launch_ck_scan(covgpu_plan* pl, cudaStream_t st) {
  const long long n = pl->batch * pl->pr.Q * 2LL * pl->pr.P * pl->pr.P;
  if (ft_nck(pl->pr.Q, pl->ft_ck) > 1)  // one chunk: nothing to add
    k_ck_scan<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl->d_ck, (int)pl->batch, pl->pr.P, pl->pr.Q, pl->ft_ck);
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
  pl->launches = 0;
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

  if (set_attrs() != cudaSuccess)
    return fail(COVGPU_ECUDA, std::string("kernel attributes: ") + cudaGetErrorString(set_attrs()) + " " + g_attr_fail);
  pl->nev = 0;
  auto mark = [&](const char* name) {
    if (pl->timing && pl->nev < covgpu_plan::kMaxEv) {
      pl->ev_name[pl->nev] = name;
      cudaEventRecord(pl->ev[pl->nev++], st);
    }
  };
  // The edge-row and corner kernels do not depend on the bulk kernel: run
  // them on a side stream so they fill the SMs the bulk kernel's last wave
  // leaves idle (fork/join with events).  With per-kernel timing enabled
  // everything stays on `st` so the event intervals are per kernel.
  const bool fork = !pl->timing && pl->side_stream != nullptr;
  cudaStream_t es = fork ? pl->side_stream : st;
  if (fork) {
    CUDA_TRY(cudaEventRecord(pl->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(es, pl->ev_fork, 0));
  }
  // (spectral host path: the side stream's kernels read only the early-copied
  // edge columns / strip rows and spectra made from them)
  if (pl->band_wait)
    CUDA_TRY(cudaStreamWaitEvent(es, pl->use_spec && pl->batch == 1 ? pl->ev_strips : pl->ev_h2d, 0));
  mark("start");
  bool dfork = false;
  if (pl->use_tile && !pl->ks_out) {
    // the tile walk's corner blocks and per-chunk state updates need only the
    // corners of A: on a stream of their own, under the sums and beside the
    // edge sums of the side stream
    cudaStream_t ds = fork && pl->delta_stream ? pl->delta_stream : es;
    if (ds != es) {
      CUDA_TRY(cudaEventRecord(pl->ev_djoin, es));  // (es already follows the fork and the host-path copies)
      CUDA_TRY(cudaStreamWaitEvent(ds, pl->ev_djoin, 0));
      dfork = true;
    }
    const int PP = 8 * pl->ft_nwarp;
    const long long nc = (long long)(pr.Q - 1) * ft_colw(pr.P, PP) * B;
    if (nc > 0) {
      k_corners_d<T><<<(unsigned)((nc + 255) / 256), 256, 0, ds>>>(A, pr, B, PP, (double2*)pl->d_corners);
      ++launches;
    }
    if (pl->n_dunits > 0) {
      launch_ck_delta<T>(pl, pl->d_dunits, pl->n_dunits, ds);
      launch_ck_scan(pl, ds);
      launches += 2;
    }
    pl->cur_ds = dfork ? ds : nullptr;
    if (!fork) mark("fin_delta");
  }
  // core sums: FP64 tensor cores when the plan allows, else the CUDA-core
  // bulk over every column block (which also yields the edge-column sums)
  bool mma = false;
  if (pl->use_spec) {
    // (band_wait: launch_spectral waits per band for the row FFTs, then for all of A)
    pl->spec_launches = 0;
    launch_spectral<T>(pl, A, st, es, mark);
    launches += pl->spec_launches;
    mma = true;
  }
  if constexpr (sizeof(T) == 8) {
    if (pl->use_mma && !mma) {
      const double2* Ad = (const double2*)A;
      switch (pl->mma_kind) {
        case 1: mma = launch_dmma3<2, 4, 2, 2, 2>(pl, Ad, st); break;
        case 2: mma = launch_dmma3<4, 4, 2, 2, 1>(pl, Ad, st); break;
        case 3: mma = launch_dmma3<2, 2, 2, 2, 2>(pl, Ad, st); break;
        case 4: mma = launch_dmma3<4, 4, 2, 2, 1, true>(pl, Ad, st); break;
        case 5: mma = launch_dmma3<2, 4, 2, 2, 2, true, 8>(pl, Ad, st); break;
        default:
          mma = pl->mma_dc == 32 ? launch_dmma<32>(pl, Ad, st) : launch_dmma<64>(pl, Ad, st);
      }
    }
  }
  if (!mma && pl->ks_nparts > 1) return fail(COVGPU_ECUDA, "row-band sums: tensor-core kernel unavailable");
  bool snap = false;
  if constexpr (sizeof(T) == 4) {
    if (!mma && pl->use_snap) {
      if (pl->band_wait) CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_h2d, 0));
      static cudaError_t attr = cudaFuncSetAttribute(k_snap_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
      if (attr != cudaSuccess) return fail(COVGPU_ECUDA, "k_snap_spec shared-memory attribute");
      k_snap_spec<<<(unsigned)B, K2_THREADS, k2_smem_bytes(pr.N, pr.P, pr.Q), st>>>(
          (const float2*)A, pr, B, pl->nclasses, pl->d_cls_slot, pl->d_cls, pl->d_ccpart, pl->d_ccol, pl->tot_ccol,
          pl->d_rc, pl->tot_rc);
      snap = true;
    }
  }
  if (!mma && !snap) {
    if (pl->band_wait) CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_h2d, 0));  // no per-band waits here
    launch_bulk_variant<T>(pl, A, st, pl->bulk_variant);
  }
  const int npart = pl->use_spec ? (pl->spec_sym && pl->ks_nparts == 1 ? 3 : 1) : snap ? 1 : mma ? pl->mma_g : pl->ncb * pl->nrs;
  ++launches;
  mark(pl->use_spec ? (pl->spec_edges ? (npart == 3 ? "spec_strips" : "spec_rc") : "spec_dft")
                    : mma ? "bulk_dmma" : snap ? "snap_spec" : "bulk");
  if (mma && !pl->spec_edges) {  // edge-column sums: tensor cores, else CUDA-core bulk on the edge column blocks
    if (!(pl->use_ecm && launch_edge_cols_dmma(pl, (const double2*)A, es))) {
      if (pl->ks_nparts > 1) return fail(COVGPU_ECUDA, "row-band sums: edge-column kernel unavailable");
      launch_bulk_variant<T>(pl, A, es, pl->edge_variant, pl->ncb_l, pl->ncb_r);
    }
    ++launches;
    mark("edge_cols");
  }
  if (pl->S > 0 && !pl->spec_edges && !snap) {  // (the snapshot kernel also yields RC')
    switch (pl->D) {
      case 4: launch_edge<T, 4>(pl, A, es); break;
      case 8: launch_edge<T, 8>(pl, A, es); break;
      default: launch_edge<T, 16>(pl, A, es);
    }
    ++launches;
    mark("edge_rows");
  }
  if (pl->ks_out) {
    // row-band partial sums (multi-GPU): reduce the per-CTA / per-segment
    // partials into [CC | CCol | RC'] and stop before the finalize
    if (fork) {
      CUDA_TRY(cudaEventRecord(pl->ev_join, es));
      CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_join, 0));
    }
    const long long ncc = (long long)B * pl->nclasses, ncl = (long long)B * pl->tot_ccol,
                    nrc = (long long)B * pl->tot_rc;
    const long long tot = ncc + ncl + nrc;
    k_reduce_sums<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->d_ccpart, npart, ncc, pl->d_ccol,
                                                                ncl, pl->d_rc, pl->nseg, nrc, pl->ks_out);
    ++launches;
    mark("reduce_sums");
    CUDA_TRY(cudaGetLastError());
    pl->launches = launches;
    return COVGPU_OK;
  }
  if (pl->fin_kr > 0 && !pl->use_tile) {
    const int ckr = fin_corner_kr(pl, layout, layout != COVGPU_COMPACT && !pl->no_direct);
    const long long nc = 4LL * corner_rows(pr.P, ckr) * (pr.Q - 1) * B;
    if (nc > 0) {
      k_corners<T><<<(unsigned)((nc + 255) / 256), 256, 0, es>>>(A, pr, B, ckr, (C2*)pl->d_corners);
      ++launches;
    }
  }
  if (fork) {
    CUDA_TRY(cudaEventRecord(pl->ev_join, es));
    CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_join, 0));
  }
  if (dfork) {
    CUDA_TRY(cudaEventRecord(pl->ev_djoin, pl->cur_ds));
    CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_djoin, 0));
    pl->cur_ds = nullptr;
  }
  if (pl->use_tile) {
    // tile finalize straight into the requested layout; u-chunks for the
    // host path (rows [P u0, P u1) of R are complete after a chunk, an event
    // per chunk lets the copy-out start while the walk continues)
    const int nch = (layout != COVGPU_COMPACT && pl->fin_nchunks > 1 && pl->d_fin_state) ? pl->fin_nchunks : 1;
    for (int ch = 0; ch < nch; ++ch) {
      const int u0 = nch > 1 ? pl->fin_ubound[ch] : 0, u1 = nch > 1 ? pl->fin_ubound[ch + 1] : (1 << 30);
      launch_fin_tile<T>(pl, pl->d_units, pl->n_units, pl->d_ccpart, npart, pl->d_ccol, pl->d_rc, pl->nseg, R,
                         r_bstride, scale, layout, u0, u1, nch > 1 ? pl->d_fin_state : nullptr, 0, INT_MAX, st);
      if (nch > 1) CUDA_TRY(cudaEventRecord(pl->ev_fin_chunk[ch], st));
    }
  } else if (pl->fin_kr > 0) {
    const unsigned blocks = (unsigned)((pl->ntasks + FIN_WARPS - 1) / FIN_WARPS);
    // finalize into the compact layout (R itself, or the plan's scratch),
    // then expand to dense / packed with coalesced stores
    // dense R: write it directly from the walk (the scattered diagonal stores
    // merge in L2; with longest-walk-first tasks this beats finalize into
    // the compact layout + a coalesced expand: cfg5 0.325 -> 0.257 ms, cfg4
    // 0.255 -> 0.249 ms; packed: cfg4 0.224 -> 0.170 ms)
    const bool direct = layout != COVGPU_COMPACT && !pl->no_direct;
    C2* cdst = (layout == COVGPU_COMPACT || direct) ? R : (C2*)pl->d_slots;
    const long long rstride = direct ? r_bstride : pl->compact_elems;
#define FINV(KR, DIR)                                                                        \
  do {                                                                                       \
    if (contig)                                                                              \
      k_finalize_v<T, KR, DIR, true><<<blocks, FIN_WARPS * 32, 0, st>>>(FINV_ARGS);                \
    else                                                                                     \
      k_finalize_v<T, KR, DIR, false><<<blocks, FIN_WARPS * 32, 0, st>>>(FINV_ARGS);               \
  } while (0)
#define FINV_ARGS                                                                               \
      (const C2*)pl->d_corners, pr, pl->d_cls, pl->d_tasks, pl->ntasks, pl->nclasses,           \
      npart, pl->nrs, B, pl->d_ccpart, pl->d_ccol, pl->tot_ccol, pl->d_rc, pl->tot_rc, \
      pl->nseg, cdst, rstride, scale, direct ? layout : (int)COVGPU_COMPACT, u0, u1, wst
    const bool contig = fin_contig(pl, layout, direct);
    // u-chunks (host path: rows [P u0, P u1) of R are complete after a chunk;
    // an event per chunk lets the copy-out start while the walk continues)
    const int nch = (direct && pl->fin_nchunks > 1 && pl->d_fin_state) ? pl->fin_nchunks : 1;
    for (int ch = 0; ch < nch; ++ch) {
      const int u0 = nch > 1 ? pl->fin_ubound[ch] : 0, u1 = nch > 1 ? pl->fin_ubound[ch + 1] : (1 << 30);
      double2* wst = nch > 1 ? pl->d_fin_state : nullptr;
      if (direct) {
        switch (pl->fin_kr) {
          case 1: FINV(1, true); break;
          case 2: FINV(2, true); break;
          default: FINV(4, true);
        }
      } else {
        switch (pl->fin_kr) {
          case 1: FINV(1, false); break;
          case 2: FINV(2, false); break;
          default: FINV(4, false);
        }
      }
      if (nch > 1) CUDA_TRY(cudaEventRecord(pl->ev_fin_chunk[ch], st));
    }
#undef FINV
#undef FINV_ARGS
    if (layout != COVGPU_COMPACT && !direct) {
      ++launches;
      mark("finalize");
      const long long per = layout == COVGPU_DENSE ? (long long)pr.PQ * pr.PQ
                                                   : (long long)pr.PQ * (pr.PQ + 1) / 2;
      const long long tot = per * B;
      k_expand<T><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
          cdst, pl->compact_elems, pl->d_uc_off, pr, B, layout, R);
    }
  } else {
    const long long ntasks = (long long)B * pl->nclasses;
    k_finalize<T><<<(unsigned)((ntasks + FIN_WARPS - 1) / FIN_WARPS), FIN_WARPS * 32, pl->fin_smem, st>>>(
        A, pr, pl->d_cls, pl->nclasses, npart, pl->nrs, pl->d_ccpart, pl->d_ccol,
        pl->tot_ccol, pl->d_rc, pl->tot_rc, pl->nseg, pl->d_slots, pl->tot_slots, R, layout,
        r_bstride, scale, ntasks, pr.Q);
  }
  ++launches;
  mark(pl->nev >= 1 && pl->ev_name[pl->nev - 1] && !strcmp(pl->ev_name[pl->nev - 1], "finalize") ? "expand"
                                                                                                  : "finalize");
  CUDA_TRY(cudaGetLastError());
  pl->launches = launches;
  return COVGPU_OK;
}

// Finalize from reduced sums [CC | CCol | RC'] (covgpu_plan_finalize_sums):
// corners + the diagonal-segment walk for classes [c_lo, c_hi) of the plan.
template <typename T>
int finalize_from_sums(covgpu_plan* pl, const void* A_dev, const double2* sums, void* R_dev, int layout,
                       double scale, int c_lo, int c_hi, cudaStream_t st) {
  using C2 = typename CT<T>::c;
  const Problem& pr = pl->pr;
  const int B = (int)pl->batch;
  if (!pl->clean || pl->fin_kr == 0)
    return fail(COVGPU_ECAPACITY, "finalize from sums needs the clean path with P <= 128");
  const bool full = c_lo == 0 && c_hi == pl->nclasses;
  if (!full && layout != COVGPU_COMPACT)
    return fail(COVGPU_EINVAL, "a class range finalizes into the compact layout");
  const int2* tasks = pl->d_tasks;
  long long ntasks = pl->ntasks;
  if (!full && !pl->use_tile) {
    if (pl->rtask_lo != c_lo || pl->rtask_hi != c_hi) {
      std::vector<int2> sub;
      for (const int2& t : pl->h_tasks)
        if (t.x >= c_lo && t.x < c_hi) sub.push_back(t);
      cudaFree(pl->d_rtasks);
      pl->d_rtasks = nullptr;
      CUDA_TRY(cudaMalloc((void**)&pl->d_rtasks, sizeof(int2) * std::max<size_t>(sub.size(), 1)));
      if (!sub.empty())
        CUDA_TRY(cudaMemcpy(pl->d_rtasks, sub.data(), sizeof(int2) * sub.size(), cudaMemcpyHostToDevice));
      pl->n_rtasks = (long long)sub.size();
      pl->rtask_lo = c_lo;
      pl->rtask_hi = c_hi;
    }
    tasks = pl->d_rtasks;
    ntasks = pl->n_rtasks;
  }
  long long r_bstride;
  if (layout == COVGPU_DENSE)
    r_bstride = (long long)pr.PQ * pr.PQ;
  else if (layout == COVGPU_PACKED)
    r_bstride = (long long)pr.PQ * (pr.PQ + 1) / 2;
  else
    r_bstride = pl->compact_elems;
  const C2* A = (const C2*)A_dev;
  const int ckr = pl->use_tile ? 1 : fin_corner_kr(pl, layout, layout != COVGPU_COMPACT);
  const long long nc = 4LL * corner_rows(pr.P, ckr) * (pr.Q - 1) * B;
  if (pl->use_tile) {
    const int PP = 8 * pl->ft_nwarp;
    const long long ncd = (long long)(pr.Q - 1) * ft_colw(pr.P, PP) * B;
    if (ncd > 0)
      k_corners_d<T><<<(unsigned)((ncd + 255) / 256), 256, 0, st>>>(A, pr, B, PP, (double2*)pl->d_corners);
  } else if (nc > 0) {
      k_corners<T><<<(unsigned)((nc + 255) / 256), 256, 0, st>>>(A, pr, B, ckr, (C2*)pl->d_corners);
  }
  if (pl->use_tile) {
    const double2* cc = sums;
    const double2* cl = sums + (long long)B * pl->nclasses;
    const double2* rc = cl + (long long)B * pl->tot_ccol;
    const int4* dunits = pl->d_dunits;
    long long ndunits = pl->n_dunits;
    const int4* units = pl->d_units;
    long long nunits = pl->n_units;
    if (!full) {
      if (pl->rtask_lo != c_lo || pl->rtask_hi != c_hi) {
        const std::vector<int4> sub = fin_tile_units(pl, c_lo, c_hi);
        const std::vector<int4> dsub = fin_tile_units(pl, c_lo, c_hi, true);
        cudaFree(pl->d_runits);
        cudaFree(pl->d_rdunits);
        pl->d_runits = pl->d_rdunits = nullptr;
        CUDA_TRY(cudaMalloc((void**)&pl->d_runits, sizeof(int4) * std::max<size_t>(sub.size(), 1)));
        CUDA_TRY(cudaMalloc((void**)&pl->d_rdunits, sizeof(int4) * std::max<size_t>(dsub.size(), 1)));
        if (!sub.empty())
          CUDA_TRY(cudaMemcpy(pl->d_runits, sub.data(), sizeof(int4) * sub.size(), cudaMemcpyHostToDevice));
        if (!dsub.empty())
          CUDA_TRY(cudaMemcpy(pl->d_rdunits, dsub.data(), sizeof(int4) * dsub.size(), cudaMemcpyHostToDevice));
        pl->n_runits = (long long)sub.size();
        pl->n_rdunits = (long long)dsub.size();
        pl->rtask_lo = c_lo;
        pl->rtask_hi = c_hi;
      }
      units = pl->d_runits;
      nunits = pl->n_runits;
      dunits = pl->d_rdunits;
      ndunits = pl->n_rdunits;
    }
    if (ndunits > 0) {
      launch_ck_delta<T>(pl, dunits, ndunits, st);
      launch_ck_scan(pl, st);
    }
    launch_fin_tile<T>(pl, units, nunits, cc, 1, cl, rc, 1, (C2*)R_dev, r_bstride, scale, layout, 0, 1 << 30,
                       nullptr, c_lo, c_hi, st);
    CUDA_TRY(cudaGetLastError());
    return COVGPU_OK;
  }
  if (ntasks > 0) {
    const double2* cc = sums;
    const double2* cl = sums + (long long)B * pl->nclasses;
    const double2* rc = cl + (long long)B * pl->tot_ccol;
    const unsigned blocks = (unsigned)((ntasks + FIN_WARPS - 1) / FIN_WARPS);
    const bool direct = layout != COVGPU_COMPACT;
#define FINS(KR, DIR)                                                                        \
  do {                                                                                       \
    if (contig)                                                                              \
      k_finalize_v<T, KR, DIR, true><<<blocks, FIN_WARPS * 32, 0, st>>>(FINS_ARGS);                \
    else                                                                                     \
      k_finalize_v<T, KR, DIR, false><<<blocks, FIN_WARPS * 32, 0, st>>>(FINS_ARGS);               \
  } while (0)
#define FINS_ARGS                                                                                 \
      (const C2*)pl->d_corners, pr, pl->d_cls, tasks, ntasks, pl->nclasses, 1, 1, B, cc, cl,      \
      pl->tot_ccol, rc, pl->tot_rc, 1, (C2*)R_dev, r_bstride, scale, direct ? layout : (int)COVGPU_COMPACT, \
      0, 1 << 30, nullptr
    const bool contig = fin_contig(pl, layout, direct);
    if (direct) {
      switch (pl->fin_kr) {
        case 1: FINS(1, true); break;
        case 2: FINS(2, true); break;
        default: FINS(4, true);
      }
    } else {
      switch (pl->fin_kr) {
        case 1: FINS(1, false); break;
        case 2: FINS(2, false); break;
        default: FINS(4, false);
      }
    }
#undef FINS
#undef FINS_ARGS
  }
  CUDA_TRY(cudaGetLastError());
  return COVGPU_OK;
}

struct PlanKey {
  int device, dtype;
  long long batch, n, m;
  int p, q;
  std::vector<int32_t> ids;
  std::string env;  // the COVGPU_* path switches the plan was made under
  bool operator<(const PlanKey& o) const {
    return std::tie(device, dtype, batch, n, m, p, q, ids, env) <
           std::tie(o.device, o.dtype, o.batch, o.n, o.m, o.p, o.q, o.ids, o.env);
  }
};

std::string path_env() {
  std::string e;
  for (const char* k : {"COVGPU_SPECTRAL", "COVGPU_NO_SPECTRAL", "COVGPU_NO_MMA", "COVGPU_NO_MMA_EDGE",
                        "COVGPU_NO_TMA", "COVGPU_MMA_KIND", "COVGPU_SPEC_NO_SMEM", "COVGPU_NO_DIRECT", "COVGPU_SPEC_E", "COVGPU_NO_GRAPH", "COVGPU_NO_SNAP", "COVGPU_FT_CK", "COVGPU_CK_WALK", "COVGPU_EDGES_LAST", "COVGPU_NO_FUSE_D0", "COVGPU_D0_SIDE", "COVGPU_NO_SYM", "COVGPU_SYM",
                        "COVGPU_SPEC_NO_PRUNE", "COVGPU_EDGE_PAIRFFT"}) {
    const char* v = getenv(k);
    e += v ? v : "-";
    e += ',';
  }
  return e;
}

// Plans cached per shape for the one-shot calls, held by shared ownership:
// evicting an entry never frees a plan another thread is still executing
// (the last holder's release destroys it).
std::mutex g_cache_mu;
std::map<PlanKey, std::shared_ptr<covgpu_plan>> g_cache;

}  // namespace

extern "C" {
static int plan_execute_locked(covgpu_plan_t pl, const void* A_dev, void* R_dev, int32_t layout, double scale,
                               cudaStream_t st);
}

// Order this execute after the plan's previous one when it runs on another
// stream (the workspace is per plan), and record its completion.
static int plan_stream_enter(covgpu_plan* pl, cudaStream_t st) {
  if (!pl->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_done, cudaEventDisableTiming));
  if (pl->has_last && pl->last_stream != st) CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_done, 0));
  return COVGPU_OK;
}
static int plan_stream_leave(covgpu_plan* pl, cudaStream_t st, int rc) {
  const cudaError_t e = cudaEventRecord(pl->ev_done, st);
  if (e == cudaSuccess) {
    pl->last_stream = st;
    pl->has_last = true;
  } else {
    cudaGetLastError();
    if (!rc) rc = fail(COVGPU_ECUDA, std::string("completion event: ") + cudaGetErrorString(e));
  }
  return rc;
}

extern "C" {

int covgpu_plan_execute_host(covgpu_plan_t pl, const void* A_host, void* R_host, int32_t layout,
                             double scale);

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
    std::vector<char> seen(nuc, 0);
    for (int k = 0; k < n_classes; ++k) {
      const int uc = class_ids[k];
      if (uc < 0 || uc >= nuc) return -1;
      if (seen[uc]) continue;
      seen[uc] = 1;
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
  {
    const int v = pick_bulk_variant(n, m, p, q, batch, dtype);
    pl->bulk_variant = v;
    if (const char* nt = hook_env("COVGPU_NO_TMA")) pl->use_tma = atoi(nt) == 0;
    if (const char* nd = hook_env("COVGPU_NO_DIRECT")) pl->no_direct = atoi(nd) != 0;
    if (const char* ng = hook_env("COVGPU_NO_GRAPH")) pl->use_graph = atoi(ng) == 0;
    pl->E = kBulkVariants[v].E;
    pl->NW = kBulkVariants[v].NW;
  }
  pl->D = pick_lags(q);
  pl->ncb = (int)((m + 31) / 32);
  pl->n_drg = (2 * p - 1 + pl->E - 1) / pl->E;
  pl->n_dcb = (q + pl->NW - 1) / pl->NW;
  {
    // split the bulk row walk when the grid would be under ~4 waves
    const int minb = kBulkVariants[pl->bulk_variant].MINB;
    const long long ctas = batch * (long long)pl->n_drg * pl->n_dcb * pl->ncb;
    const long long want = 148LL * minb * 4;
    const long long max_split = std::max(1LL, (long long)((n - p + 1) / 64));  // >= 2 chunks each
    long long r = ctas >= want ? 1 : (want + ctas - 1) / ctas;
    // measured: with a CTA per (unit, segment) the per-CTA pipeline fill
    // outweighs the better wave fill (cfg3 bulk 0.197 -> 0.223 ms), so the
    // split is off until work units are scheduled persistently
    r = 1;  // (ccol would need a pre-reduction over segments before the finalize)
    pl->nrs = (int)std::max(1LL, std::min(r, std::min(max_split, 16LL)));
  }
  {
    // FP64 tensor cores for the core sums: complex128, all classes (class
    // subsets — shards — keep the CUDA-core bulk, whose work units follow
    // the selection), windows wide enough to fill the 32-lag x DC tiles and
    // edge column blocks that stay a small share of the columns
    const int ncb_l = (q - 2) / 32 + 1;
    const int ncb_r = pl->ncb - (int)((m - q + 1) / 32);
    bool ok = dtype == COVGPU_C128 && pl->clean && class_ids == nullptr && p >= 16 && q >= 24 &&
              p <= FINV_MAX_P && q >= 2 && ncb_l + ncb_r <= pl->ncb && pl->use_tma;
    if (const char* nm = hook_env("COVGPU_NO_MMA")) ok = ok && atoi(nm) == 0;
    if (ok) {
      pl->use_mma = true;
      pl->mma_dc = q <= 32 ? 32 : 64;
      // kernel: Gauss 3-DMMA tiles (1: 32x64 lags, 8 warps, 2 CTAs/SM; 2: 64x64,
      // 16 warps, 1 CTA/SM; 3: 32x32 for Q <= 32; 4: kind 2 + producer-warp
      // operand sums (PREP); 5: kind 1 + PREP with 8-row chunks), 0: 4-DMMA k_bulk_dmma
      // (cfg5 bulk: kind 0 7.06 ms, 1 5.74, 2 5.90, 4 5.75, 5 5.65)
      pl->mma_kind = q <= 32 ? 3 : 5;
      if (const char* mk = hook_env("COVGPU_MMA_KIND")) {
        const int k = atoi(mk);
        if (k >= 0 && k <= 5) pl->mma_kind = k;
      }
      int dr_tile = MMA_DR, ctas_per_sm = 2;
      if (pl->mma_kind == 2 || pl->mma_kind == 4) {
        dr_tile = 64;
        ctas_per_sm = 1;
      }
      if (pl->mma_kind == 1 || pl->mma_kind == 2 || pl->mma_kind == 4 || pl->mma_kind == 5) pl->mma_dc = 64;
      if (pl->mma_kind == 3) pl->mma_dc = 32;
      pl->n_drt = (2 * p - 1 + dr_tile - 1) / dr_tile;
      pl->n_dct = (q + pl->mma_dc - 1) / pl->mma_dc;
      // one wave of CTAs; each CTA >= 2 chunks
      const long long tiles = batch * (long long)pl->n_drt * pl->n_dct;
      const long long chunks = (long long)((n + MMA_RC - 1) / MMA_RC + 2) * ((m - q + 1 + MMA_W - 1) / MMA_W);
      long long g = std::max(1LL, (148LL * ctas_per_sm + tiles - 1) / tiles);
      g = std::min(g, std::max(1LL, chunks / 2));
      pl->mma_g = (int)g;
      pl->ncb_l = ncb_l;
      pl->ncb_r = ncb_r;
      pl->edge_variant = pick_bulk_variant(n, 32LL * (ncb_l + ncb_r), p, q, batch, dtype);
      // (the 8x8 tile map of the strip Gram needs >= 7 tile rows to keep the
      // 4 warps balanced: cfg5 edge columns 0.647 -> 0.337 ms, but cfg3
      // (Q=32) 0.037 -> 0.074 ms)
      bool ecm = q >= 50 && q <= 65;
      if (const char* ne = hook_env("COVGPU_NO_MMA_EDGE")) ecm = ecm && atoi(ne) == 0;
      if (ecm) {
        // items (snapshot, strip, dr) x G row splits: pick G in [1, 16] for
        // the best fill of 2 CTAs/SM waves (>= 2 chunks of 16 rows per CTA)
        pl->use_ecm = true;
        pl->ecm_items = batch * 2LL * (2 * p - 1);
        const long long rows = n - 2LL * p + 2;
        int best_g = 1;
        double best = 0.0;
        for (int g = 1; g <= 16; ++g) {
          if (g > 1 && rows / ECM_RC / g < 2) break;
          const double ctas = (double)pl->ecm_items * g;
          const double waves = std::ceil(ctas / 296.0);
          const double eff = ctas / (waves * 296.0);
          if (eff > best + 0.02) {
            best = eff;
            best_g = g;
          }
        }
        pl->ecm_g = best_g;
      }
    }
  }
  {
    // spectral core and edge sums (spectral.cuh): any dtype and class
    // selection, Q <= 64 (the dr = 0 space-domain kernel), FFT lengths
    // 2^6 .. 2^12 along rows (>= M) and columns (>= N), the walk finalize
    // (P <= FINV_MAX_P); small problems stay on the direct kernels (fewer
    // launches) unless COVGPU_SPECTRAL=1
    bool spec = pl->clean && p >= 2 && q >= 2 && q <= SPEC_MAX_Q && p <= FINV_MAX_P;
    int logL = 6, logLr = 6;
    while ((1LL << logL) < m) ++logL;
    while ((1LL << logLr) < n) ++logLr;
    spec = spec && logL <= 12 && logLr <= 12;
    const double direct_work = (2.0 * p - 1) * q * (double)n * (double)m;  // per snapshot
    // (class shards: every shard would repeat the FFTs and the correlation of
    // all lags — the multi-GPU split for this path is row bands)
    bool want = direct_work >= kSpecMinWork && class_ids == nullptr;
    if (const char* fs = hook_env("COVGPU_SPECTRAL")) want = want || atoi(fs) != 0;
    spec = spec && want;
    if (const char* ns = hook_env("COVGPU_NO_SPECTRAL")) spec = spec && atoi(ns) == 0;
    if (spec) {
      pl->use_spec = true;
      pl->spec_edges = true;
      pl->spec_logLr = logLr;
      pl->spec_logL = logL;
      // edge sums: blocked short-lag correlation (COVGPU_EDGE_PAIRFFT=1, a test
      // hook, keeps one full-length FFT per line pair)
      pl->spec_blk = p <= 128 && q <= 128;
      if (const char* pf = hook_env("COVGPU_EDGE_PAIRFFT")) pl->spec_blk = pl->spec_blk && atoi(pf) == 0;
      if (pl->spec_blk) {
        pl->ebc = eb_geom((int)p, (int)q - 1, (int)n, (int)(n - p), (int)p - 1);  // strip columns, row lags
        pl->ebr = eb_geom((int)q, (int)p - 1, (int)m, (int)(m - q), 0);            // strip rows, column lags
      }
      pl->spec_L = 1 << logL;
      if (const char* se = hook_env("COVGPU_SPEC_E")) pl->spec_e = atoi(se) == 8 ? 8 : 16;
      pl->spec_ngrp = (2 * p - 1 + SPEC_E - 1) / SPEC_E;
      pl->spec_nfb = (pl->spec_L + SPEC_CW * 32 - 1) / (SPEC_CW * 32);
      // row segments: ~6 CTAs of 4 warps per SM, >= 4 windows of rows each.
      // Every split below is chosen per snapshot (not from the batch size), so a
      // snapshot's sums run in the same order alone or in a batch (bitwise equal)
      const long long per = (long long)pl->spec_ngrp * pl->spec_nfb;
      const long long rows = n - 2LL * p + 2 + SPEC_E;
      long long seg = std::max(1LL, (148LL * 6 + per - 1) / per);
      seg = std::min(seg, std::max(1LL, rows / (4LL * SPEC_E)));
      pl->spec_nseg = (int)std::min(seg, 64LL);
      pl->spec_lay.nfb = pl->spec_L / 32;
      pl->spec_lay.padr = p - 1 + SC_RC;
      pl->spec_lay.np = (int)n + 2 * pl->spec_lay.padr;
      const size_t stb = spec_corr_stage_bytes(p);
      pl->spec_smem = pl->spec_ngrp <= 8 && 2 * stb + 64 <= SC_SMEM_BUDGET;
      // warps of the SMEM kernel: negative and non-negative lags in separate groups
      if (pl->spec_smem) pl->spec_ngrp = (p - 1 + pl->spec_e - 1) / pl->spec_e + (p + pl->spec_e - 1) / pl->spec_e;
      if (const char* nsm = hook_env("COVGPU_SPEC_NO_SMEM")) pl->spec_smem = pl->spec_smem && atoi(nsm) == 0;
      if (pl->spec_smem) {
        pl->spec_stages = (int)std::min<size_t>(4, SC_SMEM_BUDGET / (stb + 16));
        // row segments: whole waves of 1-CTA/SM blocks, >= 4 chunks per segment
        const long long per2 = (long long)pl->spec_lay.nfb;
        const long long nch = (n + SC_RC - 1) / SC_RC;
        int best = 1;
        double best_eff = 0.0;
        for (int sg = 1; sg <= 32 && (sg == 1 || nch / sg >= 4); ++sg) {
          const double ctas = (double)per2 * sg, waves = std::ceil(ctas / 148.0);
          const double eff = ctas / (waves * 148.0) * std::min(1.0, ctas / 296.0);
          if (eff > best_eff + 0.01) {
            best_eff = eff;
            best = sg;
          }
        }
        pl->spec_nseg = best;
        // single snapshots the host path streams in row bands: one row segment
        // per band, so the band-wise correlation under the H2D adds the same
        // partials in the same order as the device path (bitwise equal)
        if (batch == 1 && pl->use_mma && n * m * 16 >= (8LL << 20)) {
          const long long nb = (n + host_band_rows(n) - 1) / host_band_rows(n);
          if (nb <= kMaxBandSlots) pl->spec_nseg = (int)nb;
        }
      }
      const long long d0rows = n - 2LL * p + 2;
      pl->spec_nd0 = (int)std::max(1LL, d0rows);  // N = 2P-2: no core rows
      // symmetric core sums: one mask [Q-1, M-Q] for both elements makes the
      // row-lag correlation conjugate-symmetric in dr (half the lags, one
      // spectrum per row); CC = that + the correlations inside the first and
      // the last 2Q-2 columns (second problem: the two strips as a batch of
      // two, FFT length >= 2Q-2), one extra CC partial per strip.  Needs the staged
      // correlation kernel, the blocked edge sums (they read A, not the X
      // spectra) and non-overlapping strips (M >= 3Q)
      int lg2 = 6;
      while ((1 << lg2) < 2 * q - 2) ++lg2;
      // (not the smallest spectral plans: launch-latency chains where the extra
      // strip launches cancel the gain — 512 x 512, P = Q = 32: 0.0880 vs
      // 0.0883 ms; 1024 x 1024, P = Q = 32: 0.132 -> 0.110 ms; 2048 x 2048,
      // P = Q = 16: 0.263 -> 0.183 ms)
      pl->spec_sym = pl->spec_smem && pl->spec_blk && m >= 3LL * q && q >= 2 && lg2 <= 12 && n * m >= (1LL << 19);
      if (const char* nsy = hook_env("COVGPU_NO_SYM")) pl->spec_sym = pl->spec_sym && atoi(nsy) == 0;
      if (const char* fsy = hook_env("COVGPU_SYM"))  // (test hook: also below the size gate)
        if (atoi(fsy) != 0) pl->spec_sym = pl->spec_smem && pl->spec_blk && m >= 3LL * q && q >= 2 && lg2 <= 12;
      if (pl->spec_sym) {
        pl->spec2_logL = lg2;
        pl->spec2_lay.nfb = (1 << lg2) / 32;
        pl->spec2_lay.padr = pl->spec_lay.padr;
        pl->spec2_lay.np = pl->spec_lay.np;
        // row segments of the strips' correlation: one wave of 1-CTA/SM blocks,
        // >= 2 chunks each (per-CTA pipeline fill and epilogue are as long as ~2 chunks)
        const long long nch2 = (n + SC_RC - 1) / SC_RC;
        const long long per2 = 2 * batch * pl->spec2_lay.nfb;
        pl->spec2_nseg = (int)std::max(1LL, std::min({148 / std::max(1LL, per2), nch2 / 2, 32LL}));
      }
    }
  }
  // small complex64 snapshots: the sums of a whole snapshot inside one CTA
  // (snap.cuh).  A function of the shape only (never of the batch), so a
  // snapshot alone and in a batch run the same arithmetic
  pl->use_snap = !pl->use_spec && dtype == COVGPU_C64 && pl->clean && class_ids == nullptr && m <= K2_L && p >= 2 &&
                 p <= K2_E && q >= 2 && q <= K2_MAXQ && k2_smem_bytes((int)n, (int)p, (int)q) <= 110 * 1024;
  if (const char* ns = hook_env("COVGPU_NO_SNAP")) pl->use_snap = pl->use_snap && atoi(ns) == 0;  // (test hook)
  pl->S = p - 1;
  pl->ndg = (q + pl->D - 1) / pl->D;
  pl->edge_tma = pl->S >= 16 && pl->use_tma;
  if (pl->edge_tma) {
    // TMA edge kernel: CTA = (strip, lag group, r2 group, column segment);
    // aim for ~4 waves of 1-CTA/SM blocks
    pl->r2g = std::max(1, std::min(pl->S, (EDGE_WARPS * 32) / pl->S));
    pl->n_r2g = (pl->S + pl->r2g - 1) / pl->r2g;
    const long long per = batch * 2LL * pl->ndg * pl->n_r2g;
    const long long want = 148LL * 4;
    const long long chunks = std::max(1LL, (long long)((m - q + 1 + EDGE_CW - 1) / EDGE_CW));
    long long seg = std::max(1LL, (want + per - 1) / per);
    pl->nseg = (int)std::max(1LL, std::min(seg, std::min(chunks, 16LL)));
  } else {
    // split the edge-row column walk so the launch has >= ~4 waves of warps
    const long long threads = batch * 2LL * pl->ndg * (long long)pl->S * pl->S;
    const long long want = 148LL * 32 * 16 * 4;
    const long long len = std::max(1LL, m - 2LL * q + 2);
    long long seg = threads > 0 ? (want + threads - 1) / threads : 1;
    seg = std::min(seg, std::max(1LL, len / 16));  // (short chains: the walk is latency-bound)
    pl->nseg = (int)std::max(1LL, std::min(seg, 16LL));
  }

  if (pl->use_mma && p >= 48 && p <= 65) {  // the 64-row strip tile: P-1 in [47, 64]
    bool erm = true;
    if (const char* ne = hook_env("COVGPU_NO_MMA_EDGE")) erm = atoi(ne) == 0;
    if (erm) {
      // CTA = (snapshot, strip, r2, lag tile, column segment), 1 CTA/SM: the
      // segment count with the best wave fill (>= 2 column chunks each;
      // cfg5: 126 x 7 = 882 CTAs = 5.96 waves)
      pl->use_erm = true;
      pl->erm_dct = (q + ERM_DC - 1) / ERM_DC;
      const long long per = batch * 2LL * (p - 1) * pl->erm_dct;
      const long long chunks = (m - q + 1 + MMA_W - 1) / MMA_W;
      long long seg = 1;
      double best = 0.0;
      for (long long g = 1; g <= 16 && (g == 1 || chunks / g >= 2); ++g) {
        const double ctas = (double)per * g, waves = std::ceil(ctas / 148.0);
        const double eff = ctas / (waves * 148.0) * std::min(1.0, ctas / 444.0);
        if (eff > best + 0.01) {
          best = eff;
          seg = g;
        }
      }
      pl->nseg = (int)std::min(seg, 16LL);
    }
  }
  if (pl->use_spec || pl->use_snap) pl->nseg = 1;  // RC' in one piece (k_spec_rc / k_snap_spec)
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

  long long ws = 0;
  const size_t nc = (size_t)std::max(pl->nclasses, 1);
  if ((rc = dalloc(&pl->d_cls, nc, &ws)) || (rc = dalloc(&pl->d_cls_slot, (size_t)nuc, &ws))) {
    plan_free(pl.get());
    return rc;
  }
  if (pl->use_ecm && pl->ecm_g > 1) {
    if ((rc = dalloc(&pl->d_ecm_part, (size_t)(pl->ecm_items * pl->ecm_g * ECM_PART), &ws)) ||
        (rc = dalloc(&pl->d_ecm_tickets, (size_t)pl->ecm_items, &ws))) {
      plan_free(pl.get());
      return rc;
    }
    if (cudaMemset(pl->d_ecm_tickets, 0, sizeof(unsigned) * (size_t)pl->ecm_items) != cudaSuccess) {
      plan_free(pl.get());
      return fail(COVGPU_ECUDA, "ticket reset");
    }
  }
  if (pl->use_spec) {
    const size_t L = (size_t)pl->spec_L;
    const std::vector<double2> tw = spec_twiddles(pl->spec_logL);
    const size_t fxe = (size_t)batch * pl->spec_lay.nfb * pl->spec_lay.np * 32;
    auto full_table = [&](int logn) {
      std::vector<double2> t((size_t)1 << logn);
      const long double pi2 = 6.283185307179586476925286766559L;
      for (size_t j = 0; j < t.size(); ++j) {
        const long double a = -pi2 * (long double)j / (long double)t.size();
        t[j] = make_double2((double)cosl(a), (double)sinl(a));
      }
      return t;
    };
    const std::vector<double2> twf = full_table(pl->spec_logL);
    const std::vector<double2> twrf = full_table(pl->spec_logLr);
    pl->spec_prune_q = q <= (1 << SPEC_LOGOUT) && pl->spec_logL >= SPEC_LOGOUT + 3;
    pl->spec_prune_p = p <= (1 << SPEC_LOGOUT) && pl->spec_logLr >= SPEC_LOGOUT + 3;
    if (const char* np = hook_env("COVGPU_SPEC_NO_PRUNE"))
      if (atoi(np) != 0) pl->spec_prune_q = pl->spec_prune_p = false;
    if ((rc = dalloc(&pl->d_twf, twf.size(), &ws)) || (rc = dalloc(&pl->d_twrf, twrf.size(), &ws))) {
      plan_free(pl.get());
      return rc;
    }
    if (cudaMemcpy(pl->d_twf, twf.data(), sizeof(double2) * twf.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_twrf, twrf.data(), sizeof(double2) * twrf.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      plan_free(pl.get());
      return fail(COVGPU_ECUDA, "twiddle upload");
    }
    if ((rc = dalloc(&pl->d_tw, L, &ws)) || (rc = dalloc(&pl->d_fx, fxe, &ws)) ||
        (rc = dalloc(&pl->d_fy, fxe, &ws)) ||
        (rc = dalloc(&pl->d_gp, (size_t)batch * std::max(pl->spec_nseg, batch == 1 ? kMaxBandSlots : 1) *
                                    (2 * p - 1) * L, &ws)) ||
        (rc = dalloc(&pl->d_d0p, (size_t)batch * pl->spec_nd0 * q, &ws))) {
      plan_free(pl.get());
      return rc;
    }
    if (cudaMemset(pl->d_fx, 0, sizeof(double2) * fxe) != cudaSuccess ||
        cudaMemset(pl->d_fy, 0, sizeof(double2) * fxe) != cudaSuccess ||
        cudaMemcpy(pl->d_tw, tw.data(), sizeof(double2) * L, cudaMemcpyHostToDevice) != cudaSuccess) {
      plan_free(pl.get());
      return fail(COVGPU_ECUDA, "twiddle upload");
    }
    if (pl->spec_sym) {
      const size_t L2 = (size_t)1 << pl->spec2_logL;
      const std::vector<double2> tw2 = spec_twiddles(pl->spec2_logL), twf2 = full_table(pl->spec2_logL);
      const size_t fxe2 = (size_t)2 * batch * pl->spec2_lay.nfb * pl->spec2_lay.np * 32;
      if ((rc = dalloc(&pl->d_tw2, L2, &ws)) || (rc = dalloc(&pl->d_twf2, L2, &ws)) ||
          (rc = dalloc(&pl->d_fx2, fxe2, &ws)) || (rc = dalloc(&pl->d_fy2, fxe2, &ws)) ||
          (rc = dalloc(&pl->d_gp2, (size_t)2 * batch * std::max(pl->spec2_nseg, 1) * (2 * p - 1) * L2, &ws))) {
        plan_free(pl.get());
        return rc;
      }
      if (cudaMemset(pl->d_fx2, 0, sizeof(double2) * fxe2) != cudaSuccess ||
          cudaMemset(pl->d_fy2, 0, sizeof(double2) * fxe2) != cudaSuccess ||
          cudaMemcpy(pl->d_tw2, tw2.data(), sizeof(double2) * tw2.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(pl->d_twf2, twf2.data(), sizeof(double2) * L2, cudaMemcpyHostToDevice) != cudaSuccess) {
        plan_free(pl.get());
        return fail(COVGPU_ECUDA, "strip twiddle upload");
      }
    }
    if (pl->spec_edges && pl->spec_blk) {
      const std::vector<double2> twc = spec_twiddles(pl->ebc.logLb), twr2 = spec_twiddles(pl->ebr.logLb);
      if ((rc = dalloc(&pl->d_twbc, twc.size(), &ws)) || (rc = dalloc(&pl->d_twbr, twr2.size(), &ws)) ||
          (rc = dalloc(&pl->d_ebc, std::max<size_t>(1, (size_t)batch * eb_spec_elems(pl->ebc)), &ws)) ||
          (rc = dalloc(&pl->d_ebr, std::max<size_t>(1, (size_t)batch * eb_spec_elems(pl->ebr)), &ws))) {
        plan_free(pl.get());
        return rc;
      }
      if (cudaMemcpy(pl->d_twbc, twc.data(), sizeof(double2) * twc.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(pl->d_twbr, twr2.data(), sizeof(double2) * twr2.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        plan_free(pl.get());
        return fail(COVGPU_ECUDA, "twiddle upload");
      }
    } else if (pl->spec_edges) {
      const size_t Lr = (size_t)1 << pl->spec_logLr;
      const std::vector<double2> twr = spec_twiddles(pl->spec_logLr);
      if ((rc = dalloc(&pl->d_twr, Lr, &ws)) ||
          (rc = dalloc(&pl->d_fc, (size_t)batch * 8 * (q - 1) * Lr, &ws)) ||
          (rc = dalloc(&pl->d_fy0, (size_t)batch * 2 * (p - 1) * L, &ws))) {
        plan_free(pl.get());
        return rc;
      }
      if (cudaMemcpy(pl->d_twr, twr.data(), sizeof(double2) * Lr, cudaMemcpyHostToDevice) != cudaSuccess) {
        plan_free(pl.get());
        return fail(COVGPU_ECUDA, "twiddle upload");
      }
    }
  }
  if (pl->clean) {
    // (symmetric spectral sums: three CC partials per class — core, left strip, right strip)
    const size_t npart = (size_t)std::max({pl->ncb * pl->nrs, pl->use_mma ? pl->mma_g : 0, pl->spec_sym ? 3 : 1});
    if ((rc = dalloc(&pl->d_ccpart, (size_t)batch * nc * npart, &ws)) ||
        (rc = dalloc(&pl->d_ccol, (size_t)(batch * std::max(pl->tot_ccol, 1LL) * pl->nrs), &ws)) ||
        (rc = dalloc(&pl->d_rc, (size_t)(batch * std::max(pl->tot_rc, 1LL) * pl->nseg), &ws)) ||
        (rc = dalloc(&pl->d_slots, (size_t)(batch * std::max(pl->tot_slots, 1LL)), &ws))) {
      plan_free(pl.get());
      return rc;
    }
    pl->fin_smem = sizeof(double2) * (size_t)FIN_WARPS * 4 * (size_t)q;
    if (p <= FINV_MAX_P) {
      pl->fin_kr = p <= 32 ? 1 : p <= 64 ? 2 : 4;
      pl->use_tile = hook_env("COVGPU_FIN_WALK") == nullptr || atoi(hook_env("COVGPU_FIN_WALK")) == 0;
      pl->ft_nwarp = ft_nwarp(p);
      pl->ft_ck = ft_ckstep(p, q);
      if (const char* ce = hook_env("COVGPU_FT_CK")) {  // (test hook)
        const int v = atoi(ce);
        if (v == 4 || v == 8 || v == 16) pl->ft_ck = v;
      }
      pl->ck_tiled = p >= 32 && hook_env("COVGPU_CK_WALK") == nullptr;  // (hook: chunk updates by the walk kernel)
      pl->h_units = fin_tile_units(pl.get(), 0, pl->nclasses);
      pl->n_units = (long long)pl->h_units.size();
      if (pl->use_tile && ft_nck(q, pl->ft_ck) > 0) {
        const size_t ckn = (size_t)batch * q * ft_nck(q, pl->ft_ck) * 2 * (size_t)p * p;
        const std::vector<int4> du = fin_tile_units(pl.get(), 0, pl->nclasses, true);
        pl->n_dunits = (long long)du.size();
        if ((rc = dalloc(&pl->d_ck, ckn, &ws)) || (rc = dalloc(&pl->d_dunits, std::max<size_t>(du.size(), 1), &ws))) {
          plan_free(pl.get());
          return rc;
        }
        if (!du.empty() && cudaMemcpy(pl->d_dunits, du.data(), sizeof(int4) * du.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
          plan_free(pl.get());
          return fail(COVGPU_ECUDA, "delta units upload");
        }
      }
      // tasks: (class, snapshot group of 32/W snapshots), W = min(32, pow2ceil(pv))
      std::vector<int2> tasks;
      for (int ci = 0; ci < pl->nclasses; ++ci) {
        int W = 1;
        while (W < pl->h_cls[ci].pv && W < 32) W <<= 1;
        const int per = 32 / W;
        const long long ng = (batch + per - 1) / per;
        for (long long g = 0; g < ng; ++g) tasks.push_back(make_int2(ci, (int)g));
      }
      // longest walks first (a warp's time ~ its qu column steps): the last
      // wave then holds only short tasks
      std::stable_sort(tasks.begin(), tasks.end(), [&](const int2& x, const int2& y) {
        return pl->h_cls[x.x].qu > pl->h_cls[y.x].qu;
      });
      pl->ntasks = (long long)tasks.size();
      pl->h_tasks = tasks;
      const size_t esz = (dtype == COVGPU_C128 || pl->use_tile) ? 16 : 8;  // tile walk: corners widened to double
      const size_t cbytes = pl->use_tile
          ? (size_t)batch * (size_t)std::max(q - 1, 0) * ft_colw(p, 8 * pl->ft_nwarp) * 16
          : (size_t)batch * 4 * (size_t)corner_rows(p, std::max(pl->fin_kr, 1)) * (size_t)std::max(q - 1, 0) * esz;
      std::vector<long long> uc_off(nuc, -1);
      for (const auto& cd : pl->h_cls) uc_off[cd.uc] = cd.slot_off;
      cudaError_t e1 = cudaMalloc(&pl->d_corners, std::max<size_t>(cbytes, 16));
      if (e1 == cudaSuccess) e1 = cudaMalloc((void**)&pl->d_uc_off, sizeof(long long) * nuc);
      if (e1 == cudaSuccess)
        e1 = cudaMemcpy(pl->d_uc_off, uc_off.data(), sizeof(long long) * nuc, cudaMemcpyHostToDevice);
      if (e1 == cudaSuccess) e1 = cudaMalloc((void**)&pl->d_units, sizeof(int4) * std::max<size_t>(pl->h_units.size(), 1));
      if (e1 == cudaSuccess && !pl->h_units.empty())
        e1 = cudaMemcpy(pl->d_units, pl->h_units.data(), sizeof(int4) * pl->h_units.size(), cudaMemcpyHostToDevice);
      if (e1 == cudaSuccess) e1 = cudaMalloc((void**)&pl->d_tasks, sizeof(int2) * std::max<size_t>(tasks.size(), 1));
      if (e1 == cudaSuccess && !tasks.empty())
        e1 = cudaMemcpy(pl->d_tasks, tasks.data(), sizeof(int2) * tasks.size(), cudaMemcpyHostToDevice);
      if (e1 != cudaSuccess) {
        plan_free(pl.get());
        return fail(COVGPU_ENOMEM, std::string("finalize workspace: ") + cudaGetErrorString(e1));
      }
      ws += (long long)cbytes + (long long)(sizeof(int2) * tasks.size());
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
  if (pl->clean) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // small estimates are launch- / latency-bound chains: the walk's chunk
    // updates get a stream of their own beside the edge sums (cfg3 0.094 ->
    // 0.087 ms, cfg2 0.092 -> 0.084); large ones are throughput-bound and lose
    // ~1 % to the extra concurrency (cfg5 0.463 -> 0.469 ms), so they keep one
    // side stream — unless they run the symmetric core sums, whose side work
    // (edge sums + the strips' correction) is longer than the main chain
    const bool small = batch * n * m <= (1LL << 20);
    if (cudaStreamCreateWithPriority(&pl->side_stream, cudaStreamNonBlocking, lo) != cudaSuccess ||
        ((small || pl->spec_sym) && cudaStreamCreateWithPriority(&pl->delta_stream, cudaStreamNonBlocking, lo) != cudaSuccess) ||
        cudaEventCreateWithFlags(&pl->ev_djoin, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&pl->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&pl->ev_d0, cudaEventDisableTiming) != cudaSuccess) {
      plan_free(pl.get());
      return fail(COVGPU_ECUDA, "side stream");
    }
  }
  cudaError_t e = cudaMemcpy(pl->d_cls, pl->h_cls.data(), sizeof(ClassDesc) * pl->h_cls.size(),
                             cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(pl->d_cls_slot, cls_slot.data(), sizeof(int) * cls_slot.size(),
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
  std::lock_guard<std::mutex> lk(pl->exec_mu);
  if (int rc0 = plan_stream_enter(pl, st)) return rc0;
  const int rc = plan_execute_locked(pl, A_dev, R_dev, layout, scale, st);
  return plan_stream_leave(pl, st, rc);
}

static int plan_execute_locked(covgpu_plan_t pl, const void* A_dev, void* R_dev, int32_t layout, double scale,
                               cudaStream_t st) {
  auto run = [&](cudaStream_t s) {
    return pl->dtype == COVGPU_C128 ? launch_all<double>(pl, A_dev, R_dev, layout, scale, s)
                                    : launch_all<float>(pl, A_dev, R_dev, layout, scale, s);
  };
  if (!pl->use_graph || pl->timing || pl->band_wait || pl->ks_out || !pl->clean || pl->fin_nchunks > 1)
    return run(st);
  const bool same = A_dev == pl->g_A && R_dev == pl->g_R && layout == pl->g_layout && scale == pl->g_scale;
  if (same && pl->gexec) {
    CUDA_TRY(cudaGraphLaunch(pl->gexec, st));
    return COVGPU_OK;
  }
  if (!same) {
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
    pl->g_A = A_dev;
    pl->g_R = R_dev;
    pl->g_layout = layout;
    pl->g_scale = scale;
    pl->g_hits = 0;
  }
  if (++pl->g_hits < 2) return run(st);  // first call: plain launches (attributes, tensor maps settle)
  // second identical call: capture on a private stream (the caller's may be the
  // legacy default stream, which cannot be captured), then launch on the caller's
  if (!pl->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->cap_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int rc = run(pl->cap_stream);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(pl->cap_stream, &g);
  if (rc || ce != cudaSuccess || !g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    pl->use_graph = false;  // capture not possible here: plain launches from now on
    return rc ? rc : run(st);
  }
  const cudaError_t ie = cudaGraphInstantiate(&pl->gexec, g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    pl->gexec = nullptr;
    pl->use_graph = false;
    return run(st);
  }
  CUDA_TRY(cudaGraphLaunch(pl->gexec, st));
  return COVGPU_OK;
}

int64_t covgpu_plan_workspace_bytes(covgpu_plan_t pl) { return pl ? pl->ws_bytes : -1; }
int32_t covgpu_plan_num_groups(covgpu_plan_t pl) {
  return pl ? (int32_t)(pl->batch * pl->n_drg * pl->n_dcb * pl->ncb * pl->nrs) : -1;
}
int32_t covgpu_plan_launches(covgpu_plan_t pl) { return pl ? pl->launches : -1; }

int covgpu_plan_set_timing(covgpu_plan_t pl, int32_t enable) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  CUDA_TRY(cudaSetDevice(pl->device));
  if (enable)
    for (auto& e : pl->ev)
      if (!e) CUDA_TRY(cudaEventCreate(&e));
  pl->timing = enable != 0;
  return COVGPU_OK;
}

int32_t covgpu_plan_kernel_times(covgpu_plan_t pl, float* ms, int32_t max_n) {
  if (!pl || !pl->timing || pl->nev < 2) return 0;
  if (cudaEventSynchronize(pl->ev[pl->nev - 1]) != cudaSuccess) return fail(COVGPU_ECUDA, "event sync");
  int n = 0;
  for (int i = 0; i + 1 < pl->nev && n < max_n; ++i, ++n)
    if (cudaEventElapsedTime(&ms[n], pl->ev[i], pl->ev[i + 1]) != cudaSuccess) ms[n] = -1.0f;
  return n;
}

static bool rowband_ok(const covgpu_plan* pl) {
  return pl->use_spec || (pl->use_mma && pl->use_ecm && pl->use_erm && pl->mma_kind != 0);
}

int32_t covgpu_plan_path(covgpu_plan_t pl) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  int32_t f = 0;
  if (pl->use_spec) f |= COVGPU_PATH_SPECTRAL;
  else if (pl->use_mma) f |= COVGPU_PATH_TENSOR;
  else if (pl->use_snap) f |= COVGPU_PATH_SNAPSHOT;
  if (rowband_ok(pl)) f |= COVGPU_PATH_ROWBAND;
  return f;
}

int64_t covgpu_plan_sums_elems(covgpu_plan_t pl) {
  if (!pl) return -1;
  return pl->batch * ((long long)pl->nclasses + pl->tot_ccol + pl->tot_rc);
}

int covgpu_plan_execute_sums(covgpu_plan_t pl, const void* A_dev, void* sums_dev, int32_t part,
                             int32_t nparts, void* stream) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  if (!A_dev || !sums_dev) return fail(COVGPU_EINVAL, "A and sums must be device pointers");
  if (nparts < 1 || part < 0 || part >= nparts) return fail(COVGPU_EINVAL, "part must be in [0, nparts)");
  if (!rowband_ok(pl))
    return fail(COVGPU_ECAPACITY,
                "row-band partial sums need the spectral path or the complex128 tensor-core path with "
                "tensor-core edge kernels (all classes, P in [48, 65], Q in [50, 65])");
  CUDA_TRY(cudaSetDevice(pl->device));
  std::lock_guard<std::mutex> lk(pl->exec_mu);
  if ((uintptr_t)A_dev % 16 != 0) return fail(COVGPU_EINVAL, "A must be 16-byte aligned");
  if (int rc0 = plan_stream_enter(pl, (cudaStream_t)stream)) return rc0;
  pl->ks_part = part;
  pl->ks_nparts = nparts;
  pl->ks_out = (double2*)sums_dev;
  pl->ks_failed = false;
  int rc = pl->dtype == COVGPU_C128
               ? launch_all<double>(pl, A_dev, nullptr, COVGPU_COMPACT, 1.0, (cudaStream_t)stream)
               : launch_all<float>(pl, A_dev, nullptr, COVGPU_COMPACT, 1.0, (cudaStream_t)stream);
  if (!rc && pl->ks_failed) rc = COVGPU_ECUDA;
  pl->ks_part = 0;
  pl->ks_nparts = 1;
  pl->ks_out = nullptr;
  return plan_stream_leave(pl, (cudaStream_t)stream, rc);
}

int covgpu_plan_finalize_sums(covgpu_plan_t pl, const void* A_dev, const void* sums_dev, void* R_dev,
                              int32_t layout, double scale, int32_t class_lo, int32_t class_hi,
                              void* stream) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  if (!A_dev || !sums_dev || !R_dev) return fail(COVGPU_EINVAL, "A, sums and R must be device pointers");
  if (layout < COVGPU_DENSE || layout > COVGPU_COMPACT) return fail(COVGPU_EINVAL, "unknown layout");
  if (class_lo < 0 || class_hi > pl->nclasses || class_lo > class_hi)
    return fail(COVGPU_EINVAL, "class range outside the plan");
  CUDA_TRY(cudaSetDevice(pl->device));
  std::lock_guard<std::mutex> lk(pl->exec_mu);
  CUDA_TRY(set_attrs());
  cudaStream_t st = (cudaStream_t)stream;
  if (int rc0 = plan_stream_enter(pl, st)) return rc0;
  const int rc = pl->dtype == COVGPU_C128
                     ? finalize_from_sums<double>(pl, A_dev, (const double2*)sums_dev, R_dev, layout, scale,
                                                  class_lo, class_hi, st)
                     : finalize_from_sums<float>(pl, A_dev, (const double2*)sums_dev, R_dev, layout, scale,
                                                 class_lo, class_hi, st);
  return plan_stream_leave(pl, st, rc);
}

int covgpu_plan_sums_range(covgpu_plan_t pl, int32_t class_lo, int32_t class_hi, int64_t* out) {
  if (!pl || !out) return fail(COVGPU_EINVAL, "plan or output is NULL");
  if (class_lo < 0 || class_hi > pl->nclasses || class_lo > class_hi)
    return fail(COVGPU_EINVAL, "class range outside the plan");
  const long long B = pl->batch;
  auto ccol = [&](int c) { return c < pl->nclasses ? pl->h_cls[c].ccol_off : pl->tot_ccol; };
  auto rcof = [&](int c) { return c < pl->nclasses ? pl->h_cls[c].rc_off : pl->tot_rc; };
  const long long base_cl = B * pl->nclasses, base_rc = base_cl + B * pl->tot_ccol;
  out[0] = class_lo;
  out[1] = class_hi;
  out[2] = base_cl + ccol(class_lo);
  out[3] = base_cl + ccol(class_hi);
  out[4] = base_rc + rcof(class_lo);
  out[5] = base_rc + rcof(class_hi);
  return COVGPU_OK;
}

int covgpu_plan_band_rows(covgpu_plan_t pl, int32_t part, int32_t nparts, int32_t* row_begin, int32_t* row_end) {
  if (!pl || !row_begin || !row_end) return fail(COVGPU_EINVAL, "plan or output is NULL");
  if (nparts < 1 || part < 0 || part >= nparts) return fail(COVGPU_EINVAL, "part must be in [0, nparts)");
  const Problem& pr = pl->pr;
  *row_begin = 0;
  *row_end = pr.N;
  if (!pl->use_spec || !pl->spec_smem || nparts == 1) return COVGPU_OK;  // (the whole of A)
  // launch_spectral's row-band ranges: correlation chunks +- P-1, dr = 0 rows
  const int rows_lo = pr.P - 1, nrows = pr.N - 2 * pr.P + 2;
  const int ra = rows_lo + (int)((long long)nrows * part / nparts);
  const int rz = rows_lo + (int)((long long)nrows * (part + 1) / nparts) - 1;
  const int nch = (pr.N + SC_RC - 1) / SC_RC;
  const int pieces = nparts * pl->spec_nseg;
  const int c0 = (int)((long long)nch * part * pl->spec_nseg / pieces);
  const int c1 = (int)((long long)nch * (part + 1) * pl->spec_nseg / pieces);
  int lo = std::max(0, c0 * SC_RC - (pr.P - 1)), hi = std::min(pr.N, c1 * SC_RC + pr.P - 1);
  if (rz >= ra) {
    lo = std::min(lo, ra);
    hi = std::max(hi, rz + 1);
  }
  *row_begin = lo;
  *row_end = hi;
  return COVGPU_OK;
}

int64_t covgpu_plan_class_slot_offset(covgpu_plan_t pl, int32_t class_index) {
  if (!pl || class_index < 0 || class_index > pl->nclasses) return -1;
  if (class_index == pl->nclasses) return pl->compact_elems;
  return pl->h_cls[class_index].slot_off;
}

int32_t covgpu_plan_kernel_names(covgpu_plan_t pl, char* buf, int32_t len) {
  if (!pl || !buf || len < 1) return fail(COVGPU_EINVAL, "plan or buffer is NULL");
  std::string s;
  int n = 0;
  for (int i = 1; i < pl->nev; ++i, ++n) {
    if (i > 1) s += ",";
    s += pl->ev_name[i] ? pl->ev_name[i] : "?";
  }
  std::snprintf(buf, (size_t)len, "%s", s.c_str());
  return n;
}

int covgpu_plan_destroy(covgpu_plan_t pl) {
  if (!pl) return COVGPU_OK;
  cudaSetDevice(pl->device);
  plan_free(pl);
  delete pl;
  return COVGPU_OK;
}

static int cached_plan(std::shared_ptr<covgpu_plan>* out, int device, int64_t batch, int64_t n, int64_t m,
                       int32_t p, int32_t q, int32_t dtype, const int32_t* ids, int32_t nids) {
  PlanKey key{device, dtype, batch, n, m, p, q, {}, path_env()};
  if (ids) key.ids.assign(ids, ids + nids);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *out = it->second;
    return COVGPU_OK;
  }
  if (g_cache.size() >= 32) g_cache.erase(g_cache.begin());  // (freed when its last user is done)
  covgpu_plan_t raw = nullptr;
  int rc = covgpu_plan_create(&raw, device, batch, n, m, p, q, dtype, ids, nids);
  if (rc) return rc;
  std::shared_ptr<covgpu_plan> sp(raw, [](covgpu_plan* x) { covgpu_plan_destroy(x); });
  g_cache[key] = sp;
  *out = std::move(sp);
  return COVGPU_OK;
}

int covgpu_estimate(const void* A_dev, int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q,
                    int32_t dtype, int32_t layout, const int32_t* class_ids, int32_t n_classes,
                    double scale, void* R_dev, void* stream) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::shared_ptr<covgpu_plan> pl;
  int rc = cached_plan(&pl, dev, batch, n, m, p, q, dtype, class_ids, n_classes);
  if (rc) return rc;
  return covgpu_plan_execute(pl.get(), A_dev, R_dev, layout, scale, stream);
}

int covgpu_estimate_host(const void* A_host, int64_t batch, int64_t n, int64_t m, int32_t p,
                         int32_t q, int32_t dtype, int32_t layout, double scale, void* R_host,
                         int device) {
  int rc = validate(batch, n, m, p, q, dtype);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(device));
  std::shared_ptr<covgpu_plan> pl;
  rc = cached_plan(&pl, device, batch, n, m, p, q, dtype, nullptr, 0);
  if (rc) return rc;
  return covgpu_plan_execute_host(pl.get(), A_host, R_host, layout, scale);
}

namespace {
// kind 0: FP64 FMA loop, 1: FP32 FMA loop, 2: FP64 DMMA loop
int probe_peak(int device, int kind, double seconds, double* tflops) {
  if (!tflops) return fail(COVGPU_EINVAL, "tflops is NULL");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  const int blocks = prop.multiProcessorCount * 2, threads = 256;
  void* out = nullptr;
  CUDA_TRY(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int iters) -> float {
    cudaEventRecord(e0);
    if (kind == 2)
      k_dmma_probe<<<blocks, threads>>>((double*)out, iters, 0.999999);
    else if (kind == 0)
      k_fma_probe<double><<<blocks, threads>>>((double*)out, iters, 0.999999);
    else
      k_fma_probe<float><<<blocks, threads>>>((float*)out, iters, 0.999999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  int iters = 1024;
  float ms = run(iters);
  while (ms < 20.f && iters < (1 << 26)) {
    iters *= 2;
    ms = run(iters);
  }
  // repeat for ~`seconds`, keep the best (sustained clocks, not a cold burst)
  const int reps = std::max(3, (int)(seconds * 1000.0 / std::max(ms, 1.f)));
  float best = ms;
  for (int r = 0; r < reps; ++r) best = std::min(best, run(iters));
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return fail(COVGPU_ECUDA, cudaGetErrorString(e));
  // FMA loop: 64 FMA per thread-iteration; DMMA loop: 8 x 256 FMA per warp-iteration
  const double fma_per = kind == 2 ? 8.0 * 256.0 / 32.0 : 64.0;
  const double flops = 2.0 * fma_per * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return COVGPU_OK;
}
}  // namespace

int covgpu_probe_fma_peak(int device, int32_t dtype, double seconds, double* tflops) {
  return probe_peak(device, dtype == COVGPU_C128 ? 0 : 1, seconds, tflops);
}

int covgpu_probe_dmma_peak(int device, double seconds, double* tflops) {
  return probe_peak(device, 2, seconds, tflops);
}

// Batched host path: the batch is cut into sub-batches that flow through
// kPipeSlots streams, so the H2D of one sub-batch, the kernels of another and
// the D2H of a third overlap (full-duplex PCIe copy engines + SMs).  Each
// slot owns its sub-batch plan (workspaces are per plan) and device buffers.
static int execute_host_pipelined(covgpu_plan_t pl, const void* A_host, void* R_host, int32_t layout,
                                  double scale) {
  const Problem& pr = pl->pr;
  const size_t esz = pl->dtype == COVGPU_C128 ? 16 : 8;
  const long long B = pl->batch;
  long long nsub = 32;  // cfg4: 16 -> 3.38 ms, 32 -> 3.03 ms, 64 -> 3.72 ms (bidirectional PCIe floor 2.68 ms)
  if (const char* e = hook_env("COVGPU_PIPE_SUBBATCHES")) nsub = std::max(2, atoi(e));
  const long long nch = std::min<long long>(nsub, B);
  const long long sub = (B + nch - 1) / nch;
  const long long tail = B - (B - 1) / sub * sub;  // size of the last sub-batch
  long long r_per_b;
  if (layout == COVGPU_DENSE)
    r_per_b = (long long)pr.PQ * pr.PQ;
  else if (layout == COVGPU_PACKED)
    r_per_b = (long long)pr.PQ * (pr.PQ + 1) / 2;
  else
    r_per_b = pl->compact_elems;
  const size_t a_per_b = (size_t)pr.N * pr.M * esz;
  std::vector<int32_t> ids;
  for (const auto& c : pl->h_cls) ids.push_back(c.uc);
  const bool all = (long long)ids.size() == covgpu_num_classes(pr.P, pr.Q);
  auto make = [&](covgpu_plan** dst, long long nb) -> int {
    const int rc = covgpu_plan_create(dst, pl->device, nb, pr.N, pr.M, pr.P, pr.Q, pl->dtype,
                                      all ? nullptr : ids.data(), all ? 0 : (int32_t)ids.size());
    // sub-batches overlapped on 3 streams: finalize into the compact layout
    // and expand (measured: cfg4 e2e 3.0 ms vs 3.2 ms with the direct write)
    if (!rc) (*dst)->no_direct = true;
    return rc;
  };
  if (pl->pipe_sub != sub || (tail != sub && pl->pipe_tail_b != tail)) {
    plan_free_pipe(pl);
    for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
      int rc = make(&pl->pipe[k], sub);
      if (rc) return rc;
      CUDA_TRY(cudaStreamCreateWithFlags(&pl->pipe_stream[k], cudaStreamNonBlocking));
    }
    if (tail != sub) {
      int rc = make(&pl->pipe_tail, tail);
      if (rc) return rc;
    }
    pl->pipe_sub = sub;
    pl->pipe_tail_b = tail;
  }
  const size_t ab = (size_t)sub * a_per_b, rb = (size_t)sub * r_per_b * esz;
  if (pl->pipe_Ab < ab || pl->pipe_Rb < rb) {
    for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
      cudaFree(pl->pipe_A[k]);
      cudaFree(pl->pipe_R[k]);
      pl->pipe_A[k] = pl->pipe_R[k] = nullptr;
    }
    pl->pipe_Ab = pl->pipe_Rb = 0;
    for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
      CUDA_TRY(cudaMalloc(&pl->pipe_A[k], ab));
      CUDA_TRY(cudaMalloc(&pl->pipe_R[k], rb));
    }
    pl->pipe_Ab = ab;
    pl->pipe_Rb = rb;
  }
  const char* ah = static_cast<const char*>(A_host);
  char* rh = static_cast<char*>(R_host);
  // copy-in on one stream, each slot's estimate on its own stream, copy-out on
  // one stream, chained by events: a slot's next copy-in waits only for the
  // estimate that read its A buffer (not for its copy-out), so the H2D engine
  // streams back to back (cfg4: 134 MB in, 67 MB out)
  if (!pl->pipe_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&pl->pipe_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&pl->pipe_out, cudaStreamNonBlocking));
    for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) {
      CUDA_TRY(cudaEventCreateWithFlags(&pl->pipe_ev_in[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&pl->pipe_ev_comp[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&pl->pipe_ev_out[k], cudaEventDisableTiming));
    }
  }
  int c = 0;
  for (long long b0 = 0; b0 < B; b0 += sub, ++c) {
    const long long nb = std::min(sub, B - b0);
    const int k = c % covgpu_plan::kPipeSlots;
    const bool reuse = c >= covgpu_plan::kPipeSlots;
    covgpu_plan* sp = nb == sub ? pl->pipe[k] : pl->pipe_tail;
    cudaStream_t st = pl->pipe_stream[k];
    if (reuse) CUDA_TRY(cudaStreamWaitEvent(pl->pipe_in, pl->pipe_ev_comp[k], 0));
    CUDA_TRY(cudaMemcpyAsync(pl->pipe_A[k], ah + (size_t)b0 * a_per_b, (size_t)nb * a_per_b,
                             cudaMemcpyHostToDevice, pl->pipe_in));
    CUDA_TRY(cudaEventRecord(pl->pipe_ev_in[k], pl->pipe_in));
    CUDA_TRY(cudaStreamWaitEvent(st, pl->pipe_ev_in[k], 0));
    if (reuse) CUDA_TRY(cudaStreamWaitEvent(st, pl->pipe_ev_out[k], 0));
    const int rc = covgpu_plan_execute(sp, pl->pipe_A[k], pl->pipe_R[k], layout, scale, st);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(pl->pipe_ev_comp[k], st));
    CUDA_TRY(cudaStreamWaitEvent(pl->pipe_out, pl->pipe_ev_comp[k], 0));
    CUDA_TRY(cudaMemcpyAsync(rh + (size_t)b0 * r_per_b * esz, pl->pipe_R[k],
                             (size_t)nb * r_per_b * esz, cudaMemcpyDeviceToHost, pl->pipe_out));
    CUDA_TRY(cudaEventRecord(pl->pipe_ev_out[k], pl->pipe_out));
  }
  CUDA_TRY(cudaStreamSynchronize(pl->pipe_out));
  for (int k = 0; k < covgpu_plan::kPipeSlots; ++k) CUDA_TRY(cudaStreamSynchronize(pl->pipe_stream[k]));
  CUDA_TRY(cudaStreamSynchronize(pl->pipe_in));
  return COVGPU_OK;
}

// cuStreamWriteValue32 through the runtime's driver entry point (no -lcuda)
static PFN_cuStreamWriteValue32_v11070 stream_write_value() {
  static PFN_cuStreamWriteValue32_v11070 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
  }();
  return fn;
}

// Stream A in row bands?  Single snapshot on the tensor-core path, A large
// enough for the overlap to matter, the driver's stream write available.
// Sets up the copy stream, band flag and event on first use.
static bool stream_a_in_bands(covgpu_plan* pl, size_t a_bytes) {
  if (!pl->use_mma || pl->batch != 1 || a_bytes < (8u << 20) || !stream_write_value()) return false;
  if (const char* e = hook_env("COVGPU_NO_BAND_H2D"))
    if (atoi(e) != 0) return false;
  if (!pl->d_band_flag) {
    if (cudaMalloc(&pl->d_band_flag, sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(pl->d_band_flag, 0, sizeof(unsigned)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&pl->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&pl->ev_h2d, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    pl->band_base = 0;
  }
  pl->band_rows = host_band_rows(pl->pr.N);
  return true;
}

static bool chunked_copy_out(covgpu_plan* pl, int layout);
static int copy_out_chunks(covgpu_plan* pl, void* R_host, int layout, size_t esz);

int covgpu_plan_execute_host(covgpu_plan_t pl, const void* A_host, void* R_host, int32_t layout,
                             double scale) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  if (!A_host || !R_host) return fail(COVGPU_EINVAL, "host buffers must be non-NULL");
  if (layout < COVGPU_DENSE || layout > COVGPU_COMPACT) return fail(COVGPU_EINVAL, "unknown layout");
  CUDA_TRY(cudaSetDevice(pl->device));
  const Problem& pr = pl->pr;
  const size_t esz = pl->dtype == COVGPU_C128 ? 16 : 8;
  const size_t a_bytes = (size_t)pl->batch * pr.N * pr.M * esz;
  long long r_elems;
  if (layout == COVGPU_DENSE)
    r_elems = pl->batch * (long long)pr.PQ * pr.PQ;
  else if (layout == COVGPU_PACKED)
    r_elems = pl->batch * ((long long)pr.PQ * (pr.PQ + 1) / 2);
  else
    r_elems = pl->batch * pl->compact_elems;
  const size_t r_bytes = (size_t)r_elems * esz;
  std::lock_guard<std::mutex> lk(pl->host_mu);
  if (pl->batch >= 8) return execute_host_pipelined(pl, A_host, R_host, layout, scale);
  if (!pl->host_stream) {
    // greatest priority: in the tail after the last band of A the main chain
    // (last correlation, output FFTs, walk) goes before the side stream's edge sums
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUDA_TRY(cudaStreamCreateWithPriority(&pl->host_stream, cudaStreamNonBlocking, hi));
  }
  if (pl->hA_bytes < a_bytes) {
    cudaFree(pl->hA);
    pl->hA = nullptr;
    pl->hA_bytes = 0;
    CUDA_TRY(cudaMalloc(&pl->hA, a_bytes));
    pl->hA_bytes = a_bytes;
  }
  if (pl->hR_bytes < r_bytes) {
    cudaFree(pl->hR);
    pl->hR = nullptr;
    pl->hR_bytes = 0;
    CUDA_TRY(cudaMalloc(&pl->hR, r_bytes));
    pl->hR_bytes = r_bytes;
  }
  cudaStream_t st = pl->host_stream;
  int rc;
  struct ChunkReset {  // the chunked walk is this call's only: reset on every exit path
    covgpu_plan* p;
    ~ChunkReset() { p->fin_nchunks = 1; }
  } chunk_reset{pl};
  chunked_copy_out(pl, layout);  // sets fin_nchunks > 1 when the walk can be chunked
  if (stream_a_in_bands(pl, a_bytes)) {
    // A in row bands on the copy stream, overlapped with the tensor-core
    // bulk kernel (which waits per chunk for the band it reads)
    const int nb = (pr.N + pl->band_rows - 1) / pl->band_rows;
    const size_t row_bytes = (size_t)pr.M * esz;
    auto wv = stream_write_value();
    const unsigned base = pl->band_base;
    const bool strips_first = pl->use_spec && pl->batch == 1;
    const int S = pr.P - 1;
    char* dA = (char*)pl->hA;
    const char* hA = (const char*)A_host;
    if (strips_first) {
      // spectral engine: the top / bottom strip rows first (whole rows, two
      // contiguous copies) — the edge-row sums, the strip-row spectra and the
      // walk's corner blocks need only these — then the other rows in bands
      // of whole rows (contiguous copies at the full link rate; the
      // edge-column sums wait for the last band and run beside the last
      // band's correlation)
      if (!pl->ev_strips) CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_strips, cudaEventDisableTiming));
      if (S > 0) {
        CUDA_TRY(cudaMemcpyAsync(dA, hA, (size_t)S * row_bytes, cudaMemcpyHostToDevice, pl->copy_stream));
        CUDA_TRY(cudaMemcpyAsync(dA + (size_t)(pr.N - S) * row_bytes, hA + (size_t)(pr.N - S) * row_bytes,
                                 (size_t)S * row_bytes, cudaMemcpyHostToDevice, pl->copy_stream));
      }
      CUDA_TRY(cudaEventRecord(pl->ev_strips, pl->copy_stream));
    }
    for (int k = 0; k < nb; ++k) {
      int r0 = k * pl->band_rows, r1 = std::min(pr.N, r0 + pl->band_rows);
      if (strips_first) {
        r0 = std::max(r0, S);
        r1 = std::min(r1, pr.N - S);
      }
      if (r1 > r0)
        CUDA_TRY(cudaMemcpyAsync(dA + r0 * row_bytes, hA + r0 * row_bytes, (r1 - r0) * row_bytes,
                                 cudaMemcpyHostToDevice, pl->copy_stream));
      if (strips_first) {
        // the spectral path waits per band on the host side: an event per band
        if ((int)pl->ev_band.size() < nb) pl->ev_band.resize(nb, nullptr);
        if (!pl->ev_band[k]) CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_band[k], cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(pl->ev_band[k], pl->copy_stream));
      } else if (wv(pl->copy_stream, (CUdeviceptr)pl->d_band_flag, base + (unsigned)k + 1u, 0) != CUDA_SUCCESS) {
        return fail(COVGPU_ECUDA, "cuStreamWriteValue32");
      }
    }
    CUDA_TRY(cudaEventRecord(pl->ev_h2d, pl->copy_stream));
    pl->band_wait = true;
    rc = covgpu_plan_execute(pl, pl->hA, pl->hR, layout, scale, st);
    pl->band_wait = false;
    pl->band_base = base + (unsigned)nb;
    // every later use of hA on `st` (the next execute's copies run on the
    // copy stream) must follow this execute
    if (!rc) CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_h2d, 0));
  } else {
    CUDA_TRY(cudaMemcpyAsync(pl->hA, A_host, a_bytes, cudaMemcpyHostToDevice, st));
    rc = covgpu_plan_execute(pl, pl->hA, pl->hR, layout, scale, st);
  }
  if (rc) return rc;
  if (pl->fin_nchunks > 1) {  // chunked walk: the copy-out follows each chunk
    rc = copy_out_chunks(pl, R_host, layout, esz);
    pl->fin_nchunks = 1;
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(pl->out_stream));
    CUDA_TRY(cudaStreamSynchronize(st));
    return COVGPU_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(R_host, pl->hR, r_bytes, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return COVGPU_OK;
}

// Synchronous host path with the copy-out overlapped with the finalize walk:
// the walk runs in u-chunks (state saved between them); rows [P u_c, P u_c+1)
// of R are complete after chunk c, so their D2H starts on out_stream while
// the next chunk runs.  Single snapshot, dense / packed, direct finalize.
static bool chunked_copy_out(covgpu_plan* pl, int layout) {
  if (pl->batch != 1 || !pl->clean || pl->fin_kr == 0 || pl->no_direct || layout == COVGPU_COMPACT) return false;
  // large outputs only (cfg5 packed 134 MB: 4.44 -> 4.30 ms; cfg3 8 MB: the
  // chunk launches cost more than the overlap gains, 0.353 -> 0.447 ms)
  const long long D = pl->pr.PQ;
  if (pl->pr.Q < 24 || D * (D + 1) / 2 * 16 < (32LL << 20)) return false;
  if (const char* e = hook_env("COVGPU_NO_CHUNKED_D2H"))
    if (atoi(e) != 0) return false;
  if (!pl->d_fin_state) {
    // events first: the state buffer marks a completed setup
    for (auto& e : pl->ev_fin_chunk)
      if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        e = nullptr;
        return false;
      }
    const size_t n = pl->use_tile ? (size_t)pl->n_units * 32 * pl->ft_nwarp * FT_STATE
                                  : (size_t)pl->ntasks * 32 * (2 * pl->fin_kr + 1);
    if (cudaMalloc((void**)&pl->d_fin_state, sizeof(double2) * std::max<size_t>(n, 1)) != cudaSuccess) {
      cudaGetLastError();
      pl->d_fin_state = nullptr;
      return false;
    }
  }
  if (!pl->out_stream && cudaStreamCreateWithFlags(&pl->out_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // small first chunks: the copy-out starts early (the first rows are the longest)
  const int Q = pl->pr.Q;
  pl->fin_ubound[0] = 0;
  pl->fin_ubound[1] = std::max(1, Q / 32);
  pl->fin_ubound[2] = std::max(pl->fin_ubound[1] + 1, Q / 6);
  pl->fin_ubound[3] = Q;
  pl->fin_nchunks = 3;
  return true;
}

static int copy_out_chunks(covgpu_plan* pl, void* R_host, int layout, size_t esz) {
  const long long D = pl->pr.PQ;
  auto row_off = [&](long long k1) -> long long {
    return layout == COVGPU_DENSE ? k1 * D : k1 * D - (k1 * (k1 - 1)) / 2;
  };
  for (int c = 0; c < pl->fin_nchunks; ++c) {
    const long long k0 = std::min(D, (long long)pl->pr.P * pl->fin_ubound[c]);
    const long long k1 = std::min(D, (long long)pl->pr.P * pl->fin_ubound[c + 1]);
    CUDA_TRY(cudaStreamWaitEvent(pl->out_stream, pl->ev_fin_chunk[c], 0));
    const long long o0 = row_off(k0), o1 = c + 1 == pl->fin_nchunks ? row_off(D) : row_off(k1);
    if (o1 > o0)
      CUDA_TRY(cudaMemcpyAsync((char*)R_host + o0 * esz, (const char*)pl->hR + o0 * esz, (size_t)(o1 - o0) * esz,
                               cudaMemcpyDeviceToHost, pl->out_stream));
  }
  return COVGPU_OK;
}

int covgpu_plan_execute_host_async(covgpu_plan_t pl, const void* A_host, void* R_host, int32_t layout,
                                   double scale) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  if (!A_host || !R_host) return fail(COVGPU_EINVAL, "host buffers must be non-NULL");
  if (layout < COVGPU_DENSE || layout > COVGPU_COMPACT) return fail(COVGPU_EINVAL, "unknown layout");
  if (pl->batch >= 8) {
    const int rc = covgpu_plan_execute_host(pl, A_host, R_host, layout, scale);
    if (rc && !pl->as_err) pl->as_err = rc;
    return rc;
  }
  CUDA_TRY(cudaSetDevice(pl->device));
  const Problem& pr = pl->pr;
  const size_t esz = pl->dtype == COVGPU_C128 ? 16 : 8;
  const size_t a_bytes = (size_t)pl->batch * pr.N * pr.M * esz;
  long long r_elems;
  if (layout == COVGPU_DENSE)
    r_elems = pl->batch * (long long)pr.PQ * pr.PQ;
  else if (layout == COVGPU_PACKED)
    r_elems = pl->batch * ((long long)pr.PQ * (pr.PQ + 1) / 2);
  else
    r_elems = pl->batch * pl->compact_elems;
  const size_t r_bytes = (size_t)r_elems * esz;
  std::lock_guard<std::mutex> lk(pl->host_mu);
  if (!pl->host_stream) {
    // greatest priority: in the tail after the last band of A the main chain
    // (last correlation, output FFTs, walk) goes before the side stream's edge sums
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUDA_TRY(cudaStreamCreateWithPriority(&pl->host_stream, cudaStreamNonBlocking, hi));
  }
  if (!pl->as_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&pl->as_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&pl->as_out, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaEventCreateWithFlags(&pl->as_ev_in[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&pl->as_ev_comp[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&pl->as_ev_out[k], cudaEventDisableTiming));
    }
  }
  if (pl->asA_bytes < a_bytes || pl->asR_bytes < r_bytes) {
    CUDA_TRY(cudaDeviceSynchronize());  // (re)size only with nothing in flight
    for (int k = 0; k < 2; ++k) {
      cudaFree(pl->asA[k]);
      cudaFree(pl->asR[k]);
      pl->asA[k] = pl->asR[k] = nullptr;
    }
    pl->asA_bytes = pl->asR_bytes = 0;
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaMalloc(&pl->asA[k], a_bytes));
      CUDA_TRY(cudaMalloc(&pl->asR[k], r_bytes));
    }
    pl->asA_bytes = a_bytes;
    pl->asR_bytes = r_bytes;
    pl->as_n = 0;
  }
  const int sl = (int)(pl->as_n & 1);
  const bool reuse = pl->as_n >= 2;  // slot used by call k-2
  // copy-in: A slot free once call k-2's estimate has read it
  if (reuse) CUDA_TRY(cudaStreamWaitEvent(pl->as_in, pl->as_ev_comp[sl], 0));
  CUDA_TRY(cudaMemcpyAsync(pl->asA[sl], A_host, a_bytes, cudaMemcpyHostToDevice, pl->as_in));
  CUDA_TRY(cudaEventRecord(pl->as_ev_in[sl], pl->as_in));
  // estimate: after its copy-in, and after call k-2's copy-out freed the R slot
  CUDA_TRY(cudaStreamWaitEvent(pl->host_stream, pl->as_ev_in[sl], 0));
  if (reuse) CUDA_TRY(cudaStreamWaitEvent(pl->host_stream, pl->as_ev_out[sl], 0));
  int rc = covgpu_plan_execute(pl, pl->asA[sl], pl->asR[sl], layout, scale, pl->host_stream);
  if (rc) {
    if (!pl->as_err) pl->as_err = rc;
    return rc;
  }
  CUDA_TRY(cudaEventRecord(pl->as_ev_comp[sl], pl->host_stream));
  // copy-out
  CUDA_TRY(cudaStreamWaitEvent(pl->as_out, pl->as_ev_comp[sl], 0));
  CUDA_TRY(cudaMemcpyAsync(R_host, pl->asR[sl], r_bytes, cudaMemcpyDeviceToHost, pl->as_out));
  CUDA_TRY(cudaEventRecord(pl->as_ev_out[sl], pl->as_out));
  ++pl->as_n;
  return COVGPU_OK;
}

int covgpu_plan_wait(covgpu_plan_t pl) {
  if (!pl) return fail(COVGPU_EINVAL, "plan is NULL");
  CUDA_TRY(cudaSetDevice(pl->device));
  std::lock_guard<std::mutex> lk(pl->host_mu);
  if (pl->as_out) CUDA_TRY(cudaStreamSynchronize(pl->as_out));
  if (pl->host_stream) CUDA_TRY(cudaStreamSynchronize(pl->host_stream));
  if (pl->as_in) CUDA_TRY(cudaStreamSynchronize(pl->as_in));
  const int e = pl->as_err;
  pl->as_err = 0;
  return e;
}

int covgpu_bulk_geometry(int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q, int32_t dtype,
                         int32_t* lags, int32_t* warps) {
  if (p < 1 || q < 1 || batch < 1 || !lags || !warps) return fail(COVGPU_EINVAL, "bad arguments");
  const int v = pick_bulk_variant(n, m, p, q, batch, dtype);
  *lags = kBulkVariants[v].E;
  *warps = kBulkVariants[v].NW;
  return COVGPU_OK;
}

int covgpu_scatter_compact(const void* compact_dev, int64_t batch, int64_t n, int64_t m, int32_t p,
                           int32_t q, int32_t dtype, const int32_t* class_ids, int32_t n_classes,
                           void* R_dev, void* stream) {
  int rc = validate(batch, n, m, p, q, dtype);
  if (rc) return rc;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::shared_ptr<covgpu_plan> pl;
  rc = cached_plan(&pl, dev, batch, n, m, p, q, dtype, class_ids, n_classes);
  if (rc) return rc;
  if (pl->nclasses == 0 || pl->compact_elems == 0) return COVGPU_OK;
  const long long total = pl->compact_elems * batch;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == COVGPU_C128)
    k_scatter_compact<double><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        (const double2*)compact_dev, pl->pr, pl->d_cls, pl->nclasses, pl->compact_elems, (int)batch,
        (double2*)R_dev);
  else
    k_scatter_compact<float><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        (const float2*)compact_dev, pl->pr, pl->d_cls, pl->nclasses, pl->compact_elems, (int)batch,
        (float2*)R_dev);
  CUDA_TRY(cudaGetLastError());
  return COVGPU_OK;
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

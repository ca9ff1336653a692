/*
 * covgpu — B200-native windowed covariance estimation (arXiv 1303.2285).
 *
 * C ABI of libcovgpu.so.  No torch or CUDA types appear in the signatures:
 * device pointers are plain `void*`, the CUDA stream is passed as `void*`
 * (a cudaStream_t, NULL = the legacy default stream).
 *
 * Every entry point returns 0 on success and a negative COVGPU_E* code on
 * failure; nothing throws across the ABI.  covgpu_last_error() returns the
 * calling thread's last error text.  Calls are thread-safe per (device,
 * stream).  Like the reference, kernels never validate numeric content; all
 * argument checks happen here, before any launch.
 *
 * Replaces (the drop-in seam):
 *   - engine._load_kernels / engine._run_class
 *       /root/reference/pkg/src/covcomb/engine.py:78-83, :95-101
 *     and the per-class kernels they dispatch to
 *       _numba_kernels.combination_scratch  _numba_kernels.py:62-107
 *       _numba_kernels.combination_direct   _numba_kernels.py:35-59
 *       _numpy_kernels.apply_combination    _numpy_kernels.py:67-68
 *     with ONE call per estimate (covgpu_estimate / covgpu_plan_execute);
 *   - the per-class call shape itself is kept as covgpu_combination
 *     (same arguments as combination_scratch(a, dr, dc, p, q, out, ...));
 *   - _numba_kernels.warmup (_numba_kernels.py:110-119) -> covgpu_init.
 */
#ifndef COVGPU_H
#define COVGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define COVGPU_OK 0
#define COVGPU_EINVAL -1   /* bad argument (reference: ValueError)          */
#define COVGPU_ECUDA -2    /* CUDA runtime failure (reference: RuntimeError) */
#define COVGPU_ENOMEM -3   /* device allocation failed                      */
#define COVGPU_ECAPACITY -4 /* packed triangle beyond 2^31-1 (core.py:147-151) */

/* element types of A and R */
#define COVGPU_C128 0 /* complex double, interleaved re/im (numpy complex128) */
#define COVGPU_C64 1  /* complex float  (numpy complex64)                     */

/* output layouts */
#define COVGPU_DENSE 0   /* (batch, PQ, PQ) row-major, exactly Hermitian       */
#define COVGPU_PACKED 1  /* (batch, PQ(PQ+1)/2) upper triangle, row-major    */
                         /* = reference CovarianceMatrix.packed (core.py:140-162) */
#define COVGPU_COMPACT 2 /* (batch, sum_c eta_c) class-major slot order:      */
                         /* class c in UC order, then u-major, then v         */

typedef struct covgpu_plan* covgpu_plan_t;

/* Context creation + one warm launch on `device` (replaces numba warmup). */
int covgpu_init(int device);

/* Text of the calling thread's last error ("" if none). */
const char* covgpu_last_error(void);

/* Library version string. */
const char* covgpu_version(void);

/* Number of offset classes |UC| = PQ + (P-1)(Q-1) (combinations.py:53-62). */
int64_t covgpu_num_classes(int32_t p, int32_t q);

/* Elements of R for a layout (batch included).  For COVGPU_COMPACT with a
 * class subset, only the selected classes' slots are counted. */
int64_t covgpu_output_elems(int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q,
                            int32_t layout, const int32_t* class_ids, int32_t n_classes);

/* Build an execution plan: class table, bulk work groups, device workspace.
 * class_ids (UC indices, NULL = all classes) selects a shard of the classes.
 * Validation mirrors the reference: n,m >= 1; 1 <= p <= n; 1 <= q <= m
 * (core.py:82-93, :101-106); packed size <= 2^31-1 (core.py:147-151). */
int covgpu_plan_create(covgpu_plan_t* plan, int device, int64_t batch, int64_t n, int64_t m,
                       int32_t p, int32_t q, int32_t dtype, const int32_t* class_ids,
                       int32_t n_classes);

/* R = scale * sum_windows x x^H for every selected class, written in `layout`.
 * A_dev: (batch, n, m) device array of `dtype`; R_dev: covgpu_output_elems
 * elements of `dtype`.  With every class selected every element of R is
 * written exactly once (single writer, no atomics); with a subset the other
 * elements are left untouched.  Asynchronous on `stream`. */
int covgpu_plan_execute(covgpu_plan_t plan, const void* A_dev, void* R_dev, int32_t layout,
                        double scale, void* stream);

/* Bytes of device workspace the plan holds. */
int64_t covgpu_plan_workspace_bytes(covgpu_plan_t plan);

/* Number of bulk work groups and kernel launches one execute issues. */
int32_t covgpu_plan_num_groups(covgpu_plan_t plan);
int32_t covgpu_plan_launches(covgpu_plan_t plan);

/* Environment: the library reads no configuration from the environment.  The
 * COVGPU_* switches in csrc/covgpu.cu (engine forcing and kernel variants for
 * the parity tests and for the comparison runs of bench.py) are test hooks,
 * honoured only when COVGPU_TEST_HOOKS=1 is set before the first plan is made;
 * cached plans are keyed on them. */

/* Which sum kernels the plan runs (bit flags): COVGPU_PATH_SPECTRAL — the
 * core / edge sums in the frequency domain (row and column FFTs, per-frequency
 * row-lag correlation); COVGPU_PATH_TENSOR — the core sums as Toeplitz GEMMs
 * on the FP64 tensor cores; COVGPU_PATH_SNAPSHOT — the sums of each small
 * complex64 snapshot inside one CTA in FP32 (batched per-snapshot kernel);
 * none of the three — the CUDA-core recurrence kernels;
 * COVGPU_PATH_ROWBAND — covgpu_plan_execute_sums is available.  Replaces the
 * reference's backend query (backend.resolve_backend, backend.py:45-57). */
#define COVGPU_PATH_SPECTRAL 1
#define COVGPU_PATH_TENSOR 2
#define COVGPU_PATH_ROWBAND 4
#define COVGPU_PATH_SNAPSHOT 8
int32_t covgpu_plan_path(covgpu_plan_t plan);

/* Record CUDA events around every kernel of subsequent executes (on the
 * execute's stream) so covgpu_plan_kernel_times can report per-kernel times. */
int covgpu_plan_set_timing(covgpu_plan_t plan, int32_t enable);

/* Per-kernel durations (ms) of the last timed execute, in launch order
 * (bulk, edge rows, finalize); waits for it.  Returns the count written. */
int32_t covgpu_plan_kernel_times(covgpu_plan_t plan, float* ms, int32_t max_n);

/* Comma-separated kernel names of those intervals ("bulk_dmma,edge_cols,
 * edge_rows,finalize,expand" or "bulk,edge_rows,finalize,expand" ...) into
 * buf (NUL-terminated, truncated to len).  Returns the count. */
int32_t covgpu_plan_kernel_names(covgpu_plan_t plan, char* buf, int32_t len);

/* Multi-GPU row bands (the core / edge sums are sums over rows and columns
 * of A, so they split over the K dimension with one exchange of the per-band
 * sums; replaces the reference's per-class work split, engine.py:158-190,
 * with a split that keeps every GPU on the spectral / tensor-core sums).
 * sums_elems: complex128 values of the sums buffer [CC | CCol | RC'].
 * execute_sums: part `part` of `nparts` of every sum (the driver runs a
 * FIXED number of parts, independent of the GPU count, and adds the parts of
 * a class range in part order, so R is bitwise the same on any number of
 * GPUs; distributed.py).  finalize_sums:
 * corners + diagonal-segment walk from the reduced sums for plan classes
 * [class_lo, class_hi) (a sub-range writes its slots of the COMPACT layout;
 * the full range may write DENSE / PACKED).  class_slot_offset: compact
 * offset of a plan class (class_index == #classes: total).  Requires the
 * spectral path or the complex128 tensor-core path (COVGPU_PATH_ROWBAND;
 * COVGPU_ECAPACITY otherwise). */
int64_t covgpu_plan_sums_elems(covgpu_plan_t plan);
int covgpu_plan_execute_sums(covgpu_plan_t plan, const void* A_dev, void* sums_dev, int32_t part,
                             int32_t nparts, void* stream);
int covgpu_plan_finalize_sums(covgpu_plan_t plan, const void* A_dev, const void* sums_dev, void* R_dev,
                              int32_t layout, double scale, int32_t class_lo, int32_t class_hi,
                              void* stream);
int64_t covgpu_plan_class_slot_offset(covgpu_plan_t plan, int32_t class_index);

/* Where the sums of plan classes [class_lo, class_hi) of snapshot 0 sit in
 * the sums buffer: out[0..5] = [cc_begin, cc_end, ccol_begin, ccol_end,
 * rc_begin, rc_end) — the slices a GPU finalizing that range needs (the
 * row-band exchange sends only those).  Returns 0 or an error code. */
int covgpu_plan_sums_range(covgpu_plan_t plan, int32_t class_lo, int32_t class_hi, int64_t* out);

/* Rows of A that part `part` of `nparts` of execute_sums reads besides the
 * top / bottom P-1 strip rows and the first / last Q-1 columns of every row:
 * [*row_begin, *row_end).  A GPU holding only those regions of A (the rest
 * unset) computes the same part bit for bit: the row-band input split. */
int covgpu_plan_band_rows(covgpu_plan_t plan, int32_t part, int32_t nparts, int32_t* row_begin,
                          int32_t* row_end);

int covgpu_plan_destroy(covgpu_plan_t plan);

/* One-shot estimate on device buffers (plan cached per shape internally). */
int covgpu_estimate(const void* A_dev, int64_t batch, int64_t n, int64_t m, int32_t p,
                    int32_t q, int32_t dtype, int32_t layout, const int32_t* class_ids,
                    int32_t n_classes, double scale, void* R_dev, void* stream);

/* End-to-end estimate on HOST buffers: H2D of A, compute, D2H of R on a
 * library-owned stream (device buffers cached with the plan); returns after
 * the result is in R_host.  Pinned host buffers give full PCIe bandwidth. */
int covgpu_estimate_host(const void* A_host, int64_t batch, int64_t n, int64_t m, int32_t p,
                         int32_t q, int32_t dtype, int32_t layout, double scale, void* R_host,
                         int device);

/* End-to-end execute of a plan on HOST buffers (its class shard only; for a
 * shard use COVGPU_COMPACT to receive just the shard's slots). */
int covgpu_plan_execute_host(covgpu_plan_t plan, const void* A_host, void* R_host, int32_t layout,
                             double scale);

/* Streaming form of covgpu_plan_execute_host for a sequence of estimates
 * (e.g. one per radar dwell / image frame): enqueues the H2D of A, the
 * estimate and the D2H of R and returns; up to two calls are in flight (the
 * device buffers are double-buffered), so call k+1's copy-in and compute run
 * under call k's copy-out.  The host must not write A_host or read R_host
 * until covgpu_plan_wait returns (later calls may reuse the same buffers:
 * the copies of calls sharing a device slot are ordered); pinned memory for
 * full PCIe bandwidth.  Batched
 * plans (batch >= 8) run synchronously (they pipeline internally).
 * covgpu_plan_wait blocks until every enqueued call has finished and returns
 * the first error.  The reference's API is synchronous (SPEC.md:341,
 * engine.py:108-147); this is an addition for throughput. */
int covgpu_plan_execute_host_async(covgpu_plan_t plan, const void* A_host, void* R_host, int32_t layout,
                                   double scale);
int covgpu_plan_wait(covgpu_plan_t plan);

/* Bench utility: FP64 (dtype COVGPU_C128) or FP32 (COVGPU_C64) FMA-pipe
 * throughput in TFLOP/s, measured for about `seconds` on `device` — the
 * roofline denominator of the covariance kernels. */
int covgpu_probe_fma_peak(int device, int32_t dtype, double seconds, double* tflops);

/* Bench utility: FP64 tensor-core (DMMA) throughput in TFLOP/s — the
 * roofline denominator of the tensor-core bulk kernel (complex128). */
int covgpu_probe_dmma_peak(int device, double seconds, double* tflops);

/* Bulk-kernel work unit of a shape: `lags` row lags x `warps` column lags
 * per CTA.  The partitioner shards classes in whole units. */
int covgpu_bulk_geometry(int64_t batch, int64_t n, int64_t m, int32_t p, int32_t q, int32_t dtype,
                         int32_t* lags, int32_t* warps);

/* Scatter a COVGPU_COMPACT shard (the slots of `class_ids`, class-major) into
 * a dense Hermitian R_dev (both triangles) — the root's half of the multi-GPU
 * gather (reference CovarianceMatrix.dense(), core.py:170-176). */
int covgpu_scatter_compact(const void* compact_dev, int64_t batch, int64_t n, int64_t m, int32_t p,
                           int32_t q, int32_t dtype, const int32_t* class_ids, int32_t n_classes,
                           void* R_dev, void* stream);

/* Per-class call with the reference kernel's argument shape
 * (combination_scratch(a, dr, dc, p, q, out, ...), _numba_kernels.py:62-107):
 * writes ONLY class (dr, dc)'s slots of the packed upper triangle `out_dev`
 * (unnormalised, as the reference does).  A_dev is (n, m) complex128. */
int covgpu_combination(const void* A_dev, int64_t n, int64_t m, int32_t dr, int32_t dc,
                       int32_t p, int32_t q, void* out_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* COVGPU_H */

/*
 * covoracle.c — C restatement of the reference's class-decomposition
 * estimator.  TEST INFRASTRUCTURE ONLY: loaded by tests/ (parity spot checks
 * at full size) and by bench.py's CPU-baseline leg; never by the product.
 *
 * Algorithm = the reference's vectorised class kernel
 * (pkg/src/covcomb/_numpy_kernels.py:30-53, driven per class by
 * engine.py:132-145): for class (dr, dc) form the product pane
 *   prod[i,j] = A[i+s1, j] * conj(A[i+s2, j+dc])   (|a|^2 for class (0,0))
 * take its 2-D prefix sum X, and read every slot as the four-corner box sum
 *   S(v,u) = X[v+bh][u+bw] - X[v][u+bw] - X[v+bh][u] + X[v][u].
 * The prefix table is streamed row by row and only the rows/columns the
 * four-corner reads touch are kept, so memory is O(M + P*Q) per class.
 * Classes are independent (disjoint slots), so a pthread pool pulls them from
 * a shared atomic cursor — the reference's thread pool over classes
 * (engine.py:158-190).
 *
 * Complex numbers are interleaved (re, im) doubles, numpy complex128 layout.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

static void class_dr_dc(int uc, int p, int q, int* dr, int* dc) {
  /* UC order, combinations.py:53-62 */
  if (uc < p * q) {
    *dr = uc / q;
    *dc = uc % q;
  } else {
    int r = uc - p * q;
    *dr = r / (q - 1) - (p - 1);
    *dc = r % (q - 1) + 1;
  }
}

/* Slot sums of one class, u-major then v (reference slot order), unnormalised. */
int cov_class_slots(const double* A, int n, int m, int p, int q, int dr, int dc, double* out) {
  const int adr = dr < 0 ? -dr : dr;
  const int s1 = dr < 0 ? -dr : 0, s2 = dr > 0 ? dr : 0;
  const int H = n - adr, W = m - dc;
  const int bh = n - p + 1, bw = m - q + 1;
  const int pv = p - adr, qu = q - dc;
  /* running 2-D prefix row X[i][0..W] and the kept rows / columns */
  double* xrow = (double*)calloc((size_t)2 * (W + 1), sizeof(double));
  double* keep = (double*)calloc((size_t)2 * pv * 2 * (2 * qu), sizeof(double)); /* [2 sets][pv][2qu] */
  if (!xrow || !keep) {
    free(xrow);
    free(keep);
    return -1;
  }
  const int self = (dr == 0 && dc == 0);
  for (int i = 0; i <= H; ++i) {
    if (i > 0) {
      const double* x = A + 2 * ((size_t)(i - 1 + s1) * m);
      const double* y = A + 2 * ((size_t)(i - 1 + s2) * m + dc);
      double rr = 0.0, ri = 0.0; /* row prefix of prod[i-1, :] */
      for (int j = 0; j < W; ++j) {
        const double xr = x[2 * j], xi = x[2 * j + 1];
        if (self) {
          rr += xr * xr + xi * xi;
        } else {
          const double yr = y[2 * j], yi = y[2 * j + 1];
          rr += xr * yr + xi * yi;
          ri += xi * yr - xr * yi;
        }
        xrow[2 * (j + 1)] += rr;
        xrow[2 * (j + 1) + 1] += ri;
      }
    }
    /* rows v (set 0) and v + bh (set 1) of the table are read by the slots */
    for (int set = 0; set < 2; ++set) {
      const int v = i - (set ? bh : 0);
      if (v < 0 || v >= pv) continue;
      double* k = keep + 2 * ((size_t)(set * pv + v) * 2 * qu);
      for (int u = 0; u < qu; ++u) {
        k[2 * u] = xrow[2 * u];
        k[2 * u + 1] = xrow[2 * u + 1];
        k[2 * (qu + u)] = xrow[2 * (u + bw)];
        k[2 * (qu + u) + 1] = xrow[2 * (u + bw) + 1];
      }
    }
  }
  for (int u = 0; u < qu; ++u) {
    for (int v = 0; v < pv; ++v) {
      const double* top = keep + 2 * ((size_t)(0 * pv + v) * 2 * qu);
      const double* bot = keep + 2 * ((size_t)(1 * pv + v) * 2 * qu);
      /* X[v+bh][u+bw] - X[v][u+bw] - X[v+bh][u] + X[v][u] */
      double re = ((bot[2 * (qu + u)] - top[2 * (qu + u)]) - bot[2 * u]) + top[2 * u];
      double im = ((bot[2 * (qu + u) + 1] - top[2 * (qu + u) + 1]) - bot[2 * u + 1]) + top[2 * u + 1];
      if (self) im = 0.0;
      double* o = out + 2 * ((size_t)u * pv + v);
      o[0] = re;
      o[1] = im;
    }
  }
  free(xrow);
  free(keep);
  return 0;
}

struct job {
  const double* A;
  int n, m, p, q;
  const int* ids;
  int count;
  double* packed;
  atomic_int cursor;
  atomic_int status;
};

static void run_class(struct job* jb, int k) {
  const int p = jb->p, q = jb->q;
  const long long dim = (long long)p * q;
  const int uc = jb->ids ? jb->ids[k] : k;
  int dr, dc;
  class_dr_dc(uc, p, q, &dr, &dc);
  const int adr = dr < 0 ? -dr : dr;
  const int pv = p - adr, qu = q - dc;
  const int s1 = dr < 0 ? -dr : 0;
  double* slots = (double*)malloc(sizeof(double) * 2 * (size_t)pv * qu);
  if (!slots || cov_class_slots(jb->A, jb->n, jb->m, p, q, dr, dc, slots)) {
    atomic_store(&jb->status, -1);
    free(slots);
    return;
  }
  for (int u = 0; u < qu; ++u) {
    for (int v = 0; v < pv; ++v) {
      const long long k1 = (long long)p * u + s1 + v;
      const long long k2 = k1 + (long long)dc * p + dr;
      const long long off = k1 * dim - (k1 * (k1 - 1)) / 2 + (k2 - k1);
      jb->packed[2 * off] = slots[2 * ((size_t)u * pv + v)];
      jb->packed[2 * off + 1] = slots[2 * ((size_t)u * pv + v) + 1];
    }
  }
  free(slots);
}

static void* worker(void* arg) {
  struct job* jb = (struct job*)arg;
  for (;;) {
    const int k = atomic_fetch_add(&jb->cursor, 1);
    if (k >= jb->count) return NULL;
    run_class(jb, k);
  }
}

int cov_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* Packed upper triangle (core.py:60-72 layout) for the listed classes
 * (class_ids == NULL: all of UC), unnormalised.  `packed` must be zeroed by
 * the caller when only a subset is computed.  threads <= 0: all online CPUs. */
int cov_estimate_packed(const double* A, int n, int m, int p, int q, const int* class_ids, int ncls,
                        double* packed, int threads) {
  struct job jb;
  jb.A = A;
  jb.n = n;
  jb.m = m;
  jb.p = p;
  jb.q = q;
  jb.ids = class_ids;
  jb.count = class_ids ? ncls : p * q + (p - 1) * (q - 1);
  jb.packed = packed;
  atomic_init(&jb.cursor, 0);
  atomic_init(&jb.status, 0);
  if (threads <= 0) threads = cov_max_threads();
  if (threads > jb.count) threads = jb.count > 0 ? jb.count : 1;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  if (!tid) return -1;
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[t], NULL, worker, &jb) == 0) tid[started++ + 1] = tid[t];
  worker(&jb);
  for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
  free(tid);
  return atomic_load(&jb.status);
}

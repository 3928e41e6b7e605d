/* CSR sparse matrix-vector product y = A x, complex128, row-parallel over
 * POSIX threads.  TEST INFRASTRUCTURE ONLY (CPU baseline / oracle).
 * Restates the arithmetic of scipy's sparsetools csr_matvec (C++, scipy
 * 1.18.1, not vendored), which the reference reaches through
 * LatticeOperator.apply (lattice.py:214-217: `self.matrix @ x`): for row i,
 *   y[i] = sum_{k = indptr[i]}^{indptr[i+1]-1} data[k] * x[indices[k]]
 * accumulated in index order.  Rows are split into contiguous chunks, so each
 * row's summation order is the sequential one. */
#include <complex.h>
#include <pthread.h>
#include <stdint.h>
#include <unistd.h>

typedef struct {
  int64_t r0, r1;
  const int64_t *indptr, *indices;
  const double _Complex *data, *x;
  double _Complex *y;
} chunk_t;

static void *run_chunk(void *arg) {
  const chunk_t *c = (const chunk_t *)arg;
  for (int64_t i = c->r0; i < c->r1; ++i) {
    double _Complex s = 0.0;
    for (int64_t k = c->indptr[i]; k < c->indptr[i + 1]; ++k) s += c->data[k] * c->x[c->indices[k]];
    c->y[i] = s;
  }
  return 0;
}

int oracle_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 256) n = 256;
  return (int)n;
}

void oracle_csr_matvec_c128(int64_t nrows, const int64_t *indptr, const int64_t *indices,
                            const double _Complex *data, const double _Complex *x, double _Complex *y,
                            int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  chunk_t ch[256];
  for (int t = 0; t < nthreads; ++t) {
    ch[t].r0 = nrows * t / nthreads;
    ch[t].r1 = nrows * (t + 1) / nthreads;
    ch[t].indptr = indptr;
    ch[t].indices = indices;
    ch[t].data = data;
    ch[t].x = x;
    ch[t].y = y;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, run_chunk, &ch[t]);
  run_chunk(&ch[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
}

/* TEST INFRASTRUCTURE ONLY (see oracle/helmdef_oracle.py): the oracle's sparse
 * matrix-vector product y = A x for complex CSR matrices, in C with POSIX
 * threads over row blocks, so the full-size C5 oracle run fits a GPU test's
 * time budget.
 *
 * It restates the reference's `(*A) * v` (Eigen sparse x dense, every `*` on
 * SpMat in src/precond.cpp:103-107, :140, :147-151, :238, :262) exactly the
 * way the oracle's scipy product evaluates it (sparsetools csr_matvec: per row,
 * sum = 0; sum += a_jj * x_j in column order; complex product
 * (ar xr - ai xi, ar xi + ai xr)), compiled without FMA contraction, so the
 * result is bit-identical to scipy's for any thread count
 * (tests/test_oracle.py checks it).  Rows are independent, so threads only
 * split the row range. */
#include <pthread.h>
#include <stdint.h>

typedef struct {
  long r0, r1;
  const void* indptr;
  const void* indices;
  int wide;  /* 1: int64 indices */
  const double* a;
  const double* x;
  double* y;
} job_t;

static void* run(void* p) {
  const job_t* j = (const job_t*)p;
  for (long i = j->r0; i < j->r1; ++i) {
    long b, e;
    if (j->wide) {
      b = (long)((const int64_t*)j->indptr)[i];
      e = (long)((const int64_t*)j->indptr)[i + 1];
    } else {
      b = (long)((const int32_t*)j->indptr)[i];
      e = (long)((const int32_t*)j->indptr)[i + 1];
    }
    double sr = 0.0, si = 0.0;
    for (long jj = b; jj < e; ++jj) {
      const long c = j->wide ? (long)((const int64_t*)j->indices)[jj] : (long)((const int32_t*)j->indices)[jj];
      const double ar = j->a[2 * jj], ai = j->a[2 * jj + 1];
      const double xr = j->x[2 * c], xi = j->x[2 * c + 1];
      const double pr = ar * xr - ai * xi;
      const double pi = ar * xi + ai * xr;
      sr += pr;
      si += pi;
    }
    j->y[2 * i] = sr;
    j->y[2 * i + 1] = si;
  }
  return 0;
}

static void spmv(long nrows, const void* indptr, const void* indices, int wide, const double* a, const double* x,
                 double* y, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  job_t jobs[256];
  pthread_t tid[256];
  const long chunk = (nrows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    jobs[t].r0 = t * chunk < nrows ? t * chunk : nrows;
    jobs[t].r1 = (t + 1) * chunk < nrows ? (t + 1) * chunk : nrows;
    jobs[t].indptr = indptr;
    jobs[t].indices = indices;
    jobs[t].wide = wide;
    jobs[t].a = a;
    jobs[t].x = x;
    jobs[t].y = y;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], 0, run, &jobs[t]);
  run(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], 0);
}

void csr_spmv_c128_i32(long nrows, const int32_t* indptr, const int32_t* indices, const double* a, const double* x,
                       double* y, int threads) {
  spmv(nrows, indptr, indices, 0, a, x, y, threads);
}

void csr_spmv_c128_i64(long nrows, const int64_t* indptr, const int64_t* indices, const double* a, const double* x,
                       double* y, int threads) {
  spmv(nrows, indptr, indices, 1, a, x, y, threads);
}

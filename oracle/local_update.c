/* oracle/local_update.c -- TEST INFRASTRUCTURE ONLY (CPU baseline legs of
 * bench.py; never linked into or called by the product library).
 *
 * The two operator passes of one sensor's local update in Woodbury form
 * (oracle/admm_ref.py LocalSolve.solve, restating solver_core.hpp:47-51 for
 * KM < N):  v = A_J rhs  and  z = A_J^H w, written the way a tuned host
 * implementation would stream them: the complex64 operator is read once per
 * pass as stored (no complex128 copy, no materialised conjugate transpose),
 * OpenMP across column ranges, fp64 accumulation.  SURVEY section 8d asks for
 * a compiled OpenMP figure next to the NumPy oracle's.  The two triangular
 * solves in between (lu_chol_solve) are compiled too: SciPy's cho_solve turned
 * out to be 80 % of the NumPy oracle's local update at config 2 (72 of 88 ms for
 * a 2048 x 2048 factor), which a compiled reference (Eigen LLT) would not pay.
 *
 * Summation order: fixed for a given thread count (per-thread partial vectors
 * added in thread order), so results are reproducible run to run; they differ
 * from NumPy's zgemv in the last bits only (tests/test_oracle_c_port.py).
 */
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#define LU_CLONES __attribute__((target_clones("avx2,fma", "default")))
#else
#define LU_CLONES
#endif

/* part[0..2*rows) += sum_{j in [j0, j1)} A[:, cols[j]] * x[j]   (interleaved re/im) */
LU_CLONES
static void forward_range(const float *A, long ld, int rows, const int *cols, const double *x, long j0, long j1,
                          double *part) {
  for (long j = j0; j < j1; ++j) {
    const float *a = A + 2 * ld * (long)(cols ? cols[j] : j);
    const double xr = x[2 * j], xi = x[2 * j + 1];
    for (int r = 0; r < rows; ++r) {
      const double ar = a[2 * r], ai = a[2 * r + 1];
      part[2 * r] += ar * xr - ai * xi;
      part[2 * r + 1] += ar * xi + ai * xr;
    }
  }
}

/* out[j] = sum_r conj(A[r, cols[j]]) * w[r] for j in [j0, j1) */
LU_CLONES
static void adjoint_range(const float *A, long ld, int rows, const int *cols, const double *w, long j0, long j1,
                          double *out) {
  for (long j = j0; j < j1; ++j) {
    const float *a = A + 2 * ld * (long)(cols ? cols[j] : j);
    double sr = 0.0, si = 0.0;
    for (int r = 0; r < rows; ++r) {
      const double ar = a[2 * r], ai = a[2 * r + 1], wr = w[2 * r], wi = w[2 * r + 1];
      sr += ar * wr + ai * wi;
      si += ar * wi - ai * wr;
    }
    out[2 * j] = sr;
    out[2 * j + 1] = si;
  }
}

/* v = A[:, cols] x.  A: complex64 column-major (ld complex elements per column),
 * cols: n column indices (NULL: 0..n-1), x: n complex128, v: rows complex128. */
void lu_forward(const float *A, long ld, int rows, int n, const int *cols, const double *x, double *v) {
  const int tmax = omp_get_max_threads();
  double *parts = (double *)calloc((size_t)tmax * 2 * rows, sizeof(double));
  int used = 1;
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
#pragma omp single
    used = nt;
    const long j0 = (long)n * t / nt, j1 = (long)n * (t + 1) / nt;
    forward_range(A, ld, rows, cols, x, j0, j1, parts + (size_t)t * 2 * rows);
  }
  memset(v, 0, sizeof(double) * 2 * rows);
  for (int t = 0; t < used; ++t) {
    const double *p = parts + (size_t)t * 2 * rows;
    for (int i = 0; i < 2 * rows; ++i) v[i] += p[i];
  }
  free(parts);
}

/* z = A[:, cols]^H w.  w: rows complex128, z: n complex128. */
void lu_adjoint(const float *A, long ld, int rows, int n, const int *cols, const double *w, double *z) {
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const long j0 = (long)n * t / nt, j1 = (long)n * (t + 1) / nt;
    adjoint_range(A, ld, rows, cols, w, j0, j1, z);
  }
}

/* b <- (L L^H)^{-1} b for the lower Cholesky factor L (complex128, column-major,
 * ld complex elements per column; entries above the diagonal are ignored): the
 * two triangular solves of solver_core.hpp:47-51 / LAPACK zpotrs, written
 * column-oriented so both sweeps stream L's lower triangle once (the forward
 * sweep as column axpys, the backward sweep as column dots).  One thread: each
 * column depends on the previous one. */
LU_CLONES
void lu_chol_solve(const double *L, long ld, int n, double *b) {
  for (int j = 0; j < n; ++j) {  /* L z = b */
    const double *c = L + 2 * ld * (long)j;
    const double d = c[2 * j];  /* real positive diagonal */
    const double zr = b[2 * j] / d, zi = b[2 * j + 1] / d;
    b[2 * j] = zr;
    b[2 * j + 1] = zi;
    for (int i = j + 1; i < n; ++i) {
      const double lr = c[2 * i], li = c[2 * i + 1];
      b[2 * i] -= lr * zr - li * zi;
      b[2 * i + 1] -= lr * zi + li * zr;
    }
  }
  for (int j = n - 1; j >= 0; --j) {  /* L^H w = z */
    const double *c = L + 2 * ld * (long)j;
    double sr = 0.0, si = 0.0;
    for (int i = j + 1; i < n; ++i) {  /* conj(L[i, j]) * w[i] */
      const double lr = c[2 * i], li = c[2 * i + 1], wr = b[2 * i], wi = b[2 * i + 1];
      sr += lr * wr + li * wi;
      si += lr * wi - li * wr;
    }
    const double d = c[2 * j];
    b[2 * j] = (b[2 * j] - sr) / d;
    b[2 * j + 1] = (b[2 * j + 1] - si) / d;
  }
}

int lu_threads(void) { return omp_get_max_threads(); }
void lu_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }

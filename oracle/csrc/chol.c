/* Numeric sparse Cholesky and triangular solves (oracle, plain C).
 *
 * TEST INFRASTRUCTURE ONLY -- the CPU checker for the CUDA factor/solve.
 * Restates the reference's two numba kernels:
 *   oracle_chol  <- _chol_kernel  (reference src/gridnlp/sparse/cholesky.py:147-172)
 *   oracle_solve <- _solve_kernel (reference src/gridnlp/sparse/cholesky.py:175-186)
 * Up-looking factorization on a fixed pattern: row k of L is the sparse
 * triangular solve of row k of the permuted matrix against the leading
 * factor; the pivot test `!(d > floor)` also rejects NaN pivots.
 * Single-threaded, like the reference.
 */
#include <math.h>
#include <stdint.h>

int64_t oracle_chol(int64_t n, const int64_t *a_rowptr, const int64_t *a_rowcol,
                    const double *a_vals, const int64_t *row_ptr, const int64_t *row_cols,
                    const int64_t *l_colptr, const int64_t *l_rowidx, double *l_vals,
                    int64_t *cpos, double *x, double pivot_floor) {
  for (int64_t k = 0; k < n; ++k) {
    double d = 0.0;
    for (int64_t t = a_rowptr[k]; t < a_rowptr[k + 1]; ++t) {
      int64_t j = a_rowcol[t];
      if (j == k) d = a_vals[t];
      else x[j] = a_vals[t];
    }
    for (int64_t t = row_ptr[k]; t < row_ptr[k + 1]; ++t) {
      int64_t j = row_cols[t];
      double xj = x[j];
      x[j] = 0.0;
      double lkj = xj / l_vals[l_colptr[j]];
      for (int64_t p = l_colptr[j] + 1; p < cpos[j]; ++p) x[l_rowidx[p]] -= l_vals[p] * lkj;
      d -= lkj * lkj;
      l_vals[cpos[j]] = lkj;
      cpos[j] += 1;
    }
    if (!(d > pivot_floor)) return k;
    l_vals[l_colptr[k]] = sqrt(d);
    cpos[k] = l_colptr[k] + 1;
  }
  return -1;
}

void oracle_solve(int64_t n, const int64_t *l_colptr, const int64_t *l_rowidx,
                  const double *l_vals, double *x) {
  for (int64_t j = 0; j < n; ++j) {
    double xj = x[j] / l_vals[l_colptr[j]];
    x[j] = xj;
    for (int64_t p = l_colptr[j] + 1; p < l_colptr[j + 1]; ++p) x[l_rowidx[p]] -= l_vals[p] * xj;
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    double xj = x[j];
    for (int64_t p = l_colptr[j] + 1; p < l_colptr[j + 1]; ++p) xj -= l_vals[p] * x[l_rowidx[p]];
    x[j] = xj / l_vals[l_colptr[j]];
  }
}

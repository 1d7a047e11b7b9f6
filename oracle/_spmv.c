/* Row-parallel CSR sparse matrix-vector product for the oracle (TEST
 * INFRASTRUCTURE ONLY; shares nothing with the CUDA path).  y_i = sum_j a_ij x_j
 * with the row's nonzeros summed in storage order, exactly like scipy's
 * csr_matvec, so results are bit-identical to the single-threaded oracle for any
 * thread count (each row is summed by one thread; compiled with
 * -ffp-contract=off: no fused multiply-add).  Used only to time the oracle on
 * all host cores (SURVEY 8(d) "OpenMP row-parallel CSR SpMV"). */
#include <stdint.h>
#include <omp.h>

#define MATVEC(NAME, IT)                                                                  \
  void NAME(int64_t n, const IT *indptr, const IT *indices, const double *data,          \
            const double *x, double *y, int nthreads) {                                  \
    _Pragma("omp parallel for schedule(static) num_threads(nthreads)")                   \
    for (int64_t i = 0; i < n; ++i) {                                                    \
      double s = 0.0;                                                                    \
      for (IT jj = indptr[i]; jj < indptr[i + 1]; ++jj) s += data[jj] * x[indices[jj]]; \
      y[i] = s;                                                                          \
    }                                                                                    \
  }

MATVEC(csr_matvec_i32, int32_t)
MATVEC(csr_matvec_i64, int64_t)

int spmv_max_threads(void) { return omp_get_max_threads(); }

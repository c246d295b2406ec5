/* ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * The fp64 Chebyshev low-pass filter of oracle/chebyshev.py (cheb_filter), written out in
 * plain C so that the oracle can finish full-size columns (BASELINE configs[4]: N = 10^7,
 * 2e8 nonzeros, p = 300) and use every host core for bench.py's cpu_baseline.  Rows are
 * independent within a recurrence step, so the rows of each step are split across OpenMP
 * threads; every row is computed exactly as the definition states, sequentially in CSR
 * order -- no blocking, fusion or reordering beyond the definition.
 *
 *   L = S - W, s_i = sum_k W_ik                       PAPER.md §2.1 (lines 66-72)
 *   L~ = (2 / lambda_max) L - I                        DESIGN.md R1 (Chebyshev basis of
 *   T_0 = X, T_1 = L~ X, T_{j+1} = 2 L~ T_j - T_{j-1}    the fast filter, §2.4 Eq. (3),
 *   Y = sum_{j=0}^{p} d_j T_j                            lines 135-147; §4.1 step 5
 *                                                        Eq. (10))
 *
 * It shares no code with the CUDA path (paper_1509_08863_b200/) and is pinned in
 * tests/test_oracle_pins.py against the numpy oracle and against closed forms.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* (L~ T)[i][q] for row i: (2/lmax) * (s_i T[i][q] - sum_k W_ik T[k][q]) - T[i][q] */
static void lt_row(int64_t i, const int64_t* rp, const int32_t* col, const double* val, const double* s,
                   int R, const double* T, double a, double* out) {
  for (int q = 0; q < R; ++q) out[q] = 0.0;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
    const double w = val ? val[e] : 1.0;
    const double* tk = T + (int64_t)col[e] * R;
    for (int q = 0; q < R; ++q) out[q] += w * tk[q];
  }
  const double* ti = T + i * R;
  for (int q = 0; q < R; ++q) out[q] = a * (s[i] * ti[q] - out[q]) - ti[q];
}

/* Y (n x R row-major) = sum_j d[j] T_j(L~) X; returns 0, or -1 on allocation failure.
 * nthreads <= 0: OpenMP default. */
int oracle_cheb_filter(int64_t n, const int64_t* rp, const int32_t* col, const double* val, int R,
                       const double* X, const double* d, int p, double lambda_max, double* Y, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const double a = 2.0 / lambda_max;
  double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* T0 = (double*)malloc(sizeof(double) * (size_t)(n * R > 0 ? n * R : 1));
  double* T1 = (double*)malloc(sizeof(double) * (size_t)(n * R > 0 ? n * R : 1));
  double* T2 = (double*)malloc(sizeof(double) * (size_t)(n * R > 0 ? n * R : 1));
  if (!s || !T0 || !T1 || !T2) {
    free(s); free(T0); free(T1); free(T2);
    return -1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc += val ? val[e] : 1.0;
    s[i] = acc;
  }
  memcpy(T0, X, sizeof(double) * (size_t)(n * R));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n * R; ++i) Y[i] = d[0] * T0[i];
  if (p >= 1) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) lt_row(i, rp, col, val, s, R, T0, a, T1 + i * R);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n * R; ++i) Y[i] += d[1] * T1[i];
  }
  for (int j = 1; j < p; ++j) {
    /* T2 = 2 L~ T1 - T0 */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      double* t2 = T2 + i * R;
      lt_row(i, rp, col, val, s, R, T1, a, t2);
      const double* t0 = T0 + i * R;
      for (int q = 0; q < R; ++q) t2[q] = 2.0 * t2[q] - t0[q];
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n * R; ++i) Y[i] += d[j + 1] * T2[i];
    double* tmp = T0;
    T0 = T1;
    T1 = T2;
    T2 = tmp;
  }
  free(s); free(T0); free(T1); free(T2);
  return 0;
}

/* threads OpenMP would use */
int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

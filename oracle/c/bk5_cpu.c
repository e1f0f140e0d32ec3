/* CPU oracle: BK5 element-local stiffness apply in plain C + OpenMP.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/ (checked
 * against oracle/operators.py:bk5 to 1e-13) and as bench.py's CPU baseline /
 * `--impl reference` arm.  Never linked into the product library.
 *
 * Restates the same operator as oracle/operators.py:bk5:
 *   w^e = [D1;D2;D3]^T G^e [D1;D2;D3] u^e       (
 *   PAPER.md:1150-1162 tensor contractions, PAPER.md:1240-1266 six G factors)
 *   D1 = I x I x D (along i), D2 along j, D3 along k; G order G11 G12 G13 G22
 *   G23 G33; layout u, w [e][k][j][i], G [e][6][k][j][i].
 *   Optional Helmholtz term w = lam0 A u + lam1 B u.
 * Every contraction is written with the contiguous index i innermost so the
 * compiler vectorises it; elements are distributed over OpenMP threads.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NQ_MAX 17

static inline __attribute__((always_inline)) void bk5_element(int nq, const double* restrict D, const double* restrict DT,
                        const double* restrict G, const double* restrict u, double* restrict w,
                        double lam0, const double* restrict B, double lam1, double* restrict buf) {
  const int n2 = nq * nq, n3 = n2 * nq;
  double* ur = buf;
  double* us = buf + n3;
  double* ut = buf + 2 * n3;
  memset(buf, 0, 3 * (size_t)n3 * sizeof(double));
  /* ur[k][j][i] = sum_m D[i][m] u[k][j][m] = sum_m DT[m][i] u[kj][m] */
  for (int kj = 0; kj < n2; ++kj)
    for (int m = 0; m < nq; ++m) {
      const double um = u[kj * nq + m];
      for (int i = 0; i < nq; ++i) ur[kj * nq + i] += DT[m * nq + i] * um;
    }
  /* us[k][j][i] = sum_m D[j][m] u[k][m][i] */
  for (int k = 0; k < nq; ++k)
    for (int j = 0; j < nq; ++j)
      for (int m = 0; m < nq; ++m) {
        const double d = D[j * nq + m];
        const double* um = u + k * n2 + m * nq;
        double* o = us + k * n2 + j * nq;
        for (int i = 0; i < nq; ++i) o[i] += d * um[i];
      }
  /* ut[k][j][i] = sum_m D[k][m] u[m][j][i] */
  for (int k = 0; k < nq; ++k)
    for (int m = 0; m < nq; ++m) {
      const double d = D[k * nq + m];
      const double* um = u + m * n2;
      double* o = ut + k * n2;
      for (int q = 0; q < n2; ++q) o[q] += d * um[q];
    }
  /* (gr, gs, gt) = G (ur, us, ut), in place */
  for (int q = 0; q < n3; ++q) {
    const double a = ur[q], b = us[q], c = ut[q];
    ur[q] = G[0 * n3 + q] * a + G[1 * n3 + q] * b + G[2 * n3 + q] * c;
    us[q] = G[1 * n3 + q] * a + G[3 * n3 + q] * b + G[4 * n3 + q] * c;
    ut[q] = G[2 * n3 + q] * a + G[4 * n3 + q] * b + G[5 * n3 + q] * c;
  }
  memset(w, 0, (size_t)n3 * sizeof(double));
  /* w[k][j][i] += sum_m D[m][i] gr[k][j][m] */
  for (int kj = 0; kj < n2; ++kj)
    for (int m = 0; m < nq; ++m) {
      const double g = ur[kj * nq + m];
      for (int i = 0; i < nq; ++i) w[kj * nq + i] += D[m * nq + i] * g;
    }
  /* w[k][j][i] += sum_m D[m][j] gs[k][m][i] */
  for (int k = 0; k < nq; ++k)
    for (int j = 0; j < nq; ++j)
      for (int m = 0; m < nq; ++m) {
        const double d = D[m * nq + j];
        const double* g = us + k * n2 + m * nq;
        double* o = w + k * n2 + j * nq;
        for (int i = 0; i < nq; ++i) o[i] += d * g[i];
      }
  /* w[k][j][i] += sum_m D[m][k] gt[m][j][i] */
  for (int k = 0; k < nq; ++k)
    for (int m = 0; m < nq; ++m) {
      const double d = D[m * nq + k];
      const double* g = ut + m * n2;
      double* o = w + k * n2;
      for (int q = 0; q < n2; ++q) o[q] += d * g[q];
    }
  if (lam0 != 1.0)
    for (int q = 0; q < n3; ++q) w[q] *= lam0;
  if (B != NULL && lam1 != 0.0)
    for (int q = 0; q < n3; ++q) w[q] += lam1 * B[q] * u[q];
}

/* One copy of the element kernel per order with nq a compile-time constant
 * (fully unrolled / vectorised inner loops). */
#define NK_CASE(Q) \
  case Q:          \
    bk5_element(Q, D, DT, G, u, w, lam0, B, lam1, buf); \
    break;
static void bk5_dispatch(int nq, const double* restrict D, const double* restrict DT,
                         const double* restrict G, const double* restrict u, double* restrict w,
                         double lam0, const double* restrict B, double lam1, double* restrict buf) {
  switch (nq) {
    NK_CASE(2) NK_CASE(3) NK_CASE(4) NK_CASE(5) NK_CASE(6) NK_CASE(7) NK_CASE(8) NK_CASE(9)
    NK_CASE(10) NK_CASE(11) NK_CASE(12) NK_CASE(13) NK_CASE(14) NK_CASE(15) NK_CASE(16)
    default:
      bk5_element(nq, D, DT, G, u, w, lam0, B, lam1, buf);
  }
}
#undef NK_CASE

/* w = lam0 A_L u + lam1 B u over elements [e0, e1) (all when e1 <= e0 ... E).
 * nthreads <= 0: OpenMP default.  Returns the number of threads used, or
 * -1 on invalid arguments. */
int bk5_cpu(int N, int64_t E, const double* D, const double* G, const double* u, double* w,
            double lam0, const double* B, double lam1, int nthreads) {
  const int nq = N + 1;
  if (N < 1 || nq > NQ_MAX || E < 0 || !D || !G || !u || !w) return -1;
  double DT[NQ_MAX * NQ_MAX];
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b) DT[b * nq + a] = D[a * nq + b];
  const int64_t n3 = (int64_t)nq * nq * nq;
  int used = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
    double buf[3 * NQ_MAX * NQ_MAX * NQ_MAX];
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e)
      bk5_dispatch(nq, D, DT, G + e * 6 * n3, u + e * n3, w + e * n3, lam0,
                   B ? B + e * n3 : NULL, lam1, buf);
  }
#else
  (void)nthreads;
  double* buf = (double*)malloc(3 * (size_t)n3 * sizeof(double));
  for (int64_t e = 0; e < E; ++e)
    bk5_dispatch(nq, D, DT, G + e * 6 * n3, u + e * n3, w + e * n3, lam0, B ? B + e * n3 : NULL,
                 lam1, buf);
  free(buf);
#endif
  return used;
}

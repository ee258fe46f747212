/* oracle_sanitize.c -- drives every oracle/ entry point on small inputs so the
 * oracle can be built and run under AddressSanitizer + UndefinedBehavior-
 * Sanitizer (memory / UB checking of the C code).  Test
 * infrastructure: built and run by tests/test_oracle_sanitize.py.  Exits 0
 * when every call returns what the mathematics says (exact integer checks);
 * any sanitizer report aborts with a non-zero status. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle/oracle.h"

static uint64_t rng_state = 0x9e3779b97f4a7c15ull;
static int64_t rint_in(int64_t lo, int64_t hi) { /* splitmix64, inclusive range */
  uint64_t z = (rng_state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return lo + (int64_t)(z % (uint64_t)(hi - lo + 1));
}

static double* int_matrix(int64_t n, int64_t ld, int64_t lim) {
  double* X = (double*)malloc(sizeof(double) * n * ld);
  for (int64_t i = 0; i < n * ld; ++i) X[i] = (double)rint_in(-lim, lim);
  return X;
}

#define CHECK(cond, ...)                         \
  do {                                           \
    if (!(cond)) {                               \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);              \
      fprintf(stderr, "\n");                     \
      return 1;                                  \
    }                                            \
  } while (0)

/* exact integer product of integer-valued A, B (n x n, ld lda / ldb) */
static void int_product(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      int64_t s = 0;
      for (int64_t k = 0; k < n; ++k) s += (int64_t)A[i * lda + k] * (int64_t)B[k * ldb + j];
      C[i * n + j] = (double)s;
    }
}

static int run_triple(const char* name, int levels, int64_t n, int64_t pad) {
  int p = 0, R = 0;
  CHECK(or_catalog(name, &p, &R, NULL, NULL, NULL) == 0, "catalog size %s", name);
  const size_t sz = (size_t)p * p * R;
  double *U = malloc(sizeof(double) * sz), *V = malloc(sizeof(double) * sz), *W = malloc(sizeof(double) * sz);
  CHECK(or_catalog(name, &p, &R, U, V, W) == 0, "catalog %s", name);
  int64_t first[3] = {-1, -1, -1};
  CHECK(or_brent_check(p, R, U, V, W, first) == 0, "brent %s", name);
  const int64_t ld = n + pad;
  double* A = int_matrix(n, ld, 8);
  double* B = int_matrix(n, ld, 8);
  double* C = calloc((size_t)n * ld, sizeof(double));
  double* E = malloc(sizeof(double) * n * n);
  int_product(n, A, ld, B, ld, E);
  CHECK(or_fmm(n, 1.0, A, ld, B, ld, C, ld, p, R, U, V, W, levels) == 0, "fmm %s", name);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) CHECK(C[i * ld + j] == E[i * n + j], "fmm %s (%lld,%lld)", name, (long long)i, (long long)j);
  CHECK(or_fmm(n, -2.0, A, ld, B, ld, C, ld, p, R, U, V, W, levels) == 0, "fmm alpha %s", name);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) CHECK(C[i * ld + j] == -2.0 * E[i * n + j], "fmm alpha %s", name);
  /* one level in steps: premix, classical products, postmix */
  const int64_t m = n / p, mm = m * m;
  double* T = malloc(sizeof(double) * mm * R);
  double* S = malloc(sizeof(double) * mm * R);
  double* P = malloc(sizeof(double) * mm * R);
  or_premix(n, A, ld, p, R, U, T);
  or_premix(n, B, ld, p, R, V, S);
  for (int q = 0; q < R; ++q) or_classical(m, T + q * mm, m, S + q * mm, m, P + q * mm, m);
  or_postmix(n, 0.5, P, p, R, W, C, ld);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) CHECK(C[i * ld + j] == 0.5 * E[i * n + j], "steps %s", name);
  /* Freivalds and sampled entries on the contiguous product */
  double* Ac = malloc(sizeof(double) * n * n);
  double* Bc = malloc(sizeof(double) * n * n);
  for (int64_t i = 0; i < n; ++i) {
    memcpy(Ac + i * n, A + i * ld, sizeof(double) * n);
    memcpy(Bc + i * n, B + i * ld, sizeof(double) * n);
  }
  CHECK(or_freivalds_int(n, Ac, Bc, E, 3, 7) == 0, "freivalds %s", name);
  E[n + 1] += 1.0;
  CHECK(or_freivalds_int(n, Ac, Bc, E, 3, 7) > 0, "freivalds must see a planted error");
  E[n + 1] -= 1.0;
  int64_t rows[16], cols[16];
  double got[16];
  for (int s = 0; s < 16; ++s) { rows[s] = rint_in(0, n - 1); cols[s] = rint_in(0, n - 1); }
  or_sample_entries(n, A, ld, B, ld, 16, rows, cols, got);
  for (int s = 0; s < 16; ++s) CHECK(got[s] == E[rows[s] * n + cols[s]], "sample %s", name);
  free(U); free(V); free(W); free(A); free(B); free(C); free(E); free(T); free(S); free(P);
  free(Ac); free(Bc);
  return 0;
}

int main(void) {
  /* triples, one and two levels, ragged and strided views */
  if (run_triple("strassen-winograd", 1, 34, 3)) return 1;
  if (run_triple("strassen-winograd", 2, 36, 0)) return 1;
  if (run_triple("paper-strassen", 1, 22, 1)) return 1;
  if (run_triple("strassen-1969", 2, 20, 2)) return 1;
  if (run_triple("laderman", 1, 27, 5)) return 1;
  if (run_triple("classical-p3", 1, 12, 0)) return 1;
  /* Kronecker composition: SW (x) LD is a valid <6,6,6;161> */
  int p1, R1, p2, R2;
  or_catalog("strassen-winograd", &p1, &R1, NULL, NULL, NULL);
  or_catalog("laderman", &p2, &R2, NULL, NULL, NULL);
  double *U1 = malloc(8 * p1 * p1 * R1), *V1 = malloc(8 * p1 * p1 * R1), *W1 = malloc(8 * p1 * p1 * R1);
  double *U2 = malloc(8 * p2 * p2 * R2), *V2 = malloc(8 * p2 * p2 * R2), *W2 = malloc(8 * p2 * p2 * R2);
  or_catalog("strassen-winograd", &p1, &R1, U1, V1, W1);
  or_catalog("laderman", &p2, &R2, U2, V2, W2);
  const int P = p1 * p2, R = R1 * R2;
  double *U = malloc(8 * (size_t)P * P * R), *V = malloc(8 * (size_t)P * P * R), *W = malloc(8 * (size_t)P * P * R);
  or_kron(p1, R1, U1, V1, W1, p2, R2, U2, V2, W2, U, V, W);
  CHECK(or_brent_check(P, R, U, V, W, NULL) == 0, "kron brent");
  W[5] += 1.0;
  CHECK(or_brent_check(P, R, U, V, W, NULL) > 0, "mutated kron must fail");
  CHECK(or_catalog("no-such-triple", &p1, &R1, NULL, NULL, NULL) == -1, "unknown name");
  double* A = int_matrix(10, 10, 1);
  double C[100];
  CHECK(or_fmm(10, 1.0, A, 10, A, 10, C, 10, p2, R2, U2, V2, W2, 1) == -1, "indivisible n");
  free(U1); free(V1); free(W1); free(U2); free(V2); free(W2); free(U); free(V); free(W); free(A);
  printf("oracle sanitize ok (%d threads)\n", or_num_threads());
  return 0;
}

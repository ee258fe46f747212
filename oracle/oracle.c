/* oracle.c -- plain, slow, obviously correct CPU oracle for the Matrix Flow
 * hot path (arXiv 2312.12732, "Strassen's Matrix Multiplication Algorithm Is
 * Still Faster", PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY: see oracle.h.  Nothing in the product path calls
 * this code; it shares no code, header or table with it.
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fPIC -shared
 *        -o liboracle.so oracle.c          (never -ffast-math)
 *
 * Every function cites the passage it follows.  Pins live in
 * tests/test_oracle.py.  Parity-unpinned items are listed in DESIGN.md §3.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* O1: catalog.  Coefficients typed in from the sources named per triple.   */
/* ------------------------------------------------------------------------ */

/* the DeepMind-format Strassen matrices a, b, c^t.
 * a and b are copied verbatim (rows A0..A3 / B0..B3, columns T0..T6).
 * The printed c^t lists its rows as C0, C2, C1, C3 (L245-248); honouring
 * those labels, the natural-order W below is rows [C0, C1, C2, C3] =
 * printed rows [0, 2, 1, 3]. */
static const int PS_U[4][7] = {{0, 1, 1, 0, 1, 1, 0},
                               {0, 0, -1, 1, 0, 0, 0},
                               {1, 1, 1, 0, 1, 0, 0},
                               {-1, -1, -1, 0, 0, 0, 1}};
static const int PS_V[4][7] = {{0, 0, 0, 0, 1, 1, 0},
                               {1, 1, 0, 0, 1, 0, 1},
                               {0, 1, 1, 1, 1, 0, 0},
                               {0, 1, 1, 0, 1, 0, 1}};
static const int PS_CT_PRINTED[4][7] = {{0, 0, 0, 1, 0, 1, 0},     /* C0 */
                                        {0, -1, 0, 0, 1, -1, -1},  /* C2 */
                                        {-1, 1, -1, -1, 0, 0, 0},  /* C1 */
                                        {1, 0, 0, 0, 0, 0, 1}};    /* C3 */
static const int PS_CT_LABEL[4] = {0, 2, 1, 3};

/* Strassen-Winograd <2,2,2;7> (the variant north_star names; not printed in
 * the paper).  Products, blocks 0=(1,1) 1=(1,2) 2=(2,1) 3=(2,2):
 *   P0 = A0*B0                P1 = A1*B2
 *   P2 = (A0+A1-A2-A3)*B3     P3 = A3*(B0-B1-B2+B3)
 *   P4 = (A2+A3)*(B1-B0)      P5 = (A2+A3-A0)*(B0-B1+B3)
 *   P6 = (A0-A2)*(B3-B1)
 *   C0 = P0+P1   C1 = P0+P2+P4+P5   C2 = P0-P3+P5+P6   C3 = P0+P4+P5+P6 */
static const int SW_U[4][7] = {{1, 0, 1, 0, 0, -1, 1},
                               {0, 1, 1, 0, 0, 0, 0},
                               {0, 0, -1, 0, 1, 1, -1},
                               {0, 0, -1, 1, 1, 1, 0}};
static const int SW_V[4][7] = {{1, 0, 0, 1, -1, 1, 0},
                               {0, 0, 0, -1, 1, -1, -1},
                               {0, 1, 0, -1, 0, 0, 0},
                               {0, 0, 1, 1, 0, 1, 1}};
static const int SW_W[4][7] = {{1, 1, 0, 0, 0, 0, 0},
                               {1, 0, 1, 0, 1, 1, 0},
                               {1, 0, 0, -1, 0, 1, 1},
                               {1, 0, 0, 0, 1, 1, 1}};

/* Strassen 1969 (the paper's citation STRASSEN1969):
 *   M1=(A11+A22)(B11+B22) M2=(A21+A22)B11 M3=A11(B12-B22) M4=A22(B21-B11)
 *   M5=(A11+A12)B22 M6=(A21-A11)(B11+B12) M7=(A12-A22)(B21+B22)
 *   C11=M1+M4-M5+M7 C12=M3+M5 C21=M2+M4 C22=M1-M2+M3+M6 */
static const int S69_U[4][7] = {{1, 0, 1, 0, 1, -1, 0},
                                {0, 0, 0, 0, 1, 0, 1},
                                {0, 1, 0, 0, 0, 1, 0},
                                {1, 1, 0, 1, 0, 0, -1}};
static const int S69_V[4][7] = {{1, 1, 0, -1, 0, 1, 0},
                                {0, 0, 1, 0, 0, 1, 0},
                                {0, 0, 0, 1, 0, 0, 1},
                                {1, 0, -1, 0, 1, 0, 1}};
static const int S69_W[4][7] = {{1, 0, 0, 1, -1, 0, 1},
                                {0, 0, 1, 0, 1, 0, 0},
                                {0, 1, 0, 1, 0, 0, 0},
                                {1, -1, 1, 0, 0, 1, 0}};

/* Laderman 1976 <3,3,3;23>; the paper only names "3 as 23 products"
 * (PAPER.md L275).  Blocks 0..8 row-major over the 3x3 grid.  Listed as
 * (term list of T_q) x (term list of S_q); C rows below. */
typedef struct { int nt; int k[9]; int c[9]; } lin9;
static const lin9 LD_T[23] = {
    {7, {0, 1, 2, 3, 4, 7, 8}, {1, 1, 1, -1, -1, -1, -1}},  /* P0  */
    {2, {0, 3}, {1, -1}},                                  /* P1  */
    {1, {4}, {1}},                                         /* P2  */
    {3, {0, 3, 4}, {-1, 1, 1}},                            /* P3  */
    {2, {3, 4}, {1, 1}},                                   /* P4  */
    {1, {0}, {1}},                                         /* P5  */
    {3, {0, 6, 7}, {-1, 1, 1}},                            /* P6  */
    {2, {0, 6}, {-1, 1}},                                  /* P7  */
    {2, {6, 7}, {1, 1}},                                   /* P8  */
    {7, {0, 1, 2, 4, 5, 6, 7}, {1, 1, 1, -1, -1, -1, -1}},  /* P9  */
    {1, {7}, {1}},                                         /* P10 */
    {3, {2, 7, 8}, {-1, 1, 1}},                            /* P11 */
    {2, {2, 8}, {1, -1}},                                  /* P12 */
    {1, {2}, {1}},                                         /* P13 */
    {2, {7, 8}, {1, 1}},                                   /* P14 */
    {3, {2, 4, 5}, {-1, 1, 1}},                            /* P15 */
    {2, {2, 5}, {1, -1}},                                  /* P16 */
    {2, {4, 5}, {1, 1}},                                   /* P17 */
    {1, {1}, {1}},                                         /* P18 */
    {1, {5}, {1}},                                         /* P19 */
    {1, {3}, {1}},                                         /* P20 */
    {1, {6}, {1}},                                         /* P21 */
    {1, {8}, {1}},                                         /* P22 */
};
static const lin9 LD_S[23] = {
    {1, {4}, {1}},                                         /* P0  */
    {2, {1, 4}, {-1, 1}},                                  /* P1  */
    {7, {0, 1, 3, 4, 5, 6, 8}, {-1, 1, 1, -1, -1, -1, 1}},  /* P2  */
    {3, {0, 1, 4}, {1, -1, 1}},                            /* P3  */
    {2, {0, 1}, {-1, 1}},                                  /* P4  */
    {1, {0}, {1}},                                         /* P5  */
    {3, {0, 2, 5}, {1, -1, 1}},                            /* P6  */
    {2, {2, 5}, {1, -1}},                                  /* P7  */
    {2, {0, 2}, {-1, 1}},                                  /* P8  */
    {1, {5}, {1}},                                         /* P9  */
    {7, {0, 2, 3, 4, 5, 6, 7}, {-1, 1, 1, -1, -1, -1, 1}},  /* P10 */
    {3, {4, 6, 7}, {1, 1, -1}},                            /* P11 */
    {2, {4, 7}, {1, -1}},                                  /* P12 */
    {1, {6}, {1}},                                         /* P13 */
    {2, {6, 7}, {-1, 1}},                                  /* P14 */
    {3, {5, 6, 8}, {1, 1, -1}},                            /* P15 */
    {2, {5, 8}, {1, -1}},                                  /* P16 */
    {2, {6, 8}, {-1, 1}},                                  /* P17 */
    {1, {3}, {1}},                                         /* P18 */
    {1, {7}, {1}},                                         /* P19 */
    {1, {2}, {1}},                                         /* P20 */
    {1, {1}, {1}},                                         /* P21 */
    {1, {8}, {1}},                                         /* P22 */
};
/* C_i = sum of the listed products, all with coefficient +1. */
static const int LD_C[9][8] = {
    {3, 5, 13, 18},                          /* C0 */
    {7, 0, 3, 4, 5, 11, 13, 14},             /* C1 */
    {7, 5, 6, 8, 9, 13, 15, 17},             /* C2 */
    {7, 1, 2, 3, 5, 13, 15, 16},             /* C3 */
    {5, 1, 3, 4, 5, 19},                     /* C4 */
    {5, 13, 15, 16, 17, 20},                 /* C5 */
    {7, 5, 6, 7, 10, 11, 12, 13},            /* C6 */
    {5, 11, 12, 13, 14, 21},                 /* C7 */
    {5, 5, 6, 7, 8, 22},                     /* C8 */
};  /* first entry = number of products that follow */

static void classical_triple(int p, double* U, double* V, double* W) {
  /* Eq. (recursion), PAPER.md L183-191 generalised to factor p:
   * C_{i,j} = sum_k A_{i,k} B_{k,j}; product (i,j,k) -> index q. */
  int R = p * p * p;
  memset(U, 0, sizeof(double) * p * p * R);
  memset(V, 0, sizeof(double) * p * p * R);
  memset(W, 0, sizeof(double) * p * p * R);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        int q = (i * p + j) * p + k;
        U[(i * p + k) * R + q] = 1.0;
        V[(k * p + j) * R + q] = 1.0;
        W[(i * p + j) * R + q] = 1.0;
      }
}

static void copy47(const int (*X)[7], double* out) {
  for (int r = 0; r < 4; ++r)
    for (int q = 0; q < 7; ++q) out[r * 7 + q] = (double)X[r][q];
}

int or_catalog(const char* name, int* p, int* R, double* U, double* V, double* W) {
  if (!strcmp(name, "paper-strassen")) {
    *p = 2; *R = 7;
    if (U) {
      copy47(PS_U, U);
      copy47(PS_V, V);
      for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 7; ++q) W[PS_CT_LABEL[r] * 7 + q] = (double)PS_CT_PRINTED[r][q];
    }
    return 0;
  }
  if (!strcmp(name, "strassen-winograd")) {
    *p = 2; *R = 7;
    if (U) { copy47(SW_U, U); copy47(SW_V, V); copy47(SW_W, W); }
    return 0;
  }
  if (!strcmp(name, "strassen-1969")) {
    *p = 2; *R = 7;
    if (U) { copy47(S69_U, U); copy47(S69_V, V); copy47(S69_W, W); }
    return 0;
  }
  if (!strcmp(name, "laderman")) {
    *p = 3; *R = 23;
    if (U) {
      memset(U, 0, sizeof(double) * 9 * 23);
      memset(V, 0, sizeof(double) * 9 * 23);
      memset(W, 0, sizeof(double) * 9 * 23);
      for (int q = 0; q < 23; ++q) {
        for (int t = 0; t < LD_T[q].nt; ++t) U[LD_T[q].k[t] * 23 + q] = LD_T[q].c[t];
        for (int t = 0; t < LD_S[q].nt; ++t) V[LD_S[q].k[t] * 23 + q] = LD_S[q].c[t];
      }
      for (int i = 0; i < 9; ++i)
        for (int t = 1; t <= LD_C[i][0]; ++t) W[i * 23 + LD_C[i][t]] = 1.0;
    }
    return 0;
  }
  if (!strcmp(name, "classical-p2") || !strcmp(name, "classical-p3")) {
    int pp = name[11] - '0';
    *p = pp; *R = pp * pp * pp;
    if (U) classical_triple(pp, U, V, W);
    return 0;
  }
  return -1;
}

/* outer block b and inner block s combine to the flat
 * row-major block index of the (po*pi)-way split. */
static int kron_row(int b, int s, int po, int pi) {
  int P = po * pi;
  int row = (b / po) * pi + s / pi;
  int col = (b % po) * pi + s % pi;
  return row * P + col;
}

void or_kron(int po, int Ro, const double* Uo, const double* Vo, const double* Wo,
             int pi, int Ri, const double* Ui, const double* Vi, const double* Wi,
             double* U, double* V, double* W) {
  /* a = a_o (x) a_i, b = b_o (x) b_i, c = c_o (x) c_i. */
  int P = po * pi, R = Ro * Ri;
  memset(U, 0, sizeof(double) * P * P * R);
  memset(V, 0, sizeof(double) * P * P * R);
  memset(W, 0, sizeof(double) * P * P * R);
  for (int b = 0; b < po * po; ++b)
    for (int s = 0; s < pi * pi; ++s) {
      int row = kron_row(b, s, po, pi);
      for (int qo = 0; qo < Ro; ++qo)
        for (int qi = 0; qi < Ri; ++qi) {
          int q = qo * Ri + qi;
          U[row * R + q] = Uo[b * Ro + qo] * Ui[s * Ri + qi];
          V[row * R + q] = Vo[b * Ro + qo] * Vi[s * Ri + qi];
          W[row * R + q] = Wo[b * Ro + qo] * Wi[s * Ri + qi];
        }
    }
}

/* ------------------------------------------------------------------------ */
/* O2: exact Brent check: for x=(i,k), y=(k',j), z=(i',j'),  */
/* sum_q U[x][q] V[y][q] W[z][q] = [k==k' && i==i' && j==j'].               */
/* ------------------------------------------------------------------------ */
int64_t or_brent_check(int p, int R, const double* U, const double* V, const double* W,
                       int64_t* first) {
  int P2 = p * p;
  for (int t = 0; t < P2 * R; ++t)
    if (U[t] != floor(U[t]) || V[t] != floor(V[t]) || W[t] != floor(W[t])) return -1;
  int64_t bad = 0;
  for (int x = 0; x < P2; ++x)
    for (int y = 0; y < P2; ++y)
      for (int z = 0; z < P2; ++z) {
        int64_t s = 0;
        for (int q = 0; q < R; ++q)
          s += (int64_t)U[x * R + q] * (int64_t)V[y * R + q] * (int64_t)W[z * R + q];
        int i = x / p, k = x % p, k2 = y / p, j = y % p, i2 = z / p, j2 = z % p;
        int64_t expect = (k == k2 && i == i2 && j == j2) ? 1 : 0;
        if (s != expect) {
          if (bad == 0 && first) { first[0] = x; first[1] = y; first[2] = z; }
          ++bad;
        }
      }
  return bad;
}

/* ------------------------------------------------------------------------ */
/* O3: classical product.                               */
/* ------------------------------------------------------------------------ */
void or_classical(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double* C, int64_t ldc) {
  /* i-k-j order: row i of C accumulates A[i][k]*B[k][:] for k = 0,1,...,
   * so each C[i][j] is the k-ascending sum started from +0.0, exactly as
   * the i-j-k definition (same operations in the same order per element). */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double* c = C + i * ldc;
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      double a = A[i * lda + k];
      const double* b = B + k * ldb;
      for (int64_t j = 0; j < n; ++j) c[j] = c[j] + a * b[j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Block helpers for the partition of PAPER.md L139-165 (row-major blocks). */
/* ------------------------------------------------------------------------ */
static const double* blk(const double* X, int64_t ldx, int p, int64_t m, int b) {
  return X + (int64_t)(b / p) * m * ldx + (int64_t)(b % p) * m;
}

/* The combination rule of Eq. (strassen) used for T_q,
 * S_q and C_i: out = c_0*X_{k_0}; then out = out + c*X_k for the remaining
 * nonzero coefficients in ascending k (separate multiply and add).
 * out is m x m with leading dimension ldo. */
static void combine(int64_t m, int nterms, const double* const* src, const int64_t* lds,
                    const double* coef, double* out, int64_t ldo) {
  for (int64_t r = 0; r < m; ++r)
    for (int64_t c = 0; c < m; ++c) {
      double acc = coef[0] * src[0][r * lds[0] + c];
      for (int t = 1; t < nterms; ++t) acc = acc + coef[t] * src[t][r * lds[t] + c];
      out[r * ldo + c] = acc;
    }
}

void or_premix(int64_t n, const double* X, int64_t ldx, int p, int R, const double* M,
               double* out) {
  int64_t m = n / p;
  const double* src[64];
  int64_t lds[64];
  double coef[64];
  for (int q = 0; q < R; ++q) {
    int nt = 0;
    for (int k = 0; k < p * p; ++k)
      if (M[k * R + q] != 0.0) {
        src[nt] = blk(X, ldx, p, m, k);
        lds[nt] = ldx;
        coef[nt] = M[k * R + q];
        ++nt;
      }
    combine(m, nt, src, lds, coef, out + (int64_t)q * m * m, m);
  }
}

static void scale_block(int64_t m, double alpha, double* C, int64_t ldc) {
  for (int64_t r = 0; r < m; ++r)
    for (int64_t c = 0; c < m; ++c) C[r * ldc + c] = alpha * C[r * ldc + c];
}

void or_postmix(int64_t n, double alpha, const double* P, int p, int R, const double* W,
                double* C, int64_t ldc) {
  int64_t m = n / p;
  const double** src = (const double**)malloc(sizeof(double*) * R);
  int64_t* lds = (int64_t*)malloc(sizeof(int64_t) * R);
  double* coef = (double*)malloc(sizeof(double) * R);
  for (int i = 0; i < p * p; ++i) {
    double* Ci = (double*)blk(C, ldc, p, m, i);
    int nt = 0;
    for (int q = 0; q < R; ++q)
      if (W[i * R + q] != 0.0) {
        src[nt] = P + (int64_t)q * m * m;
        lds[nt] = m;
        coef[nt] = W[i * R + q];
        ++nt;
      }
    if (nt == 0) {
      for (int64_t r = 0; r < m; ++r)
        for (int64_t c = 0; c < m; ++c) Ci[r * ldc + c] = 0.0;
    } else {
      combine(m, nt, src, lds, coef, Ci, ldc);
    }
    if (alpha != 1.0) scale_block(m, alpha, Ci, ldc); /* alpha applied last */
  }
  free(src); free(lds); free(coef);
}

/* ------------------------------------------------------------------------ */
/* O4: recursion interpreter ("compute the  */
/* operands T_i and S_i first, recursively solve the result P_i and         */
/* distribute it").                                                         */
/* ------------------------------------------------------------------------ */
static int fmm_rec(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, int p, int R, const double* U, const double* V,
                   const double* W, int levels) {
  if (levels == 0) {
    or_classical(n, A, lda, B, ldb, C, ldc);
    return 0;
  }
  int64_t m = n / p;
  double* T = (double*)malloc(sizeof(double) * m * m);
  double* S = (double*)malloc(sizeof(double) * m * m);
  double* P = (double*)malloc(sizeof(double) * m * m * R);
  if (!T || !S || !P) { free(T); free(S); free(P); return -2; }
  const double* src[64];
  int64_t lds[64];
  double coef[64];
  int rc = 0;
  for (int q = 0; q < R && rc == 0; ++q) {
    /* T_q = sum_k a_{k,q} A_k */
    int nt = 0;
    for (int k = 0; k < p * p; ++k)
      if (U[k * R + q] != 0.0) {
        src[nt] = blk(A, lda, p, m, k); lds[nt] = lda; coef[nt] = U[k * R + q]; ++nt;
      }
    combine(m, nt, src, lds, coef, T, m);
    /* S_q = sum_l b_{l,q} B_l */
    nt = 0;
    for (int l = 0; l < p * p; ++l)
      if (V[l * R + q] != 0.0) {
        src[nt] = blk(B, ldb, p, m, l); lds[nt] = ldb; coef[nt] = V[l * R + q]; ++nt;
      }
    combine(m, nt, src, lds, coef, S, m);
    /* P_q = T_q * S_q, recursively */
    rc = fmm_rec(m, T, m, S, m, P + (int64_t)q * m * m, m, p, R, U, V, W, levels - 1);
  }
  /* C_i = sum_q c_{i,q} P_q */
  if (rc == 0) or_postmix(n, 1.0, P, p, R, W, C, ldc);
  free(T); free(S); free(P);
  return rc;
}

int or_fmm(int64_t n, double alpha, const double* A, int64_t lda, const double* B,
           int64_t ldb, double* C, int64_t ldc, int p, int R, const double* U,
           const double* V, const double* W, int levels) {
  int64_t q = 1;
  for (int l = 0; l < levels; ++l) q *= p;
  if (n % q != 0) return -1;
  int rc = fmm_rec(n, A, lda, B, ldb, C, ldc, p, R, U, V, W, levels);
  if (rc == 0 && alpha != 1.0) scale_block(n, alpha, C, ldc); /* C = alpha*(AB) */
  return rc;
}

/* ------------------------------------------------------------------------ */
/* O7: large-n checks.                                                      */
/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int as_int(double v, double bound, int64_t* out) {
  if (!(fabs(v) < bound) || v != floor(v)) return 0;
  *out = (int64_t)v;
  return 1;
}

int64_t or_freivalds_int(int64_t n, const double* A, const double* B, const double* C,
                         int trials, uint64_t seed) {
  /* Freivalds (1977): C == A*B  <=>  C x == A (B x) for random x, with
   * probability of a false pass <= 2^-20 per trial for a wrong C.
   * |A|,|B| < 2^24, |C| <= 2^53, n <= 2^16 keep every sum below 2^101. */
  int64_t bad_total = 0;
  __int128* x = (__int128*)malloc(sizeof(__int128) * n);
  __int128* Bx = (__int128*)malloc(sizeof(__int128) * n);
  uint64_t s = seed;
  int invalid = 0;
  for (int t = 0; t < trials && !invalid; ++t) {
    for (int64_t j = 0; j < n; ++j) x[j] = (__int128)(splitmix64(&s) & ((1u << 20) - 1));
#pragma omp parallel for schedule(static) reduction(| : invalid)
    for (int64_t k = 0; k < n; ++k) {
      __int128 acc = 0;
      for (int64_t j = 0; j < n; ++j) {
        int64_t b;
        if (!as_int(B[k * n + j], 16777216.0, &b)) { invalid = 1; break; }
        acc += (__int128)b * x[j];
      }
      Bx[k] = acc;
    }
    if (invalid) break;
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad) reduction(| : invalid)
    for (int64_t i = 0; i < n; ++i) {
      __int128 lhs = 0, rhs = 0;
      for (int64_t j = 0; j < n; ++j) {
        int64_t c, a;
        if (!as_int(C[i * n + j], 9007199254740992.0, &c) || !as_int(A[i * n + j], 16777216.0, &a)) { invalid = 1; break; }
        lhs += (__int128)c * x[j];
        rhs += (__int128)a * Bx[j];
      }
      if (lhs != rhs) ++bad;
    }
    bad_total += bad;
  }
  free(x); free(Bx);
  return invalid ? -1 : bad_total;
}

void or_sample_entries(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                       int64_t count, const int64_t* rows, const int64_t* cols, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < count; ++s) {
    double acc = 0.0;
    for (int64_t k = 0; k < n; ++k) acc = acc + A[rows[s] * lda + k] * B[k * ldb + cols[s]];
    out[s] = acc;
  }
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

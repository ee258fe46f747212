/* oracle.h -- CPU oracle for the Matrix Flow hot path (arXiv 2312.12732).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product path (paper_2312_12732_b200/, include/mf.h, libmf.so) never
 * includes, links or calls anything here, and this file includes nothing
 * from the product: the two share no code, headers or coefficient tables.
 *
 * Conventions (§2): square n x n fp64 matrices,
 * row-major with a leading dimension in elements; a p-way partition numbers
 * the p*p blocks in row-major order, block x covering rows (x/p)*m.. and
 * columns (x%p)*m.. with m = n/p.  A bilinear triple <U,V,W> is stored as
 * three p^2 x R row-major arrays of doubles: U[k*R+q] = a_{k,q} (paper's a),
 * V[l*R+q] = b_{l,q} (paper's b), W[i*R+q] = c_{i,q} with row i the C block
 * in NATURAL row-major order (the paper prints c^t with rows C0,C2,C1,C3,
 * PAPER.md L245-248; reading R1).
 */
#ifndef MF_ORACLE_H
#define MF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* O1: builtin triples.  Names: "paper-strassen", "strassen-winograd",
 * "strassen-1969", "laderman", "classical-p2", "classical-p3".
 * Query sizes with U=V=W=NULL.  Returns 0, or -1 for an unknown name. */
int or_catalog(const char* name, int* p, int* R, double* U, double* V, double* W);

/* O1: Kronecker composition outer (x) inner (SPEC.md L244
 * row interleave).  Output arrays hold (po*pi)^2 x (Ro*Ri) doubles; product
 * index q = qo*Ri + qi. */
void or_kron(int po, int Ro, const double* Uo, const double* Vo, const double* Wo,
             int pi, int Ri, const double* Ui, const double* Vi, const double* Wi,
             double* U, double* V, double* W);

/* O2: exact Brent check over all (p^2)^3 equations.
 * Coefficients must be integers (returns -1 otherwise).  Returns the number
 * of violated equations; the lexicographically first one goes to first[3]
 * (x, y, z) when first != NULL and there is one. */
int64_t or_brent_check(int p, int R, const double* U, const double* V, const double* W,
                       int64_t* first);

/* O3: classical product C = A*B: for every (i,j),
 * C[i][j] = sum_{k=0}^{n-1} A[i][k]*B[k][j], k ascending, accumulator
 * starting at +0.0, separate multiply and add (compiled -ffp-contract=off). */
void or_classical(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double* C, int64_t ldc);

/* O4: the recursion interpreter of Eq. (strassen) (PAPER.md L196-203,
 * L280-286): C = alpha * A*B with `levels` recursion levels of <U,V,W>,
 * classical leaves.  Returns 0, -1 if n is not divisible by p^levels,
 * -2 on allocation failure. */
int or_fmm(int64_t n, double alpha, const double* A, int64_t lda, const double* B,
           int64_t ldb, double* C, int64_t ldc, int p, int R, const double* U,
           const double* V, const double* W, int levels);

/* One level of Eq. (strassen), split into its steps so that each step can be
 * compared with the matching GPU kernel:
 *   or_premix:  X_q = sum_k M[k][q] * Blk_k(X) for every q (M = U or V),
 *               written to out[q*m*m ...] (m x m, ld m);
 *   or_postmix: C_i = alpha * sum_q W[i][q] * P_q for every C block i,
 *               P_q read from P[q*m*m ...] (m x m, ld m).
 * Same combination rule as or_fmm. */
void or_premix(int64_t n, const double* X, int64_t ldx, int p, int R, const double* M,
               double* out);
void or_postmix(int64_t n, double alpha, const double* P, int p, int R, const double* W,
                double* C, int64_t ldc);

/* O7: exact Freivalds check on integer-valued A, B, C (n x n, ld n):
 * checks C*x == A*(B*x) in __int128 for `trials` seeded vectors x with
 * entries in [0, 2^20).  Returns the number of mismatching rows over all
 * trials (0 = pass), or -1 if an entry is not an integer or out of range
 * (|A|,|B| < 2^24, |C| < 2^53). */
int64_t or_freivalds_int(int64_t n, const double* A, const double* B, const double* C,
                         int trials, uint64_t seed);

/* O7: sampled entries: out[s] = classical dot product of row rows[s] of A with
 * column cols[s] of B, k ascending, as in or_classical. */
void or_sample_entries(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                       int64_t count, const int64_t* rows, const int64_t* cols, double* out);

/* Number of OpenMP threads the oracle runs on (for the bench's `cores`). */
int or_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif

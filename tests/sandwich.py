"""Test helper: valid bilinear triples outside the catalog.

If <U,V,W> computes C = A B on p x p block matrices (Eq. "strassen", PAPER.md
L196-202), so does its "sandwich" by invertible p x p matrices X, Y, Z:

    A B = X^-1 (X A Y^-1)(Y B Z^-1) Z,

i.e. run the algorithm on A~ = X A Y^-1 and B~ = Y B Z^-1 and map its result
back.  Each operand combination stays linear in the blocks of A (B), so

    U'[(a,b), q] = sum_{i,j} U[(i,j), q] X[i,a] Yinv[b,j]
    V'[(a,b), q] = sum_{i,j} V[(i,j), q] Y[i,a] Zinv[b,j]
    W'[(a,b), q] = sum_{i,j} Xinv[a,i] W[(i,j), q] Z[j,b]

(block index row-major).  With unimodular X, Y, Z the
coefficients stay integers (e.g. 2, -3): a triple the library has no
compiled-in kernels for, with coefficients other than +-1.  Plain numpy; it
shares nothing with oracle/ or the product.
"""
import numpy as np


def sandwich(U, V, W, p, X, Y, Z):
    U, V, W = (np.asarray(M, dtype=np.float64) for M in (U, V, W))
    X, Y, Z = (np.asarray(M, dtype=np.float64) for M in (X, Y, Z))
    Xi, Yi, Zi = np.linalg.inv(X), np.linalg.inv(Y), np.linalg.inv(Z)
    # exact when the inverses are dyadic: round away the solver's noise
    Xi, Yi, Zi = (np.round(M * 1024) / 1024 for M in (Xi, Yi, Zi))
    U2, V2, W2 = np.zeros_like(U), np.zeros_like(V), np.zeros_like(W)
    for a in range(p):
        for b in range(p):
            for i in range(p):
                for j in range(p):
                    U2[a * p + b] += U[i * p + j] * X[i, a] * Yi[b, j]
                    V2[a * p + b] += V[i * p + j] * Y[i, a] * Zi[b, j]
                    W2[a * p + b] += Xi[a, i] * W[i * p + j] * Z[j, b]
    return U2, V2, W2


# unimodular (integer inverse) and dyadic choices for p = 2 and p = 3
P2_INT = ([[1, 1], [0, 1]], [[1, 0], [1, 1]], [[2, 1], [1, 1]])
P2_DYADIC = ([[1, 1], [0, 1]], [[2, 0], [0, 1]], [[1, 0], [0, 4]])
P3_INT = ([[1, 0, 1], [0, 1, 0], [0, 0, 1]], [[1, 0, 0], [1, 1, 0], [0, 0, 1]],
          [[1, 0, 0], [0, 1, 2], [0, 0, 1]])

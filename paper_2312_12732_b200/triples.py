"""Bilinear triples <U,V,W> for the product path (what a user passes to mf_plan).

Each is a p^2 x R triple of integer coefficients: U = the paper's a, V = b,
W = c with rows in NATURAL row-major C-block order.  These
tables are typed independently of oracle/ (the two sides share no tables);
tests/test_binding.py checks that both catalogs agree and mf_plan re-proves
each one with an exact Brent check before use.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Triple:
    name: str
    p: int
    U: np.ndarray
    V: np.ndarray
    W: np.ndarray

    @property
    def R(self) -> int:
        return int(self.U.shape[1])


def _t(name, p, U, V, W) -> Triple:
    arr = [np.ascontiguousarray(np.array(x, dtype=np.float64)) for x in (U, V, W)]
    for a in arr:
        a.setflags(write=False)
    return Triple(name, p, *arr)


def _from_products(name, p, prods, crows):
    """prods: list of ({block: coef} for T_q, {block: coef} for S_q);
    crows: list over C blocks of {q: coef}."""
    R = len(prods)
    U = np.zeros((p * p, R)); V = np.zeros((p * p, R)); W = np.zeros((p * p, R))
    for q, (t, s) in enumerate(prods):
        for k, c in t.items():
            U[k, q] = c
        for k, c in s.items():
            V[k, q] = c
    for i, row in enumerate(crows):
        for q, c in row.items():
            W[i, q] = c
    return _t(name, p, U, V, W)


# Strassen-Winograd <2,2,2;7>; blocks 0=(1,1) 1=(1,2) 2=(2,1) 3=(2,2).
STRASSEN_WINOGRAD = _from_products(
    "strassen-winograd", 2,
    [({0: 1}, {0: 1}),                               # P0 = A0 B0
     ({1: 1}, {2: 1}),                               # P1 = A1 B2
     ({0: 1, 1: 1, 2: -1, 3: -1}, {3: 1}),           # P2 = (A0+A1-A2-A3) B3
     ({3: 1}, {0: 1, 1: -1, 2: -1, 3: 1}),           # P3 = A3 (B0-B1-B2+B3)
     ({2: 1, 3: 1}, {0: -1, 1: 1}),                  # P4 = (A2+A3)(B1-B0)
     ({0: -1, 2: 1, 3: 1}, {0: 1, 1: -1, 3: 1}),     # P5 = (A2+A3-A0)(B0-B1+B3)
     ({0: 1, 2: -1}, {1: -1, 3: 1})],                # P6 = (A0-A2)(B3-B1)
    [{0: 1, 1: 1},                                   # C0 = P0+P1
     {0: 1, 2: 1, 4: 1, 5: 1},                       # C1 = P0+P2+P4+P5
     {0: 1, 3: -1, 5: 1, 6: 1},                      # C2 = P0-P3+P5+P6
     {0: 1, 4: 1, 5: 1, 6: 1}])                      # C3 = P0+P4+P5+P6

# The paper's DeepMind-format Strassen, W rows re-sorted from
# the printed C0,C2,C1,C3 into natural order.
PAPER_STRASSEN = _t(
    "paper-strassen", 2,
    [[0, 1, 1, 0, 1, 1, 0], [0, 0, -1, 1, 0, 0, 0], [1, 1, 1, 0, 1, 0, 0], [-1, -1, -1, 0, 0, 0, 1]],
    [[0, 0, 0, 0, 1, 1, 0], [1, 1, 0, 0, 1, 0, 1], [0, 1, 1, 1, 1, 0, 0], [0, 1, 1, 0, 1, 0, 1]],
    [[0, 0, 0, 1, 0, 1, 0], [-1, 1, -1, -1, 0, 0, 0], [0, -1, 0, 0, 1, -1, -1], [1, 0, 0, 0, 0, 0, 1]])

# Strassen 1969: M1..M7 as products 0..6.
STRASSEN_1969 = _from_products(
    "strassen-1969", 2,
    [({0: 1, 3: 1}, {0: 1, 3: 1}), ({2: 1, 3: 1}, {0: 1}), ({0: 1}, {1: 1, 3: -1}),
     ({3: 1}, {2: 1, 0: -1}), ({0: 1, 1: 1}, {3: 1}), ({2: 1, 0: -1}, {0: 1, 1: 1}),
     ({1: 1, 3: -1}, {2: 1, 3: 1})],
    [{0: 1, 3: 1, 4: -1, 6: 1}, {2: 1, 4: 1}, {1: 1, 3: 1}, {0: 1, 1: -1, 2: 1, 5: 1}])

# Laderman 1976 <3,3,3;23>, blocks 0..8 row-major over the 3x3 grid.
LADERMAN = _from_products(
    "laderman", 3,
    [({0: 1, 1: 1, 2: 1, 3: -1, 4: -1, 7: -1, 8: -1}, {4: 1}),
     ({0: 1, 3: -1}, {1: -1, 4: 1}),
     ({4: 1}, {0: -1, 1: 1, 3: 1, 4: -1, 5: -1, 6: -1, 8: 1}),
     ({0: -1, 3: 1, 4: 1}, {0: 1, 1: -1, 4: 1}),
     ({3: 1, 4: 1}, {0: -1, 1: 1}),
     ({0: 1}, {0: 1}),
     ({0: -1, 6: 1, 7: 1}, {0: 1, 2: -1, 5: 1}),
     ({0: -1, 6: 1}, {2: 1, 5: -1}),
     ({6: 1, 7: 1}, {0: -1, 2: 1}),
     ({0: 1, 1: 1, 2: 1, 4: -1, 5: -1, 6: -1, 7: -1}, {5: 1}),
     ({7: 1}, {0: -1, 2: 1, 3: 1, 4: -1, 5: -1, 6: -1, 7: 1}),
     ({2: -1, 7: 1, 8: 1}, {4: 1, 6: 1, 7: -1}),
     ({2: 1, 8: -1}, {4: 1, 7: -1}),
     ({2: 1}, {6: 1}),
     ({7: 1, 8: 1}, {6: -1, 7: 1}),
     ({2: -1, 4: 1, 5: 1}, {5: 1, 6: 1, 8: -1}),
     ({2: 1, 5: -1}, {5: 1, 8: -1}),
     ({4: 1, 5: 1}, {6: -1, 8: 1}),
     ({1: 1}, {3: 1}),
     ({5: 1}, {7: 1}),
     ({3: 1}, {2: 1}),
     ({6: 1}, {1: 1}),
     ({8: 1}, {8: 1})],
    [dict.fromkeys([5, 13, 18], 1),
     dict.fromkeys([0, 3, 4, 5, 11, 13, 14], 1),
     dict.fromkeys([5, 6, 8, 9, 13, 15, 17], 1),
     dict.fromkeys([1, 2, 3, 5, 13, 15, 16], 1),
     dict.fromkeys([1, 3, 4, 5, 19], 1),
     dict.fromkeys([13, 15, 16, 17, 20], 1),
     dict.fromkeys([5, 6, 7, 10, 11, 12, 13], 1),
     dict.fromkeys([11, 12, 13, 14, 21], 1),
     dict.fromkeys([5, 6, 7, 8, 22], 1)])


def classical(p: int) -> Triple:
    """Rank-p^3 classical triple of Eq. (recursion)."""
    R = p ** 3
    U = np.zeros((p * p, R)); V = np.zeros((p * p, R)); W = np.zeros((p * p, R))
    for i in range(p):
        for j in range(p):
            for k in range(p):
                q = (i * p + j) * p + k
                U[i * p + k, q] = V[k * p + j, q] = W[i * p + j, q] = 1.0
    return _t(f"classical-p{p}", p, U, V, W)


def kron(outer: Triple, inner: Triple) -> Triple:
    """One level of the chain outer-then-inner as a single triple (PAPER.md
    L303-313: a (x) a', b (x) b', c (x) c').  Block (b of outer, s of inner) ->
    row-major block ((b/po)*pi + s/pi, (b%po)*pi + s%pi) of the (po*pi)-way
    split; product q = q_outer * R_inner + q_inner.  Pass the
    result to Plan with levels=1; mf_plan re-proves it (Brent) before use."""
    from . import triple_kron  # the composition runs in libmf (mf_triple_kron)
    U, V, W = triple_kron(outer, inner)
    return _t(f"{outer.name}(x){inner.name}", outer.p * inner.p, U, V, W)


CATALOG = {t.name: t for t in (STRASSEN_WINOGRAD, PAPER_STRASSEN, STRASSEN_1969, LADERMAN,
                               classical(2), classical(3))}


def get(name: str) -> Triple:
    try:
        return CATALOG[name]
    except KeyError:
        raise KeyError(f"unknown triple {name!r}; available: {', '.join(CATALOG)}") from None

"""CPU oracle for the Matrix Flow hot path (arXiv 2312.12732) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  It wraps ``liboracle.so``
(built from ``oracle.c`` by :func:`build`) with numpy; it never imports the
product package and the product never imports it.

Every wrapper names the C function (and through it the paper passage) it calls.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

TRIPLES = ("paper-strassen", "strassen-winograd", "strassen-1969", "laderman",
           "classical-p2", "classical-p3")


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, OpenMP, -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off",
                               "-fPIC", "-shared", "-Wall", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        d, i32, i64, u64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
        P = ctypes.c_void_p
        L.or_catalog.argtypes = [ctypes.c_char_p, ctypes.POINTER(i32), ctypes.POINTER(i32), P, P, P]
        L.or_catalog.restype = i32
        L.or_kron.argtypes = [i32, i32, P, P, P, i32, i32, P, P, P, P, P, P]
        L.or_kron.restype = None
        L.or_brent_check.argtypes = [i32, i32, P, P, P, P]
        L.or_brent_check.restype = i64
        L.or_classical.argtypes = [i64, P, i64, P, i64, P, i64]
        L.or_classical.restype = None
        L.or_fmm.argtypes = [i64, d, P, i64, P, i64, P, i64, i32, i32, P, P, P, i32]
        L.or_fmm.restype = i32
        L.or_premix.argtypes = [i64, P, i64, i32, i32, P, P]
        L.or_premix.restype = None
        L.or_postmix.argtypes = [i64, d, P, i32, i32, P, P, i64]
        L.or_postmix.restype = None
        L.or_freivalds_int.argtypes = [i64, P, P, P, i32, u64]
        L.or_freivalds_int.restype = i64
        L.or_sample_entries.argtypes = [i64, P, i64, P, i64, i64, P, P, P]
        L.or_sample_entries.restype = None
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


class Triple:
    """A bilinear triple <U,V,W>: p^2 x R arrays, W rows natural."""

    def __init__(self, name: str, p: int, U, V, W):
        self.name, self.p = name, int(p)
        self.U, self.V, self.W = _f64(U), _f64(V), _f64(W)
        self.R = self.U.shape[1]
        assert self.U.shape == self.V.shape == self.W.shape == (self.p * self.p, self.R)

    def __repr__(self):
        return f"Triple({self.name!r}, p={self.p}, R={self.R})"


def catalog(name: str) -> Triple:
    """or_catalog (O1): the builtin triples."""
    L = lib()
    p, R = ctypes.c_int(), ctypes.c_int()
    if L.or_catalog(name.encode(), ctypes.byref(p), ctypes.byref(R), None, None, None) != 0:
        raise KeyError(f"unknown triple {name!r}; available: {', '.join(TRIPLES)}")
    U = np.zeros((p.value ** 2, R.value))
    V, W = np.zeros_like(U), np.zeros_like(U)
    L.or_catalog(name.encode(), ctypes.byref(p), ctypes.byref(R), _ptr(U), _ptr(V), _ptr(W))
    return Triple(name, p.value, U, V, W)


def kron(outer: Triple, inner: Triple) -> Triple:
    """or_kron (O1): outer (x) inner with SPEC.md L244's row interleave."""
    P, R = outer.p * inner.p, outer.R * inner.R
    U = np.zeros((P * P, R))
    V, W = np.zeros_like(U), np.zeros_like(U)
    lib().or_kron(outer.p, outer.R, _ptr(outer.U), _ptr(outer.V), _ptr(outer.W),
                  inner.p, inner.R, _ptr(inner.U), _ptr(inner.V), _ptr(inner.W),
                  _ptr(U), _ptr(V), _ptr(W))
    return Triple(f"{outer.name}(x){inner.name}", P, U, V, W)


def kron_power(t: Triple, levels: int) -> Triple:
    """levels-fold Kronecker flattening (the product index stays outer-major)."""
    out = t
    for _ in range(levels - 1):
        out = kron(out, t)
    return out


def brent_check(t: Triple):
    """or_brent_check (O2): returns (violations, first (x,y,z) or None)."""
    first = np.zeros(3, dtype=np.int64)
    bad = lib().or_brent_check(t.p, t.R, _ptr(t.U), _ptr(t.V), _ptr(t.W), _ptr(first))
    if bad < 0:
        raise ValueError("non-integer coefficients")
    return int(bad), (tuple(int(v) for v in first) if bad else None)


def classical(A, B) -> np.ndarray:
    """or_classical (O3): C = A*B, k-ascending, no FMA."""
    A, B = _f64(A), _f64(B)
    n = A.shape[0]
    C = np.empty((n, n))
    lib().or_classical(n, _ptr(A), n, _ptr(B), n, _ptr(C), n)
    return C


def fmm(A, B, t: Triple, levels: int, alpha: float = 1.0) -> np.ndarray:
    """or_fmm (O4): C = alpha*A*B through `levels` levels of Eq. (strassen)."""
    A, B = _f64(A), _f64(B)
    n = A.shape[0]
    C = np.empty((n, n))
    rc = lib().or_fmm(n, float(alpha), _ptr(A), n, _ptr(B), n, _ptr(C), n, t.p, t.R,
                      _ptr(t.U), _ptr(t.V), _ptr(t.W), int(levels))
    if rc == -1:
        raise ValueError(f"n={n} is not divisible by p^levels = {t.p}^{levels}")
    if rc != 0:
        raise MemoryError("or_fmm allocation failed")
    return C


def premix(X, t: Triple, side: str) -> np.ndarray:
    """or_premix: all R operands T_q (side='A', coefficients U) or S_q (side='B', V)."""
    X = _f64(X)
    n = X.shape[0]
    m = n // t.p
    M = t.U if side == "A" else t.V
    out = np.empty((t.R, m, m))
    lib().or_premix(n, _ptr(X), n, t.p, t.R, _ptr(M), _ptr(out))
    return out


def postmix(P, t: Triple, n: int, alpha: float = 1.0) -> np.ndarray:
    """or_postmix: C_i = alpha * sum_q W[i][q] P_q."""
    P = _f64(P)
    C = np.empty((n, n))
    lib().or_postmix(n, float(alpha), _ptr(P), t.p, t.R, _ptr(t.W), _ptr(C), n)
    return C


def freivalds_int(A, B, C, trials: int = 3, seed: int = 1) -> int:
    """or_freivalds_int (O7): exact __int128 Freivalds; 0 = pass, -1 = non-integer input."""
    A, B, C = _f64(A), _f64(B), _f64(C)
    return int(lib().or_freivalds_int(A.shape[0], _ptr(A), _ptr(B), _ptr(C), trials, seed))


def sample_entries(A, B, rows, cols) -> np.ndarray:
    """or_sample_entries (O7): classical dot products for the sampled (row, col) pairs."""
    A, B = _f64(A), _f64(B)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(len(rows))
    lib().or_sample_entries(A.shape[0], _ptr(A), A.shape[1], _ptr(B), B.shape[1], len(rows),
                            _ptr(rows), _ptr(cols), _ptr(out))
    return out


def num_threads() -> int:
    return int(lib().or_num_threads())


def scaled_error(C, C_ref, A, B) -> float:
    """North-star metric: max|C - C_ref| / (n * max|A| * max|B|)."""
    n = A.shape[0]
    den = n * float(np.abs(A).max()) * float(np.abs(B).max())
    return float(np.abs(np.asarray(C) - np.asarray(C_ref)).max()) / den if den else 0.0

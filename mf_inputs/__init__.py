"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only draws matrices.  Both
``oracle/`` (through tests and bench) and the product tests feed these arrays
to their own code.  Recipe: square dense fp64, A with seed s and
B with seed s+1; value distributions

* ``uniform``   : i.i.d. Uniform[-1, 1)            (reading R12)
* ``integers``  : i.i.d. integers in [lo, hi]       ([-8, 8];
                  [-1024, 1024] stresses the mantissa, reading R15)
* ``block_impulse``: 1 on one block of a P x P partition, 0 elsewhere
                  (the GPU-level Brent check of SURVEY.md §8c)

Host arrays come from numpy's PCG64; ``device_*`` draw the same distributions
on a CUDA device with a seeded torch generator (different stream from the host
generator -- callers copy device inputs to the host when the oracle needs them).
"""
from __future__ import annotations

import numpy as np


def uniform(n: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=(n, n))


def integers(n: int, seed: int, lo: int = -1024, hi: int = 1024) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi + 1, size=(n, n)).astype(np.float64)


def block_impulse(n: int, P: int, block: int, value: float = 1.0) -> np.ndarray:
    m = n // P
    X = np.zeros((n, n))
    r, c = divmod(block, P)
    X[r * m:(r + 1) * m, c * m:(c + 1) * m] = value
    return X


def pair(kind: str, n: int, seed: int = 0):
    """(A, B) of one distribution with seeds s and s+1."""
    if kind == "uniform":
        return uniform(n, seed), uniform(n, seed + 1)
    if kind == "int8":
        return integers(n, seed, -8, 8), integers(n, seed + 1, -8, 8)
    if kind == "int1024":
        return integers(n, seed, -1024, 1024), integers(n, seed + 1, -1024, 1024)
    raise ValueError(kind)


def device_pair(kind: str, n: int, seed: int = 0, device: str = "cuda"):
    """(A, B) drawn on the device (torch, float64), for sizes where host generation is slow."""
    import torch
    g = torch.Generator(device=device)
    out = []
    for s in (seed, seed + 1):
        g.manual_seed(s)
        if kind == "uniform":
            X = torch.rand((n, n), generator=g, device=device, dtype=torch.float64) * 2.0 - 1.0
        elif kind in ("int8", "int1024"):
            lim = 8 if kind == "int8" else 1024
            X = torch.randint(-lim, lim + 1, (n, n), generator=g, device=device,
                              dtype=torch.int64).to(torch.float64)
        else:
            raise ValueError(kind)
        out.append(X)
    return out[0], out[1]

"""Host views of the universal constant tables held by librqmc_b200.so.

Halton per-dimension constants depend only on the d-th prime (base, digit
capacity K = min{K : p^K >= 2^32} (halton.py:59-66), window K + 8
(halton.py:38)), so one table serves every replication and seed.  Sobol'
direction numbers are the Joe-Kuo D6 set (sobol.py:170-173) expanded by
the m-recursion (sobol.py:61-71).
"""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import numpy as np

from . import _lib

CAP_PAD = 8  # halton.py:38
SOBOL_MAX_DIM = 421


@lru_cache(maxsize=None)
def halton_constants(dim: int):
    base = np.empty(dim, dtype=np.int32)
    K = np.empty(dim, dtype=np.int32)
    scale0 = np.empty(dim, dtype=np.float64)
    _lib.check(_lib.lib().rq_halton_constants(
        dim, base.ctypes.data_as(C.POINTER(C.c_int32)), K.ctypes.data_as(C.POINTER(C.c_int32)),
        scale0.ctypes.data_as(C.POINTER(C.c_double))))
    return base, K, scale0


def halton_layout(dim: int) -> dict:
    base, K, _ = halton_constants(dim)
    caps = K.astype(np.int64) + CAP_PAD
    return {"bases": int(base.sum()), "caps": int(caps.sum()), "sums": int((caps + 1).sum()),
            "base": base, "K": K, "cap": caps}


@lru_cache(maxsize=None)
def sobol_directions(dim: int) -> np.ndarray:
    v = np.empty((dim, 32), dtype=np.uint32)
    _lib.check(_lib.lib().rq_sobol_directions(dim, v.ctypes.data_as(C.POINTER(C.c_uint32))))
    return v

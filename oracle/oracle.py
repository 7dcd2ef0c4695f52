"""ctypes front end of the CPU oracle (oracle/rqmc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` arm -- never by the
``paper_1408_5526_b200`` package.  See rqmc_oracle.h for what each function
restates (reference file:line) and how it is pinned (tests/test_oracle.py
against tests/golden/, produced from the unmodified reference).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "librqmc_oracle.so"

GEN_IDS = {"rasrap-recursive": 0, "rasrap-counter": 1, "philox": 2, "sobol-gray": 3,
           "sobol-counter": 4, "sfc64": 5, "twister": 6, "xorwow": 7,
           "kakutani": 8}
MODEL_IDS = {"libor": 0, "mbs": 1, "x1": 2, "const1": 3, "xhash": 5}
FAMILY_IDS = {"twister": 1, "xorwow": 2, "philox": 3, "rasrap": 4, "sobol": 5, "kakutani": 6,
              "sfc64": 7}

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _declare(L):
    u64, i64, i32, dbl = C.c_uint64, C.c_int64, C.c_int, C.c_double
    P = C.POINTER
    L.orc_splitmix64.restype = u64
    L.orc_splitmix64.argtypes = [u64]
    L.orc_derive_key.restype = u64
    L.orc_derive_key.argtypes = [P(u64), i32]
    L.orc_derive_words.argtypes = [u64, i32, P(C.c_uint32)]
    L.orc_pcg64_u32_stream.argtypes = [u64, i32, P(C.c_uint32)]
    L.orc_primes.argtypes = [i32, P(i64)]
    L.orc_digit_capacity.argtypes = [i64]
    L.orc_invert_radical.restype = u64
    L.orc_invert_radical.argtypes = [dbl, i64, i32]
    L.orc_rasrap_config.argtypes = [i32, u64, P(i64), P(dbl), P(i64), i32]
    L.orc_rasrap_recursive_points.argtypes = [i32, u64, i64, P(dbl)]
    L.orc_rasrap_counter_points.argtypes = [i32, u64, P(i64), i64, P(dbl)]
    L.orc_philox_block.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
    L.orc_philox_words.argtypes = [u64, P(i64), i64, i32, P(C.c_uint32)]
    L.orc_sobol_scramble.argtypes = [i32, P(C.c_uint32), u64, i64, P(C.c_uint32),
                                     P(C.c_uint32)]
    L.orc_sobol_counter_words.argtypes = [i32, P(C.c_uint32), P(C.c_uint32), P(i64), i64,
                                          P(C.c_uint32)]
    L.orc_inv_normal.restype = dbl
    L.orc_inv_normal.argtypes = [dbl]
    L.orc_inv_normal_n.argtypes = [P(dbl), i64, P(dbl)]
    L.orc_libor_payoffs.argtypes = [P(dbl), i64, i32, P(dbl), dbl, dbl, dbl, dbl, P(dbl)]
    L.orc_mbs_payoffs.argtypes = [P(dbl), i64, i32] + [dbl] * 8 + [P(dbl), P(dbl)]
    L.orc_coord_hash.restype = dbl
    L.orc_coord_hash.argtypes = [P(dbl), i32]
    L.orc_pairwise_sum.restype = dbl
    L.orc_pairwise_sum.argtypes = [P(dbl), i64]
    L.orc_run_replication.argtypes = [i32, i32, i32, P(dbl), u64, i64, P(i64), i32,
                                      P(C.c_uint32), P(dbl)]
    L.orc_run_replications.argtypes = [i32, i32, i32, P(dbl), u64, i64, i64, P(i64), i32,
                                       P(C.c_uint32), i32, P(dbl)]
    L.orc_sfc64_path_uniforms.argtypes = [u64, i64, P(i64), i64, i32, P(dbl)]
    L.orc_mt19937_init.argtypes = [C.c_void_p, C.c_uint32]
    L.orc_mt19937_words.argtypes = [C.c_void_p, i64, P(C.c_uint32)]
    L.orc_xorwow_init.argtypes = [C.c_void_p, u64]
    L.orc_xorwow_words.argtypes = [C.c_void_p, i64, P(C.c_uint32)]
    L.orc_kakutani_set_tables.argtypes = [P(dbl), P(dbl), i32]
    L.orc_kakutani_points.argtypes = [i32, u64, i64, P(dbl)]
    _set_kakutani_tables(L)


# ---------------------------------------------------------------- seeding
def derive_key(*parts: int) -> int:
    arr = np.array([int(p) & 0xFFFFFFFFFFFFFFFF for p in parts], dtype=np.uint64)
    return int(lib().orc_derive_key(_p(arr, C.c_uint64), len(parts)))


def derive_words(key: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint32)
    lib().orc_derive_words(key, count, _p(out, C.c_uint32))
    return out


def pcg64_u32(key: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    lib().orc_pcg64_u32_stream(key, n, _p(out, C.c_uint32))
    return out


# ---------------------------------------------------------------- Halton
def primes(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    lib().orc_primes(n, _p(out, C.c_int64))
    return out


def digit_capacity(base: int) -> int:
    return int(lib().orc_digit_capacity(base))


def invert_radical(omega: float, base: int, k: int) -> int:
    return int(lib().orc_invert_radical(omega, base, k))


def rasrap_config(dim: int, key: int):
    ps = primes(dim)
    mb = int(ps[-1])
    start = np.empty(dim, dtype=np.int64)
    omega = np.empty(dim)
    sigma = np.empty((dim, mb), dtype=np.int64)
    lib().orc_rasrap_config(dim, key, _p(start, C.c_int64), _p(omega, C.c_double),
                            _p(sigma, C.c_int64), mb)
    return start, omega, sigma


def rasrap_recursive(dim: int, key: int, count: int) -> np.ndarray:
    out = np.empty((count, dim))
    lib().orc_rasrap_recursive_points(dim, key, count, _p(out, C.c_double))
    return out


def rasrap_counter(dim: int, key: int, idx) -> np.ndarray:
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty((idx.size, dim))
    lib().orc_rasrap_counter_points(dim, key, _p(idx, C.c_int64), idx.size,
                                    _p(out, C.c_double))
    return out


# ---------------------------------------------------------------- Philox / Sobol / SFC64
def philox_block(counter, key):
    c = np.array(counter, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    out = np.empty(4, dtype=np.uint32)
    lib().orc_philox_block(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return tuple(int(x) for x in out)


def philox_words(key: int, paths, nwords: int) -> np.ndarray:
    paths = np.ascontiguousarray(paths, dtype=np.int64)
    out = np.empty((paths.size, nwords), dtype=np.uint32)
    lib().orc_philox_words(key, _p(paths, C.c_int64), paths.size, nwords, _p(out, C.c_uint32))
    return out


def sobol_scramble(v: np.ndarray, key: int, replication: int):
    v = np.ascontiguousarray(v, dtype=np.uint32)
    dim = v.shape[0]
    gen_v = np.empty((dim, 32), dtype=np.uint32)
    shift = np.empty(dim, dtype=np.uint32)
    lib().orc_sobol_scramble(dim, _p(v, C.c_uint32), key, replication, _p(gen_v, C.c_uint32),
                             _p(shift, C.c_uint32))
    return gen_v, shift


def sobol_counter_words(gen_v, shift, idx) -> np.ndarray:
    gen_v = np.ascontiguousarray(gen_v, dtype=np.uint32)
    shift = np.ascontiguousarray(shift, dtype=np.uint32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    dim = gen_v.shape[0]
    out = np.empty((idx.size, dim), dtype=np.uint32)
    lib().orc_sobol_counter_words(dim, _p(gen_v, C.c_uint32), _p(shift, C.c_uint32),
                                  _p(idx, C.c_int64), idx.size, _p(out, C.c_uint32))
    return out


def sfc64_uniforms(seed: int, m: int, paths, dim: int) -> np.ndarray:
    paths = np.ascontiguousarray(paths, dtype=np.int64)
    out = np.empty((paths.size, dim))
    lib().orc_sfc64_path_uniforms(seed, m, _p(paths, C.c_int64), paths.size, dim,
                                  _p(out, C.c_double))
    return out


KK_TAB = 64
_KK = {}


def kakutani_tables(dims: int = 512):
    """KakutaniState._grow_tables (halton.py:178-193) for the first `dims`
    primes: thr = float(Fraction(1, p^k)) + 1e-11, b = float(Fraction(p + 1 - p^k, p^k)),
    k = 1..64 -> arrays [dims, 64]."""
    from fractions import Fraction

    if dims not in _KK:
        thr = np.empty((dims, KK_TAB))
        b = np.empty((dims, KK_TAB))
        ps = [int(p) for p in _primes_py(dims)]
        for d, p in enumerate(ps):
            pk = 1
            for k in range(1, KK_TAB + 1):
                pk *= p
                b[d, k - 1] = float(Fraction(p + 1 - pk, pk))
                thr[d, k - 1] = float(Fraction(1, pk)) + 1e-11
        _KK[dims] = (thr, b)
    return _KK[dims]


def _primes_py(n: int):
    out, c = [], 2
    while len(out) < n:
        if all(c % q for q in out if q * q <= c):
            out.append(c)
        c += 1
    return out


_KK_SET = [0]


def _set_kakutani_tables(L, dims: int = 512):
    thr, b = kakutani_tables(dims)
    L.orc_kakutani_set_tables(_p(thr, C.c_double), _p(b, C.c_double), thr.shape[0])
    _KK_SET[0] = dims


def _ensure_kakutani(dim: int):
    """Bracket tables of at least `dim` dims in the C oracle (grown in 512s)."""
    if dim > _KK_SET[0]:
        _set_kakutani_tables(lib(), (dim + 511) // 512 * 512)


def kakutani_points(dim: int, key: int, count: int) -> np.ndarray:
    """KakutaniSampler(dim, key).fill of `count` rows (halton.py:521-542)."""
    out = np.empty((count, dim))
    _ensure_kakutani(dim)
    if lib().orc_kakutani_points(dim, key & 0xFFFFFFFFFFFFFFFF, count, _p(out, C.c_double)):
        raise ValueError("kakutani orbit left the 64-entry bracket tables")
    return out


class _WordStream:
    """Sequential word generator state owned by Python (prng.py:63-149)."""

    def __init__(self, nbytes: int, init, seed: int, fill):
        self._buf = C.create_string_buffer(nbytes)
        self._fill = fill
        init(self._buf, seed)

    def words(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        self._fill(self._buf, n, _p(out, C.c_uint32))
        return out


def mt19937(seed32: int) -> _WordStream:
    """prng.MT19937(seed) (prng.py:63-72)."""
    return _WordStream(624 * 4 + 8, lib().orc_mt19937_init, seed32 & 0xFFFFFFFF,
                       lib().orc_mt19937_words)


def xorwow(seed: int) -> _WordStream:
    """prng.Xorwow(seed) (prng.py:128-134)."""
    return _WordStream(6 * 4, lib().orc_xorwow_init, seed & 0xFFFFFFFFFFFFFFFF,
                       lib().orc_xorwow_words)


# ---------------------------------------------------------------- models
def inv_normal(u) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    lib().orc_inv_normal_n(_p(u, C.c_double), u.size, _p(out, C.c_double))
    return out


def libor_payoffs(u, l0, delta, sigma, strike, front_factor) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    l0 = np.ascontiguousarray(l0, dtype=np.float64)
    out = np.empty(u.shape[0])
    lib().orc_libor_payoffs(_p(u, C.c_double), u.shape[0], u.shape[1], _p(l0, C.c_double),
                            delta, sigma, strike, front_factor, _p(out, C.c_double))
    return out


def mbs_payoffs(u, i0, k0, k1, k2, k3, k4, sigma_xi, payment, ck) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    ck = np.ascontiguousarray(ck, dtype=np.float64)
    out = np.empty(u.shape[0])
    lib().orc_mbs_payoffs(_p(u, C.c_double), u.shape[0], u.shape[1], i0, k0, k1, k2, k3, k4,
                          sigma_xi, payment, _p(ck, C.c_double), _p(out, C.c_double))
    return out


def coord_hash(u) -> np.ndarray:
    """xhash test-integrand payoffs of uniforms u[n, dim] (rqmc_oracle.c)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    return np.array([lib().orc_coord_hash(_p(r, C.c_double), u.shape[1]) for r in u])


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum(_p(a, C.c_double), a.size))


def model_params(model) -> tuple[int, int, np.ndarray]:
    """(model id, dim, packed params) for a package or reference model object."""
    name = model.name
    if name == "libor":
        c = model.config
        ff = 1.0 / (1.0 + c.accrual * model.front_rate)
        p = np.concatenate([[c.accrual, c.sigma, c.strike, ff], model.initial_rates])
    elif name == "mbs":
        c = model.config
        p = np.concatenate([[c.initial_rate, c.k0, c.k1, c.k2, c.k3, c.k4, c.sigma_xi,
                             c.payment], c.annuity_ratios()])
    else:
        p = np.zeros(1)
    return MODEL_IDS[name], model.dim, np.ascontiguousarray(p, dtype=np.float64)


def run_replications(generator: str, model, seed: int, first: int, count: int, grid,
                     threads: int = 1, sobol_v=None) -> np.ndarray:
    """theta[count, len(grid)] for replications first..first+count-1."""
    mid, dim, params = model_params(model)
    grid = np.ascontiguousarray(grid, dtype=np.int64)
    theta = np.empty((count, grid.size))
    if sobol_v is None:
        sobol_v = np.zeros((1, 32), dtype=np.uint32)
    sobol_v = np.ascontiguousarray(sobol_v, dtype=np.uint32)
    if generator == "kakutani":
        _ensure_kakutani(dim)
    rc = lib().orc_run_replications(GEN_IDS[generator], mid, dim, _p(params, C.c_double), seed,
                                    first, count, _p(grid, C.c_int64), grid.size,
                                    _p(sobol_v, C.c_uint32), threads, _p(theta, C.c_double))
    if rc:
        raise ValueError(f"oracle run_replications failed ({rc})")
    return theta


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1

"""The C-ABI library (CPU-side checks, no CUDA calls).

* it loads without a GPU and exports every entry point declared in
  include/rqmc_b200.h;
* its host-built constant tables match the reference: Halton bases /
  digit capacities / Python-pow scales (halton.py:59-66, 273-274), the
  division magic the kernels use, Joe-Kuo direction numbers (sobol.py);
* the numpy pairwise-sum plan it uploads reproduces np.sum bit for bit;
* argument validation fails with the reference's error class before any
  device work.
"""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "rqmc_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_1408_5526_b200 import _lib

    return _lib.lib()


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), f"{n} declared in rqmc_b200.h but not exported"
    assert lib.rq_abi_version() == 1


def test_halton_constants_match_reference(lib, oracle):
    from paper_1408_5526_b200.tables import halton_constants

    base, K, scale0 = halton_constants(512)
    assert np.array_equal(base, oracle.primes(512))
    for p, k, s in zip(base, K, scale0):
        p, k = int(p), int(k)
        assert p**k >= 2**32 > p ** (k - 1)  # digit_capacity, halton.py:59-66
        assert s == (1.0 / p) ** k  # Python float ** int (halton.py:274)


def test_division_magic_is_exact(lib):
    from paper_1408_5526_b200.tables import halton_constants

    base, _, _ = halton_constants(512)
    rng = np.random.default_rng(3)
    q64, q32 = C.c_uint64(), C.c_uint32()
    for d in list(range(40)) + list(range(40, 512, 37)) + [511]:
        p = int(base[d])
        xs = [0, 1, p - 1, p, p + 1, 2**32 - 1, 2**46 - 1, p**3 - 1 if p**3 < 2**46 else p]
        xs += [int(x) for x in rng.integers(0, 2**46, size=200, dtype=np.int64)]
        xs += list(range(0, 65536, 997)) + [65535, p * 100 - 1, p * 100]  # 16-bit magic
        for x in xs:
            assert lib.rq_halton_divide(d, x, C.byref(q64), C.byref(q32)) == 0
            assert q64.value == x // p, (d, x)
            assert q32.value == (x & 0xFFFFFFFF) // p, (d, x)


def test_sobol_directions_match_reference(golden):
    from paper_1408_5526_b200.tables import sobol_directions

    assert np.array_equal(sobol_directions(421), golden("sobol")["table421_v"])
    assert np.array_equal(sobol_directions(20), golden("sobol")["table421_v"][:20])


@pytest.mark.parametrize("n", list(range(1, 260)) + [1000, 10_000, 99_991, 2**20, 10**6])
def test_pairwise_plan_matches_numpy(lib, n):
    rng = np.random.default_rng(n)
    a = rng.random(n) * np.exp(rng.normal(size=n) * 3)
    out = C.c_double()
    assert lib.rq_pairwise_sum_host(a.ctypes.data_as(C.POINTER(C.c_double)), n,
                                    C.byref(out)) == 0
    assert out.value == np.sum(a)


def test_validation_errors_before_device_work(lib):
    h = C.c_void_p()
    assert lib.rq_sampler_create(C.byref(h), 99, 4, 0, 1, 1, None) == -1
    assert b"generator" in lib.rq_last_error()
    assert lib.rq_sampler_create(C.byref(h), 0, 0, 0, 1, 1, None) == -1
    assert lib.rq_sampler_create(C.byref(h), 3, 500, 0, 1, 1, None) == -1
    assert b"421" in lib.rq_last_error()
    assert lib.rq_sampler_create(C.byref(h), 0, 4, 0, 1, 0, None) == -1
    from paper_1408_5526_b200._lib import RqModel

    m = RqModel()
    m.kind, m.dim = 2, 2
    theta = np.zeros(4)
    bad = np.array([10, 5], dtype=np.int64)
    rc = lib.rq_run_replications(0, C.byref(m), 0, 1, 2, bad.ctypes.data_as(C.POINTER(C.c_int64)),
                                 2, theta.ctypes.data_as(C.POINTER(C.c_double)), None)
    assert rc == -1 and b"increasing" in lib.rq_last_error()
    big = np.array([2**41], dtype=np.int64)  # beyond the 2^40 cap
    rc = lib.rq_run_replications(0, C.byref(m), 0, 1, 2, big.ctypes.data_as(C.POINTER(C.c_int64)),
                                 1, theta.ctypes.data_as(C.POINTER(C.c_double)), None)
    assert rc == -3
    big = np.array([2**33], dtype=np.int64)  # beyond Sobol's 2^32 index range
    rc = lib.rq_run_replications(3, C.byref(m), 0, 1, 2, big.ctypes.data_as(C.POINTER(C.c_int64)),
                                 1, theta.ctypes.data_as(C.POINTER(C.c_double)), None)
    assert rc == -3 and b"index range" in lib.rq_last_error()


def test_error_codes_map_to_reference_exceptions():
    from paper_1408_5526_b200 import _lib
    from paper_1408_5526_b200.harness import ConfigurationError

    _lib.lib().rq_sampler_create(C.byref(C.c_void_p()), 99, 4, 0, 1, 1, None)
    with pytest.raises(ConfigurationError):
        _lib.check(-1)
    with pytest.raises(ArithmeticError):
        _lib.check(-4)
    with pytest.raises(_lib.DeviceError):
        _lib.check(-2)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1408_5526_b200 import _lib, models

    with pytest.raises(_lib.DeviceError):
        models.inv_normal(np.array([0.3]))
    import paper_1408_5526_b200 as P

    with pytest.raises(_lib.DeviceError):
        P.run_experiment(P.ExperimentConfig(model="x1", generator="philox", n_grid=(8,),
                                            replications=2))


def test_kakutani_tables_exact(lib, oracle):
    """The library's big-integer rounding == the reference's Fraction tables."""
    import ctypes as C

    dims = 512
    thr = np.empty((dims, 64))
    b = np.empty((dims, 64))
    assert lib.rq_kakutani_tables(dims, thr.ctypes.data_as(C.POINTER(C.c_double)),
                                  b.ctypes.data_as(C.POINTER(C.c_double))) == 0
    rthr, rb = oracle.kakutani_tables(dims)
    assert np.array_equal(thr, rthr)
    assert np.array_equal(b, rb)

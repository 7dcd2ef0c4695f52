"""CPU: the oracle and the host tables beyond 512 dimensions / 160 LIBOR steps,
pinned to tests/golden/bigdim.npz (written by the unmodified reference)."""
import ctypes as C

import numpy as np
import pytest

from conftest import SEED


@pytest.fixture(scope="module")
def G(golden):
    return golden("bigdim")


def test_oracle_rasrap_1000_dims(oracle, G):
    tag = "rasrap_d1000_m2"
    key = oracle.derive_key(SEED, 4, 2)
    cols = G[f"{tag}_cols"]
    assert np.array_equal(oracle.rasrap_recursive(1000, key, 300)[:, cols], G[f"{tag}_recursive"])
    assert np.array_equal(oracle.rasrap_counter(1000, key, G[f"{tag}_idx"])[:, cols],
                          G[f"{tag}_counter"])


def test_oracle_kakutani_700_dims(oracle, G):
    tag = "kakutani_d700_m1"
    rows, cols = G[f"{tag}_rows"], G[f"{tag}_cols"]
    pts = oracle.kakutani_points(700, oracle.derive_key(SEED, 6, 1), int(rows[-1]) + 1)
    assert np.array_equal(pts[rows][:, cols], G[f"{tag}_points"])


def _models(G):
    from paper_1408_5526_b200 import models as M

    curve = M.YieldCurve(G["long_curve"][0], G["long_curve"][1])
    return {
        "libor200": M.LiborModel(M.LiborConfig(maturity=25.0, accrual=0.125)),
        "libor600": M.LiborModel(M.LiborConfig(maturity=150.0, accrual=0.25), curve=curve),
        "mbs600": M.MbsModel(M.MbsConfig(months=600)),
    }


@pytest.mark.parametrize("tag,gen,mk", [
    ("libor200_rasrap", "rasrap-recursive", "libor200"),
    ("libor200_philox", "philox", "libor200"),
    ("libor600_rasrap", "rasrap-recursive", "libor600"),
    ("libor600_counter", "rasrap-counter", "libor600"),
    ("mbs600_rasrap", "rasrap-recursive", "mbs600"),
    ("libor200_kakutani", "kakutani", "libor200"),
])
def test_oracle_big_estimates_bit_exact(oracle, G, tag, gen, mk):
    model = _models(G)[mk]
    theta = G[f"{tag}_theta"]
    mine = oracle.run_replications(gen, model, SEED, 1, theta.shape[1], G[f"{tag}_grid"],
                                   threads=2)
    assert np.array_equal(mine.T, theta)


def test_libor_steps_beyond_shared_memory_model():
    from paper_1408_5526_b200 import models as M

    assert M.LiborModel(M.LiborConfig(maturity=25.0, accrual=0.125)).dim == 200
    assert M.LIBOR_MAX_STEPS == 6542


def test_host_tables_all_bases_below_2_16(oracle):
    from paper_1408_5526_b200 import _lib

    L = _lib.lib()
    n = 6542
    base = np.zeros(n, np.int32)
    K = np.zeros(n, np.int32)
    s0 = np.zeros(n)
    assert L.rq_halton_constants(n, base.ctypes.data_as(C.POINTER(C.c_int32)),
                                 K.ctypes.data_as(C.POINTER(C.c_int32)),
                                 s0.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert np.array_equal(base, oracle.primes(n))
    assert base[-1] == 65521 and base.max() < 2**16
    assert all(K[d] == oracle.digit_capacity(int(base[d])) for d in (0, 511, 512, 4000, n - 1))
    assert L.rq_halton_constants(n + 1, None, None, None) != 0
    # the division magic past the constant-bank dims
    for d in (512, 3000, n - 1):
        q64 = C.c_uint64()
        q32 = C.c_uint32()
        x = 2**39 + 12345
        assert L.rq_halton_divide(d, x, C.byref(q64), C.byref(q32)) == 0
        assert q64.value == x // int(base[d])
        assert q32.value == (x & 0xFFFFFFFF) // int(base[d])


def test_kakutani_tables_past_512(oracle):
    from paper_1408_5526_b200 import _lib

    dims = 1024
    thr = np.zeros((dims, 64))
    b = np.zeros((dims, 64))
    assert _lib.lib().rq_kakutani_tables(dims, thr.ctypes.data_as(C.POINTER(C.c_double)),
                                         b.ctypes.data_as(C.POINTER(C.c_double))) == 0
    rthr, rb = oracle.kakutani_tables(dims)
    assert np.array_equal(thr, rthr) and np.array_equal(b, rb)

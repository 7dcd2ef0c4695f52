"""Pin the CPU oracle (oracle/rqmc_oracle.c) to the reference.

Every check compares the oracle with golden fixtures written by
tests/golden/make_golden.py from the unmodified reference package, or with
numpy itself for the third-party algorithms the reference calls.  All
comparisons are bit-exact.
"""
import numpy as np
import pytest

from conftest import SEED

FAM = {"philox": 3, "rasrap": 4, "sobol": 5}


def test_derive_key_and_words(oracle, golden):
    g = golden("seeding")
    for i, f in enumerate(g["families"]):
        for m in range(9):
            assert oracle.derive_key(SEED, int(f), m) == int(g["keys"][i, m])
    for i in range(len(g["families"])):
        assert np.array_equal(oracle.derive_words(int(g["keys"][i, 1]), 7), g["words"][i])


@pytest.mark.parametrize("key", [0, 1, 2**32 - 1, 2**32, 0xDEADBEEFCAFEF00D, 2**64 - 1])
def test_pcg64_matches_numpy(oracle, key):
    rng = np.random.Generator(np.random.PCG64(key))
    expect = rng.integers(0, 2**32, size=1001, dtype=np.uint32)
    assert np.array_equal(oracle.pcg64_u32(key, 1001), expect)


def test_numpy_random_and_permutation(oracle):
    # rasrap_config draws rng.random() then rng.permutation(p) (halton.py:357-359)
    ps = oracle.primes(360)
    s, om, sg = oracle.rasrap_config(360, 123)
    for d in (0, 1, 2, 3, 19, 79, 359):
        p = int(ps[d])
        key = oracle.derive_key(123, d)
        rng = np.random.Generator(np.random.PCG64(key))
        w = rng.random()
        perm = rng.permutation(p)
        assert om[d] == w
        assert np.array_equal(sg[d, :p], perm)


def test_primes_and_capacity(oracle):
    ps = oracle.primes(360)
    assert list(ps[:10]) == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]
    assert ps[-1] == 2423
    for p in ps[:50]:
        k = oracle.digit_capacity(int(p))
        assert p**k >= 2**32 > p ** (k - 1)


def test_invert_radical_hand_values(oracle):
    # test_halton.py:93-96
    assert oracle.invert_radical(0.0, 2, 32) == 0
    assert oracle.invert_radical(0.5, 2, 32) == 1
    assert oracle.invert_radical(0.375, 2, 32) == 6


RASRAP_CASES = ["d20_m1", "d20_m2", "d80_m1", "d80_m3", "d360_m1", "d360_m2"]


def _tag(tag):
    dim, m = tag[1:].split("_m")
    return int(dim), int(m)


@pytest.mark.parametrize("tag", RASRAP_CASES)
def test_rasrap_config_and_points(oracle, golden, tag):
    g = golden("rasrap")
    dim, m = _tag(tag)
    key = oracle.derive_key(SEED, FAM["rasrap"], m)
    start, omega, sigma = oracle.rasrap_config(dim, key)
    assert np.array_equal(start, g[f"{tag}_start"])
    assert np.array_equal(omega, g[f"{tag}_omega"])
    assert np.array_equal(sigma, g[f"{tag}_sigma"])
    rows = g[f"{tag}_rows"]
    assert np.array_equal(oracle.rasrap_counter(dim, key, rows), g[f"{tag}_counter"])
    assert np.array_equal(oracle.rasrap_counter(dim, key, g[f"{tag}_bigidx"]),
                          g[f"{tag}_counter_big"])
    nmax = int(rows[-1]) + 1
    if nmax * dim <= 30_000_000:  # the long d360 stream is checked in test_gpu_parity
        pts = oracle.rasrap_recursive(dim, key, nmax)
        assert np.array_equal(pts[rows], g[f"{tag}_recursive"])


def test_philox_kat(oracle):
    # Random123 known-answer vectors (test_prng.py:15-25)
    kat = [
        (((0, 0, 0, 0), (0, 0)), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        (((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        (((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for (c, k), e in kat:
        assert oracle.philox_block(c, k) == e


@pytest.mark.parametrize("tag", ["d20_m1", "d20_m2", "d80_m1", "d360_m1"])
def test_philox_paths(oracle, golden, tag):
    g = golden("philox")
    dim, m = _tag(tag)
    key = oracle.derive_key(SEED, FAM["philox"], m)
    assert np.array_equal(oracle.philox_words(key, g[f"{tag}_rows"], dim), g[f"{tag}_words"])
    u = oracle.philox_words(key, np.arange(300), dim) * 2.0**-32 + 2.0**-33
    assert np.array_equal(u, g[f"{tag}_fill300"])


@pytest.mark.parametrize("tag", ["d20_m1", "d20_m2", "d80_m1", "d360_m1"])
def test_sobol(oracle, golden, tag):
    g = golden("sobol")
    dim, m = _tag(tag)
    key = oracle.derive_key(SEED, FAM["sobol"], m)
    gen_v, shift = oracle.sobol_scramble(g["table421_v"][:dim], key, m)
    assert np.array_equal(gen_v, g[f"{tag}_gen_v"])
    assert np.array_equal(shift, g[f"{tag}_shift"])
    rows = g[f"{tag}_rows"]
    gray = oracle.sobol_counter_words(gen_v, shift, rows ^ (rows >> 1)) * 2.0**-32
    assert np.array_equal(gray, g[f"{tag}_gray"])
    cnt = oracle.sobol_counter_words(gen_v, shift, rows) * 2.0**-32
    assert np.array_equal(cnt, g[f"{tag}_counter"])


def test_inv_normal(oracle, golden):
    g = golden("inv_normal")
    assert np.array_equal(oracle.inv_normal(g["u"]), g["x"])


@pytest.mark.parametrize("tag", ["s10", "s20", "s80"])
def test_libor_payoffs(oracle, golden, tag):
    g = golden("models")
    mat, acc, K, sig, fr = g[f"libor_{tag}_params"]
    p = oracle.libor_payoffs(g[f"libor_{tag}_u"], g[f"libor_{tag}_l0"], acc, sig, K,
                             1.0 / (1.0 + acc * fr))
    assert np.array_equal(p, g[f"libor_{tag}_payoffs"])


def test_mbs_payoffs(oracle, golden):
    g = golden("models")
    k0, sx = g["mbs_k0_sigxi"]
    p = oracle.mbs_payoffs(g["mbs_u"], 0.007, k0, 0.01, -0.005, 10.0, 0.5, sx, 1.0, g["mbs_ck"])
    assert np.array_equal(p, g["mbs_payoffs"])


@pytest.mark.parametrize("n", list(range(1, 300)) + [1000, 4097, 10_000, 65_537, 1_000_000])
def test_pairwise_sum_matches_numpy(oracle, n):
    rng = np.random.default_rng(n)
    a = rng.random(n) * np.exp(rng.normal(size=n) * 4)
    assert oracle.pairwise_sum(a) == np.sum(a)


def _golden_models(golden):
    from types import SimpleNamespace as NS

    g = golden("models")

    def libor(tag):
        mat, acc, K, sig, fr = g[f"libor_{tag}_params"]
        return NS(name="libor", dim=len(g[f"libor_{tag}_l0"]),
                  config=NS(accrual=acc, sigma=sig, strike=K), front_rate=fr,
                  initial_rates=g[f"libor_{tag}_l0"])

    k0, sx = g["mbs_k0_sigxi"]
    mbs = NS(name="mbs", dim=360, config=NS(initial_rate=0.007, k0=k0, k1=0.01, k2=-0.005,
                                            k3=10.0, k4=0.5, sigma_xi=sx, payment=1.0,
                                            annuity_ratios=lambda: g["mbs_ck"]))
    return {"s20": libor("s20"), "s80": libor("s80"), "mbs": mbs,
            "x1": NS(name="x1", dim=2), "const1": NS(name="const1", dim=2)}


THETA_RUNS = {
    "c1_rasrap_recursive": ("rasrap-recursive", "s20"),
    "c1_rasrap_counter": ("rasrap-counter", "s20"),
    "libor20_prefix_rasrap": ("rasrap-recursive", "s20"),
    "libor20_philox": ("philox", "s20"),
    "libor20_sobol_gray": ("sobol-gray", "s20"),
    "libor20_sobol_counter": ("sobol-counter", "s20"),
    "libor80_rasrap": ("rasrap-recursive", "s80"),
    "libor80_philox": ("philox", "s80"),
    "mbs_rasrap": ("rasrap-recursive", "mbs"),
    "mbs_philox": ("philox", "mbs"),
    "mbs_sobol_gray": ("sobol-gray", "mbs"),
    "x1_rasrap": ("rasrap-recursive", "x1"),
    "x1_philox": ("philox", "x1"),
    "x1_sobol_gray": ("sobol-gray", "x1"),
    "const1_rasrap": ("rasrap-recursive", "const1"),
}


@pytest.mark.parametrize("tag", sorted(THETA_RUNS))
def test_replication_estimates_bit_exact(oracle, golden, tag):
    gen, mk = THETA_RUNS[tag]
    model = _golden_models(golden)[mk]
    t = golden("theta")
    theta = t[f"{tag}_theta"]  # [grid, M]
    sob = golden("sobol")["table421_v"][: model.dim]
    mine = oracle.run_replications(gen, model, SEED, 1, theta.shape[1], t[f"{tag}_grid"],
                                   threads=4, sobol_v=sob)
    assert np.array_equal(mine.T, theta)
    # thread-count invariance (test_harness.py:127-132)
    one = oracle.run_replications(gen, model, SEED, 1, theta.shape[1], t[f"{tag}_grid"],
                                  threads=1, sobol_v=sob)
    assert np.array_equal(one, mine)


def test_sfc64_matches_numpy(oracle):
    """SFC64 has no reference: numpy's SFC64 with the state set is the oracle."""
    seed, m = SEED, 3
    paths = np.array([0, 1, 2, 1000, 2**31 + 5])
    mine = oracle.sfc64_uniforms(seed, m, paths, 37)
    for r, p in enumerate(paths):
        w = oracle.derive_words(oracle.derive_key(seed, 7, m, int(p)), 6).astype(np.uint64)
        bg = np.random.SFC64()
        st = bg.state
        st["state"]["state"] = np.array([w[0] | (w[1] << np.uint64(32)),
                                         w[2] | (w[3] << np.uint64(32)),
                                         w[4] | (w[5] << np.uint64(32)), 1], dtype=np.uint64)
        st["has_uint32"] = 0
        bg.state = st
        bg.random_raw(12)
        expect = np.random.Generator(bg).random(37)
        assert np.array_equal(mine[r], expect)


# ---------------------------------------------------------------- MT19937 / XORWOW
def test_mt19937_words(oracle, golden):
    g = golden("prng_seq")
    for s, w in zip(g["mt_seeds"], g["mt_words"]):
        assert np.array_equal(oracle.mt19937(int(s)).words(len(w)), w)


def test_mt19937_kat(oracle):
    # test_prng.py:43-53: 10000th output of the classic 5489 seeding
    assert oracle.mt19937(5489).words(10000)[-1] == 4123659995
    # numpy's legacy RandomState seeding is the same init_genrand recursion
    rs = np.random.RandomState(20120224)
    assert np.array_equal(oracle.mt19937(20120224).words(2000),
                          rs.randint(0, 2**32, size=2000, dtype=np.uint64).astype(np.uint32))


def test_xorwow_words(oracle, golden):
    g = golden("prng_seq")
    for s, w in zip(g["xw_seeds"], g["xw_words"]):
        assert np.array_equal(oracle.xorwow(int(s)).words(len(w)), w)


def test_xorwow_matches_independent_recurrence(oracle):
    # test_prng.py:28-39 style: Marsaglia's recurrence written out in Python ints
    st = [int(x) for x in oracle.derive_words(987654321, 6)]
    x, y, z, w, v, d = st
    ref = []
    for _ in range(500):
        t = (x ^ (x >> 2)) & 0xFFFFFFFF
        x, y, z, w = y, z, w, v
        v = (v ^ ((v << 4) & 0xFFFFFFFF)) ^ (t ^ ((t << 1) & 0xFFFFFFFF))
        d = (d + 362437) & 0xFFFFFFFF
        ref.append((d + v) & 0xFFFFFFFF)
    assert list(oracle.xorwow(987654321).words(500)) == ref


THETA_SEQ_RUNS = {
    "libor20_twister": ("twister", "s20"),
    "libor20_xorwow": ("xorwow", "s20"),
    "libor80_twister": ("twister", "s80"),
    "libor80_xorwow": ("xorwow", "s80"),
    "mbs_twister": ("twister", "mbs"),
    "mbs_xorwow": ("xorwow", "mbs"),
    "x1_twister": ("twister", "x1"),
    "x1_xorwow": ("xorwow", "x1"),
}


@pytest.mark.parametrize("tag", sorted(THETA_SEQ_RUNS))
def test_sequential_prng_estimates_bit_exact(oracle, golden, tag):
    gen, mk = THETA_SEQ_RUNS[tag]
    model = _golden_models(golden)[mk]
    t = golden("theta_seq")
    theta = t[f"{tag}_theta"]
    mine = oracle.run_replications(gen, model, SEED, 1, theta.shape[1], t[f"{tag}_grid"],
                                   threads=4)
    assert np.array_equal(mine.T, theta)


# ---------------------------------------------------------------- Kakutani
def test_kakutani_points_bit_exact(oracle, golden):
    g = golden("kakutani")
    for tag in ("d20_m1", "d5_m2", "d360_m1"):
        dim, m = int(tag[1:].split("_m")[0]), int(tag.split("_m")[1])
        rows = g[f"{tag}_rows"]
        key = oracle.derive_key(SEED, 6, m)
        pts = oracle.kakutani_points(dim, key, int(rows[-1]) + 1)
        assert np.array_equal(pts[rows], g[f"{tag}_points"]), tag


def test_kakutani_estimates_bit_exact(oracle, golden):
    g = golden("kakutani")
    models = _golden_models(golden)
    for tag, mk in (("libor20", "s20"), ("mbs", "mbs"), ("x1", "x1")):
        theta = g[f"{tag}_theta"]
        mine = oracle.run_replications("kakutani", models[mk], SEED, 1, theta.shape[1],
                                       g[f"{tag}_grid"], threads=4)
        assert np.array_equal(mine.T, theta), tag


def test_xhash_model_definitions_agree(oracle):
    """The package's host definition of the coordinate hash == the oracle's."""
    from paper_1408_5526_b200 import models as M

    u = np.random.default_rng(3).random((257, 37))
    h = M.CoordinateHashModel(37).payoffs(u)
    assert np.array_equal(h, oracle.coord_hash(u))
    assert h.min() >= 0 and h.max() < 2**20 and len(np.unique(h)) > 250

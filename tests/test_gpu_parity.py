"""Device parity: the sm_100a path through the C ABI vs the reference.

Bars (BASELINE north_star):
  * point streams (Rasrap both forms, Philox, Sobol' both forms, SFC64) and
    the on-device randomisation: BIT-EXACT against the golden fixtures
    written from the reference (tests/golden/) and against the oracle;
  * inverse normal: |x_gpu - x_ref| <= 2e-13 * max(1, |x|): FMA Horner and
    a Newton reciprocal instead of the reference's two-rounding Horner and
    IEEE division; the rational's condition number (~100) amplifies the
    per-operation ulp differences;
  * per-path payoffs and per-replication estimates theta_N^m: relative
    error <= 1e-12 (PAYOFF_RTOL / THETA_RTOL below); theta of the test
    integrands x1 / const1 (no transcendental) BIT-EXACT, which pins the
    numpy pairwise reduction order;
  * grand averages within one standard error.
"""
import numpy as np
import pytest

from conftest import SEED

pytestmark = pytest.mark.gpu

THETA_RTOL = 1e-12
PAYOFF_RTOL = 1e-12
INVN_TOL = 2e-13  # FMA Horner vs the reference two-rounding Horner (cond ~ 100)


@pytest.fixture(scope="module")
def P():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1408_5526_b200 as pkg
    from paper_1408_5526_b200 import _lib

    _lib.lib()
    return pkg


def _tag(tag):
    dim, m = tag[1:].split("_m")
    return int(dim), int(m)


RASRAP_CASES = ["d20_m1", "d20_m2", "d80_m1", "d80_m3", "d360_m1", "d360_m2"]


@pytest.mark.parametrize("tag", RASRAP_CASES)
@pytest.mark.parametrize("form", ["recursive", "counter"])
def test_rasrap_points_bit_exact(P, golden, tag, form):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("rasrap")
    dim, m = _tag(tag)
    s = DeviceSampler(f"rasrap-{form}", dim, SEED, m)
    rows = g[f"{tag}_rows"]
    got = s.points_at(rows).cpu().numpy()
    assert np.array_equal(got, g[f"{tag}_{form}"])
    if form == "counter":  # indices up to 3 * 2^33 + 5 (RasrapCounter.at on int64)
        big = g[f"{tag}_bigidx"]
        assert big.max() > 2**34
        assert np.array_equal(s.points_at(big).cpu().numpy(), g[f"{tag}_counter_big"])


@pytest.mark.parametrize("tag", ["d20_m1", "d80_m3", "d360_m2"])
def test_rasrap_fill_sequence(P, golden, tag):
    """fill() in chunks reproduces the reference stream rows 0..n-1."""
    g = golden("rasrap")
    dim, m = _tag(tag)
    s = P.make_sampler("rasrap-recursive", dim, SEED, m)
    out = np.empty((512, dim))
    s.fill(out[:100])
    s.fill(out[100:])
    rows = g[f"{tag}_rows"]
    assert np.array_equal(out, g[f"{tag}_recursive"][:512])
    assert rows[511] == 511


@pytest.mark.parametrize("tag", ["d20_m1", "d80_m1", "d360_m1"])
def test_rasrap_device_tables_match_oracle(P, oracle, tag):
    from paper_1408_5526_b200.samplers import DeviceSampler
    from paper_1408_5526_b200.tables import halton_layout

    dim, m = _tag(tag)
    s = DeviceSampler("rasrap-recursive", dim, SEED, m)
    dig, sig, sums = s.rasrap_tables()
    key = oracle.derive_key(SEED, 4, m)
    start, _, sigma = oracle.rasrap_config(dim, key)
    lay = halton_layout(dim)
    so = do = 0
    for d in range(dim):
        p, cap = int(lay["base"][d]), int(lay["cap"][d])
        assert np.array_equal(sig[so:so + p], sigma[d, :p])
        n0 = sum(int(a) * p**j for j, a in enumerate(dig[do:do + cap]))
        assert n0 == start[d]
        so += p
        do += cap


@pytest.mark.parametrize("tag", ["d20_m1", "d20_m2", "d80_m1", "d360_m1"])
def test_philox_points_bit_exact(P, golden, tag):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("philox")
    dim, m = _tag(tag)
    s = DeviceSampler("philox", dim, SEED, m)
    u = s.points_at(g[f"{tag}_rows"]).cpu().numpy()
    assert np.array_equal(u, g[f"{tag}_words"] * 2.0**-32 + 2.0**-33)
    out = np.empty((300, dim))
    s.fill(out[:100])
    s.fill(out[100:])
    assert np.array_equal(out, g[f"{tag}_fill300"])


@pytest.mark.parametrize("tag", ["d20_m1", "d20_m2", "d80_m1", "d360_m1"])
def test_sobol_points_bit_exact(P, golden, tag):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("sobol")
    dim, m = _tag(tag)
    rows = g[f"{tag}_rows"]
    gray = DeviceSampler("sobol-gray", dim, SEED, m).points_at(rows).cpu().numpy()
    assert np.array_equal(gray, g[f"{tag}_gray"])
    cnt = DeviceSampler("sobol-counter", dim, SEED, m).points_at(rows).cpu().numpy()
    assert np.array_equal(cnt, g[f"{tag}_counter"])


def test_sfc64_points_match_oracle(P, oracle):
    from paper_1408_5526_b200.samplers import DeviceSampler

    paths = np.array([0, 1, 2, 127, 128, 99_999, 2**31 + 5, 2**32 - 1])
    for dim, m in ((20, 1), (360, 7)):
        got = DeviceSampler("sfc64", dim, SEED, m).points_at(paths).cpu().numpy()
        assert np.array_equal(got, oracle.sfc64_uniforms(SEED, m, paths, dim))


@pytest.mark.parametrize("gen", ["rasrap-recursive", "rasrap-counter", "philox", "sobol-gray"])
def test_large_index_blocks_match_oracle(P, oracle, gen):
    """Points deep in the stream (N = 2^20 region and near 2^32) vs the oracle."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    dim, m = 20, 5
    idx = np.concatenate([np.arange(2**20 - 300, 2**20 + 300),
                          np.arange(2**32 - 200, 2**32)]).astype(np.int64)
    got = DeviceSampler(gen, dim, SEED, m).points_at(idx).cpu().numpy()
    if gen.startswith("rasrap"):
        key = oracle.derive_key(SEED, 4, m)
        if gen == "rasrap-counter":
            ref = oracle.rasrap_counter(dim, key, idx)
            assert np.array_equal(got, ref)
        else:  # recursive form == counter form to 1e-12 (test_halton.py:161-175)
            ref = oracle.rasrap_counter(dim, key, idx)
            assert np.abs(got - ref).max() <= 1e-12
            head = oracle.rasrap_recursive(dim, key, 2**20 + 300)
            assert np.array_equal(got[:600], head[2**20 - 300:])
    elif gen == "philox":
        key = oracle.derive_key(SEED, 3, m)
        ref = oracle.philox_words(key, idx, dim) * 2.0**-32 + 2.0**-33
        assert np.array_equal(got, ref)
    else:
        from paper_1408_5526_b200.tables import sobol_directions

        key = oracle.derive_key(SEED, 5, m)
        gv, sh = oracle.sobol_scramble(sobol_directions(dim), key, m)
        ref = oracle.sobol_counter_words(gv, sh, idx ^ (idx >> 1)) * 2.0**-32
        assert np.array_equal(got, ref)


def test_index_range_per_generator(P):
    """Sobol' stops at 2^32 (32-bit direction numbers; sobol.py:181-193
    raises), the counter PRNGs and Rasrap take 64-bit indices."""
    from paper_1408_5526_b200 import _lib

    lim = {g: int(_lib.lib().rq_index_limit(i)) for g, i in _lib.GEN_IDS.items()}
    assert lim["sobol-gray"] == lim["sobol-counter"] == 2**32
    assert lim["philox"] == lim["sfc64"] == 2**62
    assert lim["rasrap-recursive"] == lim["rasrap-counter"] == 2**39
    s = P.make_sampler("sobol-gray", 4, SEED, 1)
    with pytest.raises(ValueError):
        s.points(2**32 - 2, 5)
    with pytest.raises(ValueError):
        P.make_sampler("rasrap-counter", 4, SEED, 1).at(np.array([2**39]))
    assert P.make_sampler("philox", 4, SEED, 1).points(2**32 - 2, 5).shape == (5, 4)


@pytest.mark.parametrize("gen", ["philox", "sfc64", "rasrap-counter", "rasrap-recursive"])
def test_64bit_indices_match_oracle(P, oracle, gen):
    """Points at indices beyond 2^32 (the reference takes int64 indices:
    halton.py:506-512, prng.py:180-246) vs the oracle, through at() (direct
    kernels) and fill() (tile kernels) across the 2^32 boundary."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    dim, m = 20, 3
    s = DeviceSampler(gen, dim, SEED, m)
    hi = 2**61 if gen in ("philox", "sfc64") else 2**39
    idx = np.concatenate([np.arange(2**32 - 70, 2**32 + 70), np.arange(2**36 - 5, 2**36 + 5),
                          np.arange(hi - 40, hi)]).astype(np.int64)
    got = s.points_at(idx).cpu().numpy()
    run = s.points(2**32 - 300, 600).cpu().numpy()  # fill across the 2^32 boundary
    ridx = np.arange(2**32 - 300, 2**32 + 300, dtype=np.int64)
    if gen == "philox":
        key = oracle.derive_key(SEED, 3, m)
        words = lambda ix: oracle.philox_words(key, ix, dim) * 2.0**-32 + 2.0**-33  # noqa: E731
        assert np.array_equal(got, words(idx))
        assert np.array_equal(run, words(ridx))
    elif gen == "sfc64":
        assert np.array_equal(got, oracle.sfc64_uniforms(SEED, m, idx, dim))
        assert np.array_equal(run, oracle.sfc64_uniforms(SEED, m, ridx, dim))
    else:
        key = oracle.derive_key(SEED, 4, m)
        ref, rref = oracle.rasrap_counter(dim, key, idx), oracle.rasrap_counter(dim, key, ridx)
        if gen == "rasrap-counter":
            assert np.array_equal(got, ref) and np.array_equal(run, rref)
        else:
            # recursive form: fill (digit tree) == direct chain bit for bit,
            # both within 1e-12 of the counter form (test_halton.py:161-175)
            assert np.array_equal(run, s.points_at(ridx).cpu().numpy())
            assert np.abs(got - ref).max() <= 1e-12 and np.abs(run - rref).max() <= 1e-12


def test_inv_normal(P, golden):
    from paper_1408_5526_b200.models import inv_normal

    g = golden("inv_normal")
    x = inv_normal(g["u"])
    err = np.abs(x - g["x"]) / np.maximum(1.0, np.abs(g["x"]))
    assert err.max() <= INVN_TOL
    assert np.all(np.isfinite(x))
    assert inv_normal(0.5) == 0.0


@pytest.mark.parametrize("tag,mat", [("s10", None), ("s20", 5.0), ("s80", 20.0)])
def test_libor_payoffs(P, golden, tag, mat):
    from paper_1408_5526_b200 import models as M

    g = golden("models")
    model = M.LiborModel() if mat is None else M.LiborModel(M.LiborConfig(maturity=mat, accrual=0.25))
    assert np.array_equal(model.initial_rates, g[f"libor_{tag}_l0"])
    got = model.payoffs(g[f"libor_{tag}_u"])
    ref = g[f"libor_{tag}_payoffs"]
    scale = np.maximum(np.abs(ref), np.abs(ref).max() * 1e-3)
    assert (np.abs(got - ref) / scale).max() <= PAYOFF_RTOL


def test_mbs_payoffs(P, golden):
    from paper_1408_5526_b200 import models as M

    g = golden("models")
    model = M.MbsModel()
    assert np.array_equal(model.annuity, g["mbs_ck"])
    got = model.payoffs(g["mbs_u"])
    assert (np.abs(got / g["mbs_payoffs"] - 1)).max() <= PAYOFF_RTOL


THETA = {
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


def _model(kind):
    from paper_1408_5526_b200 import models as M

    return {"s20": lambda: M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)),
            "s80": lambda: M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25)),
            "mbs": M.MbsModel, "x1": M.FirstCoordinateModel, "const1": M.ConstantModel}[kind]()


@pytest.mark.parametrize("tag", sorted(THETA))
def test_theta_vs_reference(P, golden, tag):
    gen, mk = THETA[tag]
    t = golden("theta")
    grid = tuple(int(n) for n in t[f"{tag}_grid"])
    ref = t[f"{tag}_theta"]  # [grid, M]
    M_ = ref.shape[1]
    cfg = P.ExperimentConfig(model=_model(mk).name, generator=gen, n_grid=grid, replications=M_,
                             seed=SEED)
    rep = P.run_experiment(cfg, model=_model(mk))
    got = np.stack([rep.estimates(gen, n) for n in grid])
    if mk in ("x1", "const1"):
        assert np.array_equal(got, ref)
    else:
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL
    for gi, n in enumerate(grid):
        row = rep.row(gen, n)
        se = t[f"{tag}_std"][gi] / np.sqrt(M_)
        assert abs(row.mean - t[f"{tag}_mean"][gi]) <= max(se, 1e-15 * abs(row.mean))


def test_theta_invariant_to_sharding(P):
    """Replication ranges [1..8] == [1..3] + [4..8] (GPU-count invariance)."""
    from paper_1408_5526_b200.harness import estimate_replications

    model = _model("s20")
    grid = (1000, 5000)
    full = estimate_replications("rasrap-recursive", model, SEED, 1, 8, grid)
    a = estimate_replications("rasrap-recursive", model, SEED, 1, 3, grid)
    b = estimate_replications("rasrap-recursive", model, SEED, 4, 5, grid)
    assert np.array_equal(full, np.concatenate([a, b]))


def test_theta_matches_oracle_c1_full(P, oracle):
    """Config 1 exactly (M=16, N=10^4) and a 2^17 run, GPU vs oracle."""
    from paper_1408_5526_b200.harness import estimate_replications

    model = _model("s20")
    for gen, grid, M_ in (("rasrap-recursive", (10_000,), 16), ("philox", (2**17,), 4),
                          ("sobol-gray", (2**17,), 4)):
        got = estimate_replications(gen, model, SEED, 1, M_, grid)
        sob = None
        if gen.startswith("sobol"):
            from paper_1408_5526_b200.tables import sobol_directions

            sob = sobol_directions(20)
        ref = oracle.run_replications(gen, model, SEED, 1, M_, grid, threads=8, sobol_v=sob)
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


def test_x1_theta_bit_exact_large(P, oracle):
    """f = x_1 at N = 10^6 and 2^20: isolates generator + reduction, bit-exact."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.FirstCoordinateModel()
    grid = (999_983, 2**20)
    from paper_1408_5526_b200.tables import sobol_directions

    sob = sobol_directions(model.dim)
    for gen in ("rasrap-recursive", "philox", "sobol-gray", "sobol-counter"):
        got = estimate_replications(gen, model, SEED, 1, 3, grid)
        ref = oracle.run_replications(gen, model, SEED, 1, 3, grid, threads=3,
                                      sobol_v=sob if gen.startswith("sobol") else None)
        assert np.array_equal(got, ref), gen


@pytest.mark.parametrize("n", [1, 7, 8, 127, 128, 129, 1000, 10_000, 2**20, 10**6 + 3])
def test_pairwise_sum_bit_exact(P, n):
    import torch
    from paper_1408_5526_b200 import _lib

    rng = np.random.default_rng(n)
    a = rng.random(n) * np.exp(rng.normal(size=n) * 3)
    t = torch.from_numpy(a).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().rq_pairwise_sum(t.data_ptr(), n, out.data_ptr(), _lib.stream_ptr()))
    assert float(out.item()) == np.sum(a)


@pytest.mark.parametrize("gen", ["philox", "rasrap-recursive", "sfc64", "sobol-gray", "sobol-counter"])
@pytest.mark.parametrize("dim,npts,keep", [(360, 3000, True), (360, 3001, False),
                                           (7, 1000, True), (7, 999, False), (1, 77, False),
                                           (361, 700, True), (40, 20000, False)])
def test_stream_normals_sum(P, oracle, gen, dim, npts, keep):
    """Config-4 stream kernel: sum of fused normals vs oracle (small sample),
    with and without the stored normals, ragged dims and point counts."""
    import torch
    from paper_1408_5526_b200 import _lib
    from paper_1408_5526_b200.samplers import DeviceSampler

    s = DeviceSampler(gen, dim, SEED, 0)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    store = torch.empty((npts, dim), dtype=torch.float64, device="cuda") if keep else None
    _lib.check(_lib.lib().rq_stream_normals(s._h, 0, npts, out.data_ptr(),
                                             store.data_ptr() if keep else None,
                                             _lib.stream_ptr()))
    u = s.points(0, npts).cpu().numpy()
    z = oracle.inv_normal(u)
    if keep:
        st = store.cpu().numpy()
        assert np.abs(st - z).max() <= INVN_TOL * max(1.0, np.abs(z).max())
    assert abs(float(out.item()) - z.sum()) <= 1e-9


def test_errors_map_to_reference_exceptions(P):
    with pytest.raises(P.ConfigurationError):
        P.make_sampler("nope", 2, 0, 1)
    with pytest.raises(P.ConfigurationError):
        P.ExperimentConfig(model="libor", generator="philox", n_grid=(10, 5))
    from paper_1408_5526_b200 import models as M

    with pytest.raises(ValueError):
        M.LiborModel().payoffs(np.zeros((3, 4)))


# ---------------------------------------------------------------- edge cases vs the oracle
def _oracle_theta(oracle, gen, model, seed, first, count, grid):
    sob = None
    if gen.startswith("sobol"):
        from paper_1408_5526_b200.tables import sobol_directions

        sob = sobol_directions(model.dim)
    return oracle.run_replications(gen, model, seed, first, count, grid, threads=8, sobol_v=sob)


@pytest.mark.parametrize("gen", ["rasrap-recursive", "rasrap-counter", "philox", "sobol-gray",
                                 "sobol-counter", "sfc64"])
def test_ragged_grids_and_big_ids(P, oracle, gen):
    """N not a multiple of the 128-path tile, N = 1, several grid points,
    replication ids far from 1, a 64-bit seed: theta vs the oracle."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    grid = (1, 2, 7, 127, 129, 1000, 4099)
    for seed, first in ((SEED, 1), (2**63 + 12345, 1_000_003)):
        got = estimate_replications(gen, model, seed, first, 3, grid)
        ref = _oracle_theta(oracle, gen, model, seed, first, 3, grid)
        scale = np.maximum(np.abs(ref), 1e-3 * np.abs(ref).max())
        assert (np.abs(got - ref) / scale).max() <= THETA_RTOL, (seed, first)


@pytest.mark.parametrize("mat,acc", [(5.0, 0.5), (10.0, 0.25), (20.0, 0.25)])
def test_libor_steps_vs_oracle(P, oracle, mat, acc):
    """All compiled LIBOR widths (S = 10, 40, 80) through the fused kernel."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.LiborModel(M.LiborConfig(maturity=mat, accrual=acc))
    for gen in ("rasrap-recursive", "philox", "sobol-gray", "sobol-counter"):
        got = estimate_replications(gen, model, SEED, 5, 2, (3000,))
        ref = _oracle_theta(oracle, gen, model, SEED, 5, 2, (3000,))
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


@pytest.mark.parametrize("mat,acc", [(0.25, 0.25), (3.0, 0.25), (7.5, 0.25), (15.0, 0.5),
                                     (20.0, 0.125)])
def test_libor_any_steps_vs_oracle(P, oracle, mat, acc):
    """Step counts without a register kernel (S = 1, 12, 30, 30, 160): the
    shared-memory LIBOR model, fused paths and model.payoffs(u)."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.LiborModel(M.LiborConfig(maturity=mat, accrual=acc))
    for gen in ("rasrap-recursive", "philox", "xorwow", "kakutani", "sobol-gray", "sobol-counter"):
        got = estimate_replications(gen, model, SEED, 3, 2, (2000,))
        ref = _oracle_theta(oracle, gen, model, SEED, 3, 2, (2000,))
        # (S = 1: the caplet is out of the money on every path, theta == 0)
        assert (np.abs(got - ref) <= THETA_RTOL * np.abs(ref)).all(), gen
    u = np.random.default_rng(5).random((700, model.dim))
    mid, dim, par = oracle.model_params(model)
    ref = oracle.libor_payoffs(u, par[4:], par[0], par[1], par[2], par[3])
    got = model.payoffs(u)
    # per path the caplet's (L - K)^+ cancels near the money (an ulp of L is
    # ~1e-12 of a small payoff); theta above holds the 1e-12 bar
    scale = np.maximum(np.abs(ref), np.abs(ref).max() * 1e-3)
    assert (np.abs(got - ref) <= 10 * PAYOFF_RTOL * scale).all()


@pytest.mark.parametrize("sigma,mat,acc", [(0.0, 5.0, 0.25), (1e-160, 5.0, 0.25), (0.5, 5.0, 0.25),
                                           (0.04, 3.0, 0.3), (0.2, 20.0, 0.25)])
def test_libor_volatility_edges_vs_oracle(P, oracle, sigma, mat, acc):
    """The kernels hold the rates as z = sigma^2 delta * delta L (the drift
    weight folded in, scale clamped at 2^-900): sigma = 0 and tiny sigma
    (no drift), a large sigma, a non-dyadic accrual (delta L rounded)."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.LiborModel(M.LiborConfig(maturity=mat, accrual=acc, sigma=sigma))
    for gen in ("rasrap-recursive", "philox"):
        got = estimate_replications(gen, model, SEED, 3, 2, (2000,))
        ref = _oracle_theta(oracle, gen, model, SEED, 3, 2, (2000,))
        assert (np.abs(got - ref) <= THETA_RTOL * np.abs(ref)).all(), gen


@pytest.mark.parametrize("cfg", [dict(months=24), dict(months=360, variance=0.0),
                                 dict(months=100, variance=0.0009, initial_rate=0.01)])
def test_mbs_variants_vs_oracle(P, oracle, cfg):
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.MbsModel(M.MbsConfig(**cfg))
    for gen in ("rasrap-recursive", "sobol-gray"):
        got = estimate_replications(gen, model, SEED, 1, 2, (777,))
        ref = _oracle_theta(oracle, gen, model, SEED, 1, 2, (777,))
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


def test_x1_dim1_and_const_bit_exact(P, oracle):
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    for gen in ("rasrap-recursive", "sobol-gray", "philox", "sfc64", "rasrap-counter"):
        m = M.FirstCoordinateModel(dim=1)
        got = estimate_replications(gen, m, SEED, 1, 4, (5, 128, 131, 70_001))
        ref = _oracle_theta(oracle, gen, m, SEED, 1, 4, (5, 128, 131, 70_001))
        assert np.array_equal(got, ref), gen
    c = estimate_replications("philox", M.ConstantModel(), SEED, 1, 3, (9, 1000))
    assert np.all(c == 1.0)


def test_many_replications_batched(P, oracle):
    """More replications than one payoff batch / sampler group: theta of a
    500-replication run equals per-replication oracle values."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    m = M.FirstCoordinateModel()
    got = estimate_replications("rasrap-recursive", m, SEED, 1, 500, (300_000,))
    idx = [0, 1, 137, 255, 256, 499]
    for i in idx:
        ref = _oracle_theta(oracle, "rasrap-recursive", m, SEED, 1 + i, 1, (300_000,))
        assert got[i, 0] == ref[0, 0]


def test_rasrap_counter_tiles_bit_exact(P, oracle):
    """The tiled counter form (low digits per point + shared high terms) at
    large and ragged N, and through indices above 2^32 - n0: f = x1 theta is
    bit-exact against the oracle's per-point counter sums."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    x1 = M.FirstCoordinateModel()
    grid = (999_983, 2**20 + 77)
    got = estimate_replications("rasrap-counter", x1, SEED, 7, 3, grid)
    ref = oracle.run_replications("rasrap-counter", x1, SEED, 7, 3, grid, threads=3)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("dim", [1, 20, 37, 360])
def test_rasrap_counter_fill_tiles_vs_oracle(P, oracle, dim):
    """sampler.fill of the counter form (tiled: shared high terms per tile)
    from unaligned starts, up to indices near 2^32, == the oracle's counter sums."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    key = oracle.derive_key(SEED, 4, 3)
    s = DeviceSampler("rasrap-counter", dim, SEED, 3)
    for first, count in ((0, 777), (12_345, 1000), (2**32 - 1500, 1500)):
        got = s.points(first, count).cpu().numpy()
        ref = oracle.rasrap_counter(dim, key, np.arange(first, first + count, dtype=np.int64))
        assert np.array_equal(got, ref), (dim, first)


def test_inv_normal_tail_edges(P, oracle):
    """The tail's own log (pl = m 2^e, atanh series) over every binade of
    [2^-53, 0.0465] and at the clamp, against the reference formula."""
    from paper_1408_5526_b200.models import inv_normal

    e = np.arange(-53, -4)
    u = np.concatenate([2.0 ** e, np.nextafter(2.0 ** e, 1), 2.0 ** e * 1.4142135,
                        2.0 ** e * 1.41421357, 2.0 ** e * 1.9999999, [0.0465, 0.04649999999],
                        1.0 - 2.0 ** e[e > -53], [np.nan, -1.0, 2.0]])
    u = u[(u < 0.0465) | (u > 0.95) | ~np.isfinite(u) | (u < 0) | (u > 1)]
    got = inv_normal(u)
    ref = oracle.inv_normal(u)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    err = np.abs(got[fin] - ref[fin]) / np.maximum(1.0, np.abs(ref[fin]))
    assert err.max() <= INVN_TOL

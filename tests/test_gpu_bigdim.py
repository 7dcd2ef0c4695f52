"""Dimensions beyond the constant-bank tables and LIBOR beyond 160 steps.

The reference takes any number of primes (halton.py:40-56) and any number of
accrual periods (models.py:172-193).  The device covers Rasrap and Kakutani
up to the 6542nd prime (every base below 2^16: digits and sigma entries are
uint16) -- dims >= 512 read their constants from global memory instead of
the constant bank -- and LIBOR up to 6542 steps (rates in shared memory up to
160 steps, in a per-CTA slice of global memory beyond).  Pinned against
tests/golden/bigdim.npz, written by the unmodified reference
(make_golden.py --only bigdim): points bit-exact, theta within 1e-12.
"""
import numpy as np
import pytest

from conftest import SEED

pytestmark = pytest.mark.gpu

THETA_RTOL = 1e-12


@pytest.fixture(scope="module")
def P():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1408_5526_b200 as pkg
    from paper_1408_5526_b200 import _lib

    _lib.lib()
    return pkg


@pytest.fixture(scope="module")
def G(golden):
    return golden("bigdim")


@pytest.mark.parametrize("dim,m", [(6542, 1), (1000, 2)])
def test_rasrap_wide_points_bit_exact(P, G, dim, m):
    from paper_1408_5526_b200.samplers import DeviceSampler

    tag = f"rasrap_d{dim}_m{m}"
    cols = G[f"{tag}_cols"]
    assert cols.max() == dim - 1 and (cols >= 512).any()
    s = DeviceSampler("rasrap-recursive", dim, SEED, m)
    rec = s.points(0, 300).cpu().numpy()
    assert np.array_equal(rec[:, cols], G[f"{tag}_recursive"])
    s.close()
    c = DeviceSampler("rasrap-counter", dim, SEED, m)
    idx = G[f"{tag}_idx"]
    assert np.array_equal(c.points_at(idx).cpu().numpy()[:, cols], G[f"{tag}_counter"])
    c.close()


def test_rasrap_dimension_limit(P):
    from paper_1408_5526_b200.samplers import DeviceSampler

    with pytest.raises(ValueError):
        DeviceSampler("rasrap-recursive", 6543, SEED, 1)


def test_kakutani_wide_points_bit_exact(P, G):
    from paper_1408_5526_b200.samplers import DeviceSampler

    tag = "kakutani_d700_m1"
    rows, cols = G[f"{tag}_rows"], G[f"{tag}_cols"]
    s = DeviceSampler("kakutani", 700, SEED, 1)
    pts = s.points(0, int(rows[-1]) + 1).cpu().numpy()
    assert np.array_equal(pts[rows][:, cols], G[f"{tag}_points"])
    k = rows.size // 2  # a far row alone (segment snapshot mid-stream)
    assert np.array_equal(s.points(int(rows[k]), 1).cpu().numpy()[0][cols], G[f"{tag}_points"][k])
    s.close()


def _models(P, G):
    M = P.models
    curve = M.YieldCurve(G["long_curve"][0], G["long_curve"][1])
    return {
        "libor200": M.LiborModel(M.LiborConfig(maturity=25.0, accrual=0.125)),
        "libor600": M.LiborModel(M.LiborConfig(maturity=150.0, accrual=0.25), curve=curve),
        "mbs600": M.MbsModel(M.MbsConfig(months=600)),
    }


BIG_THETA = {
    "libor200_rasrap": ("rasrap-recursive", "libor200"),
    "libor200_philox": ("philox", "libor200"),
    "libor600_rasrap": ("rasrap-recursive", "libor600"),
    "libor600_counter": ("rasrap-counter", "libor600"),
    "mbs600_rasrap": ("rasrap-recursive", "mbs600"),
    "libor200_kakutani": ("kakutani", "libor200"),
}


@pytest.mark.parametrize("tag", sorted(BIG_THETA))
def test_big_theta_vs_reference(P, G, tag):
    gen, mk = BIG_THETA[tag]
    model = _models(P, G)[mk]
    assert model.dim in (200, 600)
    grid = tuple(int(n) for n in G[f"{tag}_grid"])
    ref = G[f"{tag}_theta"]
    cfg = P.ExperimentConfig(model=model.name, generator=gen, n_grid=grid,
                             replications=ref.shape[1], seed=SEED)
    rep = P.run_experiment(cfg, model=model)
    got = np.stack([rep.estimates(gen, n) for n in grid])
    assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


@pytest.mark.parametrize("gen", ["rasrap-recursive", "philox", "xorwow", "kakutani"])
def test_big_libor_vs_oracle(P, oracle, gen):
    """S = 239 (global-memory rates) through the fused, counter-tile and
    sequential path kernels against the C oracle."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    model = M.LiborModel(M.LiborConfig(maturity=30.0 - 0.125, accrual=0.125))
    assert model.dim == 239
    got = estimate_replications(gen, model, SEED, 1, 3, (129, 2000))
    ref = oracle.run_replications(gen, model, SEED, 1, 3, (129, 2000), threads=3)
    assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


def test_big_libor_payoffs_from_uniforms(P, oracle, G):
    """model.payoffs(u) for S = 600 (grid-stride over the state slices)."""
    model = _models(P, G)["libor600"]
    u = np.random.default_rng(7).random((3000, model.dim))
    mid, dim, par = oracle.model_params(model)
    ref = oracle.libor_payoffs(u, par[4:], par[0], par[1], par[2], par[3])
    got = model.payoffs(u)
    # per-path tolerance as test_gpu_parity.test_libor_any_steps_vs_oracle
    scale = np.maximum(np.abs(ref), np.abs(ref).max() * 1e-3)
    assert (np.abs(got - ref) <= 10 * 1e-12 * scale).all()

"""The reference's acceptance study (tests/test_acceptance.py:1-46: desk
scale N = 2^10..2^18, M = 50, seed 20120224) run on the B200 path.

The convergence slopes and the Black-consistency difference are functions of
theta, which agrees with the reference to 1e-12, so they must reproduce the
values the reference recorded in pkg/test_output.txt:12-36 (printed to three
decimals) -- including the two criteria that FAIL there by design
(README.md:40-54): MBS Sobol' slope -0.655 and Rasrap-vs-Sobol' ordering.
"""
import math

import numpy as np
import pytest

from conftest import SEED

pytestmark = pytest.mark.gpu

DESK_GRID = tuple(2**k for k in range(10, 19))
REPS = 50
# test_output.txt:12-36
RECORDED = {
    ("libor", "twister"): -0.488, ("libor", "rasrap-recursive"): -0.938,
    ("libor", "sobol-gray"): -1.010,
    ("mbs", "philox"): -0.518, ("mbs", "xorwow"): -0.521, ("mbs", "sobol-gray"): -0.655,
    ("mbs", "rasrap-recursive"): -0.885,
}


@pytest.fixture(scope="module")
def desk():
    import paper_1408_5526_b200 as P

    out = {}
    for (model, gen) in RECORDED:
        cfg = P.ExperimentConfig(model=model, generator=gen, n_grid=DESK_GRID,
                                 replications=REPS, seed=SEED, workers=2)
        out[(model, gen)] = P.run_experiment(cfg)
    return out


@pytest.mark.parametrize("key", sorted(RECORDED))
def test_slope_reproduces_reference_record(desk, key):
    s = desk[key].slopes[0].slope
    assert abs(s - RECORDED[key]) <= 0.0005 + 1e-9, (key, s)


def test_criteria_1_2_verdicts(desk):
    sl = {k: v.slopes[0].slope for k, v in desk.items()}
    assert -0.62 <= sl[("libor", "twister")] <= -0.38
    assert sl[("libor", "rasrap-recursive")] <= -0.72
    assert sl[("libor", "sobol-gray")] <= -0.78
    assert -0.62 <= sl[("mbs", "philox")] <= -0.38
    assert -0.62 <= sl[("mbs", "xorwow")] <= -0.38
    assert sl[("mbs", "rasrap-recursive")] <= -0.55
    assert not sl[("mbs", "sobol-gray")] <= -0.70  # FAILs in the reference too


def test_criterion_3_ordering_fails_as_recorded(desk):
    wins = sum(desk[("mbs", "rasrap-recursive")].row("rasrap-recursive", n).std
               < desk[("mbs", "sobol-gray")].row("sobol-gray", n).std for n in DESK_GRID)
    assert wins == 0  # "FAIL (0 of 9)", test_output.txt:33


def test_criterion_4_black_consistency(desk):
    from paper_1408_5526_b200 import models

    row = desk[("libor", "sobol-gray")].row("sobol-gray", 2**18)
    black = models.LiborModel().black_price()
    tol = max(3 * row.std / math.sqrt(REPS), 0.005 * black)
    diff = abs(row.mean - black)
    assert diff <= tol
    assert abs(diff - 1.404e-10) <= 0.001e-10  # "|diff| 1.404e-10", test_output.txt:36


def test_criterion_7_paradigm_equivalence():
    import paper_1408_5526_b200 as P

    for gen in ("philox", "rasrap-counter", "sobol-counter"):
        rows = []
        for workers, paradigm in ((1, "replication-parallel"), (2, "stride-parallel"),
                                  (8, "stride-parallel")):
            cfg = P.ExperimentConfig(model="libor", generator=gen, n_grid=(1024, 4096),
                                     replications=6, seed=SEED, workers=workers,
                                     paradigm=paradigm)
            rep = P.run_experiment(cfg)
            rows.append([(rep.row(gen, n).mean, rep.row(gen, n).std) for n in (1024, 4096)])
        assert rows[0] == rows[1] == rows[2]


@pytest.mark.parametrize("gen", ["sobol-counter", "sobol-gray"])
def test_criterion_10_dyadic_equidistribution(gen):
    """test_acceptance.py:270-280 on the device's scrambled points: a linear
    scramble plus digital shift keeps each coordinate a (0, m, 1)-net, so the
    first 2^12 points hit every dyadic cell of width 2^-12 once (the Gray
    order is a permutation of the counter order)."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    n = 2**12
    u = DeviceSampler(gen, 360, SEED, 1).points(0, n).cpu().numpy()
    cells = np.floor(u * n).astype(np.int64)
    assert all(np.array_equal(np.sort(cells[:, d]), np.arange(n)) for d in range(360))


def test_criterion_9_single_month_collapse():
    """test_acceptance.py:232-237: one month, PV = payment / (1 + i0) for any shock."""
    from paper_1408_5526_b200 import models as M

    m = M.MbsModel(M.MbsConfig(months=1))
    u = np.array([[1e-9], [0.5], [0.999], [0.25]])
    pv = m.payoffs(u)
    expected = m.config.payment / (1 + m.config.initial_rate)
    assert np.allclose(pv, expected, rtol=0, atol=1e-15)


def test_report_timing_is_measured_per_mark():
    """time_s per grid mark is the measured mean wall time per replication of
    a call that stops at that mark (harness.py:300-313), so it grows with N;
    efficiency = std x time_s (harness.py:364-385)."""
    import paper_1408_5526_b200 as P
    from paper_1408_5526_b200 import models as M

    cfg = P.ExperimentConfig(model="libor", generator="rasrap-recursive",
                             n_grid=(2**12, 2**16, 2**20), replications=64, seed=SEED)
    rep = P.run_experiment(cfg, model=M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)))
    t = [rep.row("rasrap-recursive", n).seconds for n in cfg.n_grid]
    assert t[0] < t[2] and t[1] < t[2]
    for n in cfg.n_grid:
        r = rep.row("rasrap-recursive", n)
        assert r.efficiency == r.std * r.seconds
    with pytest.raises(ValueError):
        P.run_experiment(cfg, timing="guess")

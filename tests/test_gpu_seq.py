"""Device parity of the sequential word streams: MT19937 and
XORWOW (prng.py:40-149) behind make_sampler("twister" / "xorwow")
(harness.py:110-113) and in the fused replication engine.

Bars as in test_gpu_parity.py: uniforms BIT-EXACT against the reference's
chunked ``fill`` (golden fixtures) and the oracle; theta of f = x_1
BIT-EXACT; LIBOR / MBS theta within 1e-12 relative.  The device positions
MT19937 by snapshots and XORWOW by GF(2) jump matrices, so the far-row and
segment-boundary cases below are what pin those.
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


def _model(kind):
    from paper_1408_5526_b200 import models as M

    return {"s20": lambda: M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25)),
            "s80": lambda: M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25)),
            "mbs": M.MbsModel, "x1": M.FirstCoordinateModel}[kind]()


CASES = ["twister_d20_m1", "xorwow_d20_m1", "twister_d80_m2", "xorwow_d360_m3",
         "twister_d360_m1"]


def _case(tag):
    gen, d, m = tag.split("_")
    return gen, int(d[1:]), int(m[1:])


@pytest.mark.parametrize("tag", CASES)
def test_points_bit_exact_far_rows(P, golden, tag):
    """points(first, count) anywhere in the stream == the reference's fill."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("prng_seq")
    gen, dim, m = _case(tag)
    rows, ref = g[f"{tag}_rows"], g[f"{tag}_points"]
    s = DeviceSampler(gen, dim, SEED, m)
    # contiguous head block, then every sampled far row one at a time
    head = rows[rows < 300]
    assert np.array_equal(s.points(0, 300).cpu().numpy()[head], ref[: head.size])
    far = np.nonzero(rows >= 300)[0]
    for k in far[:: max(1, far.size // 40)]:
        got = s.points(int(rows[k]), 1).cpu().numpy()[0]
        assert np.array_equal(got, ref[k]), (tag, int(rows[k]))


@pytest.mark.parametrize("gen", ["twister", "xorwow"])
def test_fill_sequence_matches_reference(P, golden, gen):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("prng_seq")
    tag = f"{gen}_d20_m1"
    rows, ref = g[f"{tag}_rows"], g[f"{tag}_points"]
    s = DeviceSampler(gen, 20, SEED, 1)
    out = np.empty((20000, 20))
    for a, b in ((0, 137), (137, 8192), (8192, 8193), (8193, 20000)):  # ragged chunks
        s.fill(out[a:b])
    sel = rows < 20000
    assert np.array_equal(out[rows[sel]], ref[sel])


@pytest.mark.parametrize("gen", ["twister", "xorwow", "kakutani"])
def test_fill_readahead_refills(P, gen, monkeypatch):
    """Consecutive fills of a sequential stream are served from a read-ahead
    block (repeated fills re-walked the stream from its start);
    a small block forces refills across its boundaries."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    monkeypatch.setattr(DeviceSampler, "READAHEAD_BYTES", 8 * 5 * 1000)  # 1000-row blocks
    s = DeviceSampler(gen, 5, SEED, 2)
    out = np.empty((5000, 5))
    for a in range(0, 5000, 777):
        s.fill(out[a:a + 777])
    ref = DeviceSampler(gen, 5, SEED, 2).points(0, 5000).cpu().numpy()
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("gen", ["twister", "xorwow"])
def test_word_streams_vs_oracle_many_segments(P, oracle, gen):
    """A long fill that spans many device segments (and jump/snapshot starts)."""
    from paper_1408_5526_b200.samplers import DeviceSampler

    dim, m, first, count = 7, 5, 123_457, 300_001
    key = oracle.derive_key(SEED, 1 if gen == "twister" else 2, m)
    ws = oracle.mt19937(key & 0xFFFFFFFF) if gen == "twister" else oracle.xorwow(key)
    w = ws.words((first + count) * dim)[first * dim:].reshape(count, dim)
    got = DeviceSampler(gen, dim, SEED, m).points(first, count).cpu().numpy()
    assert np.array_equal(got, w * 2.0**-32 + 2.0**-33)


def test_at_is_not_available(P):
    from paper_1408_5526_b200.samplers import DeviceSampler

    for gen in ("twister", "xorwow"):
        s = DeviceSampler(gen, 4, SEED, 1)
        assert not s.counter_based
        with pytest.raises(TypeError):
            s.at(np.arange(3))


THETA_SEQ = {
    "libor20_twister": ("twister", "s20"),
    "libor20_xorwow": ("xorwow", "s20"),
    "libor80_twister": ("twister", "s80"),
    "libor80_xorwow": ("xorwow", "s80"),
    "mbs_twister": ("twister", "mbs"),
    "mbs_xorwow": ("xorwow", "mbs"),
    "x1_twister": ("twister", "x1"),
    "x1_xorwow": ("xorwow", "x1"),
}


@pytest.mark.parametrize("tag", sorted(THETA_SEQ))
def test_theta_vs_reference(P, golden, tag):
    gen, mk = THETA_SEQ[tag]
    t = golden("theta_seq")
    grid = tuple(int(n) for n in t[f"{tag}_grid"])
    ref = t[f"{tag}_theta"]  # [grid, M]
    M_ = ref.shape[1]
    cfg = P.ExperimentConfig(model=_model(mk).name, generator=gen, n_grid=grid, replications=M_,
                             seed=SEED)
    rep = P.run_experiment(cfg, model=_model(mk))
    got = np.stack([rep.estimates(gen, n) for n in grid])
    if mk == "x1":
        assert np.array_equal(got, ref)
    else:
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


@pytest.mark.parametrize("gen", ["twister", "xorwow"])
def test_theta_vs_oracle_large(P, oracle, gen):
    """N large enough for several segments per replication; ragged N."""
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    x1 = M.FirstCoordinateModel()
    grid = (65_537, 999_983)
    got = estimate_replications(gen, x1, SEED, 3, 3, grid)
    ref = oracle.run_replications(gen, x1, SEED, 3, 3, grid, threads=3)
    assert np.array_equal(got, ref)
    lib = _model("s20")
    got = estimate_replications(gen, lib, SEED, 1, 4, (300_001,))
    ref = oracle.run_replications(gen, lib, SEED, 1, 4, (300_001,), threads=4)
    assert (np.abs(got / ref - 1)).max() <= THETA_RTOL
    mbs = _model("mbs")
    got = estimate_replications(gen, mbs, SEED, 2, 2, (20_011,))
    ref = oracle.run_replications(gen, mbs, SEED, 2, 2, (20_011,), threads=2)
    assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


def test_theta_invariant_to_sharding(P):
    from paper_1408_5526_b200.harness import estimate_replications

    model = _model("s20")
    for gen in ("twister", "xorwow"):
        full = estimate_replications(gen, model, SEED, 1, 6, (4096,))
        a = estimate_replications(gen, model, SEED, 1, 2, (4096,))
        b = estimate_replications(gen, model, SEED, 3, 4, (4096,))
        assert np.array_equal(full, np.concatenate([a, b]))


# ---------------------------------------------------------------- Kakutani
@pytest.mark.parametrize("tag", ["d20_m1", "d5_m2", "d360_m1"])
def test_kakutani_points_bit_exact(P, golden, tag):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("kakutani")
    dim, m = int(tag[1:].split("_m")[0]), int(tag.split("_m")[1])
    rows, ref = g[f"{tag}_rows"], g[f"{tag}_points"]
    s = DeviceSampler("kakutani", dim, SEED, m)
    pts = s.points(0, int(rows[-1]) + 1).cpu().numpy()
    assert np.array_equal(pts[rows], ref)
    k = rows.size // 2  # a single far row (snapshot start mid-stream)
    assert np.array_equal(s.points(int(rows[k]), 1).cpu().numpy()[0], ref[k])


def test_kakutani_fill_sequence(P, golden):
    from paper_1408_5526_b200.samplers import DeviceSampler

    g = golden("kakutani")
    rows, ref = g["d5_m2_rows"], g["d5_m2_points"]
    s = DeviceSampler("kakutani", 5, SEED, 2)
    out = np.empty((50_000, 5))
    for a, b in ((0, 1), (1, 8192), (8192, 8300), (8300, 50_000)):
        s.fill(out[a:b])
    sel = rows < 50_000
    assert np.array_equal(out[rows[sel]], ref[sel])


@pytest.mark.parametrize("tag,mk", [("libor20", "s20"), ("mbs", "mbs"), ("x1", "x1")])
def test_kakutani_theta_vs_reference(P, golden, tag, mk):
    g = golden("kakutani")
    grid = tuple(int(n) for n in g[f"{tag}_grid"])
    ref = g[f"{tag}_theta"]
    cfg = P.ExperimentConfig(model=_model(mk).name, generator="kakutani", n_grid=grid,
                             replications=ref.shape[1], seed=SEED)
    rep = P.run_experiment(cfg, model=_model(mk))
    got = np.stack([rep.estimates("kakutani", n) for n in grid])
    if mk == "x1":
        assert np.array_equal(got, ref)
    else:
        assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


def test_kakutani_theta_vs_oracle_large(P, oracle):
    from paper_1408_5526_b200 import models as M
    from paper_1408_5526_b200.harness import estimate_replications

    x1 = M.FirstCoordinateModel()
    got = estimate_replications("kakutani", x1, SEED, 1, 3, (65_537, 700_001))
    ref = oracle.run_replications("kakutani", x1, SEED, 1, 3, (65_537, 700_001), threads=3)
    assert np.array_equal(got, ref)
    lib = _model("s20")
    got = estimate_replications("kakutani", lib, SEED, 2, 3, (200_003,))
    ref = oracle.run_replications("kakutani", lib, SEED, 2, 3, (200_003,), threads=3)
    assert (np.abs(got / ref - 1)).max() <= THETA_RTOL


@pytest.mark.parametrize("gen", ["twister", "xorwow", "kakutani", "rasrap-recursive"])
def test_small_batches_and_snapshot_groups(P, gen, monkeypatch):
    """Many payoff batches and snapshot groups give the same theta as one."""
    from paper_1408_5526_b200.harness import estimate_replications

    model = _model("s20")
    ref = estimate_replications(gen, model, SEED, 1, 7, (5000, 20_000))
    monkeypatch.setenv("RQ_BATCH_PATHS", "40000")      # 2 replications per batch
    monkeypatch.setenv("RQ_SNAP_GROUP_BYTES", "1")      # one batch per snapshot group
    got = estimate_replications(gen, model, SEED, 1, 7, (5000, 20_000))
    assert np.array_equal(got, ref)

"""Parity at the BENCHMARK sizes (BASELINE.json configs 2, 3, 5).

The fused path kernels run in a different regime at the bench sizes than at
the small N of test_gpu_parity.py: at N = 2^20 a persistent CTA advances its
Rasrap odometer / Sobol' state through ~1,400 contiguous tiles and across
replication boundaries inside a 128-replication batch.  These tests run the
GPU exactly as bench.py does (all M replications of the config through
rq_run_replications) and compare replications at both ends of the range —
first ids and ids in the LAST payoff batch — with the oracle (oracle/, a
bit-exact C restatement of the reference numba path, harness.py:291-315):

  * LIBOR / MBS theta: relative error <= 1e-12 (north_star tolerance);
  * the xhash test integrand (a hash of every coordinate's bits, exact sums):
    theta BIT-EXACT, so all 20 / 80 / 360 coordinates of every path of the
    device streams are pinned at N = 2^20 / 10^6, not only dimension 0.
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

    return pkg


def _threads(oracle):
    return max(4, oracle.host_cores())


def _sobol_v(gen, dim):
    if not gen.startswith("sobol"):
        return None
    from paper_1408_5526_b200.tables import sobol_directions

    return sobol_directions(dim)


def _oracle_ids(oracle, gen, model, ids, grid):
    """Oracle theta for the replication ids (runs of consecutive ids)."""
    rows = []
    runs = np.split(ids, np.where(np.diff(ids) != 1)[0] + 1)
    for r in runs:
        rows.append(oracle.run_replications(gen, model, SEED, int(r[0]), len(r), grid,
                                            threads=_threads(oracle),
                                            sobol_v=_sobol_v(gen, model.dim)))
    return np.concatenate(rows)


def _libor(mat):
    from paper_1408_5526_b200 import models as M

    return M.LiborModel(M.LiborConfig(maturity=mat, accrual=0.25))


def _gpu(gen, model, M, grid):
    from paper_1408_5526_b200.harness import estimate_replications

    return estimate_replications(gen, model, SEED, 1, M, grid)


C2_IDS = np.r_[1:9, 1017:1025]


@pytest.mark.parametrize("gen", ["rasrap-recursive", "rasrap-counter", "philox", "sobol-gray",
                                 "sobol-counter", "sfc64", "twister", "xorwow", "kakutani"])
def test_c2_theta_at_bench_size(P, oracle, gen):
    """Config 2: LIBOR S=20, M=1024 x N=2^20 on the GPU (8 payoff batches of
    128 replications), ids 1-8 and 1017-1024 vs the oracle."""
    model = _libor(5.0)
    grid = (2**20,)
    got = _gpu(gen, model, 1024, grid)
    ref = _oracle_ids(oracle, gen, model, C2_IDS, grid)
    err = np.abs(got[C2_IDS - 1] / ref - 1).max()
    assert err <= THETA_RTOL, (gen, err)


def test_c2_prefix_grid_at_bench_size(P, oracle):
    """Several grid marks of one stream (harness.py:282-315) at the C2 size."""
    model = _libor(5.0)
    grid = (10_000, 2**18 + 3, 999_983, 2**20)
    got = _gpu("rasrap-recursive", model, 130, grid)
    ids = np.r_[1:3, 128:131]
    ref = _oracle_ids(oracle, "rasrap-recursive", model, ids, grid)
    assert np.abs(got[ids - 1] / ref - 1).max() <= THETA_RTOL


@pytest.mark.parametrize("gen", ["rasrap-recursive", "philox", "sobol-gray", "xorwow"])
def test_c3_mbs_theta_at_bench_size(P, oracle, gen):
    """Config 3: MBS 360 months, M=256 x N=10^6 (two payoff batches), ids
    1-4 and 253-256 vs the oracle (Rasrap is the config's generator; the
    others are the reference's MBS acceptance set)."""
    from paper_1408_5526_b200 import models as M

    model = M.MbsModel()
    grid = (10**6,)
    got = _gpu(gen, model, 256, grid)
    ids = np.r_[1:5, 253:257]
    ref = _oracle_ids(oracle, gen, model, ids, grid)
    err = np.abs(got[ids - 1] / ref - 1).max()
    assert err <= THETA_RTOL, (gen, err)


@pytest.mark.parametrize("gen", ["rasrap-recursive", "philox", "sobol-gray"])
def test_c5_theta_at_bench_size(P, oracle, gen):
    """Config 5: LIBOR S=80 at N=2^20 (the first 256 of its 8192
    replications: two payoff batches), ids 1-4 and 253-256 vs the oracle."""
    model = _libor(20.0)
    assert model.dim == 80
    grid = (2**20,)
    got = _gpu(gen, model, 256, grid)
    ids = np.r_[1:5, 253:257]
    ref = _oracle_ids(oracle, gen, model, ids, grid)
    err = np.abs(got[ids - 1] / ref - 1).max()
    assert err <= THETA_RTOL, (gen, err)


XHASH = [
    # (generator, dim, N, M on the GPU, oracle ids)
    ("rasrap-recursive", 20, 2**20, 256, np.r_[1:5, 253:257]),
    ("rasrap-counter", 20, 2**20, 256, np.r_[1:3, 255:257]),
    ("philox", 20, 2**20, 256, np.r_[1:3, 255:257]),
    ("sobol-gray", 20, 2**20, 256, np.r_[1:3, 255:257]),
    ("sobol-counter", 20, 2**20, 256, np.r_[1:3, 255:257]),
    ("sfc64", 20, 2**20, 256, np.r_[1:3, 255:257]),
    ("rasrap-recursive", 80, 2**20, 130, np.r_[1:3, 129:131]),
    ("philox", 80, 2**20, 130, np.r_[1:2, 130:131]),
    ("sobol-gray", 80, 2**20, 130, np.r_[1:2, 130:131]),
    ("rasrap-recursive", 360, 10**6, 136, np.r_[1:3, 135:137]),
    ("rasrap-counter", 360, 10**6, 4, np.r_[1:3]),
    ("sobol-gray", 360, 10**6, 136, np.r_[1:2, 136:137]),
    ("philox", 360, 10**6, 4, np.r_[1:3]),
    ("twister", 20, 2**20, 8, np.r_[1:3, 8:9]),
    ("xorwow", 20, 2**20, 8, np.r_[1:3, 8:9]),
    ("kakutani", 20, 2**18, 4, np.r_[1:3]),
    ("twister", 360, 2**17, 4, np.r_[1:3]),
    ("xorwow", 360, 2**17, 4, np.r_[1:3]),
    ("kakutani", 80, 2**16, 2, np.r_[1:3]),
]


@pytest.mark.parametrize("gen,dim,n,M_,ids", XHASH,
                         ids=[f"{g}-d{d}-n{n}" for g, d, n, _, _ in XHASH])
def test_xhash_theta_bit_exact(P, oracle, gen, dim, n, M_, ids):
    """Every coordinate of every path of the production path kernel: theta of
    the coordinate-hash integrand is bit-exact against the oracle."""
    from paper_1408_5526_b200 import models as M

    model = M.CoordinateHashModel(dim)
    grid = (n // 3, n)
    got = _gpu(gen, model, M_, grid)
    ref = _oracle_ids(oracle, gen, model, ids, grid)
    assert np.array_equal(got[ids - 1], ref), (gen, dim, got[ids - 1], ref)


MBS_EDGE = [
    # (MbsConfig overrides, tolerance): forced out-of-range branches
    ({"variance": 0.04}, THETA_RTOL),       # |sigma_xi z| > 0.1 for |z| > 0.5: exp fallback
    ({"k4": 1.2}, THETA_RTOL),              # atan argument above the two series centres
    ({"k4": 0.1}, THETA_RTOL),              # ... and below them
    ({"k3": -30.0, "k4": 0.6}, THETA_RTOL), # negative atan arguments
    ({"variance": 0.25}, THETA_RTOL),       # prod(1 + i) overflows without rescaling
]


@pytest.mark.parametrize("over,tol", MBS_EDGE, ids=[str(o) for o, _ in MBS_EDGE])
def test_mbs_fallback_branches(P, oracle, over, tol):
    """MBS configs that force the exp / atan fallbacks (models.py:430-449)
    and a high-variance config whose discount product overflows a double:
    theta finite and within tolerance of the oracle."""
    from paper_1408_5526_b200 import models as M

    model = M.MbsModel(M.MbsConfig(**over))
    grid = (1000, 4096)
    for gen in ("rasrap-recursive", "philox"):
        got = _gpu(gen, model, 4, grid)
        ref = oracle.run_replications(gen, model, SEED, 1, 4, grid, threads=4)
        assert np.all(np.isfinite(ref)) and np.all(np.isfinite(got))
        err = np.abs(got / ref - 1).max()
        assert err <= tol, (gen, over, err)


@pytest.mark.parametrize("var", [0.0004, 0.04, 0.25])
def test_mbs_payoffs_high_variance(P, oracle, var):
    """Per-path MBS payoffs (model.payoffs, models.py:462-469) of 4096 Philox
    paths vs the oracle, including paths whose discount product passes
    2^512 (rescaled on the device)."""
    from paper_1408_5526_b200 import models as M

    m = M.MbsModel(M.MbsConfig(variance=var))
    c = m.config
    u = oracle.philox_words(oracle.derive_key(SEED, 3, 1), np.arange(4096), 360) * 2.0**-32 \
        + 2.0**-33
    ref = oracle.mbs_payoffs(u, c.initial_rate, c.k0, c.k1, c.k2, c.k3, c.k4, c.sigma_xi,
                             c.payment, m.annuity)
    got = m.payoffs(u)
    assert np.all(np.isfinite(got))
    assert np.abs(got / ref - 1).max() <= 1e-12


SEG_GENS = ["rasrap-recursive", "rasrap-counter", "philox", "sobol-gray", "sfc64"]


@pytest.mark.parametrize("gen", SEG_GENS)
def test_segmented_estimates_match(P, oracle, gen, monkeypatch):
    """Grid marks longer than RQ_SEG_PATHS are evaluated in segments, each a
    subtree of numpy's pairwise tree (harness.py:314), combined in tree
    order: forcing tiny segments must reproduce the single-pass theta bit for
    bit (x1 against the oracle, LIBOR against the unsegmented device run)."""
    from paper_1408_5526_b200 import models as M

    grid = (1000, 50_000, 100_003)
    x1 = M.FirstCoordinateModel()
    libor = _libor(5.0)
    base_x1 = _gpu(gen, x1, 3, grid)
    base_l = _gpu(gen, libor, 3, grid)
    for seg in ("4096", "128"):
        monkeypatch.setenv("RQ_SEG_PATHS", seg)
        assert np.array_equal(_gpu(gen, x1, 3, grid), base_x1)
        assert np.array_equal(_gpu(gen, libor, 3, grid), base_l)
    monkeypatch.delenv("RQ_SEG_PATHS")
    ref = oracle.run_replications(gen, x1, SEED, 1, 3, grid, threads=3,
                                  sobol_v=_sobol_v(gen, x1.dim))
    assert np.array_equal(base_x1, ref)


def test_estimates_beyond_2_32_paths(P):
    """N > 2^32 paths per replication (the reference sums any N): segmented
    on the device; f = 1 is exact, f = x1 within 6 standard errors of 1/2,
    and Sobol' (32-bit direction numbers) is refused."""
    from paper_1408_5526_b200 import models as M

    n = 2**32 + 1000
    th = _gpu("philox", M.ConstantModel(), 2, (2**31 + 8, n))
    assert np.array_equal(th, np.ones_like(th))
    th = _gpu("philox", M.FirstCoordinateModel(), 2, (2**31 + 8, n))
    assert np.all(np.abs(th - 0.5) < 6 * (1 / np.sqrt(12 * 2**31)))
    with pytest.raises(ValueError):
        _gpu("sobol-gray", M.FirstCoordinateModel(), 1, (n,))


@pytest.mark.timeout(900)
def test_sharded_device_pipeline_under_torchrun(P):
    """The device pipeline under torchrun with 3 ranks (sharing the box's
    GPU over gloo): a fixed M=37 split 13/12/12, theta gathered once --
    bit-identical to one process (harness.py:349-358 worker-count invariance)."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "3", "--master-addr", "127.0.0.1",
                        "--master-port", "29547", "tests/_torchrun_device.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    one = _gpu("rasrap-recursive", _libor(5.0), 37, (1000, 2**17))
    assert d["world"] == 3 and np.array_equal(np.array(d["theta"]), one)

"""Host-side logic of the drop-in API (no GPU): configuration validation,
statistics and reports (mirroring the reference's test_harness.py), model
setup parity with the reference, and replication sharding over a 2-process
gloo group (the CPU stand-in for NCCL over NVLink)."""
import math
import os

import numpy as np
import pytest

from conftest import SEED

import paper_1408_5526_b200 as P
from paper_1408_5526_b200 import distributed as D
from paper_1408_5526_b200 import harness as H
from paper_1408_5526_b200 import models as M


# ------------------------------------------------------------ config / stats
def test_config_validation_mirrors_reference():
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="philox", n_grid=())
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="philox", n_grid=(10, 10))
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="philox", n_grid=(0, 10))
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="philox", n_grid=(10,), replications=1)
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="philox", n_grid=(10,), workers=0)
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="nope", n_grid=(10,))
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="rasrap-recursive", n_grid=(10,),
                           paradigm="stride-parallel")
    cfg = H.ExperimentConfig(model="libor", generator="philox", n_grid=[10, 20],
                             paradigm="stride-parallel")
    assert cfg.n_grid == (10, 20)
    assert isinstance(H.ConfigurationError("x"), ValueError)


def test_generators_without_device_path_raise():
    with pytest.raises(H.ConfigurationError):
        H.make_sampler("bogus", 2, 0, 1)
    # every reference generator has a device path; the sequential ones are not counter-based
    assert set(H.DEVICE_GENERATORS) >= set(H.GENERATOR_NAMES)
    assert not ({"twister", "xorwow", "kakutani"} & H.COUNTER_BASED)
    with pytest.raises(H.ConfigurationError):
        H.ExperimentConfig(model="libor", generator="xorwow", n_grid=(10,),
                           paradigm="stride-parallel")


def test_sample_std_and_slope():
    assert H.sample_std([1.0, 2.0, 3.0]) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        H.sample_std([1.0])
    pts = [(2**k, 3.0 * (2**k) ** -0.5) for k in range(4, 10)]
    slope, icpt, res = H.fit_slope(pts)
    assert slope == pytest.approx(-0.5, abs=1e-12)
    assert icpt == pytest.approx(math.log(3.0), abs=1e-12)
    with pytest.raises(ValueError):
        H.fit_slope([(1, 0.0), (2, 0.0), (4, 1.0)])


def test_assign_stride_partitions():
    W, n = 3, 20
    idx = sorted(H.assign_stride(w, W, k) for w in range(W) for k in range(n) if
                 H.assign_stride(w, W, k) < n)
    assert idx == list(range(n))
    with pytest.raises(ValueError):
        H.assign_stride(3, 3, 0)


def test_report_roundtrip(tmp_path):
    rep = H.ConvergenceReport(
        rows=[H.GridRow("philox", "libor", 1024, 4, 0.1234567890123, 1e-5, 0.5, 5e-6)],
        slopes=[H.SlopeFit("philox", "libor", -0.5, 1.0, 1e-3)])
    out = tmp_path / "r.csv"
    H.write_report(rep, out)
    lines = out.read_text().splitlines()
    assert lines[0] == "generator,model,N,M,mean,std,time_s,efficiency"
    assert lines[1].startswith("philox,libor,1024,4,0.123456789012,")
    assert (tmp_path / "r_summary.csv").read_text().splitlines()[1] == "philox,libor,-0.5,0.001"
    assert H.summary_path("x.csv") == "x_summary.csv"
    with pytest.raises(OSError):
        H.write_report(rep, tmp_path / "missing" / "r.csv")


# ------------------------------------------------------------ model setup
@pytest.mark.parametrize("tag,mat", [("s10", None), ("s20", 5.0), ("s80", 20.0)])
def test_libor_setup_matches_reference(golden, tag, mat):
    g = golden("models")
    model = M.LiborModel() if mat is None else M.LiborModel(M.LiborConfig(maturity=mat,
                                                                        accrual=0.25))
    assert np.array_equal(model.bonds, g[f"libor_{tag}_bonds"])
    assert np.array_equal(model.initial_rates, g[f"libor_{tag}_l0"])
    assert model.front_rate == g[f"libor_{tag}_params"][4]
    assert model.black_price() == g[f"libor_{tag}_black"][0]


def test_mbs_setup_matches_reference(golden):
    g = golden("models")
    m = M.MbsModel()
    assert np.array_equal(m.annuity, g["mbs_ck"])
    assert (m.config.k0, m.config.sigma_xi) == tuple(g["mbs_k0_sigxi"])
    with pytest.raises(ValueError):
        M.MbsConfig(initial_rate=0.0)


def test_libor_config_validation():
    with pytest.raises(ValueError):
        M.LiborConfig(maturity=5.0, accrual=0.3)
    with pytest.raises(ValueError):
        M.LiborModel(M.LiborConfig(maturity=50.0, accrual=0.25))  # S=200 > 160
    assert M.LiborModel(M.LiborConfig(maturity=7.5, accrual=0.25)).dim == 30  # generic model


# ------------------------------------------------------------ aggregation
def test_run_experiment_aggregation_matches_reference(golden, monkeypatch, oracle):
    """Device engine swapped for the oracle: the host aggregation
    (mean, unbiased std, slope rows) must reproduce the reference's report."""
    t = golden("theta")
    tag, grid = "libor20_prefix_rasrap", tuple(int(n) for n in golden("theta")[
        "libor20_prefix_rasrap_grid"])
    model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))

    def fake(gen, mdl, seed, first, count, grid_, launches=None):
        return oracle.run_replications(gen, mdl, seed, first, count, grid_, threads=4)

    monkeypatch.setattr(H, "estimate_replications", fake)
    cfg = P.ExperimentConfig(model="libor", generator="rasrap-recursive", n_grid=grid,
                             replications=8, seed=SEED)
    rep = P.run_experiment(cfg, model=model, distributed=False)
    for gi, n in enumerate(grid):
        assert rep.row("rasrap-recursive", n).mean == t[f"{tag}_mean"][gi]
        assert rep.row("rasrap-recursive", n).std == t[f"{tag}_std"][gi]
        assert np.array_equal(rep.estimates("rasrap-recursive", n), t[f"{tag}_theta"][gi])
    assert len(rep.slopes) == 1


def test_nonfinite_estimate_raises():
    with pytest.raises(ArithmeticError):
        H.ReplicationResult(3, float("nan"), 0.1)


# ------------------------------------------------------------ sharding
def test_shard_partition():
    for total in (1, 7, 16, 256, 8192):
        for world in (1, 2, 3, 4, 8):
            parts = [D.shard(total, world, r) for r in range(world)]
            assert parts[0][0] == 0
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f0 + c0 == f1
            assert sum(c for _, c in parts) == total
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def _worker(rank, world, port, total, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def est(gen, model, seed, first, count, grid):
        # deterministic stand-in for the device: theta = f(replication id, N)
        return np.array([[first + r + n * 1e-6 for n in grid] for r in range(count)])

    theta = D.estimate_sharded("philox", None, SEED, total, (10, 20), estimator=est)
    q.put((rank, theta))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 16), (2, 7), (3, 5)])
def test_gather_over_gloo_is_world_size_invariant(world, total):
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.array([[1 + r + n * 1e-6 for n in (10, 20)] for r in range(total)])
    for _, theta in res:
        assert np.array_equal(theta, expect)


def _failing_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def est(gen, model, seed, first, count, grid):
        if first > 1:  # only the last rank's shard "produces a NaN"
            raise ArithmeticError(f"replication {first} produced a non-finite estimate")
        return np.ones((count, len(grid)))

    try:
        D.estimate_sharded("philox", None, SEED, 8, (10,), estimator=est)
        q.put((rank, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, (type(e).__name__, str(e))))
    dist.destroy_process_group()


def test_sharded_error_reaches_every_rank():
    """one rank's ArithmeticError must not leave the others
    blocked in the gather -- every rank re-raises the same error type."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_failing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert res[r] is not None and res[r][0] == "ArithmeticError", res
        assert "rank 1" in res[r][1]


@pytest.mark.timeout(600)
def test_sharded_oracle_under_torchrun_matches_one_process(oracle):
    """Strong-scaling host path under torchrun (2 ranks, gloo, CPU): the
    fixed M split over ranks, real estimator (the oracle standing in for the
    device), theta gathered once -- bit-identical to one process."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29541", "tests/_torchrun_sharded.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    from paper_1408_5526_b200 import models as M

    model = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    ref = oracle.run_replications("philox", model, SEED, 1, 7, (1000, 4096), threads=4)
    assert d["world"] == 2 and d["counts"] == [4, 3]
    assert np.array_equal(np.array(d["theta"]), ref)

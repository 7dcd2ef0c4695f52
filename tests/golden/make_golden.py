"""Generate the golden fixtures the oracle and the CUDA path are pinned to.

Runs the UNMODIFIED reference package (`rqmcbench`, /root/reference/pkg)
from a writable copy (numba writes its cache next to the sources) and
records its outputs on seeded inputs into ``tests/golden/*.npz``.  Only
this script touches the reference; the committed fixtures are what the
tests read (the GPU box has no /root/reference).

    python tests/golden/make_golden.py [--ref /root/reference/pkg]

Versions of numpy / numba / scipy used are stored in every fixture
(``versions`` key) because the randomisation goes through numpy's PCG64.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SEED = 20120224  # reference acceptance seed, test_acceptance.py:19


def _import_reference(ref: Path):
    tmp = Path(tempfile.mkdtemp(prefix="rqmc_ref_"))
    shutil.copytree(ref, tmp / "pkg")
    sys.path.insert(0, str(tmp / "pkg" / "src"))
    import rqmcbench  # noqa: F401
    from rqmcbench import halton, harness, models, prng, seeding, sobol

    return halton, harness, models, prng, seeding, sobol


def _rows(nmax: int, head: int = 512, step: int = 1999, tail: int = 32) -> np.ndarray:
    idx = set(range(min(head, nmax)))
    idx.update(range(head, nmax, step))
    idx.update(range(max(0, nmax - tail), nmax))
    return np.array(sorted(idx), dtype=np.int64)


def _fill_rows(sampler, dim: int, nmax: int, rows: np.ndarray, chunk: int = 8192):
    """Run sampler.fill sequentially (as the harness does) keeping `rows`."""
    out = np.empty((rows.size, dim))
    buf = np.empty((chunk, dim))
    done = 0
    k = 0
    while done < nmax:
        n = min(chunk, nmax - done)
        sampler.fill(buf[:n])
        while k < rows.size and rows[k] < done + n:
            out[k] = buf[rows[k] - done]
            k += 1
        done += n
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--out", default=str(HERE))
    ap.add_argument("--only", default="", help="comma list of sections (e.g. seq)")
    args = ap.parse_args()
    halton, H, M, prng, seeding, sobol = _import_reference(Path(args.ref))
    import numba
    import scipy

    versions = json.dumps(
        {"numpy": np.__version__, "numba": numba.__version__, "scipy": scipy.__version__}
    )
    out = Path(args.out)
    if args.only:
        for sec in args.only.split(","):
            globals()[f"_section_{sec}"](out, versions, H, M, prng, seeding)
        return
    _section_seq(out, versions, H, M, prng, seeding)
    _section_kak(out, versions, H, M, prng, seeding)

    # ---------------- seeding + randomisation ---------------------------
    fams = sorted(seeding.GENERATOR_IDS.values())
    keys = np.array(
        [[seeding.derive_key(SEED, f, m) for m in range(0, 9)] for f in fams], dtype=np.uint64
    )
    words = np.array([seeding.derive_words(int(k), 7) for k in keys[:, 1]], dtype=np.uint32)
    np.savez_compressed(out / "seeding.npz", versions=versions, families=np.array(fams),
                        keys=keys, words=words)

    # ---------------- Rasrap (random start + permutations) --------------
    rz = {"versions": versions}
    cases = [(20, 1, 2**20 + 1024), (20, 2, 20000), (80, 1, 2**18), (80, 3, 20000),
             (360, 1, 10**6 + 64), (360, 2, 4096)]
    for dim, m, nmax in cases:
        key = seeding.derive_key(SEED, seeding.GENERATOR_IDS["rasrap"], m)
        cfg = halton.rasrap_config(dim, key)
        tag = f"d{dim}_m{m}"
        rz[f"{tag}_start"] = np.array(cfg.start_indices, dtype=np.int64)
        rz[f"{tag}_omega"] = np.array(cfg.starts)
        rz[f"{tag}_sigma"] = halton._pack_sigmas(cfg).astype(np.int16)
        rows = _rows(nmax, step=9973 if dim == 360 else 1999)
        rz[f"{tag}_rows"] = rows
        rz[f"{tag}_recursive"] = _fill_rows(H.make_sampler("rasrap-recursive", dim, SEED, m),
                                            dim, nmax, rows)
        cs = H.make_sampler("rasrap-counter", dim, SEED, m)
        rz[f"{tag}_counter"] = cs.at(rows)
        big = np.array([2**32 - 7, 2**32 + 12345, 3 * 2**33 + 5], dtype=np.int64)
        rz[f"{tag}_bigidx"] = big
        rz[f"{tag}_counter_big"] = cs.at(big)
    np.savez_compressed(out / "rasrap.npz", **rz)

    # ---------------- Philox ------------------------------------------
    pz = {"versions": versions}
    for dim, m in ((20, 1), (20, 2), (80, 1), (360, 1)):
        key = seeding.derive_key(SEED, seeding.GENERATOR_IDS["philox"], m)
        rows = _rows(2**20 + 100, head=128, step=8191)
        pp = prng.PhiloxPaths(key)
        pz[f"d{dim}_m{m}_rows"] = rows
        pz[f"d{dim}_m{m}_words"] = pp.words_at(rows, dim)
        s = H.make_sampler("philox", dim, SEED, m)
        u = np.empty((300, dim))
        s.fill(u[:100]); s.fill(u[100:])
        pz[f"d{dim}_m{m}_fill300"] = u
    np.savez_compressed(out / "philox.npz", **pz)

    # ---------------- Sobol (scrambled) ---------------------------------
    sz = {"versions": versions}
    sz["table421_v"] = sobol.default_table(421).v
    for dim, m, nmax in ((20, 1, 2**20 + 1024), (20, 2, 30000), (80, 1, 40000), (360, 1, 10000)):
        tag = f"d{dim}_m{m}"
        g = H.make_sampler("sobol-gray", dim, SEED, m)
        sz[f"{tag}_gen_v"] = g.table._gen_v
        sz[f"{tag}_shift"] = g.table._gen_shift
        rows = _rows(nmax)
        sz[f"{tag}_rows"] = rows
        sz[f"{tag}_gray"] = _fill_rows(g, dim, nmax, rows)
        c = H.make_sampler("sobol-counter", dim, SEED, m)
        sz[f"{tag}_counter"] = c.at(rows)
    np.savez_compressed(out / "sobol.npz", **sz)

    # ---------------- inverse normal -----------------------------------
    rng = np.random.default_rng(11)
    u = np.concatenate([
        np.array([0.0, 2.0**-1074, 1e-300, 2.0**-60, 2.0**-53, 2.0**-52, 1e-10, 0.0465,
                  np.nextafter(0.0465, 0), np.nextafter(0.0465, 1), 0.5, np.nextafter(0.5, 1),
                  np.nextafter(0.5, 0), 1 - 0.0465, 1 - 2.0**-53, 1 - 2.0**-52, 1.0]),
        np.linspace(0, 1, 20001), rng.random(20000), rng.random(2000) * 0.0465,
    ])
    np.savez_compressed(out / "inv_normal.npz", versions=versions, u=u, x=M.inv_normal(u))

    # ---------------- models -------------------------------------------
    mz = {"versions": versions}
    for tag, mat in (("s10", None), ("s20", 5.0), ("s80", 20.0)):
        model = M.LiborModel() if mat is None else M.LiborModel(M.LiborConfig(maturity=mat, accrual=0.25))
        c = model.config
        n = {"s10": 500, "s20": 2000, "s80": 400}[tag]
        uu = rng.random((n, model.dim))
        mz[f"libor_{tag}_params"] = np.array([c.maturity, c.accrual, c.strike, c.sigma,
                                              model.front_rate])
        mz[f"libor_{tag}_l0"] = model.initial_rates
        mz[f"libor_{tag}_bonds"] = model.bonds
        mz[f"libor_{tag}_black"] = np.array([model.black_price()])
        mz[f"libor_{tag}_u"] = uu
        mz[f"libor_{tag}_payoffs"] = model.payoffs(uu)
    mbs = M.MbsModel()
    uu = rng.random((300, 360))
    mz["mbs_ck"] = mbs._ck
    mz["mbs_u"] = uu
    mz["mbs_payoffs"] = mbs.payoffs(uu)
    mz["mbs_k0_sigxi"] = np.array([mbs.config.k0, mbs.config.sigma_xi])
    np.savez_compressed(out / "models.npz", **mz)

    # ---------------- per-replication estimates -------------------------
    tz = {"versions": versions}
    s20 = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    s80 = M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25))
    runs = [
        ("c1_rasrap_recursive", "libor", "rasrap-recursive", (10_000,), 16, s20),
        ("c1_rasrap_counter", "libor", "rasrap-counter", (10_000,), 16, s20),
        ("libor20_prefix_rasrap", "libor", "rasrap-recursive", (100, 1000, 4096, 10_000), 8, s20),
        ("libor20_philox", "libor", "philox", (1000, 8192, 20_000), 8, s20),
        ("libor20_sobol_gray", "libor", "sobol-gray", (1000, 8192, 20_000), 8, s20),
        ("libor20_sobol_counter", "libor", "sobol-counter", (1000, 8192), 4, s20),
        ("libor80_rasrap", "libor", "rasrap-recursive", (2048,), 4, s80),
        ("libor80_philox", "libor", "philox", (2048,), 4, s80),
        ("mbs_rasrap", "mbs", "rasrap-recursive", (500, 3000), 4, M.MbsModel()),
        ("mbs_philox", "mbs", "philox", (3000,), 4, M.MbsModel()),
        ("mbs_sobol_gray", "mbs", "sobol-gray", (3000,), 4, M.MbsModel()),
        ("x1_rasrap", "x1", "rasrap-recursive", (7, 100, 1000, 10_000, 100_003), 8,
         M.FirstCoordinateModel()),
        ("x1_philox", "x1", "philox", (129, 65_536), 8, M.FirstCoordinateModel()),
        ("x1_sobol_gray", "x1", "sobol-gray", (1000, 65_536), 8, M.FirstCoordinateModel()),
        ("const1_rasrap", "const1", "rasrap-recursive", (10, 1000), 4, M.ConstantModel()),
    ]
    for tag, mname, gen, grid, reps, model in runs:
        cfg = H.ExperimentConfig(model=mname, generator=gen, n_grid=grid, replications=reps,
                                 seed=SEED, workers=4)
        rep = H.run_experiment(cfg, model=model)
        tz[f"{tag}_grid"] = np.array(grid, dtype=np.int64)
        tz[f"{tag}_theta"] = np.stack([rep.estimates(gen, n) for n in grid])  # [grid, M]
        tz[f"{tag}_mean"] = np.array([rep.row(gen, n).mean for n in grid])
        tz[f"{tag}_std"] = np.array([rep.row(gen, n).std for n in grid])
        print(tag, tz[f"{tag}_mean"], flush=True)
    # stride paradigm must equal replication paradigm (test_harness.py:134-143)
    cfg = H.ExperimentConfig(model="libor", generator="philox", n_grid=(5000,), replications=3,
                             seed=SEED, workers=3, paradigm="stride-parallel")
    rep = H.run_experiment(cfg, model=s20)
    tz["stride_philox_theta"] = rep.estimates("philox", 5000)
    np.savez_compressed(out / "theta.npz", **tz)
    print("golden fixtures written to", out)


def _section_seq(out, versions, H, M, prng, seeding):
    """MT19937 / XORWOW word streams and replication estimates (prng.py:40-149,
    harness.py:37-50, 99-125)."""
    z = {"versions": versions}
    mt_seeds = np.array([0, 1, 5489, 2**32 - 1, 20120224], dtype=np.uint64)
    xw_seeds = np.array([0, 1, 123456789, 2**64 - 1, 20120224], dtype=np.uint64)
    z["mt_seeds"] = mt_seeds
    z["mt_words"] = np.stack([_words(prng.MT19937(int(s)), 5000) for s in mt_seeds])
    z["xw_seeds"] = xw_seeds
    z["xw_words"] = np.stack([_words(prng.Xorwow(int(s)), 5000) for s in xw_seeds])
    # far into a stream: rows of the harness samplers (chunked fill)
    for gen, dim, m, nmax in (("twister", 20, 1, 2**20 + 1024), ("xorwow", 20, 1, 2**20 + 1024),
                              ("twister", 80, 2, 50000), ("xorwow", 360, 3, 20000),
                              ("twister", 360, 1, 20000)):
        tag = f"{gen}_d{dim}_m{m}"
        rows = _rows(nmax, head=300, step=7919)
        z[f"{tag}_rows"] = rows
        z[f"{tag}_points"] = _fill_rows(H.make_sampler(gen, dim, SEED, m), dim, nmax, rows)
    np.savez_compressed(out / "prng_seq.npz", **z)

    tz = {"versions": versions}
    s20 = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    s80 = M.LiborModel(M.LiborConfig(maturity=20.0, accrual=0.25))
    runs = [
        ("libor20_twister", "libor", "twister", (1000, 8192, 20_000), 8, s20),
        ("libor20_xorwow", "libor", "xorwow", (1000, 8192, 20_000), 8, s20),
        ("libor80_twister", "libor", "twister", (2048,), 4, s80),
        ("libor80_xorwow", "libor", "xorwow", (2048,), 4, s80),
        ("mbs_twister", "mbs", "twister", (500, 3000), 4, M.MbsModel()),
        ("mbs_xorwow", "mbs", "xorwow", (3000,), 4, M.MbsModel()),
        ("x1_twister", "x1", "twister", (7, 1000, 65_536), 4, M.FirstCoordinateModel()),
        ("x1_xorwow", "x1", "xorwow", (129, 65_536), 4, M.FirstCoordinateModel()),
    ]
    for tag, mname, gen, grid, reps, model in runs:
        cfg = H.ExperimentConfig(model=mname, generator=gen, n_grid=grid, replications=reps,
                                 seed=SEED, workers=4)
        rep = H.run_experiment(cfg, model=model)
        tz[f"{tag}_grid"] = np.array(grid, dtype=np.int64)
        tz[f"{tag}_theta"] = np.stack([rep.estimates(gen, n) for n in grid])  # [grid, M]
        tz[f"{tag}_mean"] = np.array([rep.row(gen, n).mean for n in grid])
        tz[f"{tag}_std"] = np.array([rep.row(gen, n).std for n in grid])
        print(tag, tz[f"{tag}_mean"], flush=True)
    np.savez_compressed(out / "theta_seq.npz", **tz)


def _section_kak(out, versions, H, M, prng, seeding):
    """Kakutani orbits (halton.py:163-239, 521-542): points and estimates."""
    import time

    z = {"versions": versions}
    for dim, m, nmax in ((20, 1, 60_000), (5, 2, 200_000), (360, 1, 2000)):
        tag = f"d{dim}_m{m}"
        rows = _rows(nmax, head=300, step=997)
        z[f"{tag}_rows"] = rows
        t0 = time.time()
        z[f"{tag}_points"] = _fill_rows(H.make_sampler("kakutani", dim, SEED, m), dim, nmax, rows)
        print(tag, f"{time.time() - t0:.1f}s", flush=True)
    s20 = M.LiborModel(M.LiborConfig(maturity=5.0, accrual=0.25))
    for tag, mname, grid, reps, model in (
            ("libor20", "libor", (1000, 8192), 4, s20),
            ("mbs", "mbs", (500,), 2, M.MbsModel()),
            ("x1", "x1", (7, 1000, 20_000), 4, M.FirstCoordinateModel())):
        cfg = H.ExperimentConfig(model=mname, generator="kakutani", n_grid=grid,
                                 replications=reps, seed=SEED, workers=4)
        rep = H.run_experiment(cfg, model=model)
        z[f"{tag}_grid"] = np.array(grid, dtype=np.int64)
        z[f"{tag}_theta"] = np.stack([rep.estimates("kakutani", n) for n in grid])
        print(tag, z[f"{tag}_theta"][:, 0], flush=True)
    np.savez_compressed(out / "kakutani.npz", **z)


BIG_COLS_STEP = 97
LONG_CURVE = ((0.25, 1.0, 2.0, 5.0, 10.0, 30.0, 60.0, 100.0, 160.0),
              (1.0, 1.2, 1.5, 2.0, 2.5, 3.0, 3.2, 3.3, 3.4))  # tenor years, rate percent


def _big_cols(dim: int) -> np.ndarray:
    """Columns kept of a wide row: the first and last 24, the constant-bank
    edge (512), and every BIG_COLS_STEP-th."""
    cols = set(range(min(24, dim))) | set(range(max(0, dim - 24), dim))
    cols |= {c for c in range(500, 530) if c < dim} | set(range(0, dim, BIG_COLS_STEP))
    return np.array(sorted(cols), dtype=np.int64)


def _section_bigdim(out, versions, H, M, prng, seeding):
    """Dimensions beyond the first 512 primes (up to every base < 2^16) and
    LIBOR beyond 160 steps: points of the reference's own samplers (selected
    columns) and per-replication estimates."""
    import time

    z = {"versions": versions}
    for gen, dim, m in (("rasrap", 6542, 1), ("rasrap", 1000, 2), ("kakutani", 700, 1)):
        tag = f"{gen}_d{dim}_m{m}"
        cols = _big_cols(dim)
        z[f"{tag}_cols"] = cols
        t0 = time.time()
        if gen == "rasrap":
            rows = np.arange(300, dtype=np.int64)
            z[f"{tag}_recursive"] = _fill_rows(H.make_sampler("rasrap-recursive", dim, SEED, m),
                                               dim, 300, rows)[:, cols]
            idx = np.array([0, 1, 127, 128, 300, 12345, 2**20 + 3, 2**32 + 7, 3 * 2**33 + 5],
                           dtype=np.int64)
            z[f"{tag}_idx"] = idx
            z[f"{tag}_counter"] = H.make_sampler("rasrap-counter", dim, SEED, m).at(idx)[:, cols]
        else:
            rows = _rows(3000, head=300, step=997)
            z[f"{tag}_rows"] = rows
            z[f"{tag}_points"] = _fill_rows(H.make_sampler(gen, dim, SEED, m), dim, 3000,
                                            rows)[:, cols]
        print(tag, f"{time.time() - t0:.1f}s", flush=True)
    # 200 steps on the default curve (it ends at 30 years); 600 on a longer
    # user curve (YieldCurve takes any tenors, models.py:96-112)
    s200 = M.LiborModel(M.LiborConfig(maturity=25.0, accrual=0.125))
    z["long_curve"] = np.array([LONG_CURVE[0], LONG_CURVE[1]])
    s600 = M.LiborModel(M.LiborConfig(maturity=150.0, accrual=0.25),
                        curve=M.YieldCurve(np.array(LONG_CURVE[0]), np.array(LONG_CURVE[1])))
    for tag, mname, gen, grid, reps, model in (
            ("libor200_rasrap", "libor", "rasrap-recursive", (300, 1000), 2, s200),
            ("libor200_philox", "libor", "philox", (1000,), 2, s200),
            ("libor600_rasrap", "libor", "rasrap-recursive", (257,), 2, s600),
            ("libor600_counter", "libor", "rasrap-counter", (257,), 2, s600),
            ("mbs600_rasrap", "mbs", "rasrap-recursive", (500,), 2, M.MbsModel(M.MbsConfig(months=600))),
            ("libor200_kakutani", "libor", "kakutani", (500,), 2, s200)):
        t0 = time.time()
        cfg = H.ExperimentConfig(model=mname, generator=gen, n_grid=grid, replications=reps,
                                 seed=SEED, workers=2)
        rep = H.run_experiment(cfg, model=model)
        z[f"{tag}_grid"] = np.array(grid, dtype=np.int64)
        z[f"{tag}_theta"] = np.stack([rep.estimates(gen, n) for n in grid])
        print(tag, z[f"{tag}_theta"][:, 0], f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(out / "bigdim.npz", **z)


def _words(gen, n: int) -> np.ndarray:
    w = np.empty(n, dtype=np.uint32)
    gen.fill_words(w)
    return w


if __name__ == "__main__":
    main()

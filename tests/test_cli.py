"""CLI mirror of the reference (cli.py:1-152): parsing and exit codes on CPU,
device output in test_gpu_parity-style checks (marked gpu)."""
import io
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, SEED


def test_parse_n_grid_matches_reference_forms():
    from paper_1408_5526_b200.cli import parse_n_grid

    assert parse_n_grid("2^10..2^12") == (1024, 2048, 4096)
    assert parse_n_grid("1000..8000") == (1000, 2000, 4000, 8000)
    assert parse_n_grid("1024, 2^11,4096") == (1024, 2048, 4096)


def test_configuration_errors_exit_1(capsys):
    from paper_1408_5526_b200 import cli

    # unknown generator inside the comma list -> ConfigurationError before device work
    rc = cli.main(["libor", "--generator", "nope", "--n-grid", "10,20", "--out", "/tmp/x.csv"])
    assert rc == 1
    assert "configuration error" in capsys.readouterr().err
    rc = cli.main(["mbs", "--generator", "philox", "--n-grid", "20,10", "--out", "/tmp/x.csv"])
    assert rc == 1
    rc = cli.main(["gen", "--generator", "kakutani", "--dim", "0", "--count", "3"])
    assert rc == 1


def test_argparse_rejects_unknown_generator():
    with pytest.raises(SystemExit):
        from paper_1408_5526_b200 import cli

        cli.build_parser().parse_args(["gen", "--generator", "bogus", "--dim", "1", "--count", "1"])


def test_module_entry_point_runs():
    r = subprocess.run([sys.executable, "-m", "paper_1408_5526_b200", "--help"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0 and "gen" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("gen,tagfile,tag", [("rasrap-recursive", "rasrap", "d20_m1"),
                                             ("xorwow", "prng_seq", "xorwow_d20_m1")])
def test_gen_dump_bit_exact(golden, gen, tagfile, tag):
    from paper_1408_5526_b200 import cli

    g = golden(tagfile)
    rows = g[f"{tag}_rows"]
    ref = g[f"{tag}_recursive"] if gen.startswith("rasrap") else g[f"{tag}_points"]
    n = 1000
    buf = io.StringIO()
    args = cli.build_parser().parse_args(["gen", "--generator", gen, "--dim", "20", "--count",
                                          str(n), "--seed", str(SEED), "--replication", "1"])
    assert cli._run_gen(args, out=buf) == 0
    pts = np.array([[float(x) for x in ln.split("\t")] for ln in buf.getvalue().splitlines()])
    sel = rows < n
    assert np.array_equal(pts[rows[sel]], ref[sel])


@pytest.mark.gpu
def test_libor_experiment_writes_report(tmp_path):
    from paper_1408_5526_b200 import cli

    out = tmp_path / "r.csv"
    rc = cli.main(["libor", "--generator", "philox,xorwow", "--n-grid", "2^10..2^12",
                   "--reps", "4", "--seed", str(SEED), "--out", str(out)])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "generator,model,N,M,mean,std,time_s,efficiency"
    assert len(lines) == 1 + 2 * 3
    assert (tmp_path / "r_summary.csv").exists()


@pytest.mark.gpu
@pytest.mark.parametrize("gen", ["rasrap-recursive", "philox", "sobol-gray", "twister",
                                 "kakutani"])
def test_bench_throughput_runs(gen):
    """harness.bench_throughput (harness.py:401-429): raw generation rate."""
    from paper_1408_5526_b200 import harness

    rate = harness.bench_throughput(gen, 20, 2_000_000, runs=3)
    assert rate > 1e8  # coordinates/s (the reference's CPU rate is ~1e8 at best)


@pytest.mark.gpu
def test_cli_bench_prints_rate(capsys):
    from paper_1408_5526_b200 import cli

    assert cli.main(["bench", "--generator", "xorwow", "--dim", "8", "--count", "100000",
                     "--runs", "2"]) == 0
    out = capsys.readouterr().out
    assert out.startswith("xorwow\tdim=8\t") and out.strip().endswith("numbers/s")

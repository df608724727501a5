"""CLI drop-in and file interchange, host side (no GPU): parser surface and
defaults vs the reference CLI (cli.py:297-356), MatrixMarket round trips
(io.py:33-54), manifests (io.py:129-152), exit codes (cli.py:376-380), and
the reference's output schemas recorded in tests/golden/cli/."""

import json
import os

import numpy as np
import pytest

from paper_1403_7458_b200 import cli, io

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")


def test_parser_defaults_match_reference():
    p = cli.build_parser()
    a = p.parse_args(["multiply", "a.mtx", "b.mtx", "--out", "c.mtx"])
    assert (a.tau, a.block_size, a.chunk_size, a.mode, a.workers, a.deterministic,
            a.format, a.stats) == (0.0, 16, None, "serial", None, True, "auto", None)
    s = p.parse_args(["sp2", "f.mtx", "--n-occ", "3", "--out", "p.mtx"])
    assert (s.tau, s.max_iter, s.idem_tol, s.report, s.criterion) == (0.0, 100, 1e-9, None,
                                                                       "trace")
    t = p.parse_args(["sweep", "tau", "--f", "f.mtx", "--n-occ", "3", "--out", "o.csv"])
    assert t.taus == [1e-6, 1e-8, 1e-10] and t.max_iter == 100
    t = p.parse_args(["sweep", "tau", "--f", "f.mtx", "--n-occ", "3", "--taus", "1e-4,1e-6",
                      "--out", "o.csv"])
    assert t.taus == [1e-4, 1e-6]
    assert p.parse_args(["multiply", "a", "b", "--out", "c", "--no-deterministic"]).deterministic is False


def test_version_and_usage_errors(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["--version"])
    assert e.value.code == 0
    with pytest.raises(SystemExit) as e:
        cli.main(["multiply", "a.mtx"])          # argparse: missing operands -> 2
    assert e.value.code == 2


def test_missing_input_exits_2(tmp_path, capsys):
    rc = cli.main(["multiply", str(tmp_path / "nope.mtx"), str(tmp_path / "nope.mtx"),
                   "--out", str(tmp_path / "c.mtx")])
    assert rc == 2 and "error:" in capsys.readouterr().err


@pytest.mark.parametrize("fmt", ["auto", "array", "coordinate"])
def test_matrix_market_round_trip_exact(tmp_path, rng, fmt):
    d = rng.standard_normal((23, 23)) * 10.0 ** rng.integers(-300, 300, (23, 23))
    d[rng.random((23, 23)) < 0.6] = 0.0
    path = tmp_path / "m.mtx"
    io.write_matrix_market(path, d, fmt=fmt)
    back = io.read_matrix_market(path)
    assert np.array_equal(back, d)
    head = path.read_text().splitlines()[0]
    want = "coordinate" if fmt == "coordinate" or (fmt == "auto" and np.count_nonzero(d) < d.size / 2) else "array"
    assert want in head
    with pytest.raises(ValueError):
        io.write_matrix_market(path, d, fmt="dense")


def test_reads_reference_written_files():
    a = io.read_matrix_market(os.path.join(GOLD, "A.mtx"))
    f = io.read_matrix_market(os.path.join(GOLD, "F.mtx"))
    assert a.shape == (100, 100) and f.shape == (200, 200)
    assert np.array_equal(f, f.T)
    from paper_1403_7458_b200.synth import decay_pair, water_cluster
    assert np.array_equal(a, decay_pair(100, lam=0.15, seeds=(3, 4))[0])
    assert np.array_equal(f, water_cluster(8, seed=2)[0])


def test_manifest_fields(tmp_path):
    m = io.build_manifest("multiply", {"tau": 1e-3}, {}, ["a.mtx"], ["c.mtx"],
                          argv=["multiply", "a.mtx", "b.mtx"])
    assert set(m) == {"command", "argv", "parameters", "seeds", "inputs", "outputs",
                      "library_version", "timestamp", "user"}
    io.write_manifest(tmp_path / "x.manifest.json", m)
    assert io.read_manifest(tmp_path / "x.manifest.json")["argv"] == ["multiply", "a.mtx", "b.mtx"]


def test_reference_schemas_recorded():
    st = json.load(open(os.path.join(GOLD, "C_ref.stats.json")))
    assert list(st) == ["tau", "tiers", "leaf_products", "flop_estimate", "wall_seconds"]
    rep = json.load(open(os.path.join(GOLD, "P_ref.report.json")))
    assert list(rep) == ["n", "n_occ", "tau", "iterations", "converged", "trace_history",
                         "branch_history", "wall_seconds_per_iteration", "idempotency_error"]
    header = open(os.path.join(GOLD, "sweep_ref.csv")).readline().strip().split(",")
    assert header == ["tau", "energy_error", "abs_energy_error", "idempotency_error",
                      "iterations", "converged", "leaf_products"]

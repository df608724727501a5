"""CLI drop-in on the GPU vs the reference CLI's recorded outputs
(tests/golden/cli, made by make_cli_golden.py with the reference):
with --leaf-kernel exact the product, the SP2 density matrix, the stats /
report JSON (wall times aside) and the tau sweep are bitwise the
reference's; the default (DMMA) path is within the BASELINE tolerance."""

import csv
import json
import os

import numpy as np
import pytest

from paper_1403_7458_b200 import cli, io

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")
G = lambda name: os.path.join(GOLD, name)  # noqa: E731
N_OCC = open(os.path.join(GOLD, "n_occ.txt")).read().strip()


def _strip_wall(d):
    return {k: v for k, v in d.items() if not k.startswith("wall_seconds")}


@pytest.mark.parametrize("kernel", ["exact", "auto"])
def test_cli_multiply(tmp_path, kernel):
    out, stats = tmp_path / "C.mtx", tmp_path / "C.stats.json"
    assert cli.main(["multiply", G("A.mtx"), G("B.mtx"), "--tau", "1e-3", "--block-size", "16",
                     "--leaf-kernel", kernel, "--out", str(out), "--stats", str(stats)]) == 0
    c, ref = io.read_matrix_market(out), io.read_matrix_market(G("C_ref.mtx"))
    if kernel == "exact":
        assert np.array_equal(c, ref)
    else:
        assert np.linalg.norm(c - ref) <= 1e-12 * np.linalg.norm(ref)
    assert _strip_wall(json.load(open(stats))) == _strip_wall(json.load(open(G("C_ref.stats.json"))))
    man = io.read_manifest(str(out) + ".manifest.json")
    assert man["command"] == "multiply" and man["outputs"] == [str(out), str(stats)]


def test_cli_sp2_and_rerun(tmp_path):
    out, rep = tmp_path / "P.mtx", tmp_path / "P.report.json"
    argv = ["sp2", G("F.mtx"), "--n-occ", N_OCC, "--tau", "1e-7", "--block-size", "16",
            "--leaf-kernel", "exact", "--out", str(out), "--report", str(rep)]
    assert cli.main(argv) == 0
    p, ref = io.read_matrix_market(out), io.read_matrix_market(G("P_ref.mtx"))
    assert np.array_equal(p, ref)
    got, want = json.load(open(rep)), json.load(open(G("P_ref.report.json")))
    assert _strip_wall(got) == _strip_wall(want)
    # one entry per X^2 (the converging square included), as the reference
    assert len(got["wall_seconds_per_iteration"]) == len(want["wall_seconds_per_iteration"])
    first = out.read_bytes()
    os.remove(out)
    assert cli.main(["rerun", str(out) + ".manifest.json"]) == 0
    assert out.read_bytes() == first          # replay is bitwise


def test_cli_sweep_tau(tmp_path):
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "tau", "--f", G("F.mtx"), "--n-occ", N_OCC, "--taus", "1e-4,1e-6",
                     "--block-size", "16", "--leaf-kernel", "exact", "--out", str(out)]) == 0
    got = list(csv.DictReader(open(out)))
    want = list(csv.DictReader(open(G("sweep_ref.csv"))))
    assert got == want


def test_cli_sp2_fro_criterion(tmp_path):
    out = tmp_path / "P.mtx"
    assert cli.main(["sp2", G("F.mtx"), "--n-occ", N_OCC, "--tau", "1e-7", "--block-size", "16",
                     "--criterion", "fro", "--out", str(out)]) == 0
    p = io.read_matrix_market(out)
    assert np.linalg.norm(p @ p - p) < 1e-5

"""Golden outputs of the REFERENCE CLI (cli.py) for the CLI drop-in tests.

Run once in the build container (the reference is importable there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Inputs come from paper_1403_7458_b200.synth (seeded, host independent) and
are written as MatrixMarket with the reference's own writer; the reference
CLI then runs `multiply`, `sp2` and `sweep tau` on them.  Everything lands in
tests/golden/cli/ (inputs, outputs, JSON, CSV); manifests are dropped (they
hold timestamps, user names and absolute paths).
"""

from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from spamm import io as ref_io  # noqa: E402  (the reference)
from spamm.cli import main as ref_main  # noqa: E402

from paper_1403_7458_b200.synth import decay_pair, water_cluster  # noqa: E402

OUT = os.path.join(HERE, "cli")


def run(argv):
    rc = ref_main(argv)
    assert rc == 0, (argv, rc)


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    p = lambda name: os.path.join(OUT, name)  # noqa: E731
    a, b = decay_pair(100, lam=0.15, seeds=(3, 4))
    ref_io.write_matrix_market(p("A.mtx"), a)
    ref_io.write_matrix_market(p("B.mtx"), b)
    h, n_occ = water_cluster(8, seed=2)
    ref_io.write_matrix_market(p("F.mtx"), h)
    with open(p("n_occ.txt"), "w") as fh:
        fh.write(f"{n_occ}\n")
    run(["multiply", p("A.mtx"), p("B.mtx"), "--tau", "1e-3", "--block-size", "16",
         "--out", p("C_ref.mtx"), "--stats", p("C_ref.stats.json")])
    run(["sp2", p("F.mtx"), "--n-occ", str(n_occ), "--tau", "1e-7", "--block-size", "16",
         "--out", p("P_ref.mtx"), "--report", p("P_ref.report.json")])
    run(["sweep", "tau", "--f", p("F.mtx"), "--n-occ", str(n_occ), "--taus", "1e-4,1e-6",
         "--block-size", "16", "--out", p("sweep_ref.csv")])
    for name in os.listdir(OUT):
        if name.endswith(".manifest.json"):
            os.remove(os.path.join(OUT, name))
    print(sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

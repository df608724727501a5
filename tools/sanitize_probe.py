"""Leaf-product kernels under compute-sanitizer (racecheck / synccheck /
memcheck): one multiply per (input, kernel), results checked against the
oracle so a run that "passes" the tool also computed the right product.

Usage (GPU box):
    compute-sanitizer --tool racecheck --racecheck-report all \
        python tools/sanitize_probe.py cfg1 dmma
inputs: cfg1 (decay pair, N=1024, Nb=32), nb64 (decay pair, N=1024, Nb=64),
cfg3x0 (cfg3 X0^2: 90 molecules, N=2250 -> 4096, Nb=32);
kernels: dmma (K4, TMA + mbarrier), ozaki (K4z / K4z32), exact."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1403_7458_b200 as sp  # noqa: E402
from oracle import spamm_oracle as O  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402


def main():
    which, kernel = sys.argv[1], sys.argv[2]
    if which == "cfg3x0":
        cfg = CONFIGS[3]
        h, _ = water_cluster(cfg.n_mol, seed=0)
        f = sp.build_from_dense(h, 32)
        a = sp.sp2_init(f, sp.gershgorin_bounds(f))
        of = O.from_dense(h, 32)
        oa = O.sp2_init(of, O.gershgorin_bounds(of))
        b, ob, tau = a, oa, cfg.tau
    else:
        nb = 64 if which == "nb64" else 32
        da, db = decay_pair(1024, 0.1, (0, 1))
        a, b = sp.build_from_dense(da, nb), sp.build_from_dense(db, nb)
        oa, ob, tau = O.from_dense(da, nb), O.from_dense(db, nb), 1e-8
    c, st = sp.multiply(a, b, tau, kernel=kernel)
    oc, ost, _ = O.multiply(oa, ob, tau, threads=os.cpu_count())
    ref = O.to_dense(oc)
    got = sp.to_dense(c)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    exact = bool(np.array_equal(got, ref))
    ok = st.visited == ost["visited"] and (exact if kernel == "exact" else err < 1e-12)
    print(f"[sanitize_probe] {which} {kernel}: leaf_products={st.leaf_products} "
          f"symmetric={st.symmetric} rel_fro={err:.3e} bitwise={exact} ok={ok}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

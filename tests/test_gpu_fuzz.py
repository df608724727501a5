"""Randomised parity sweep (seeded): shapes, block sizes, sparsity, symmetry
and tolerances drawn at random; every product is checked against the oracle
(task counters exact, exact kernel bitwise, DMMA kernel within the BASELINE
tolerance), and symmetric cases also run a short SP2 solve."""

import numpy as np
import pytest

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    nb = int(r.choice([1, 2, 4, 8, 16, 32, 64]))
    n = int(r.integers(1, 5 * nb + 40 if nb < 32 else 4 * nb + 1))
    d = r.standard_normal((n, n)) * np.exp(-0.05 * np.abs(np.subtract.outer(np.arange(n), np.arange(n))))
    d[r.random((n, n)) < r.uniform(0.0, 0.9)] = 0.0
    sym = bool(r.integers(0, 2))
    if sym:
        d = np.triu(d) + np.triu(d, 1).T
    e = r.standard_normal((n, n)) if not sym else d
    return r, nb, d, e, sym


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_multiply(seed):
    r, nb, d, e, sym = _case(seed)
    a = sp.build_from_dense(d, nb)
    b = a if sym else sp.build_from_dense(e, nb)
    oa = O.from_dense(d, nb)
    ob = oa if sym else O.from_dense(e, nb)
    norms = np.concatenate([t.ravel() for t in oa.tier_norms])
    pos = norms[norms > 0]
    taus = [0.0, float(r.uniform(0, 1)) * (pos.max() ** 2 if len(pos) else 1.0)]
    if len(pos) > 1:
        taus.append(float(pos[r.integers(len(pos))] * pos[r.integers(len(pos))]))  # a tie
    for tau in taus:
        oc, ost, _ = O.multiply(oa, ob, tau)
        c, st = sp.multiply(a, b, tau, kernel="exact")
        assert st.visited == tuple(ost["visited"]) and st.culled == tuple(ost["culled"])
        assert st.leaf_products == ost["leaf_products"]
        assert np.array_equal(sp.to_dense(c), O.to_dense(oc))
        assert np.array_equal(c._block_keys, oc.keys)
        if nb in (8, 16, 32, 64):
            cd, _ = sp.multiply(a, b, tau)
            ref = O.to_dense(oc)
            den = np.linalg.norm(ref)
            assert np.linalg.norm(sp.to_dense(cd) - ref) <= 1e-12 * max(den, 1e-300)


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_sp2(seed):
    r = np.random.default_rng(2000 + seed)
    nb = int(r.choice([4, 8, 16, 32, 64]))
    n = int(r.integers(nb + 2, 4 * nb + 3))
    a = r.standard_normal((n, n)) * np.exp(-0.1 * np.abs(np.subtract.outer(np.arange(n), np.arange(n))))
    d = (a + a.T) / 2
    n_occ = int(r.integers(1, n))
    tau = float(r.choice([0.0, 1e-8, 1e-5]))
    crit = str(r.choice(["trace", "fro"]))
    p, st = sp.sp2_solve(sp.build_from_dense(d, nb), n_occ, tau, kernel="exact", criterion=crit,
                         max_iter=60)
    ro = O.sp2_solve(O.from_dense(d, nb), n_occ, tau, criterion=crit, max_iter=60)
    assert st.iteration == ro.iterations and st.converged == ro.converged
    assert st.branch_history == ro.branches
    assert np.array_equal(sp.to_dense(p), O.to_dense(ro.x))

"""Oracle vs the live reference package (only where /root/reference exists,
i.e. in the build container).  Randomised shapes, block sizes, tolerances."""

import numpy as np
import pytest

from conftest import import_reference, pyramid_flat, reference_available
from oracle import spamm_oracle as O

pytestmark = pytest.mark.skipif(not reference_available(),
                                reason="reference package not mounted here")


def _ref():
    return import_reference()


@pytest.mark.parametrize("seed", range(6))
def test_multiply_and_storage_bitwise(seed):
    spamm = _ref()
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 160))
    nb = int(2 ** rng.integers(0, 6))
    da = rng.standard_normal((n, n)) * np.exp(rng.standard_normal((n, n)) * 2)
    db = rng.standard_normal((n, n))
    da[np.abs(da) < rng.uniform(0, 1.5)] = 0.0
    a, b = spamm.build_from_dense(da, nb), spamm.build_from_dense(db, nb)
    oa, ob = O.from_dense(da, nb), O.from_dense(db, nb)
    assert np.array_equal(oa.keys, a._block_keys)
    assert np.array_equal(pyramid_flat(oa.tier_norms), pyramid_flat(a._tier_norms))
    for tau in (0.0, float(rng.uniform(0, 1)), float(rng.uniform(1, 50))):
        c, st = spamm.multiply(a, b, tau)
        oc, ost, _ = O.multiply(oa, ob, tau, threads=3)
        assert ost["visited"] == st.visited and ost["culled"] == st.culled
        assert ost["leaf_products"] == st.leaf_products
        assert np.array_equal(O.to_dense(oc), spamm.to_dense(c))
        assert np.array_equal(pyramid_flat(oc.tier_norms), pyramid_flat(c._tier_norms))
        assert O.trace(oc) == spamm.trace(c)
    s, os_ = spamm.add_scaled(2.0, a, -1.0, b), O.add_scaled(2.0, oa, -1.0, ob)
    assert np.array_equal(O.to_dense(os_), spamm.to_dense(s))
    assert np.array_equal(pyramid_flat(os_.tier_norms), pyramid_flat(s._tier_norms))
    ident = spamm.identity(n, nb)
    oi = O.identity(n, nb)
    assert np.array_equal(O.to_dense(oi), spamm.to_dense(ident))
    assert np.array_equal(pyramid_flat(oi.tier_norms), pyramid_flat(ident._tier_norms))


def test_sp2_trace_criterion_bitwise():
    spamm = _ref()
    from paper_1403_7458_b200.synth import water_cluster
    h, n_occ = water_cluster(12, seed=3)
    f = spamm.build_from_dense(h, 16)
    p, st = spamm.sp2_solve(f, n_occ, 1e-9)
    r = O.sp2_solve(O.from_dense(h, 16), n_occ, 1e-9, threads=2)
    assert r.iterations == st.iteration and r.converged == st.converged
    assert r.branches == st.branch_history
    assert r.trace_history == st.trace_history
    assert np.array_equal(O.to_dense(r.x), spamm.to_dense(p))
    lo, hi = O.gershgorin_bounds(O.from_dense(h, 16))
    b = spamm.gershgorin_bounds(f)
    assert (lo, hi) == (b.eps_min, b.eps_max)


def test_sweep_matches_reference_sweep():
    spamm = _ref()
    rng = np.random.default_rng(9)
    d = rng.standard_normal((90, 90)) * np.exp(-0.05 * np.abs(np.subtract.outer(np.arange(90),
                                                                                np.arange(90))))
    a = spamm.build_from_dense(d, 4)
    for tau in (1e-6, 1e-3, 0.1):
        ref = spamm.kernel._sweep(a._tier_norms, a._tier_norms, tau)
        mine = O.sweep(a._tier_norms, a._tier_norms, tau)
        assert ref[0] == mine[0] and ref[1] == mine[1]
        for x, y in zip(ref[2:], mine[2:]):
            assert np.array_equal(x, y)

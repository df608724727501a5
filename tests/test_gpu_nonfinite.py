"""Non-finite operands on every leaf kernel, the default one included.

The reference propagates Inf / NaN through its FP64 leaf loop (kernel.py:64-77)
and culls on the block norms (kernel.py:108: NaN norms never pass the strict
``>``, Inf norms pass against any non-zero partner).  K4z cannot carry Inf or
NaN in integer digits: its exponent pass flags the global row / column, and
the epilogue recomputes the C elements of flagged rows / columns in FP64 in
the reference's order.  So on every kernel the Inf / NaN pattern of C equals
the reference's, flagged elements are bitwise the reference's, and the finite
rest is within the FP64 contract (rel-Fro 1e-12)."""

import numpy as np
import pytest

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402


def _sym(rng, n, scale=1.0):
    a = rng.uniform(-1, 1, (n, n)) * scale
    return np.triu(a) + np.triu(a, 1).T


def _decay(rng, n):
    i = np.arange(n)
    return _sym(rng, n) * np.exp(-0.05 * np.abs(i[:, None] - i[None, :]))


def _poison(d, cells):
    d = d.copy()
    for (r, c, v) in cells:
        d[r, c] = v
    return d


CASES = {
    # one +Inf (its own block survives; the row / column of C turn Inf / NaN)
    "inf": [(5, 70, np.inf)],
    # -Inf and +Inf in one row: Inf - Inf = NaN in the sums
    "inf_pair": [(9, 3, np.inf), (9, 100, -np.inf)],
    # NaN: its block norm is NaN, so every task reading it is culled
    "nan": [(40, 41, np.nan)],
    # mixed, several blocks
    "mixed": [(0, 0, np.inf), (130, 7, np.nan), (200, 199, -np.inf)],
}


def _compare(c_dense, ref):
    assert np.array_equal(np.isnan(c_dense), np.isnan(ref))
    inf_d, inf_r = np.isinf(c_dense), np.isinf(ref)
    assert np.array_equal(inf_d, inf_r)
    assert np.array_equal(np.sign(c_dense[inf_d]), np.sign(ref[inf_r]))
    fin = np.isfinite(ref)
    den = np.linalg.norm(ref[fin])
    err = np.linalg.norm(c_dense[fin] - ref[fin]) / (den if den > 0 else 1.0)
    assert err < 1e-12, err


@pytest.mark.parametrize("nb", [32, 64])
@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("kernel", ["auto", "ozaki", "dmma", "exact"])
def test_nonfinite_product_matches_reference(rng, nb, case, kernel):
    n = 256
    da = _poison(_decay(rng, n), CASES[case])
    db = _decay(rng, n)
    tau = 1e-10
    oa, ob = O.from_dense(da, nb), O.from_dense(db, nb)
    a, b = sp.build_from_dense(da, nb), sp.build_from_dense(db, nb)
    for (x, y, ox, oy) in ((a, b, oa, ob), (b, a, ob, oa)):   # non-finite in A, then in B
        oc, ost, _ = O.multiply(ox, oy, tau)
        ref = O.to_dense(oc)
        c, st = sp.multiply(x, y, tau, kernel=kernel)
        assert st.visited == ost["visited"] and st.culled == ost["culled"]
        got = sp.to_dense(c)
        if kernel == "exact":
            assert np.array_equal(got, ref, equal_nan=True)
        else:
            _compare(got, ref)
        # the elements of poisoned rows / columns are the reference's, bitwise
        if kernel in ("auto", "ozaki"):
            bad = ~np.isfinite(ref)
            assert np.array_equal(got[bad], ref[bad], equal_nan=True)


@pytest.mark.parametrize("nb", [32, 64])
@pytest.mark.parametrize("kernel", ["auto", "ozaki"])
def test_nonfinite_symmetric_square(rng, nb, kernel):
    """X*X with X exactly symmetric (the symmetric SpAMM path, mirrors written
    from the same accumulators): pattern and values as the reference."""
    n = 256
    d = _decay(rng, n)
    d[17, 150] = d[150, 17] = np.inf
    d[60, 61] = d[61, 60] = -np.inf
    x = sp.build_from_dense(d, nb)
    ox = O.from_dense(d, nb)
    oc, ost, _ = O.multiply(ox, ox, 1e-9)
    ref = O.to_dense(oc)
    c, st = sp.multiply(x, x, 1e-9, kernel=kernel)
    assert st.visited == ost["visited"]
    got = sp.to_dense(c)
    _compare(got, ref)
    bad = ~np.isfinite(ref)
    assert bad.any()
    assert np.array_equal(got[bad], ref[bad], equal_nan=True)

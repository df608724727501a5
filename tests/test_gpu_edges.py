"""Edge cases of the fast paths (dense cull, single-CTA finalisation, fused
idempotency residual, lazy pruning) against the oracle: tiny trees (depth 0),
products culled to nothing inside SP2, and exact-zero blocks that stay
pending across SP2 iterations."""

import numpy as np
import pytest

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402


def _solve_both(d, nb, n_occ, tau, kernel="exact", **kw):
    p, st = sp.sp2_solve(sp.build_from_dense(d, nb), n_occ, tau, kernel=kernel, **kw)
    r = O.sp2_solve(O.from_dense(d, nb), n_occ, tau, **kw)
    return p, st, r


@pytest.mark.parametrize("nb", [32, 64])
@pytest.mark.parametrize("criterion", ["fro", "trace"])
def test_sp2_depth0_single_block(rng, nb, criterion):
    n = nb - 5
    a = rng.standard_normal((n, n))
    d = (a + a.T) / 2
    p, st, r = _solve_both(d, nb, n // 3, 0.0, criterion=criterion)
    assert st.iteration == r.iterations and st.branch_history == r.branches
    assert np.array_equal(sp.to_dense(p), O.to_dense(r.x))
    if criterion == "fro":
        assert np.array_equal(np.array(st.idempotency_history), np.array(r.idem_history))


@pytest.mark.parametrize("nb", [32, 64])
def test_sp2_with_fully_culled_square(rng, nb):
    """tau above every norm product: X^2 is empty, E = 2X, the residual is ||X||."""
    n = 3 * nb
    a = rng.standard_normal((n, n))
    d = (a + a.T) / 2
    p, st, r = _solve_both(d, nb, n // 2, 1e30, criterion="fro", max_iter=4)
    assert st.iteration == r.iterations and st.branch_history == r.branches
    assert all(lp == 0 for lp in st.leaf_products)
    assert np.array_equal(np.array(st.idempotency_history), np.array(r.idem_history))
    assert np.array_equal(sp.to_dense(p), O.to_dense(r.x))


@pytest.mark.parametrize("nb", [32, 64])
def test_sp2_pending_zero_blocks_across_iterations(rng, nb):
    """X = [[I, M], [M^T, -I]] (+ small symmetric tail): (X^2)_01 cancels to an
    exact-zero block, E keeps lazily pruned blocks into the next iterations;
    the whole trajectory must stay bitwise the reference's."""
    m = rng.standard_normal((2 * nb, 2 * nb)) * 0.1
    n = 4 * nb
    x = np.zeros((n, n))
    x[: 2 * nb, : 2 * nb] = np.eye(2 * nb)
    x[2 * nb:, 2 * nb:] = -np.eye(2 * nb)
    x[: 2 * nb, 2 * nb:] = m
    x[2 * nb:, : 2 * nb] = m.T
    for criterion in ("fro", "trace"):
        p, st, r = _solve_both(x, nb, 2 * nb, 0.0, criterion=criterion, max_iter=30)
        assert st.iteration == r.iterations and st.branch_history == r.branches
        assert np.array_equal(sp.to_dense(p), O.to_dense(r.x))
        assert np.array_equal(p._block_keys, r.x.keys)        # storage settled = reference's


def test_dense_cull_max_depth_tree(rng):
    """Depth 8 (G = 256): the largest tree the dense cull takes."""
    n = 250
    d = rng.standard_normal((n, n))
    d[np.abs(d) < 1.5] = 0.0
    a = sp.build_from_dense(d, 1)
    assert a.depth == 8
    tau = 0.5
    c, st = sp.multiply(a, a, tau, kernel="exact")
    oc, ost, _ = O.multiply(O.from_dense(d, 1), O.from_dense(d, 1), tau)
    assert st.visited == tuple(ost["visited"]) and st.leaf_products == ost["leaf_products"]
    assert np.array_equal(sp.to_dense(c), O.to_dense(oc))

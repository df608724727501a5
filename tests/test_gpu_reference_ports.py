"""Remaining reference test ports (reference tests/test_kernel.py,
tests/test_quadtree.py) not covered elsewhere; see DESIGN.md §3 for the
full map of reference tests to this suite."""

import numpy as np
import pytest

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402


def test_deterministic_flag_accepts_false(rng):
    """test_kernel.py:197-201."""
    a = sp.build_from_dense(rng.standard_normal((16, 16)), block_size=4)
    c1, _ = sp.multiply(a, a, 0.0, mode="tasked", deterministic=False, workers=4)
    c2, _ = sp.multiply(a, a, 0.0, mode="serial")
    assert np.array_equal(sp.to_dense(c1), sp.to_dense(c2))


def test_submultiplicativity_witness(rng):
    """test_quadtree.py:156-163: ||AB||_F <= ||A|| ||B|| with the pyramid roots."""
    for _ in range(5):
        da, db = rng.standard_normal((24, 24)), rng.standard_normal((24, 24))
        a, b = sp.build_from_dense(da, 4), sp.build_from_dense(db, 4)
        assert np.linalg.norm(da @ db) <= a.norm() * b.norm() * (1 + 1e-12)


def test_culled_branches_and_census_against_recursion():
    """test_kernel.py:128-151: every culled branch has product <= tau, and the
    census equals the recursive oracle on a decay matrix."""
    n, nb, tau = 64, 4, 1e-6
    idx = np.arange(n)
    u = np.random.default_rng(9).uniform(0.5, 1.0, (n, n))
    dense = 0.5 ** np.abs(idx[:, None] - idx[None, :]) * (np.triu(u) + np.triu(u, 1).T)
    tree = sp.build_from_dense(dense, nb)
    pyr = tree._tier_norms
    depth = len(pyr) - 1
    visited = [0] * (depth + 1)

    def walk(t, i, k, j):
        prod = pyr[t][i, k] * pyr[t][k, j]
        if prod <= tau:
            return
        visited[t] += 1
        if t < depth:
            for di in (0, 1):
                for dk in (0, 1):
                    for dj in (0, 1):
                        walk(t + 1, 2 * i + di, 2 * k + dk, 2 * j + dj)

    walk(0, 0, 0, 0)
    st = sp.convolution_census(tree, tree, tau)
    assert st.visited == tuple(visited)
    ov, _, _, _, _ = O.sweep(O.from_dense(dense, nb).tier_norms, O.from_dense(dense, nb).tier_norms, tau)
    assert st.visited == tuple(ov)

"""Device-resident quadtree storage vs the reference semantics (quadtree.py).
Ported from the reference's test_quadtree.py against the new API, plus
bit-exact pyramid parity with the golden fixtures and the oracle."""

import numpy as np
import pytest

from conftest import golden, pyramid_flat
from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402


def test_padding_2250_to_4096():
    tree = sp.build_from_dense(np.zeros((2250, 2250)), block_size=16)
    assert tree.n_padded == 4096 and tree.n_native == 2250
    assert tree.stored_leaf_count == 0


def test_single_element_root_is_leaf():
    tree = sp.build_from_dense(np.array([[5.0]]), block_size=1)
    assert tree.root.is_leaf and tree.root.norm == 5.0 and tree.depth == 0


def test_three_four_five_norm_and_null_children():
    tree = sp.build_from_dense(np.array([[3.0, 4.0], [0.0, 0.0]]), block_size=1)
    assert tree.root.norm == pytest.approx(5.0, rel=1e-15)
    assert tree.root.children[1][0] is None and tree.root.children[1][1] is None
    assert tree.root.children[0][0].norm == 3.0 and tree.root.children[0][1].norm == 4.0


@pytest.mark.parametrize("n,nb", [(7, 2), (7, 4), (1, 1), (37, 4), (64, 16), (100, 8),
                                  (130, 64), (300, 32)])
def test_roundtrip_bitwise(rng, n, nb):
    dense = rng.standard_normal((n, n))
    tree = sp.build_from_dense(dense, block_size=nb)
    assert np.array_equal(sp.to_dense(tree), dense)


def test_empty_tree():
    tree = sp.build_from_dense(np.zeros((4, 4)), block_size=2)
    assert np.array_equal(sp.to_dense(tree), np.zeros((4, 4)))
    assert tree.root.norm == 0.0 and tree.stored_leaf_count == 0 and tree.norm() == 0.0


def test_identity_examples():
    assert np.array_equal(sp.to_dense(sp.identity(3, 2)), np.eye(3))
    assert np.array_equal(sp.to_dense(sp.identity(1, 1)), np.eye(1))
    assert sp.trace(sp.identity(5, 2)) == 5.0
    assert sp.identity(4, 2).norm() == pytest.approx(2.0, rel=1e-15)
    tree = sp.identity(8, 2)
    assert tree.root.children[0][1] is None and tree.root.children[1][0] is None


def test_add_scaled_examples(rng):
    a = sp.build_from_dense(np.arange(16.0).reshape(4, 4), block_size=2)
    z = sp.add_scaled(1.0, a, -1.0, a)
    assert z.norm() == 0.0 and z.stored_leaf_count == 0
    eye = sp.identity(4, 2)
    assert np.array_equal(sp.to_dense(sp.add_scaled(2.0, eye, -1.0, eye)), np.eye(4))
    da, db = rng.standard_normal((8, 8)), rng.standard_normal((8, 8))
    out = sp.add_scaled(0.3, sp.build_from_dense(da, 2), -1.7, sp.build_from_dense(db, 2))
    assert np.array_equal(sp.to_dense(out), 0.3 * da + (-1.7) * db)
    with pytest.raises(ValueError):
        sp.add_scaled(1.0, sp.build_from_dense(np.eye(4), 2), 1.0, sp.build_from_dense(np.eye(8), 2))


def test_trace_examples(rng):
    assert sp.trace(sp.identity(8, 2)) == 8.0
    diag = sp.build_from_dense(np.diag([1.0, 2.0, 3.0]), block_size=2)
    assert sp.trace(diag) == pytest.approx(6.0, rel=1e-15)
    for nb in (1, 2, 4, 16):
        dense = rng.standard_normal((37, 37))
        tree = sp.build_from_dense(dense, block_size=nb)
        assert sp.trace(tree) == O.trace(O.from_dense(dense, nb))


def test_verify_norms_fresh_corrupted_and_after_multiply(rng):
    tree = sp.build_from_dense(rng.standard_normal((16, 16)), block_size=4)
    ok, worst = sp.verify_norms(tree)
    assert ok and worst < 1e-12
    tree.root.children[0][0].norm += 1.0
    ok, worst = sp.verify_norms(tree)
    assert not ok and worst > 1e-12
    a = sp.build_from_dense(rng.standard_normal((32, 32)), block_size=4)
    b = sp.build_from_dense(rng.standard_normal((32, 32)), block_size=4)
    for tau in (0.0, 1e-2, 1.0):
        c, _ = sp.multiply(a, b, tau)
        assert sp.verify_norms(c)[0]


def test_padding_neutrality(rng):
    dense = rng.standard_normal((20, 20))
    small, large = sp.build_from_dense(dense, 2), sp.build_from_dense(dense, 16)
    assert np.array_equal(sp.to_dense(small), sp.to_dense(large))
    assert sp.trace(small) == pytest.approx(sp.trace(large), rel=1e-13)
    s1, s2 = sp.add_scaled(2.0, small, 3.0, small), sp.add_scaled(2.0, large, 3.0, large)
    assert np.array_equal(sp.to_dense(s1), sp.to_dense(s2))


def test_chunk_tier_geometry_and_node_tiers(rng):
    tree = sp.build_from_dense(np.eye(64), block_size=4, chunk_size=16)
    assert tree.depth == 4 and tree.chunk_tier() == 2 and tree.chunk_tier(64) == 0
    with pytest.raises(ValueError):
        tree.chunk_tier(128)
    t2 = sp.build_from_dense(rng.standard_normal((8, 8)), block_size=2)
    assert t2.root.tier == 0 and t2.root.children[0][0].tier == 1
    assert t2.root.children[0][0].children[0][0].is_leaf


def test_golden_small_cases_storage_bitwise():
    g = golden("small_cases")
    for idx in range(int(g["n_small"])):
        nb = int(g[f"s{idx}_nb"])
        a = sp.build_from_dense(g[f"s{idx}_a"], nb)
        b = sp.build_from_dense(g[f"s{idx}_b"], nb)
        assert np.array_equal(pyramid_flat(a._tier_norms), g[f"s{idx}_apyr"]), idx
        s = sp.add_scaled(0.3, a, -1.7, b)
        assert np.array_equal(sp.to_dense(s), g[f"s{idx}_add"]), idx
        assert np.array_equal(pyramid_flat(s._tier_norms), g[f"s{idx}_addpyr"]), idx


def test_norm_pyramid_bitwise_on_configs():
    from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster
    g1 = golden("cfg1")
    da, db = decay_pair(1024, 0.1, (0, 1))
    a = sp.build_from_dense(da, 32)
    assert np.array_equal(pyramid_flat(a._tier_norms), g1["a_pyramid"])
    assert a.stored_leaf_count == int(g1["a_stored"])
    g4 = golden("cfg4_sp2")
    h, _ = water_cluster(CONFIGS[4].n_mol, seed=0)
    f = sp.build_from_dense(h, 64)
    assert np.array_equal(pyramid_flat(f._tier_norms), g4["f_pyramid"])


def test_from_blocks_prunes_zero_blocks_and_reorders(rng):
    nb, depth = 4, 3
    g = 1 << depth
    keys = np.array([5, 0, 63, 17], dtype=np.int64)
    data = rng.standard_normal((4, nb, nb))
    data[2] = 0.0
    m = sp.QuadTreeMatrix.from_blocks(30, nb, 8, keys, data, depth)
    om = O.from_blocks(30, nb, 8, np.sort(keys), data[np.argsort(keys)], depth)
    assert np.array_equal(m._block_keys, om.keys)
    assert np.array_equal(m._block_data, om.data)
    assert np.array_equal(pyramid_flat(m._tier_norms), pyramid_flat(om.tier_norms))
    assert m.n_blocks == g
